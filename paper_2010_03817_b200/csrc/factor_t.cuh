// factor_t.cuh -- K2a with the pencil in lower-triangle 8 x 8 tile storage: TWO chains per SM.
//
// Same mathematics as factor_kernel (L L^T = A(x), M = -L^{-1} A(v) L^{-T};
// the Schur deflation of a boundary start, R6), with the congruence formed as
//     W = L^{-1} (blocked, in place, right to left),  M = -W B W^T,
// per 8-column panel J of M by one warp: Y^T_J = W_J: B (accumulators kept in registers),
// then M_IJ = -sum_K W_IK Y_KJ for I >= J, whose DMMA B operand is exactly the Y^T
// accumulator when the k index of the product runs over (2q, 2q+1) instead of (q, q+4).
// Both matrices are stored as the lower triangle of 8 x 8 tiles (91 tiles = 46.6 KB each at
// m = 100), so one chain needs ~111 KB of shared memory and two chains share an SM: one
// chain's latency chain (the 8 x 8 diagonal factors, barriers) overlaps the other's work.
// Tiles are XOR-swizzled (rows with bit 1 set: column ^ 5) so that the DMMA A-fragment,
// B-fragment and accumulator-pair accesses of a half-warp are all bank-conflict free.
// Outputs as factor_kernel: M (full rows of ld, zero padded) and packed L in the slot's work
// buffers, deflation vectors and status in the slot's scalar area (the Lanczos and tail
// kernels are unchanged).
#pragma once
#include "chord3.cuh"

namespace sw {

constexpr int FT_NT = 256;
constexpr int FT_TBMAX = 13;  // mdp <= 104

__device__ __forceinline__ int tph(int r, int c) { return r * 8 + (c ^ (((r >> 1) & 1) * 5)); }
__device__ __forceinline__ int tix(int i, int j) { return (i * (i + 1) / 2 + j) * 64; }  // tile (i, j), j <= i
// element (i, j) of the symmetric matrix held as lower tiles
__device__ __forceinline__ double tsym(const double* Tm, int i, int j) {
    const int a = i >= j ? i : j, b = i >= j ? j : i;
    return Tm[tix(a >> 3, b >> 3) + tph(a & 7, b & 7)];
}
__device__ __forceinline__ int tel(int i, int j) { return tix(i >> 3, j >> 3) + tph(i & 7, j & 7); }  // j <= i

__host__ __device__ inline size_t ft_smem_doubles(int mdp) {
    const int TB = mdp >> 3;
    return 2 * (size_t)TB * (TB + 1) / 2 * 64 + (size_t)TB * 64 + 8 * (size_t)(mdp + 8) + 8 * 64;
}

// (ib, jb) of the lower tile t (row-major over the lower tiles), TB <= 16: a broadcast constant load
// instead of a square root per tile (tile_of was ~10% of factor_t_kernel's stall samples, r2ft4)
__constant__ unsigned char c_tib[136] = {0, 1, 1, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 4, 5, 5, 5, 5, 5, 5, 6, 6, 6, 6, 6, 6, 6, 7, 7, 7, 7, 7, 7, 7, 7, 8, 8, 8, 8, 8, 8, 8, 8, 8, 9, 9, 9, 9, 9, 9, 9, 9, 9, 9, 10, 10, 10, 10, 10, 10, 10, 10, 10, 10, 10, 11, 11, 11, 11, 11, 11, 11, 11, 11, 11, 11, 11, 12, 12, 12, 12, 12, 12, 12, 12, 12, 12, 12, 12, 12, 13, 13, 13, 13, 13, 13, 13, 13, 13, 13, 13, 13, 13, 13, 14, 14, 14, 14, 14, 14, 14, 14, 14, 14, 14, 14, 14, 14, 14, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15};
__constant__ unsigned char c_tjb[136] = {0, 0, 1, 0, 1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 4, 0, 1, 2, 3, 4, 5, 0, 1, 2, 3, 4, 5, 6, 0, 1, 2, 3, 4, 5, 6, 7, 0, 1, 2, 3, 4, 5, 6, 7, 8, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15};
__device__ __forceinline__ void tile_of(int t, int& ib, int& jb) {
    ib = c_tib[t];
    jb = c_tjb[t];
}

// the (m - o) x (m - o) trailing block of the packed symmetric P as lower tiles, padded to
// mdp with `pad` on the diagonal (8-byte cp.async; the caller waits); o = 1 also copies row 0
// of P (m doubles) to row0
__device__ void ft_unpack(const Team& T, const double* __restrict__ P, double* Tm, int m, int o, int mdp, double pad,
                          double* row0) {
    const int TB = mdp >> 3, md = m - o;
    const int ntile = TB * (TB + 1) / 2;
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int t = T.warp; t < ntile; t += T.nwarps) {
        int ib, jb;
        tile_of(t, ib, jb);
        const int i = ib * 8 + r;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = q + 4 * h, j = jb * 8 + c;
            double* dst = Tm + tix(ib, jb) + tph(r, c);
            if (i < md && j < md) {
                const int gi = i + o, gj = j + o;
                cp_async8(dst, P + ((gj <= gi) ? pk(gi, gj) : pk(gj, gi)));
            } else {
                *dst = (i == j) ? pad : 0.0;
            }
        }
    }
    if (o)
        for (int j = T.tid; j < m; j += T.nthr) row0[j] = P[pk(j, 0)];
}

// p = beta X h - (beta/2)(h . beta X h) h for X = [[row0], [row0^T, tiles]] (m x m), for G and B
// at once: (X h) of the trailing block as row sums (a warp per block row, tiles J <= I in order)
// plus the transposed tiles' column sums (a warp per block column, tiles I > J in order) --
// deterministic: every sum in a fixed order (lane (r, q): elements (r, q), (r, q + 4))
__device__ void ft_householder_vecs(const Team& T, const double* Gt, const double* Bt, const double* g0,
                                    const double* b0, int m, int md, int TB, const double* h, double beta,
                                    double* pg, double* pb, double* cg, double* cb, double* red) {
    const int r = T.lane >> 2, q = T.lane & 3;
    const double* h1 = h + 1;  // trailing index i' = i - 1
    for (int w = T.warp; w < 2 * TB; w += T.nwarps) {
        if (w < TB) {  // block row I = w: sum_J X_IJ h_J
            const int I = w;
            double sg = 0.0, sb = 0.0;
            for (int J = 0; J <= I; ++J) {
                const double* Xg = Gt + tix(I, J);
                const double* Xb = Bt + tix(I, J);
                const int c0 = J * 8 + q, c1 = c0 + 4;
                const double hc0 = (c0 < md) ? h1[c0] : 0.0, hc1 = (c1 < md) ? h1[c1] : 0.0;
                sg = fma(Xg[tph(r, q)], hc0, sg);
                sg = fma(Xg[tph(r, 4 + q)], hc1, sg);
                sb = fma(Xb[tph(r, q)], hc0, sb);
                sb = fma(Xb[tph(r, 4 + q)], hc1, sb);
            }
            sg += __shfl_xor_sync(0xffffffffu, sg, 1);
            sb += __shfl_xor_sync(0xffffffffu, sb, 1);
            sg += __shfl_xor_sync(0xffffffffu, sg, 2);
            sb += __shfl_xor_sync(0xffffffffu, sb, 2);
            if (q == 0) {
                pg[I * 8 + r] = sg;
                pb[I * 8 + r] = sb;
            }
        } else {  // block column J = w - TB: sum_{I > J} X_IJ^T h_I
            const int J = w - TB;
            double tg0 = 0.0, tg1 = 0.0, tb0 = 0.0, tb1 = 0.0;
            for (int I = J + 1; I < TB; ++I) {
                const double* Xg = Gt + tix(I, J);
                const double* Xb = Bt + tix(I, J);
                const int ri = I * 8 + r;
                const double hr = (ri < md) ? h1[ri] : 0.0;
                tg0 = fma(Xg[tph(r, q)], hr, tg0);
                tg1 = fma(Xg[tph(r, 4 + q)], hr, tg1);
                tb0 = fma(Xb[tph(r, q)], hr, tb0);
                tb1 = fma(Xb[tph(r, 4 + q)], hr, tb1);
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                tg0 += __shfl_xor_sync(0xffffffffu, tg0, o);
                tg1 += __shfl_xor_sync(0xffffffffu, tg1, o);
                tb0 += __shfl_xor_sync(0xffffffffu, tb0, o);
                tb1 += __shfl_xor_sync(0xffffffffu, tb1, o);
            }
            if (r == 0) {
                cg[J * 8 + q] = tg0;
                cg[J * 8 + q + 4] = tg1;
                cb[J * 8 + q] = tb0;
                cb[J * 8 + q + 4] = tb1;
            }
        }
    }
    __syncthreads();
    // shift to full indices (i = i' + 1) and add the column part: trailing (X h)_i
    for (int ip = T.tid; ip < md; ip += T.nthr) {
        cg[ip] += pg[ip];
        cb[ip] += pb[ip];
    }
    __syncthreads();
    for (int i = T.tid; i < m; i += T.nthr) {
        pg[i] = (i == 0) ? 0.0 : cg[i - 1];
        pb[i] = (i == 0) ? 0.0 : cb[i - 1];
    }
    __syncthreads();
    // row / column 0 and the scaling: p = beta (X h) - K h
    double s0g = 0.0, s0b = 0.0;
    for (int j = T.tid; j < m; j += T.nthr) {
        s0g = fma(g0[j], h[j], s0g);
        s0b = fma(b0[j], h[j], s0b);
    }
    s0g = block_sum(T, s0g, red);
    s0b = block_sum(T, s0b, red);
    double hpg = 0.0, hpb = 0.0;
    for (int i = T.tid; i < m; i += T.nthr) {
        const double yg = (i == 0) ? s0g : fma(g0[i], h[0], pg[i]);
        const double yb = (i == 0) ? s0b : fma(b0[i], h[0], pb[i]);
        pg[i] = beta * yg;
        pb[i] = beta * yb;
        hpg += h[i] * pg[i];
        hpb += h[i] * pb[i];
    }
    const double Kg = 0.5 * beta * block_sum(T, hpg, red);
    const double Kb = 0.5 * beta * block_sum(T, hpb, red);
    for (int i = T.tid; i < m; i += T.nthr) {
        pg[i] -= Kg * h[i];
        pb[i] -= Kb * h[i];
    }
    __syncthreads();
}

// 8 x 8 diagonal factor of a swizzled tile and its inverse (diag_factor_inv_reg on tile storage;
// the inverse is stored as an Lv block, lv_idx swizzle)
__device__ __forceinline__ bool ft_diag_factor(double* D, double* rd8, double* V, int lane) {
    double a[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) a[r][c] = D[tph(r, c)];
    bool ok = true;
    double rd[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double d = a[c][c];
        if (!(d > 0.0)) ok = false;
        const double il = rsqrt(fmax(d, 1e-300));
        a[c][c] = d * il;
        rd[c] = il;
#pragma unroll
        for (int r = c + 1; r < 8; ++r) a[r][c] *= il;
#pragma unroll
        for (int k = c + 1; k < 8; ++k)
#pragma unroll
            for (int r = k; r < 8; ++r) a[r][k] = fma(-a[r][c], a[k][c], a[r][k]);
    }
    const int c = lane & 7;
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < r; ++k) acc = fma(a[r][k], x[k], acc);
        x[r] = ((r == c ? 1.0 : 0.0) - acc) * rd[r];
    }
    __syncwarp();
    if (lane < 8) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            V[lv_idx(r, c)] = (r >= c) ? x[r] : 0.0;
            if (r == lane) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k <= r) D[tph(r, k)] = a[r][k];
                rd8[r] = rd[r];
            }
        }
    }
    return ok;
}

__device__ __forceinline__ void ft_acc_ld(double (&acc)[2], const double* X, int r, int q) {
    acc[0] = X[tph(r, 2 * q)];
    acc[1] = X[tph(r, 2 * q + 1)];
}
__device__ __forceinline__ void ft_acc_st(const double (&acc)[2], double* X, int r, int q) {
    X[tph(r, 2 * q)] = acc[0];
    X[tph(r, 2 * q + 1)] = acc[1];
}

// blocked right-looking Cholesky of the tiles with a one-block lookahead (cholesky_inv_blocked_la)
__device__ bool ft_cholesky(const Team& T, double* Gt, int TB, double* rdiag, double* Lv, int* flag) {
    const int r = T.lane >> 2, q = T.lane & 3;
    if (T.warp == 0) {
        const bool ok = ft_diag_factor(Gt, rdiag, Lv, T.lane);
        if (T.lane == 0) *flag = ok ? 0 : 1;
    }
    __syncthreads();
    if (*flag) return false;
    for (int kb = 0; kb < TB; ++kb) {
        const double* Vk = Lv + kb * 64;
        for (int ib = kb + 1 + T.warp; ib < TB; ib += T.nwarps) {  // panel: L_ik = A_ik L_kk^{-T}
            double* Ct = Gt + tix(ib, kb);
            double acc[2] = {0.0, 0.0};
            dmma_t(acc, Ct[tph(r, q)], Vk[lv_idx(r, q)]);
            dmma_t(acc, Ct[tph(r, 4 + q)], Vk[lv_idx(r, 4 + q)]);
            __syncwarp();
            ft_acc_st(acc, Ct, r, q);
        }
        __syncthreads();
        const int Tr = TB - kb - 1;
        if (Tr == 0) break;
        if (T.warp == 0) {
            double* C = Gt + tix(kb + 1, kb + 1);
            const double* Pk = Gt + tix(kb + 1, kb);
            double acc[2];
            ft_acc_ld(acc, C, r, q);
            dmma_t(acc, -Pk[tph(r, q)], Pk[tph(r, q)]);
            dmma_t(acc, -Pk[tph(r, 4 + q)], Pk[tph(r, 4 + q)]);
            ft_acc_st(acc, C, r, q);
            __syncwarp();
            const bool ok = ft_diag_factor(C, rdiag + (kb + 1) * 8, Lv + (kb + 1) * 64, T.lane);
            if (T.lane == 0) *flag = ok ? 0 : 1;
        } else {
            int ii = 0, jj = 0, t = T.warp;
            while (ii < Tr && jj + t > ii) { t -= ii + 1 - jj; jj = 0; ++ii; }
            jj += t;
            while (ii < Tr) {
                const int ib = kb + 1 + ii, jb = kb + 1 + jj;
                double* C = Gt + tix(ib, jb);
                const double* Pi = Gt + tix(ib, kb);
                const double* Pj = Gt + tix(jb, kb);
                double acc[2];
                ft_acc_ld(acc, C, r, q);
                dmma_t(acc, -Pi[tph(r, q)], Pj[tph(r, q)]);
                dmma_t(acc, -Pi[tph(r, 4 + q)], Pj[tph(r, 4 + q)]);
                ft_acc_st(acc, C, r, q);
                jj += T.nwarps - 1;
                while (ii < Tr && jj > ii) { jj -= ii + 1; ++ii; }
            }
        }
        __syncthreads();
        if (*flag) return false;
    }
    return true;
}

// W = L^{-1} in place (right to left over the block columns): W_jj = L_jj^{-1} (the Lv blocks),
// W_ij = -(sum_{k=j+1..i} W_ik L_kj) L_jj^{-1}.  A column's tiles are formed from the original
// column of L before any of them is stored (barrier between).
__device__ void ft_trtri(const Team& T, double* Gt, int TB, const double* Lv, double (*stash)[2]) {
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int j = T.warp; j < TB; j += T.nwarps) {  // W_jj
        double* D = Gt + tix(j, j);
        for (int e = T.lane; e < 64; e += 32) D[tph(e >> 3, e & 7)] = Lv[j * 64 + lv_idx(e >> 3, e & 7)];
    }
    __syncthreads();
    for (int j = TB - 2; j >= 0; --j) {
        const double* Vj = Lv + j * 64;
        int slot = 0;
        for (int i = j + 1 + T.warp; i < TB; i += T.nwarps, ++slot) {
            double acc[2] = {0.0, 0.0};
            for (int k = j + 1; k <= i; ++k) {
                const double* Wik = Gt + tix(i, k);
                const double* Lkj = Gt + tix(k, j);
                // acc += W_ik L_kj: A = W_ik (r, q / 4+q), B[k'][n] = L_kj[k'][n] (lane: (q, r) / (4+q, r))
                dmma_t(acc, Wik[tph(r, q)], Lkj[tph(q, r)]);
                dmma_t(acc, Wik[tph(r, 4 + q)], Lkj[tph(4 + q, r)]);
            }
            // W_ij = -acc L_jj^{-1}: the accumulator is the A operand with k over (2q, 2q+1)
            double w[2] = {0.0, 0.0};
            dmma_t(w, -acc[0], Vj[lv_idx(2 * q, r)]);
            dmma_t(w, -acc[1], Vj[lv_idx(2 * q + 1, r)]);
            stash[slot][0] = w[0];
            stash[slot][1] = w[1];
        }
        __syncthreads();
        slot = 0;
        for (int i = j + 1 + T.warp; i < TB; i += T.nwarps, ++slot) {
            const double w[2] = {stash[slot][0], stash[slot][1]};
            ft_acc_st(w, Gt + tix(i, j), r, q);
        }
        __syncthreads();
    }
}

// M = -W B W^T into the slot's rows (ld), one warp per 8-column panel J
__device__ void ft_congruence(const Team& T, const double* Wt, const double* Bt, int TB, double* Mw, int ld,
                              double* scratch) {
    const int r = T.lane >> 2, q = T.lane & 3;
    double* sc = scratch + T.warp * 64;
    for (int J = T.warp; J < TB; J += T.nwarps) {
        double yt[FT_TBMAX][2];
#pragma unroll
        for (int K = 0; K < FT_TBMAX; ++K) yt[K][0] = yt[K][1] = 0.0;
        // Y^T_JK = sum_{L <= J} W_JL B_LK: one W fragment feeds 13 independent accumulators
        for (int L = 0; L <= J; ++L) {
            const double* Wl = Wt + tix(J, L);
            const double a0 = Wl[tph(r, q)], a1 = Wl[tph(r, 4 + q)];
#pragma unroll
            for (int K = 0; K < FT_TBMAX; ++K) {
                if (K < TB) {
                    double b0, b1;
                    if (L >= K) {  // B_LK stored: element (q, r) / (4+q, r)
                        const double* Bl = Bt + tix(L, K);
                        b0 = Bl[tph(q, r)];
                        b1 = Bl[tph(4 + q, r)];
                    } else {  // B_LK = B_KL^T: element (r, q) / (r, 4+q) of B_KL
                        const double* Bl = Bt + tix(K, L);
                        b0 = Bl[tph(r, q)];
                        b1 = Bl[tph(r, 4 + q)];
                    }
                    dmma_t(yt[K], a0, b0);
                    dmma_t(yt[K], a1, b1);
                }
            }
        }
        // M_IJ = -sum_{K <= I} W_IK Y_KJ, two output tiles at a time (independent chains)
        for (int I0 = J; I0 < TB; I0 += 2) {
            double accs[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
            const bool two = (I0 + 1 < TB);
#pragma unroll
            for (int K = 0; K < FT_TBMAX; ++K) {
                if (K <= I0) {
                    const double* Wk = Wt + tix(I0, K);
                    dmma_t(accs[0], -Wk[tph(r, 2 * q)], yt[K][0]);
                    dmma_t(accs[0], -Wk[tph(r, 2 * q + 1)], yt[K][1]);
                }
                if (two && K <= I0 + 1) {
                    const double* Wk = Wt + tix(I0 + 1, K);
                    dmma_t(accs[1], -Wk[tph(r, 2 * q)], yt[K][0]);
                    dmma_t(accs[1], -Wk[tph(r, 2 * q + 1)], yt[K][1]);
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
            const int I = I0 + u;
            if (I >= TB) break;
            const double* acc = accs[u];
            double* row = Mw + (size_t)(I * 8 + r) * ld + J * 8 + 2 * q;
            if (I > J) {
                *reinterpret_cast<double2*>(row) = make_double2(acc[0], acc[1]);
                Mw[(size_t)(J * 8 + 2 * q) * ld + I * 8 + r] = acc[0];
                Mw[(size_t)(J * 8 + 2 * q + 1) * ld + I * 8 + r] = acc[1];
            } else {  // diagonal tile: (M + M^T) / 2 through the warp's scratch
                sc[r * 8 + 2 * q] = acc[0];
                sc[r * 8 + 2 * q + 1] = acc[1];
                __syncwarp();
                const double m0 = 0.5 * (acc[0] + sc[(2 * q) * 8 + r]);
                const double m1 = 0.5 * (acc[1] + sc[(2 * q + 1) * 8 + r]);
                __syncwarp();
                *reinterpret_cast<double2*>(row) = make_double2(m0, m1);
            }
            }
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(FT_NT, 2) factor_t_kernel(ChordParams P) {
    extern __shared__ __align__(16) double smem_dyn[];
    Team T;
    T.tid = threadIdx.x;
    T.nthr = FT_NT;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = FT_NT >> 5;
    __shared__ double red[64];
    __shared__ int sh_i[8];
    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    const int TBmax = mp >> 3;
    const int ntmax = TBmax * (TBmax + 1) / 2 * 64;
    double* Gt = smem_dyn;
    double* Bt = Gt + ntmax;
    double* Lv = Bt + ntmax;
    double* vec = Lv + TBmax * 64;
    double* uu = vec + 0 * vl;
    double* hh = vec + 1 * vl;
    double* pw = vec + 2 * vl;
    double* rdiag = vec + 3 * vl;
    double* yy = vec + 4 * vl;
    double* bv = vec + 5 * vl;
    double* g0 = vec + 6 * vl;
    double* b0 = vec + 7 * vl;
    double* scratch = vec + 8 * vl;  // 8 warps x 64
    double stash[2][2];

    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        if (P.mode == 0 && (P.flags[slot] & CF_DONE)) continue;
        const double* av = P.AV + (size_t)slot * P.mtp;
        const double* ax = P.AX + (size_t)slot * P.mtp;
        double* S = P.wS + (size_t)slot * P.w_sstride;
        double* Mw = P.wM + (size_t)slot * P.w_mstride;
        double* Lw = P.wL + (size_t)slot * P.w_mstride;
        const int bnd = P.bound[slot];
        const bool defl = (bnd == 0);
        const int o = defl ? 1 : 0;
        const int md = m - o;
        const int mdp = (md + 7) & ~7;
        const int TB = mdp >> 3;
        __syncthreads();
        long long t_prof = clock64();
        ft_unpack(T, ax, Gt, m, o, mdp, 1.0, g0);
        ft_unpack(T, av, Bt, m, o, mdp, 0.0, b0);
        if (defl)
            for (int i = T.tid; i < m; i += T.nthr) uu[i] = P.U[(size_t)slot * m + i];
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
        PROF_MARK(0);
        double a_schur = 0.0, beta_h = 0.0;
        bool outward = false;
        if (defl) {
            double nu = 0.0;
            for (int i = T.tid; i < m; i += T.nthr) nu += uu[i] * uu[i];
            nu = sqrt(block_sum(T, nu, red));
            for (int i = T.tid; i < m; i += T.nthr) hh[i] = uu[i] / nu;
            __syncthreads();
            if (T.tid == 0) hh[0] += (hh[0] >= 0.0 ? 1.0 : -1.0);
            __syncthreads();
            double h2 = 0.0;
            for (int i = T.tid; i < m; i += T.nthr) h2 += hh[i] * hh[i];
            beta_h = 2.0 / block_sum(T, h2, red);
            ft_householder_vecs(T, Gt, Bt, g0, b0, m, md, TB, hh, beta_h, pw, yy, rdiag, bv, red);
            a_schur = b0[0] - (hh[0] * yy[0] + yy[0] * hh[0]);
            outward = !(a_schur > 0.0);
            for (int i = T.tid; i + 1 < m; i += T.nthr) bv[i] = b0[i + 1] - (hh[i + 1] * yy[0] + yy[i + 1] * hh[0]);
            __syncthreads();
            // trailing blocks (index i' = i - 1): G' = G - h p^T - p h^T; B'' = B' - b b^T / a (warp per
            // tile; diagonal tiles hold both triangles)
            {
                const int r = T.lane >> 2, q = T.lane & 3;
                const int ntile = TB * (TB + 1) / 2;
                for (int t = T.warp; t < ntile; t += T.nwarps) {
                    int ib, jb;
                    tile_of(t, ib, jb);
                    const int ip = ib * 8 + r;
                    if (ip >= md) continue;
                    const double hi = hh[ip + 1], pgi = pw[ip + 1], pbi = yy[ip + 1], bvi = bv[ip];
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        const int c = q + 4 * hf, jp = jb * 8 + c;
                        if (jp >= md) continue;
                        const int x = tix(ib, jb) + tph(r, c);
                        const double hj = hh[jp + 1];
                        Gt[x] -= hi * pw[jp + 1] + pgi * hj;
                        const double bij = Bt[x] - (hi * yy[jp + 1] + pbi * hj);
                        Bt[x] = outward ? 0.0 : bij - bvi * bv[jp] / a_schur;
                    }
                }
            }
            __syncthreads();
        }
        PROF_MARK(1);
        int status = (defl ? ST_DEFL : 0) | (outward ? ST_OUTWARD : 0);
        if (!outward && md >= 1) {
            const bool okc = ft_cholesky(T, Gt, TB, rdiag, Lv, &sh_i[2]);
            PROF_MARK(2);
            if (!okc) {
                status |= ST_FAILED;
            } else {
                // packed lower rows of L for the tail kernel
                const int r = T.lane >> 2, q = T.lane & 3;
                const int ntile = TB * (TB + 1) / 2;
                for (int t = T.warp; t < ntile; t += T.nwarps) {
                    int ib, jb;
                    tile_of(t, ib, jb);
                    const int i = ib * 8 + r;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = jb * 8 + q + 4 * h;
                        if (j <= i) Lw[pk(i, j)] = Gt[tix(ib, jb) + tph(r, q + 4 * h)];
                    }
                }
                __syncthreads();
                ft_trtri(T, Gt, TB, Lv, stash);
                PROF_MARK(3);
                ft_congruence(T, Gt, Bt, TB, Mw, ld, scratch);
            }
        }
        if (T.tid == 0) {
            S[S_A] = a_schur;
            S[S_BH] = beta_h;
            S[S_MD] = (double)md;
            S[S_ST] = (double)status;
        }
        for (int i = T.tid; i < mp; i += T.nthr) {
            S[S_VEC + i] = hh[i];
            S[S_VEC + vl + i] = bv[i];
            S[S_VEC + 2 * vl + i] = rdiag[i];
        }
        PROF_MARK(4);
    }
}

}  // namespace sw
