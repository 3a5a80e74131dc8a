// factor_g.cuh -- K2a for 104 < mp <= 208 (configs[4], m = 200): factor_t_kernel's tile algorithm with
// A(x) -- G, then L, then W = L^{-1} -- as the lower triangle of 8 x 8 tiles in ONE CTA's shared
// memory (325 tiles = 166 KB at m = 200) and A(v) = B as the same tiles in the CTA's global scratch
// slice (L2 resident: 148 x 166 KB).
//
// Same mathematics as the global-scratch factor phase (L L^T = A(x),
// M = -L^{-1} A(v) L^{-T}; the Schur deflation of a boundary start, R6): the Cholesky and
// the triangular inverse never leave shared memory, and the congruence M = -W B W^T reads every
// B tile from L2 straight into DMMA B fragments (Y^T_J = W_J: B in 2 x TBM register accumulators per
// 8-column panel J, then M_IJ = -sum_K W_IK Y_KJ with the accumulators as the B operands); the
// fragment loads run one batch of FG_KCH tiles ahead of the DMMAs (two register buffers).
// Panels are handed to the warps from a shared counter in order of decreasing cost (each panel's
// arithmetic is self-contained and ordered, so the result does not depend on the assignment).
// Outputs as the gsplit-2 factor phase: M as row-major lower 8 x 8 tiles (lanczos_t_kernel's
// layout), packed L, the deflation vectors and status in the slot's scalar area.
#pragma once
#include "factor_t.cuh"

namespace sw {

constexpr int FG_TBMAX = 26;  // mdp <= 208
#ifndef SW_FG_PIPE
#define SW_FG_PIPE 1  // software-pipelined B-fragment loads in the congruence (0: one batch at a time)
#endif
#ifndef SW_FG_S2W
#define SW_FG_S2W 2
#endif
#ifndef SW_FG_KCH
#define SW_FG_KCH 5
#endif
constexpr int FG_S2W = SW_FG_S2W;  // output tiles per step of the congruence's second stage
constexpr int FG_KCH = SW_FG_KCH;  // B tiles per load batch of the congruence (unpipelined 7: K2a 116.2 ms, 9: 114.0 ms per m = 200 round; pipelined 5: 104.4 ms)

__host__ __device__ inline size_t fg_smem_doubles(int mp, int nwarps) {
    const int TB = mp >> 3;
    return (size_t)TB * (TB + 1) / 2 * 64 + (size_t)TB * 64 + 8 * (size_t)(mp + 8) + (size_t)nwarps * 64;
}
__host__ __device__ inline size_t fg_scratch_doubles(int mp) {
    const int TB = mp >> 3;
    return (size_t)TB * (TB + 1) / 2 * 64;
}

// next lower tile (ib, jb) `step` tiles further in row-major order over the lower tiles
__device__ __forceinline__ void fg_tile_adv(int& ib, int& jb, int step) {
    jb += step;
    while (jb > ib) {
        jb -= ib + 1;
        ++ib;
    }
}

// ft_unpack for either memory: shared tiles by 8-byte cp.async; global tiles by plain loads and
// stores, four tiles per warp step so that eight loads are in flight per lane
template <bool SH>
__device__ void fg_unpack(const Team& T, const double* __restrict__ P, double* Tm, int m, int o, int mdp, double pad,
                          double* row0) {
    const int TB = mdp >> 3, md = m - o;
    const int r = T.lane >> 2, q = T.lane & 3;
    constexpr int U = SH ? 1 : 4;
    int ib = 0, jb = 0;
    fg_tile_adv(ib, jb, T.warp * U);
    while (ib < TB) {
        double val[U][2];
        double* dst[U][2];
        bool live[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = ib * 8 + r;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = q + 4 * h, j = jb * 8 + c;
                live[u][h] = (ib < TB);
                dst[u][h] = Tm + tix(ib, jb) + tph(r, c);
                val[u][h] = (i == j) ? pad : 0.0;
                if (ib < TB && i < md && j < md) {
                    const int gi = i + o, gj = j + o;
                    const double* src = P + ((gj <= gi) ? pk(gi, gj) : pk(gj, gi));
                    if (SH) {
                        cp_async8(dst[u][h], src);
                        live[u][h] = false;
                    } else {
                        val[u][h] = *src;
                    }
                }
            }
            fg_tile_adv(ib, jb, (u + 1 < U) ? 1 : (T.nwarps - 1) * U + 1);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (live[u][h]) *dst[u][h] = val[u][h];
    }
    if (o)
        for (int j = T.tid; j < m; j += T.nthr) row0[j] = P[pk(j, 0)];
}

// ft_trtri with SL register stash slots per warp (SL * nwarps >= TB - 1)
template <int SL>
__device__ void fg_trtri(const Team& T, double* Gt, int TB, const double* Lv) {
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int j = T.warp; j < TB; j += T.nwarps) {  // W_jj
        double* D = Gt + tix(j, j);
        for (int e = T.lane; e < 64; e += 32) D[tph(e >> 3, e & 7)] = Lv[j * 64 + lv_idx(e >> 3, e & 7)];
    }
    __syncthreads();
    for (int j = TB - 2; j >= 0; --j) {
        const double* Vj = Lv + j * 64;
        double st[SL][2];
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            const int i = j + 1 + T.warp + s * T.nwarps;
            st[s][0] = st[s][1] = 0.0;
            if (i < TB) {
                double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};
                int k = j + 1;
                for (; k + 1 <= i; k += 2) {  // two independent DMMA chains
                    const double* Wik = Gt + tix(i, k);
                    const double* Lkj = Gt + tix(k, j);
                    const double* Wik2 = Gt + tix(i, k + 1);
                    const double* Lkj2 = Gt + tix(k + 1, j);
                    dmma_t(acc, Wik[tph(r, q)], Lkj[tph(q, r)]);
                    dmma_t(acc2, Wik2[tph(r, q)], Lkj2[tph(q, r)]);
                    dmma_t(acc, Wik[tph(r, 4 + q)], Lkj[tph(4 + q, r)]);
                    dmma_t(acc2, Wik2[tph(r, 4 + q)], Lkj2[tph(4 + q, r)]);
                }
                if (k <= i) {
                    const double* Wik = Gt + tix(i, k);
                    const double* Lkj = Gt + tix(k, j);
                    dmma_t(acc, Wik[tph(r, q)], Lkj[tph(q, r)]);
                    dmma_t(acc, Wik[tph(r, 4 + q)], Lkj[tph(4 + q, r)]);
                }
                acc[0] += acc2[0];
                acc[1] += acc2[1];
                // W_ij = -acc L_jj^{-1}: the accumulator is the A operand with k over (2q, 2q+1)
                dmma_t(st[s], -acc[0], Vj[lv_idx(2 * q, r)]);
                dmma_t(st[s], -acc[1], Vj[lv_idx(2 * q + 1, r)]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            const int i = j + 1 + T.warp + s * T.nwarps;
            if (i < TB) ft_acc_st(st[s], Gt + tix(i, j), r, q);
        }
        __syncthreads();
    }
}

// M = -W B W^T as row-major lower 8 x 8 tiles at Mw + 64 (I (I + 1) / 2 + J); W in shared memory,
// B in global memory (both swizzled lower tiles); panels from the shared counter *ctr (zeroed by
// the caller before a barrier), most expensive (J = TB - 1) first
__device__ void fg_congruence(const Team& T, const double* Wt, const double* Bt, int TB, double* Mw, double* scratch,
                              int* ctr) {
    const int r = T.lane >> 2, q = T.lane & 3;
    double* sc = scratch + T.warp * 64;
    for (;;) {
        int t = 0;
        if (T.lane == 0) t = atomicAdd(ctr, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= TB) break;
        const int J = TB - 1 - t;
        double yt[FG_TBMAX][2];
#pragma unroll
        for (int K = 0; K < FG_TBMAX; ++K) yt[K][0] = yt[K][1] = 0.0;
        // Y^T_JK = sum_{L <= J} W_JL B_LK: one W fragment feeds TB independent accumulators.  The B
        // fragments come from L2 in branch-free batches of FG_KCH tiles (all loads of a batch in
        // flight before its DMMAs): B_LK is the stored tile (L, K), element (q, r) / (4+q, r), for
        // K <= L and the transpose of tile (K, L), element (r, q) / (r, 4+q), for K > L; K >= TB
        // reads tile (TB - 1, .) again and feeds accumulators that are never used
        const int os0 = tph(q, r), os1 = tph(4 + q, r), ot0 = tph(r, q), ot1 = tph(r, 4 + q);
#if SW_FG_PIPE
        // software pipeline over the (L, batch) sequence: the loads of the next batch are issued
        // before the DMMAs of the current one (two register buffers; FG_NCH is even, so the buffer
        // of batch c is c & 1 for every L)
        constexpr int FG_NCH = (FG_TBMAX + FG_KCH - 1) / FG_KCH;
        static_assert(FG_NCH % 2 == 0, "FG_NCH must be even");
        double b[2][FG_KCH][2];
        auto load_batch = [&](int L, int c, double (&bb)[FG_KCH][2]) {
            const double* Brow = Bt + tix(L, 0);
#pragma unroll
            for (int u = 0; u < FG_KCH; ++u) {
                const int K = c * FG_KCH + u;
                if (K < FG_TBMAX) {
                    const bool st = (L >= K);
                    const int Kc = (K < TB) ? K : TB - 1;
                    const double* Bl = st ? Brow + K * 64 : Bt + tix(Kc, L);
                    bb[u][0] = Bl[st ? os0 : ot0];
                    bb[u][1] = Bl[st ? os1 : ot1];
                }
            }
        };
        load_batch(0, 0, b[0]);
        for (int L = 0; L <= J; ++L) {
            const double* Wl = Wt + tix(J, L);
            const double a0 = Wl[tph(r, q)], a1 = Wl[tph(r, 4 + q)];
#pragma unroll
            for (int c = 0; c < FG_NCH; ++c) {
                if (c + 1 < FG_NCH)
                    load_batch(L, c + 1, b[(c + 1) & 1]);
                else if (L < J)
                    load_batch(L + 1, 0, b[0]);
#pragma unroll
                for (int u = 0; u < FG_KCH; ++u) {
                    const int K = c * FG_KCH + u;
                    if (K < FG_TBMAX) {
                        dmma_t(yt[K], a0, b[c & 1][u][0]);
                        dmma_t(yt[K], a1, b[c & 1][u][1]);
                    }
                }
            }
        }
#else
        for (int L = 0; L <= J; ++L) {
            const double* Wl = Wt + tix(J, L);
            const double a0 = Wl[tph(r, q)], a1 = Wl[tph(r, 4 + q)];
            const double* Brow = Bt + tix(L, 0);  // tiles (L, K), K <= L
#pragma unroll
            for (int K0 = 0; K0 < FG_TBMAX; K0 += FG_KCH) {
                double b[FG_KCH][2];
#pragma unroll
                for (int u = 0; u < FG_KCH; ++u) {
                    const int K = K0 + u;
                    if (K < FG_TBMAX) {
                        const bool st = (L >= K);
                        const int Kc = (K < TB) ? K : TB - 1;
                        const double* Bl = st ? Brow + K * 64 : Bt + tix(Kc, L);
                        b[u][0] = Bl[st ? os0 : ot0];
                        b[u][1] = Bl[st ? os1 : ot1];
                    }
                }
#pragma unroll
                for (int u = 0; u < FG_KCH; ++u) {
                    const int K = K0 + u;
                    if (K < FG_TBMAX) {
                        dmma_t(yt[K], a0, b[u][0]);
                        dmma_t(yt[K], a1, b[u][1]);
                    }
                }
            }
        }
#endif
        // M_IJ = -sum_{K <= I} W_IK Y_KJ, FG_S2W output tiles at a time (independent chains)
        for (int I0 = J; I0 < TB; I0 += FG_S2W) {
            double accs[FG_S2W][2];
            const double* Wr[FG_S2W];
#pragma unroll
            for (int u = 0; u < FG_S2W; ++u) {
                accs[u][0] = accs[u][1] = 0.0;
                Wr[u] = Wt + tix((I0 + u < TB) ? I0 + u : I0, 0);
            }
#pragma unroll
            for (int K = 0; K < FG_TBMAX; ++K) {
#pragma unroll
                for (int u = 0; u < FG_S2W; ++u) {
                    if (I0 + u < TB && K <= I0 + u) {
                        const double* Wk = Wr[u] + K * 64;
                        dmma_t(accs[u], -Wk[tph(r, 2 * q)], yt[K][0]);
                        dmma_t(accs[u], -Wk[tph(r, 2 * q + 1)], yt[K][1]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < FG_S2W; ++u) {
                const int I = I0 + u;
                if (I >= TB) break;
                const double* acc = accs[u];
                double* Mt = Mw + 64 * (size_t)(I * (I + 1) / 2 + J) + r * 8 + 2 * q;
                if (I > J) {
                    *reinterpret_cast<double2*>(Mt) = make_double2(acc[0], acc[1]);
                } else {  // diagonal tile: (M + M^T) / 2 through the warp's scratch
                    sc[r * 8 + 2 * q] = acc[0];
                    sc[r * 8 + 2 * q + 1] = acc[1];
                    __syncwarp();
                    const double m0 = 0.5 * (acc[0] + sc[(2 * q) * 8 + r]);
                    const double m1 = 0.5 * (acc[1] + sc[(2 * q + 1) * 8 + r]);
                    __syncwarp();
                    *reinterpret_cast<double2*>(Mt) = make_double2(m0, m1);
                }
            }
        }
    }
    __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) factor_g_kernel(ChordParams P) {
    extern __shared__ __align__(16) double smem_dyn[];
    Team T;
    T.tid = threadIdx.x;
    T.nthr = NT;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = NT >> 5;
    constexpr int SL = (FG_TBMAX - 1 + (NT >> 5) - 1) / (NT >> 5);
    __shared__ double red[64];
    __shared__ int sh_i[8];
    const int m = P.m;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    const int TBmax = mp >> 3;
    const int ntmax = TBmax * (TBmax + 1) / 2 * 64;
    double* Gt = smem_dyn;
    double* Lv = Gt + ntmax;
    double* vec = Lv + TBmax * 64;
    double* uu = vec + 0 * vl;
    double* hh = vec + 1 * vl;
    double* pw = vec + 2 * vl;
    double* rdiag = vec + 3 * vl;
    double* yy = vec + 4 * vl;
    double* bv = vec + 5 * vl;
    double* g0 = vec + 6 * vl;
    double* b0 = vec + 7 * vl;
    double* scratch = vec + 8 * vl;  // nwarps x 64
    double* Bt = P.scratch + (size_t)blockIdx.x * P.scratch_stride;

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
        fg_unpack<true>(T, ax, Gt, m, o, mdp, 1.0, g0);
        fg_unpack<false>(T, av, Bt, m, o, mdp, 0.0, b0);
        if (defl)
            for (int i = T.tid; i < m; i += T.nthr) uu[i] = P.U[(size_t)slot * m + i];
        if (T.tid == 0) sh_i[3] = 0;  // the congruence's panel counter
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
                int ib = 0, jb = 0;
                fg_tile_adv(ib, jb, T.warp);
                for (; ib < TB; fg_tile_adv(ib, jb, T.nwarps)) {
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
                int ib = 0, jb = 0;
                fg_tile_adv(ib, jb, T.warp);
                for (; ib < TB; fg_tile_adv(ib, jb, T.nwarps)) {
                    const int i = ib * 8 + r;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = jb * 8 + q + 4 * h;
                        if (j <= i) Lw[pk(i, j)] = Gt[tix(ib, jb) + tph(r, q + 4 * h)];
                    }
                }
                __syncthreads();
                fg_trtri<SL>(T, Gt, TB, Lv);
                PROF_MARK(3);
                fg_congruence(T, Gt, Bt, TB, Mw, scratch, &sh_i[3]);
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
