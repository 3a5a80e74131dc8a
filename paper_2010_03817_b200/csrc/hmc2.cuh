// hmc2.cuh -- K5 split for m <= 128: the reflective-HMC chord of hmc.cuh
// (Alg. 6, eq:boltz_ode P:1440-1446; SURVEY a-10) as
//
//   K5s hmc_setup_kernel     per chain: Weyl state s = 0; after a dense reflection the
//                            Householder vector h of the kernel u and the rank-2 terms
//                            q_k of H A_k H = A_k - h q_k^T - q_k h^T (k = A(p), A(v), A(c))
//   per Weyl iteration, over the chains still stepping (compacted lists):
//     K5a hmc_factor_kernel  G~(s) -> K K^T (blocked Cholesky, DMMA); N~_k = K^{-1} C_k K^{-T}
//                            (two TRSMs per dense C_k, two vector solves for the rank-2 border
//                            terms of the quartic); N_j = sum_k binom(k, j) s^{k-j} N~_k;
//                            -N_1 to the Lanczos buffer, |N_j|_F (j >= 2), K to the L buffer
//     K2b lanczos_kernel     lambda_min(N_1) = -theta_max(-N_1) and its Ritz vector z
//     K5b hmc_weyl_kernel    h = first root of 1 + a h - sum_j |N_j|_F h^j; s += h; stop
//                            when h <= 1e-15 s (or 60 iterations); else to the next list
//   K5c hmc_tail_kernel      y = K^{-T} z, the boundary back-transform y = H D y~, then
//                            the cube faces, selection, advance and step logic (hmc_finish)
//
// The arithmetic is hmc_kernel's (monotone Weyl stepping on the quadratic pencil /
// sqrt(t)-deflated quartic) up to the order of the congruences: hmc_kernel forms
// D_j = sum_k binom(k, j) s^{k-j} C_k first and congruences each D_j; here each C_k is
// congruenced once and the N_j are combined afterwards (same matrices up to rounding),
// and the border terms C_1, C_3 of the quartic are rank 2 (e_0 b^T + b e_0^T), so their
// congruences are p q^T + q p^T with p = K^{-1} e_0, q = K^{-1} b: two TRSM pairs per
// iteration instead of four.  The split gives each phase the whole SM (the fused K5
// ran every phase on a global scratch slice with the unblocked Lanczos).
#pragma once
#include "hmc.cuh"
#include "chord3.cuh"

namespace sw {

// per-slot Weyl state (P.wH, H_NS doubles per slot)
enum : int { H_S = 0, H_D = 1, H_IT = 2, H_ST = 3, H_C2 = 4, H_C3 = 5, H_C4 = 6, H_BH = 7, H_NS = 8 };
enum : int { HS_ITER = 0, HS_HIT = 1, HS_FAILED = 2, HS_INF = 3, HS_OUTWARD = 4, HS_CAPPED = 5 };

// X_w <- L^{-1} X_w for nv vectors (stride vl) with L lower in G and the inverse 8 x 8
// diagonal blocks Lv (cholesky_inv_blocked_la): one warp per vector, left-looking over
// 8-row blocks (lane = 4 r + q: row k0 + r, columns q mod 4 of the off-diagonal part).
__device__ void fwd_solve_vecs(const Team& T, const double* G, const double* Lv, double* X, int nv, int vl, int n,
                               int ld) {
    const int TB = n >> 3;
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int w = T.warp; w < nv; w += T.nwarps) {
        double* x = X + w * vl;
        for (int kb = 0; kb < TB; ++kb) {
            const int k0 = kb * 8;
            const double* Li = G + (k0 + r) * ld;
            double a0 = 0.0, a1 = 0.0;
            int c = q;
            for (; c + 4 < k0; c += 8) {
                a0 = fma(Li[c], x[c], a0);
                a1 = fma(Li[c + 4], x[c + 4], a1);
            }
            if (c < k0) a0 = fma(Li[c], x[c], a0);
            double acc = a0 + a1;
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            const double ri = x[k0 + r] - acc;
            const double r0 = __shfl_sync(0xffffffffu, ri, 8 * q);
            const double r1 = __shfl_sync(0xffffffffu, ri, 8 * q + 4);
            const double* V = Lv + kb * 64;
            double part = fma(V[lv_idx(r, 2 * q)], r0, V[lv_idx(r, 2 * q + 1)] * r1);
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            __syncwarp();
            if (q == 0) x[k0 + r] = part;
            __syncwarp();
        }
    }
}

// (H A H)(i, j) = a - (h_i q_j + q_i h_j), the arithmetic of householder_congruence
__device__ __forceinline__ double hconj(double a, const double* h, const double* qv, int i, int j) {
    return a - (h[i] * qv[j] + qv[i] * h[j]);
}

// ---------------------------------------------------------------- K5s
template <int NT>
__global__ void __launch_bounds__(NT) hmc_setup_kernel(ChordParams P) {
    Team T;
    T.tid = threadIdx.x;
    T.nthr = NT;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = NT >> 5;
    __shared__ double red[64];
    __shared__ double hs[128];
    __shared__ double ps[128];
    const int m = P.m;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        if (P.mode == 0 && (P.flags[slot] & CF_DONE)) continue;
        double* H = P.wH + (size_t)slot * H_NS;
        const int bnd = P.bound[slot];
        __syncthreads();
        int state = HS_ITER;
        if (bnd == 0) {
            double* S = P.wS + (size_t)slot * P.w_sstride;
            double* Qv = P.wQ + (size_t)slot * 3 * vl;
            double nu = 0.0;
            for (int i = T.tid; i < m; i += NT) {
                const double u = P.U[(size_t)slot * m + i];
                hs[i] = u;
                nu += u * u;
            }
            nu = sqrt(block_sum(T, nu, red));
            for (int i = T.tid; i < m; i += NT) hs[i] /= nu;
            __syncthreads();
            if (T.tid == 0) hs[0] += (hs[0] >= 0.0 ? 1.0 : -1.0);
            __syncthreads();
            double h2 = 0.0;
            for (int i = T.tid; i < m; i += NT) h2 += hs[i] * hs[i];
            const double beta_h = 2.0 / block_sum(T, h2, red);
            for (int i = T.tid; i < mp; i += NT) S[S_VEC + i] = (i < m) ? hs[i] : 0.0;
            for (int k = 0; k < 3; ++k) {
                const double* A = (k == 0) ? (const double*)(P.AX + (size_t)slot * P.mtp)
                                           : (k == 1) ? P.AV + (size_t)slot * P.mtp : P.Ac;
                // p = beta A h (A symmetric, packed lower), one warp per row
                for (int i = T.warp; i < m; i += T.nwarps) {
                    double s = 0.0;
                    for (int j = T.lane; j < m; j += 32) s += A[j <= i ? pk(i, j) : pk(j, i)] * hs[j];
                    s = warp_sum(s);
                    if (T.lane == 0) ps[i] = beta_h * s;
                }
                __syncthreads();
                double hp = 0.0;
                for (int i = T.tid; i < m; i += NT) hp += hs[i] * ps[i];
                const double Kc = 0.5 * beta_h * block_sum(T, hp, red);
                for (int i = T.tid; i < mp; i += NT) Qv[k * vl + i] = (i < m) ? ps[i] - Kc * hs[i] : 0.0;
                if (k == 1 && T.tid == 0) {
                    const double q0 = ps[0] - Kc * hs[0];
                    const double a1 = A[0] - (hs[0] * q0 + q0 * hs[0]);  // (H A(v) H)_00
                    red[40] = a1;
                }
                __syncthreads();
            }
            if (!(red[40] > 0.0)) state = HS_OUTWARD;
            if (T.tid == 0) H[H_BH] = beta_h;
        }
        if (T.tid == 0) {
            H[H_S] = 0.0;
            H[H_D] = (bnd == 0) ? 4.0 : 2.0;
            H[H_IT] = 0.0;
            H[H_ST] = (double)state;
            if (state == HS_ITER) {
                const int q = atomicAdd(P.nxt_count, 1);
                P.nxt_list[q] = slot;
            }
        }
    }
}

// ---------------------------------------------------------------- K5a
template <int NT>
__global__ void __launch_bounds__(NT, 1) hmc_factor_kernel(ChordParams P) {
    extern __shared__ __align__(16) double smem_dyn[];
    Team T;
    T.tid = threadIdx.x;
    T.nthr = NT;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = NT >> 5;
    __shared__ double red[64];
    __shared__ int sh_i[8];
    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    double* G = smem_dyn;
    double* B = G + (size_t)mp * ld;
    double* vec = B + (size_t)mp * ld;
    double* hh = vec + 0 * vl;
    double* q0 = vec + 1 * vl;  // q_0, q_1, q_2 consecutive
    double* rdiag = vec + 4 * vl;
    double* X = vec + 5 * vl;    // e_0, b_1, b_3 -> p, q1, q3 (3 slots)
    double* Lv = vec + 8 * vl;   // inverse diagonal blocks (8 mp)
    const double c2s = -0.5 / P.Temp;

    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        double* H = P.wH + (size_t)slot * H_NS;
        double* S = P.wS + (size_t)slot * P.w_sstride;
        __syncthreads();
        const double s = H[H_S];
        const int d = (int)H[H_D];
        const int it = (int)H[H_IT];
        const double t = s * s;
        const double* ax = P.AX + (size_t)slot * P.mtp;
        const double* av = P.AV + (size_t)slot * P.mtp;
        const double* ac = P.Ac;
        long long t_prof = clock64();
        if (d == 4) {
            const double* Qs = P.wQ + (size_t)slot * 3 * vl;
            for (int i = T.tid; i < mp; i += NT) {
                hh[i] = S[S_VEC + i];
                q0[i] = Qs[i];
                q0[vl + i] = Qs[vl + i];
                q0[2 * vl + i] = Qs[2 * vl + i];
            }
            __syncthreads();
        }
        const double* q1 = q0 + vl;
        const double* q2 = q0 + 2 * vl;
        // G = G~(s) (lower), B = the first congruence operand: C_2 = c2s A(c) (quadratic)
        // or C_4 = inner(g2) (quartic); padding: G identity, B zero
        for (int i = T.warp; i < mp; i += T.nwarps)
            for (int j = T.lane; j <= i; j += 32) {
                double gv, bv;
                if (i >= m || j >= m) {
                    gv = (i == j) ? 1.0 : 0.0;
                    bv = 0.0;
                } else if (d == 2) {
                    const int e = pk(i, j);
                    const double c2 = c2s * ac[e];
                    gv = ax[e] + s * (av[e] + s * c2);
                    bv = c2;
                } else {
                    const int e = pk(i, j);
                    const double g1 = hconj(av[e], hh, q1, i, j);
                    const double g2 = c2s * hconj(ac[e], hh, q2, i, j);
                    if (j > 0) {  // inner
                        const double g0 = hconj(ax[e], hh, q0, i, j);
                        gv = g0 + t * (g1 + t * g2);
                        bv = g2;
                    } else if (i > 0) {  // border
                        gv = s * (g1 + t * g2);
                        bv = 0.0;
                    } else {  // corner
                        gv = g1 + t * g2;
                        bv = 0.0;
                    }
                }
                G[i * ld + j] = gv;
                B[i * ld + j] = bv;
            }
        __syncthreads();
        mirror_upper(T, B, mp, ld);
        __syncthreads();
        PROF_MARK(0);
        const bool okc = cholesky_inv_blocked_la(T, G, mp, ld, rdiag, Lv, &sh_i[2]);
        PROF_MARK(2);
        if (!okc) {
            // not interior at the start, or rounding past the root: keep the last safe s
            // (its K and Ritz vector stay in the buffers)
            if (T.tid == 0) {
                H[H_ST] = (double)(it == 0 ? HS_FAILED : HS_HIT);
                S[S_ST] = (double)ST_FAILED;
            }
            continue;
        }
        congruence_inv(T, G, Lv, B, mp, ld);
        // N~_first (symmetrised) parked in the Lanczos buffer
        double* Mw = P.wM + (size_t)slot * P.w_mstride;
        for (int i = T.warp; i < mp; i += T.nwarps)
            for (int j = T.lane; j < mp; j += 32) Mw[i * ld + j] = 0.5 * (B[i * ld + j] + B[j * ld + i]);
        __syncthreads();
        PROF_MARK(3);
        // second operand: C_1 = A(v) (quadratic) or C_2 = inner(g1) + corner g2 (quartic)
        for (int i = T.warp; i < mp; i += T.nwarps)
            for (int j = T.lane; j <= i; j += 32) {
                double bv = 0.0;
                if (i < m && j < m) {
                    const int e = pk(i, j);
                    if (d == 2) bv = av[e];
                    else if (j > 0) bv = hconj(av[e], hh, q1, i, j);
                    else if (i == 0) bv = c2s * hconj(ac[e], hh, q2, 0, 0);
                }
                B[i * ld + j] = bv;
            }
        if (d == 4) {  // border columns: e_0, b_1 = g1(1:, 0), b_3 = g2(1:, 0)
            for (int i = T.tid; i < mp; i += NT) {
                double b1 = 0.0, b3 = 0.0;
                if (i > 0 && i < m) {
                    const int e = pk(i, 0);
                    b1 = hconj(av[e], hh, q1, i, 0);
                    b3 = c2s * hconj(ac[e], hh, q2, i, 0);
                }
                X[i] = (i == 0) ? 1.0 : 0.0;
                X[vl + i] = b1;
                X[2 * vl + i] = b3;
            }
        }
        __syncthreads();
        mirror_upper(T, B, mp, ld);
        __syncthreads();
        PROF_MARK(5);
        congruence_inv(T, G, Lv, B, mp, ld);
        PROF_MARK(6);
        if (d == 4) fwd_solve_vecs(T, G, Lv, X, 3, vl, mp, ld);
        __syncthreads();
        PROF_MARK(7);
        // N_1 -> -N_1 (Lanczos operand, in place over N~_first), |N_j|_F^2 for j >= 2
        double f2 = 0.0, f3 = 0.0, f4 = 0.0;
        const double* pv = X;
        const double* u1 = X + vl;
        const double* u3 = X + 2 * vl;
        for (int i = T.warp; i < mp; i += T.nwarps)
            for (int j = T.lane; j < mp; j += 32) {
                const double nf = Mw[i * ld + j];
                const double ns = 0.5 * (B[i * ld + j] + B[j * ld + i]);
                double n1;
                if (d == 2) {  // nf = N~_2, ns = N~_1
                    n1 = ns + 2.0 * s * nf;
                    f2 += nf * nf;
                } else {       // nf = N~_4, ns = N~_2, rank-2 N~_1, N~_3
                    const double r1 = pv[i] * u1[j] + u1[i] * pv[j];
                    const double r3 = pv[i] * u3[j] + u3[i] * pv[j];
                    n1 = r1 + s * (2.0 * ns + s * (3.0 * r3 + s * 4.0 * nf));
                    const double n2 = ns + s * (3.0 * r3 + s * 6.0 * nf);
                    const double n3 = r3 + 4.0 * s * nf;
                    f2 += n2 * n2;
                    f3 += n3 * n3;
                    f4 += nf * nf;
                }
                Mw[i * ld + j] = -n1;
            }
        f2 = block_sum(T, f2, red);
        if (d == 4) {
            f3 = block_sum(T, f3, red);
            f4 = block_sum(T, f4, red);
        }
        // K to the L buffer (lower rows), 1 / diag(K), the slot header for lanczos_kernel
        double* Lw = P.wL + (size_t)slot * P.w_mstride;
        for (int i = T.warp; i < mp; i += T.nwarps)
            for (int j = T.lane; j <= i; j += 32) Lw[i * ld + j] = G[i * ld + j];
        for (int i = T.tid; i < mp; i += NT) S[S_VEC + 2 * vl + i] = rdiag[i];
        if (T.tid == 0) {
            S[S_MD] = (double)m;
            S[S_ST] = 0.0;
            H[H_C2] = sqrt(f2);
            H[H_C3] = sqrt(f3);
            H[H_C4] = sqrt(f4);
        }
        PROF_MARK(4);
    }
}

// ---------------------------------------------------------------- K5b
__global__ void hmc_weyl_kernel(ChordParams P) {
    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x * blockDim.x + threadIdx.x; rr < count; rr += gridDim.x * blockDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        double* H = P.wH + (size_t)slot * H_NS;
        if ((int)H[H_ST] != HS_ITER) continue;  // the Cholesky ended it
        const double* S = P.wS + (size_t)slot * P.w_sstride;
        const int d = (int)H[H_D];
        const double a_min = -S[S_TMAX];
        double cj[5] = {0.0, 0.0, H[H_C2], H[H_C3], H[H_C4]};
        const double h = weyl_step(a_min, cj, d);
        const int it = (int)H[H_IT] + 1;
        H[H_IT] = (double)it;
        if (P.prof) atomicAdd(&P.prof[17], 1ull);
        if (!(h < SW_INF)) {
            H[H_S] = SW_INF;
            H[H_ST] = (double)HS_INF;
            continue;
        }
        const double s = H[H_S] + h;
        H[H_S] = s;
        if (h <= 1e-15 * s) {
            H[H_ST] = (double)HS_HIT;
            continue;
        }
        if (it >= HMC_MAX_IT) {  // not converged: s is a lower bound only (rejected, counted)
            H[H_ST] = (double)HS_CAPPED;
            continue;
        }
        const int q = atomicAdd(P.nxt_count, 1);
        P.nxt_list[q] = slot;
    }
}

// ---------------------------------------------------------------- K5c
template <int NT>
__global__ void __launch_bounds__(NT, 2) hmc_tail_kernel(ChordParams P) {
    extern __shared__ __align__(16) double smem_dyn[];
    Team T;
    T.tid = threadIdx.x;
    T.nthr = NT;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = NT >> 5;
    __shared__ double red[64];
    __shared__ int sh_i[8];
    __shared__ double sh_d[16];
    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    double* G = smem_dyn;  // K (lower)
    double* vec = G + (size_t)mp * ld;
    double* zz = vec + 0 * vl;
    double* yy = vec + 1 * vl;
    double* hh = vec + 2 * vl;
    double* rdiag = vec + 3 * vl;
    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        if (P.mode == 0 && (P.flags[slot] & CF_DONE)) continue;
        const long long gidv = P.gid ? P.gid[slot] : P.chain_base + slot;
        double* x = P.X + (size_t)slot * P.np;
        double* v = P.V + (size_t)slot * P.np;
        const double* av = P.AV + (size_t)slot * P.mtp;
        double* ax = P.AX + (size_t)slot * P.mtp;
        const int bnd = P.bound[slot];
        const double* H = P.wH + (size_t)slot * H_NS;
        const double* S = P.wS + (size_t)slot * P.w_sstride;
        const int st = (int)H[H_ST];
        const double s = H[H_S];
        const int d = (int)H[H_D];
        const bool outward = (st == HS_OUTWARD);
        const bool failed = (st == HS_FAILED);
        const bool hit = !outward && s < SW_INF;
        __syncthreads();
        if (hit && !failed) {
            const double* Lw = P.wL + (size_t)slot * P.w_mstride;
            for (int i = T.warp; i < mp; i += T.nwarps)
                for (int c2 = T.lane; 2 * c2 <= i; c2 += 32) cp_async16(G + i * ld + 2 * c2, Lw + i * ld + 2 * c2);
            for (int i = T.tid; i < mp; i += NT) {
                zz[i] = S[S_VEC + 3 * vl + i];
                rdiag[i] = S[S_VEC + 2 * vl + i];
                hh[i] = (d == 4) ? S[S_VEC + i] : 0.0;
            }
            cp_async_wait_all();
            __syncthreads();
            back_solve_lt(T, G, ld, mp, zz, yy, rdiag);
            // boundary start: y = H D y~, D = diag(1/s, I)
            if (T.warp == 0) {
                if (d == 4) {
                    if (T.lane == 0) yy[0] /= s;
                    __syncwarp();
                    double hy = 0.0;
                    for (int i = T.lane; i < m; i += 32) hy += hh[i] * yy[i];
                    hy = warp_sum(hy) * H[H_BH];
                    for (int i = T.lane; i < m; i += 32) yy[i] -= hy * hh[i];
                    __syncwarp();
                }
                double yn = 0.0;
                for (int i = T.lane; i < m; i += 32) yn += yy[i] * yy[i];
                yn = sqrt(warp_sum(yn));
                for (int i = T.lane; i < m; i += 32) yy[i] /= yn;
            }
        } else {
            for (int i = T.tid; i < mp; i += NT) yy[i] = 0.0;
        }
        __syncthreads();
        const double t_dense = outward ? 0.0 : (hit ? (d == 4 ? s * s : s) : SW_INF);
        hmc_finish(T, P, slot, gidv, x, v, av, ax, bnd, yy, t_dense, failed, outward, st == HS_CAPPED, red, sh_d, sh_i);
    }
}

}  // namespace sw
