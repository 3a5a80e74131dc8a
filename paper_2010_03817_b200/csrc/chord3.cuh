// chord3.cuh -- K2 split into three kernels per scheduler round (m <= 128):
//
//   K2a factor_kernel   unpack A(x), A(v); Schur deflation of a boundary start
//                       (R6); L L^T = A(x) (blocked Cholesky, DMMA
//                       trailing updates); M = -L^{-1} A(v) L^{-T} (two blocked
//                       TRSMs) -> M, L, deflation data to per-slot work buffers
//   K2b lanczos_kernel  theta_max (theta_min in oracle mode) of M by the
//                       register-resident Lanczos (lanczos_reg); z = Q s
//   K2c tail_kernel     y = L^{-T} z, the deflation back-transform, then the
//                       closed-form cube / ball constraints, selection, advance
//                       and step logic (chord_tail.inc)
//
// Same mathematics as chord_kernel2 (Alg. 2, Lemma 3
// P:587-651, the Cholesky-transformed pencil of P:1207-1215, the PEP
// eigenvector y = L^{-T} z of P:784-791).  The split gives each phase the whole
// register file (the fused kernel spilled the Lanczos loop to local memory) and
// its own launch shape; the work buffers cost ~4 x 86 KB of HBM traffic per
// chain-call at m = 100 (~3% of a round).
#pragma once
#include "chord2.cuh"
#ifndef SW_UNPACK_BOTH
#define SW_UNPACK_BOTH 1  // factor_kernel: both triangles by cp.async, no mirror pass (-1.8% factor time, r2s)
#endif
#ifndef SW_FACTOR_SYM
#define SW_FACTOR_SYM 1  // M = -(B + B^T)/2 when written, as the oracle (0: -B, rows only: -0.8% factor time, r2r)
#endif
#ifndef SW_TAIL_CTAS
#define SW_TAIL_CTAS 3  // K2c CTAs per SM (L packed: ~49 KB of shared memory each at m = 100)
#endif
#include "chol_inv.cuh"

namespace sw {

// (the per-slot scalar/vector area S_* / ST_* and s_stride live in chord.cuh)

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}

// packed lower P (row-major packing, pk(i, j) = i(i+1)/2 + j) -> rows of M (lower
// triangle) by 8-byte cp.async, one warp per row (no index arithmetic per element);
// the caller waits (cp.async.wait_all + barrier) and mirrors the upper triangle.
__device__ __forceinline__ void unpack_lower_async(const Team& T, const double* __restrict__ P, double* M, int m,
                                                   int ld) {
    for (int i = T.warp; i < m; i += T.nwarps) {
        const double* src = P + (size_t)i * (i + 1) / 2;
        for (int j = T.lane; j <= i; j += 32) cp_async8(M + i * ld + j, src + j);
    }
}
// both triangles straight from the packed lower rows (two asynchronous copies per element:
// no mirror pass and its barrier)
__device__ __forceinline__ void unpack_sym_async(const Team& T, const double* __restrict__ P, double* M, int m,
                                                 int ld) {
    for (int i = T.warp; i < m; i += T.nwarps) {
        const double* src = P + (size_t)i * (i + 1) / 2;
        for (int j = T.lane; j <= i; j += 32) {
            cp_async8(M + i * ld + j, src + j);
            if (j < i) cp_async8(M + j * ld + i, src + j);
        }
    }
}
// the same copy per 8 x 8 tile of the lower triangle (one warp per tile): lane (r, q) copies
// elements (r, q) and (r, q + 4) and their transposes, so that both the row-wise and the
// transposed 8-byte writes of a half-warp hit distinct bank slots (ld = 4 or 12 mod 16); the
// row-wise copy's transposed writes were 4-way conflicted (14% of K2a's excess shared-memory
// wavefronts, ncu r2fs)
__device__ __forceinline__ void unpack_sym_tiles_async(const Team& T, const double* __restrict__ P, double* M, int m,
                                                       int ld) {
    const int TB = (m + 7) >> 3;
    const int ntile = TB * (TB + 1) / 2;
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int t = T.warp; t < ntile; t += T.nwarps) {
        int ib = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
        while ((ib + 1) * (ib + 2) / 2 <= t) ++ib;
        while (ib * (ib + 1) / 2 > t) --ib;
        const int jb = t - ib * (ib + 1) / 2;
        const int i = ib * 8 + r;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = jb * 8 + q + 4 * h;
            if (i < m && j <= i) {
                const double* src = P + (size_t)i * (i + 1) / 2 + j;
                cp_async8(M + i * ld + j, src);
                if (j < i) cp_async8(M + j * ld + i, src);
            }
        }
    }
}
__device__ __forceinline__ void mirror_upper(const Team& T, double* M, int m, int ld) {
    for (int i = T.warp; i < m; i += T.nwarps)
        for (int j = T.lane; j < i; j += 32) M[j * ld + i] = M[i * ld + j];
}

// ---------------------------------------------------------------- K2a
template <int NT>
__global__ void __launch_bounds__(NT, 1) factor_kernel(ChordParams P) {
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
    // one spare row each: a deflated boundary start works in place on the trailing block
    // (G + ld + 1, B + ld + 1), whose padded rows reach row mp
    double* G = smem_dyn;
    double* B = G + (size_t)(mp + 1) * ld;
    double* vec = B + (size_t)(mp + 1) * ld;
    double* uu = vec + V_UU * vl;
    double* hh = vec + V_HH * vl;
    double* pw = vec + V_PW * vl;
    double* rdiag = vec + V_RDIAG * vl;
    double* yy = vec + V_YY * vl;
    double* bv = vec + V_BV * vl;
    double* Lv = vec + NVEC2 * vl + 64;  // inverse diagonal blocks (8 mp doubles)

    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        if (P.mode == 0 && (P.flags[slot] & CF_DONE)) continue;
        const double* av = P.AV + (size_t)slot * P.mtp;
        const double* ax = P.AX + (size_t)slot * P.mtp;
        double* S = P.wS + (size_t)slot * P.w_sstride;
        const int bnd = P.bound[slot];
        __syncthreads();
        long long t_prof = clock64();
#if SW_UNPACK_BOTH
        unpack_sym_tiles_async(T, ax, G, m, ld);
        unpack_sym_tiles_async(T, av, B, m, ld);
#else
        unpack_lower_async(T, ax, G, m, ld);
        unpack_lower_async(T, av, B, m, ld);
#endif
        const bool defl = (bnd == 0);
        if (defl)
            for (int i = T.tid; i < m; i += T.nthr) uu[i] = P.U[(size_t)slot * m + i];
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
#if !SW_UNPACK_BOTH
        mirror_upper(T, G, m, ld);
        mirror_upper(T, B, m, ld);
        __syncthreads();
#endif
        PROF_MARK(0);
        int md = m;
        double a_schur = 0.0, beta_h = 0.0;
        bool outward = false;
        double* Gd = G;  // the matrices of the (possibly deflated) pencil
        double* Bd = B;
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
            // H G H and H B H (H u = -+|u| e_0) as rank-2 updates X - h p^T - p h^T, applied below
            // only where needed: the trailing block, in place, fused with the Schur complement of
            // B's (0, 0) pivot a and border b (R6)
            householder_congruence2(T, G, B, m, ld, hh, beta_h, pw, yy, red, false);
            a_schur = B[0] - (hh[0] * yy[0] + yy[0] * hh[0]);
            outward = !(a_schur > 0.0);
            for (int i = T.tid; i + 1 < m; i += T.nthr) bv[i] = B[(i + 1) * ld] - (hh[i + 1] * yy[0] + yy[i + 1] * hh[0]);
            __syncthreads();
            md = m - 1;
            for (int i = 1 + T.warp; i < m; i += T.nwarps) {
                const double hi = hh[i], pxi = pw[i], pyi = yy[i], bi = bv[i - 1];
                for (int jx = 1 + T.lane; jx < m; jx += 32) {
                    const double hj = hh[jx];
                    G[i * ld + jx] -= hi * pw[jx] + pxi * hj;
                    const double bij = B[i * ld + jx] - (hi * yy[jx] + pyi * hj);
                    B[i * ld + jx] = outward ? 0.0 : bij - bi * bv[jx - 1] / a_schur;
                }
            }
            Gd = G + ld + 1;
            Bd = B + ld + 1;
        }
        const int mdp = (md + 7) & ~7;
        for (int i = md + T.warp; i < mdp; i += T.nwarps)
            for (int j = T.lane; j < mdp; j += 32) {
                Gd[i * ld + j] = (i == j) ? 1.0 : 0.0;
                Gd[j * ld + i] = (i == j) ? 1.0 : 0.0;
                Bd[i * ld + j] = 0.0;
                Bd[j * ld + i] = 0.0;
            }
        __syncthreads();
        int status = (defl ? ST_DEFL : 0) | (outward ? ST_OUTWARD : 0);
        PROF_MARK(1);
        if (!outward && md >= 1) {
            const bool okc = cholesky_inv_blocked_la(T, Gd, mdp, ld, rdiag, Lv, &sh_i[2]);
            PROF_MARK(2);
            if (!okc) {
                status |= ST_FAILED;
            } else {
                congruence_inv(T, Gd, Lv, Bd, mdp, ld);
                PROF_MARK(3);
                // M = -(B + B^T)/2 and L to the work buffers (rows of length mdp), per 8 x 8 tile
                // (lane (r, q): elements (r, q), (r, q + 4)) so that the transposed reads of B are
                // conflict-free (the row-wise pass's column reads were 4-way conflicted, ncu r2fs)
                double* Mw = P.wM + (size_t)slot * P.w_mstride;
                double* Lw = P.wL + (size_t)slot * P.w_mstride;
                const int TBd = mdp >> 3;
                const int tr = T.lane >> 2, tq = T.lane & 3;
                for (int t = T.warp; t < TBd * TBd; t += T.nwarps) {
                    const int i = (t / TBd) * 8 + tr;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int jx = (t % TBd) * 8 + tq + 4 * h;
#if SW_FACTOR_SYM
                        Mw[i * ld + jx] = -0.5 * (Bd[i * ld + jx] + Bd[jx * ld + i]);
#else
                        Mw[i * ld + jx] = -Bd[i * ld + jx];
#endif
                        if (jx <= i) Lw[pk(i, jx)] = Gd[i * ld + jx];  // packed lower rows (tail_kernel)
                    }
                }
            }
        }
        // scalars and vectors of the slot
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

// ---------------------------------------------------------------- K2b
template <int NT, int KC>
__global__ void __launch_bounds__(NT, 1) lanczos_kernel(ChordParams P) {
    extern __shared__ __align__(16) double smem_dyn[];
    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    // Q (rows of ld), vector area (NVEC2 slots) + 64 slack; no transposed basis (the smaller
    // shared-memory footprint leaves more L1 for the M loads)
    const int oQ = 0, oVec = mp * ld, oRed = oVec + NVEC2 * vl;
    const int tid = threadIdx.x;
    __shared__ int sh_deg;
    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        if (P.mode == 0 && (P.flags[slot] & CF_DONE)) continue;
        double* S = P.wS + (size_t)slot * P.w_sstride;
        const int status = (int)S[S_ST];
        const int md = (int)S[S_MD];
        __syncthreads();
        if ((status & (ST_OUTWARD | ST_FAILED)) || md < 1) {
            if (tid == 0) {
                S[S_TMAX] = -SW_INF;
                S[S_TMIN] = SW_INF;
                S[S_DEG] = 0.0;
            }
            continue;
        }
        const int mdp = (md + 7) & ~7;
        const double* Mw = P.wM + (size_t)slot * P.w_mstride;
        const int J = lanczos_reg<NT, KC, true, false>(-1, oQ, md, mdp, ld, P.need_tmin && !P.zall, oVec, vl, oRed,
                                                       P.zall ? SW_FIRST_CHECK_PCT_HMC : 0,
                                                       P.prof, Mw, 0);
        if (P.jlast && tid == 0) P.jlast[slot] = J;
        if (P.jsum && tid == 0) {
            atomicAdd(&P.jsum[0], (unsigned long long)J);
            atomicAdd(&P.jsum[1], 1ull);
        }
        const double theta_max = smem_dyn[oRed + 32 + 4];
        const double theta_min = smem_dyn[oRed + 32 + 5];
        const double* al = smem_dyn + oVec + V_AL * vl;
        const double* be = smem_dyn + oVec + V_BE * vl;
        const double* sv = smem_dyn + oVec + V_SV * vl;
        if (tid == NT - 1) {  // a thread without z = Q s work when mdp < NT
            const double th2 = theta_max - 1e-12 * fabs(theta_max);
            const int c = sturm_below(al, be, J, th2);
            sh_deg = (md >= 2 && J >= 2 && c <= J - 2) ? 1 : 0;
        }
        // z = Q s (rows of Q are the normalised Lanczos vectors)
        double* zg = S + S_VEC + 3 * vl;
        if (theta_max > 0.0 || P.zall) {
            for (int e = tid; e < mdp; e += NT) {
                double s0 = 0.0, s1 = 0.0;
                int i = 0;
                for (; i + 1 < J; i += 2) {
                    s0 = fma(sv[i], smem_dyn[oQ + i * ld + e], s0);
                    s1 = fma(sv[i + 1], smem_dyn[oQ + (i + 1) * ld + e], s1);
                }
                if (i < J) s0 = fma(sv[i], smem_dyn[oQ + i * ld + e], s0);
                zg[e] = s0 + s1;
            }
        }
        __syncthreads();
        if (tid == 0) {
            S[S_TMAX] = theta_max;
            S[S_TMIN] = theta_min;
            S[S_DEG] = (double)sh_deg;
            S[S_J] = (double)J;
            if (P.prof) atomicAdd(&P.prof[10], (unsigned long long)J);
        }
    }
}

// closed-form cube / ball constraints and the selection with the fixed tie order
// (R10) -- the same arithmetic as chord_tail.inc's block, as a function so that
// the tail kernel can run it on its last warp while the others solve for y.
__device__ __forceinline__ void select_bound_warp(const ChordParams& P, int lane, int n, const double* x,
                                                  const double* v, double theta_max, double theta_min, bool defl,
                                                  bool outward, int bnd, double* sh_d, int* sh_i) {
    double tpl = (theta_max > 0.0) ? 1.0 / theta_max : SW_INF;
    double tmi = defl ? 0.0 : ((theta_min < 0.0) ? 1.0 / theta_min : -SW_INF);
    if (outward) { tpl = 0.0; tmi = 0.0; }
    int bind = (tpl < SW_INF) ? 0 : SW_BIND_NONE_DEV;
    if (P.lo) {
        double bt = SW_INF;
        int bi = 0x7fffffff;
        double tm = -SW_INF;
        for (int i = lane; i < n; i += 32) {
            double vi = v[i], xi = x[i];
            double t = SW_INF, tn = -SW_INF;
            if (vi > 0.0) { t = (P.hi[i] - xi) / vi; tn = (P.lo[i] - xi) / vi; }
            else if (vi < 0.0) { t = (P.lo[i] - xi) / vi; tn = (P.hi[i] - xi) / vi; }
            if (t < bt) { bt = t; bi = i; }
            tm = fmax(tm, tn);
        }
        for (int o = 16; o > 0; o >>= 1) {
            double ot = __shfl_xor_sync(0xffffffffu, bt, o);
            int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ot < bt || (ot == bt && oi < bi)) { bt = ot; bi = oi; }
        }
        tm = warp_max(tm);
        if (bt < tpl) {
            tpl = bt;
            bind = (v[bi] > 0.0) ? 1 + 2 * bi : 2 + 2 * bi;
        }
        tmi = fmax(tmi, tm);
    }
    if (P.has_ball) {
        double dv = 0.0, dd2 = 0.0, vv = 0.0;
        for (int i = lane; i < n; i += 32) {
            double di = x[i] - P.ball_c[i];
            dv += di * v[i];
            dd2 += di * di;
            vv += v[i] * v[i];
        }
        dv = warp_sum(dv); dd2 = warp_sum(dd2); vv = warp_sum(vv);
        double disc = dv * dv - vv * (dd2 - P.ball_r * P.ball_r);
        double sq = sqrt(fmax(disc, 0.0));
        double tb = (-dv + sq) / vv;
        double tbm = (-dv - sq) / vv;
        if (bnd == SW_BIND_BALL_DEV && tb <= 0.0) tb = SW_INF;
        if (tb < tpl) { tpl = tb; bind = SW_BIND_BALL_DEV; }
        tmi = fmax(tmi, fmin(tbm, 0.0));
    }
    if (lane == 0) {
        sh_d[0] = tpl;
        sh_d[1] = tmi;
        sh_i[1] = bind;
    }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// y = L^{-T} z with L lower in G (rows of ld), rdiag = 1 / diag(L); blocked backwards
// over 8-row blocks (warp 0 solves the diagonal block, all threads update).  zz is
// overwritten.
__device__ __forceinline__ void back_solve_lt(const Team& T, const double* G, int ld, int mdp, double* zz, double* yy,
                                              const double* rdiag) {
    for (int kb = (mdp >> 3) - 1; kb >= 0; --kb) {
        const int k0 = kb * 8;
        if (T.warp == 0) {
            const int r = T.lane;
            double zr = (r < 8) ? zz[k0 + r] : 0.0;
#pragma unroll
            for (int c = 7; c >= 0; --c) {
                const double yc = __shfl_sync(0xffffffffu, zr, c) * rdiag[k0 + c];
                if (r == c) zr = yc;
                else if (r < c) zr -= G[(k0 + c) * ld + k0 + r] * yc;
            }
            if (r < 8) yy[k0 + r] = zr;
        }
        __syncthreads();
        for (int i = T.tid; i < k0; i += T.nthr) {
            double acc = zz[i];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc -= G[(k0 + c) * ld + i] * yy[k0 + c];
            zz[i] = acc;
        }
        __syncthreads();
    }
}

// back_solve_lt with L packed by rows (L[i][j] at pk(i, j), j <= i)
__device__ __forceinline__ void back_solve_lt_packed(const Team& T, const double* Lp, int mdp, double* zz, double* yy,
                                                     const double* rdiag) {
    for (int kb = (mdp >> 3) - 1; kb >= 0; --kb) {
        const int k0 = kb * 8;
        if (T.warp == 0) {
            const int r = T.lane;
            double zr = (r < 8) ? zz[k0 + r] : 0.0;
#pragma unroll
            for (int c = 7; c >= 0; --c) {
                const double yc = __shfl_sync(0xffffffffu, zr, c) * rdiag[k0 + c];
                if (r == c) zr = yc;
                else if (r < c) zr -= Lp[pk(k0 + c, k0 + r)] * yc;
            }
            if (r < 8) yy[k0 + r] = zr;
        }
        __syncthreads();
        for (int i = T.tid; i < k0; i += T.nthr) {
            double acc = zz[i];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc -= Lp[pk(k0 + c, i)] * yy[k0 + c];
            zz[i] = acc;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- K2c
template <int NT>
__global__ void __launch_bounds__(NT, (NT > 256) ? 1 : SW_TAIL_CTAS) tail_kernel(ChordParams P) {
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
    const int m = P.m, n = P.n;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    double* G = smem_dyn;  // L (packed lower rows)
    double* vec = G + (((size_t)mp * (mp + 1) / 2 + 1) & ~(size_t)1);
    double* zz = vec + 0 * vl;
    double* yy = vec + 1 * vl;
    double* hh = vec + 2 * vl;
    double* bv = vec + 3 * vl;
    double* rdiag = vec + 4 * vl;
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
        const double* S = P.wS + (size_t)slot * P.w_sstride;
        const int status = (int)S[S_ST];
        const int md = (int)S[S_MD];
        const double a_schur = S[S_A], beta_h = S[S_BH];
        const double theta_max = S[S_TMAX], theta_min = S[S_TMIN];
        const bool degenerate = S[S_DEG] != 0.0;
        const bool outward = (status & ST_OUTWARD) != 0;
        const bool failed = (status & ST_FAILED) != 0;
        const bool defl = (bnd == 0);
        long long t_prof = clock64();
        __syncthreads();
        // (Hit-and-Run walks never reflect: no kernel vector needed)
        const bool dense_y = !outward && !failed && md >= 1 && theta_max > 0.0 && !(P.mode == 0 && P.wkind >= 2);
        if (dense_y) {
            // L (lower rows, 16-byte segments [0, i+1]) into shared memory asynchronously
            const int mdp = (md + 7) & ~7;
            const double* Lw = P.wL + (size_t)slot * P.w_mstride;
            const int lp = mdp * (mdp + 1) / 2;
            for (int c2 = T.tid; 2 * c2 < lp; c2 += T.nthr) cp_async16(G + 2 * c2, Lw + 2 * c2);
            for (int i = T.tid; i < mdp; i += T.nthr) {
                zz[i] = S[S_VEC + 3 * vl + i];
                rdiag[i] = S[S_VEC + 2 * vl + i];
            }
            if (defl)
                for (int i = T.tid; i < m; i += T.nthr) {
                    hh[i] = S[S_VEC + i];
                    bv[i] = S[S_VEC + vl + i];
                }
        }
        // the last warp selects the binding constraint while L is in flight
        if (T.warp == T.nwarps - 1)
            select_bound_warp(P, T.lane, n, x, v, theta_max, theta_min, defl, outward, bnd, sh_d, sh_i);
        if (dense_y) {
            const int mdp = (md + 7) & ~7;
            cp_async_wait_all();
            __syncthreads();
            PROF_MARK(5);
            back_solve_lt_packed(T, G, mdp, zz, yy, rdiag);  // y = L^{-T} z
            PROF_MARK(6);
            if (T.warp == 0) {
                if (defl) {  // y = H [ -b^T yh / a ; yh ]
                    double s = 0.0;
                    for (int i = T.lane; i < md; i += 32) s += bv[i] * yy[i];
                    s = warp_sum(s);
                    double alpha0 = -s / a_schur;
                    __syncwarp();
                    for (int base_i = md - 1; base_i >= 0; base_i -= 32) {
                        int i = base_i - T.lane;
                        double val = (i >= 0) ? yy[i] : 0.0;
                        __syncwarp();
                        if (i >= 0) yy[i + 1] = val;
                        __syncwarp();
                    }
                    if (T.lane == 0) yy[0] = alpha0;
                    __syncwarp();
                    double hy = 0.0;
                    for (int i = T.lane; i < m; i += 32) hy += hh[i] * yy[i];
                    hy = warp_sum(hy) * beta_h;
                    for (int i = T.lane; i < m; i += 32) yy[i] -= hy * hh[i];
                    __syncwarp();
                }
                double yn = 0.0;
                for (int i = T.lane; i < m; i += 32) yn += yy[i] * yy[i];
                yn = sqrt(warp_sum(yn));
                for (int i = T.lane; i < m; i += 32) yy[i] /= yn;
            }
            __syncthreads();
        }
#define SW_SELECT_EARLY
#include "chord_tail.inc"
#undef SW_SELECT_EARLY
    }
}

}  // namespace sw
