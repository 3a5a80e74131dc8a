// lanczos_t.cuh -- K2b for 104 < m <= 208 (configs[4], m = 200): the largest eigenvalue theta_max
// of the Cholesky-transformed pencil M = -L^{-1} A(v) L^{-T} (Lemma 3) by
// Lanczos with M held in ONE CTA's shared memory as the lower triangle of 8 x 8 tiles (M is
// symmetric: 325 tiles = 166 KB at m = 200 instead of 320 KB of full rows), 512 threads, one chain
// per SM.  The factor phase is the global-scratch chord kernel's gsplit mode 2 (M as these lower
// tiles in the slot's work buffer), the tail is tail_kernel<256> (chord3.cuh).
//
// Why: the fused global-scratch kernel re-reads the full M from L2 / HBM in every Lanczos
// iteration (11.5k cycles per matvec, 46% of a call's cycles at m = 200, 210 GB of DRAM per
// 65536-chain round); the 2-CTA cluster variant (lanczos_cl.cuh) holds it in distributed shared
// memory but pays three cluster barriers per iteration.  Here the matvec reads 2 x 166 KB of
// shared memory (every off-diagonal tile once for its block row, once for its block column).
//
// Per iteration (partial reorthogonalisation as lanczos2.cuh, SW_PRO_TAU2):
//   A: warp w < NWM owns the block indices i = w and NB-1-w; for each, y rows [8i, 8i+8) =
//      sum_{J <= i} M_iJ q_J (row part: lane (r, cq) accumulates M[r][2cq..2cq+1] q_J[2cq..],
//      reduced over cq) + sum_{I > i} M_Ii^T q_I (column part: lane (r, cq) accumulates
//      M[r][2cq..] q_I[r], reduced over r); y' = y - beta_{j-1} q_{j-1} to shared memory with
//      the warp's partial sums of q_j.y' and |y'|^2.  Warps NWM..15 run the omega recurrence.
//   B: as lanczos2: alpha, beta^2 = |y'|^2 - alpha^2 (exact |w|^2 on cancellation, a
//      Gram-Schmidt pass against the global basis Q when due); q_{j+1} to shared memory (ring of
//      three vectors: the matvec warps read q_j and q_{j-1}) and to global Q.
// Two barriers per iteration on the plain path; checks, Ritz value / vector as lanczos2.
#pragma once
#include "lanczos2.cuh"

#ifndef SW_FIRST_CHECK_PCT_T
#define SW_FIRST_CHECK_PCT_T 15  // first convergence check at this % of md (as the global-scratch variant)
#endif

namespace sw {

constexpr int LZT_NT = 512;
constexpr int LZT_NBMAX = 26;  // block indices (mdp <= 208): at most 13 matvec warps with two each

struct LztLayout {
    int oM, oX, oY, oW, oPart, oAl, oBe, oB2, oRbe, oOm, oDp, oDm, oSv, oRed, oShd, total;
    __host__ __device__ LztLayout(int mp) {
        const int nb = mp >> 3, vl = mp + 8;
        oM = 0;
        oX = oM + 64 * (nb * (nb + 1) / 2);  // q ring: q_j at (j % 3)
        oY = oX + 3 * vl;                      // y' = M q_j - beta q_{j-1}
        oW = oY + vl;                          // w (reorthogonalisation path)
        oPart = oW + vl;                       // [0,16) alpha, [16,32) |y'|^2, 40/41 PRO flags, [48,64) |w|^2; h at 64
        oAl = oPart + 64 + vl;
        oBe = oAl + vl;
        oB2 = oBe + vl;
        oRbe = oB2 + vl;
        oOm = oRbe + vl;  // omega rows, ring of 3
        oDp = oOm + 3 * vl;
        oDm = oDp + vl;
        oSv = oDm + vl;
        oRed = oSv + vl;  // 64
        oShd = oRed + 64; // check state (CK_*) + thetas
        total = oShd + 40;
    }
};

// y' rows [8i, 8i+8) of block index i for the calling warp (see the header); returns the lane's
// contributions to q_j.y' and |y'|^2 (lanes 0..7 hold row 8i + lane, the others 0)
__device__ __forceinline__ void lzt_block(const int i, const int nb, const int md, const int lane, const int oM,
                                          const int oXj, const int oXp, const int oY, const double bjm1,
                                          double& pa, double& pn) {
    extern __shared__ __align__(16) double sm[];
    const int r = lane >> 2, cq = lane & 3;
    // row part: tiles (i, J), J = 0..i (contiguous), four independent accumulator pairs
    const double* tr = sm + oM + 64 * (i * (i + 1) / 2) + 8 * r + 2 * cq;
    const double* xq = sm + oXj + 2 * cq;
    double ra[4] = {0.0, 0.0, 0.0, 0.0}, rb[4] = {0.0, 0.0, 0.0, 0.0};
    int J = 0;
    for (; J + 3 <= i; J += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double2 m2 = *reinterpret_cast<const double2*>(tr + 64 * (J + u));
            const double2 x2 = *reinterpret_cast<const double2*>(xq + 8 * (J + u));
            ra[u] = fma(m2.x, x2.x, ra[u]);
            rb[u] = fma(m2.y, x2.y, rb[u]);
        }
    }
    for (; J <= i; ++J) {  // fixed accumulator: a J & 3 index would put ra, rb in local memory
        const double2 m2 = *reinterpret_cast<const double2*>(tr + 64 * J);
        const double2 x2 = *reinterpret_cast<const double2*>(xq + 8 * J);
        ra[0] = fma(m2.x, x2.x, ra[0]);
        rb[0] = fma(m2.y, x2.y, rb[0]);
    }
    double yr = ((ra[0] + rb[0]) + (ra[1] + rb[1])) + ((ra[2] + rb[2]) + (ra[3] + rb[3]));
    yr += __shfl_xor_sync(0xffffffffu, yr, 1);
    yr += __shfl_xor_sync(0xffffffffu, yr, 2);  // row 8i + r in lanes 4r..4r+3
    // column part: tiles (I, i), I = i+1..nb-1; tile (I, i) at I (I + 1) / 2 + i, so the next
    // tile is I + 1 tiles further on
    double ca[4] = {0.0, 0.0, 0.0, 0.0}, cb[4] = {0.0, 0.0, 0.0, 0.0};
    {
        int I = i + 1;
        const double* p = sm + oM + 8 * r + 2 * cq + 64 * ((i + 1) * (i + 2) / 2 + i);
        int st = 64 * (i + 2);
        const double* xr = sm + oXj + r;
        for (; I + 3 < nb; I += 4) {
            const double* pp[4];
            pp[0] = p;
            pp[1] = pp[0] + st;
            pp[2] = pp[1] + st + 64;
            pp[3] = pp[2] + st + 128;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double2 m2 = *reinterpret_cast<const double2*>(pp[u]);
                const double qv = xr[8 * (I + u)];
                ca[u] = fma(m2.x, qv, ca[u]);
                cb[u] = fma(m2.y, qv, cb[u]);
            }
            p = pp[3] + st + 192;
            st += 256;
        }
        for (; I < nb; ++I) {
            const double2 m2 = *reinterpret_cast<const double2*>(p);
            const double qv = xr[8 * I];
            ca[0] = fma(m2.x, qv, ca[0]);
            cb[0] = fma(m2.y, qv, cb[0]);
            p += st;
            st += 64;
        }
    }
    double cx = (ca[0] + ca[1]) + (ca[2] + ca[3]), cy = (cb[0] + cb[1]) + (cb[2] + cb[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        cx += __shfl_xor_sync(0xffffffffu, cx, o);
        cy += __shfl_xor_sync(0xffffffffu, cy, o);
    }
    // lane t < 8: row 8i + t = row part (lane 4t) + column part (column t: lane t >> 1, x / y)
    const int t = lane & 7;
    const double y_row = __shfl_sync(0xffffffffu, yr, 4 * t);
    const double c_x = __shfl_sync(0xffffffffu, cx, t >> 1);
    const double c_y = __shfl_sync(0xffffffffu, cy, t >> 1);
    if (lane < 8) {
        const int R = 8 * i + t;
        const double y = y_row + ((t & 1) ? c_y : c_x);
        const double ypr = (R < md) ? y - bjm1 * sm[oXp + R] : 0.0;
        sm[oY + R] = ypr;
        pa = fma(sm[oXj + R], ypr, pa);
        pn = fma(ypr, ypr, pn);
    }
}

__global__ void __launch_bounds__(LZT_NT, 1) lanczos_t_kernel(ChordParams P) {
    extern __shared__ __align__(16) double sm[];
    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    const LztLayout Lo(mp);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = LZT_NT / 32;
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
        const int nb = mdp >> 3;
        const int nwm = (nb + 1) >> 1;  // matvec warps (<= 13)
        double* Qg = P.wM + (size_t)slot * P.w_mstride;  // M (lower tiles) on entry; the Lanczos basis afterwards
        // ---- M (the lower 8 x 8 tiles the factor phase wrote, contiguous) into shared memory
        const int ntiles = nb * (nb + 1) / 2;
        for (int e2 = tid; e2 < 32 * ntiles; e2 += LZT_NT) cp_async16(sm + Lo.oM + 2 * e2, Qg + 2 * e2);
        // start vector u_0 (as lanczos2), |u_0|^2 partials
        const bool owner = tid < mdp;
        const bool rowok = tid < md;
        double ur = 0.0;
        if (rowok) {
            const double f = (double)tid * 0.6180339887498949;
            ur = 0.5 + (f - floor(f));
        }
        const double p0 = warp_sum(ur * ur);
        if (lane == 0) sm[Lo.oPart + warp] = p0;
        for (int e = tid; e < 3 * vl; e += LZT_NT) sm[Lo.oX + e] = 0.0;  // q_{-1} = 0, padding
        if (tid == 0) {
            sm[Lo.oShd + CK_INTOP] = -SW_INF;
            sm[Lo.oShd + CK_INBOT] = SW_INF;
            sm[Lo.oShd + CK_JPREV] = 0.0;
            sm[Lo.oShd + CK_LRES] = 0.0;
            sm[Lo.oShd + CK_TTOP] = -SW_INF;
            sm[Lo.oShd + CK_TBOT] = SW_INF;
            sm[Lo.oShd + CK_HINTED] = 0.0;
            sm[Lo.oOm] = 1.0;  // omega_{0,0}
        }
        cp_async_wait_all();
        __syncthreads();
        double nn0 = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) nn0 += sm[Lo.oPart + w];
        double qj = rowok ? ur / sqrt(nn0) : 0.0;  // q_j[r] (owners)
        __syncthreads();  // M loaded everywhere before Q overwrites the global rows
        if (tid == 0) {
            sm[Lo.oPart + 40] = 0.0;
            sm[Lo.oPart + 41] = 0.0;
        }
        if (owner) {
            sm[Lo.oX + tid] = qj;
            Qg[tid] = qj;
        }
        double bjm1 = 0.0, tnorm = 0.0;
        int reorth_left = 0;
        bool was_full = true;
        const double eps1 = 2.220446049250313e-16 * sqrt((double)md);
        int next_check = max(12, (md * SW_FIRST_CHECK_PCT_T) / 100);
        const bool need_bot = P.need_tmin && !P.zall;
        int J = 0;
        __syncthreads();
        for (int j = 0; j < md; ++j) {
            const int oXj = Lo.oX + (j % 3) * vl, oXn = Lo.oX + ((j + 1) % 3) * vl, oXp = Lo.oX + ((j + 2) % 3) * vl;
            // ---- A: y' = M q_j - beta q_{j-1} (warps < nwm), omega recurrence (the other warps)
            if (warp < nwm) {
                double pa = 0.0, pn = 0.0;
                lzt_block(warp, nb, md, lane, Lo.oM, oXj, oXp, Lo.oY, bjm1, pa, pn);
                if (nb - 1 - warp != warp) lzt_block(nb - 1 - warp, nb, md, lane, Lo.oM, oXj, oXp, Lo.oY, bjm1, pa, pn);
                pa = warp_sum(pa);
                pn = warp_sum(pn);
                if (lane == 0) {
                    sm[Lo.oPart + warp] = pa;
                    sm[Lo.oPart + 16 + warp] = pn;
                }
            } else if (j >= 1) {
                // omega_{j,k} = q_j . q_k estimates (Simon 1984), as lanczos2
                const int oRj = Lo.oOm + (j % 3) * vl, oR1 = Lo.oOm + ((j + 2) % 3) * vl,
                          oR2 = Lo.oOm + ((j + 1) % 3) * vl;
                const double sj = sm[Lo.oRbe + j - 1];  // 1 / beta_{j-1}
                const int t0 = 32 * nwm, ts = LZT_NT - t0;
                for (int k = tid - t0; k <= j; k += ts) {
                    double v;
                    if (k == j) v = 1.0;
                    else if (k == j - 1) v = eps1 * tnorm * sj;
                    else if (was_full) v = eps1;
                    else {
                        const double bk = sm[Lo.oBe + k], bkm = (k > 0) ? sm[Lo.oBe + k - 1] : 0.0;
                        double num = bk * sm[oR1 + k + 1] + (sm[Lo.oAl + k] - sm[Lo.oAl + j - 1]) * sm[oR1 + k] +
                                     ((k > 0) ? bkm * sm[oR1 + k - 1] : 0.0) - sm[Lo.oBe + j - 2] * sm[oR2 + k];
                        num += copysign(eps1 * (bk + bjm1), num);
                        v = num * sj;
                        if (fabs(v) > SW_PRO_TAU2) sm[Lo.oPart + 40 + (j & 1)] = 1.0;
                    }
                    sm[oRj + k] = v;
                }
            }
            __syncthreads();
            // ---- B: alpha, beta; q_{j+1}
            double alpha0 = 0.0, nny = 0.0;
            for (int w = 0; w < nwm; ++w) {
                alpha0 += sm[Lo.oPart + w];
                nny += sm[Lo.oPart + 16 + w];
            }
            const double ypr = rowok ? sm[Lo.oY + tid] : 0.0;
            bool reorth = (j == 0);
            if (reorth_left > 0) {
                reorth = true;
                --reorth_left;
            } else if (j >= 1 && sm[Lo.oPart + 40 + (j & 1)] != 0.0) {
                reorth = true;
                reorth_left = 1;
            }
            double alpha = alpha0;
            double wr = rowok ? ypr - alpha * qj : 0.0;
            double nn = nny - alpha0 * alpha0;  // |w|^2 by Pythagoras
            bool full = false;
            if (reorth || !(nn >= 0.25 * nny)) {
                if (!(nn >= 1e-12 * nny)) reorth = true;
                full = reorth;
                if (reorth) {
                    if (owner) sm[Lo.oW + tid] = wr;
                    if (tid == 0) sm[Lo.oPart + 40 + ((j + 1) & 1)] = 0.0;
                    __syncthreads();
                    // h_i = q_i . w, i <= j (Q rows from global / L2): 8 threads per dot, 64 dots per pass
                    for (int i0 = 0; i0 <= j; i0 += LZT_NT / 8) {
                        const int i = i0 + (tid >> 3), sub = tid & 7;
                        double s0 = 0.0, s1 = 0.0;
                        if (i <= j) {
                            const double* qi = Qg + (size_t)i * ld;
                            double2 q2[13];
#pragma unroll
                            for (int k = 0; k < 13; ++k) {
                                const int c = 2 * sub + 16 * k;
                                q2[k] = (c < mdp) ? *reinterpret_cast<const double2*>(qi + c) : make_double2(0.0, 0.0);
                            }
#pragma unroll
                            for (int k = 0; k < 13; ++k) {
                                const int c = 2 * sub + 16 * k;
                                if (c < mdp) {
                                    const double2 w2 = *reinterpret_cast<const double2*>(sm + Lo.oW + c);
                                    s0 = fma(q2[k].x, w2.x, s0);
                                    s1 = fma(q2[k].y, w2.y, s1);
                                }
                            }
                        }
                        double sd = s0 + s1;
                        sd += __shfl_xor_sync(0xffffffffu, sd, 1);
                        sd += __shfl_xor_sync(0xffffffffu, sd, 2);
                        sd += __shfl_xor_sync(0xffffffffu, sd, 4);
                        if (sub == 0 && i <= j) sm[Lo.oPart + 64 + i] = sd;
                    }
                    __syncthreads();
                    // w -= Q h: row r = tid & 255, the two thread halves take alternate rows of Q
                    const int rq = tid & 255, hq = tid >> 8;
                    double qa[4] = {0.0, 0.0, 0.0, 0.0};
                    if (rq < md) {
                        for (int i = hq; i <= j; i += 16) {
                            double qv[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const int ii = i + 2 * u;
                                qv[u] = (ii <= j) ? Qg[(size_t)ii * ld + rq] : 0.0;
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const int ii = i + 2 * u;
                                if (ii <= j) qa[u & 3] = fma(sm[Lo.oPart + 64 + ii], qv[u], qa[u & 3]);
                            }
                        }
                    }
                    const double qpart = (qa[0] + qa[1]) + (qa[2] + qa[3]);
                    if (hq == 1 && rq < mdp) sm[Lo.oW + rq] = qpart;  // w itself is no longer needed
                    __syncthreads();
                    const double qh0 = qpart, qh1 = (rowok && tid < 256) ? sm[Lo.oW + tid] : 0.0;
                    wr = rowok ? wr - (qh0 + qh1) : 0.0;
                    alpha += sm[Lo.oPart + 64 + j];
                }
                if (tid == 0) sm[Lo.oPart + 40 + ((j + 1) & 1)] = 0.0;
                const double pw = warp_sum(wr * wr);
                if (lane == 0) sm[Lo.oPart + 48 + warp] = pw;
                __syncthreads();
                nn = 0.0;
#pragma unroll
                for (int w = 0; w < NW; ++w) nn += sm[Lo.oPart + 48 + w];
                if (nn < 1e-28 * nny) nn = 0.0;  // only rounding left: invariant Krylov space
            } else if (tid == 0) {
                sm[Lo.oPart + 40 + ((j + 1) & 1)] = 0.0;
            }
            if (!(nn > 0.0)) nn = 0.0;
            const double rsb = (nn > 0.0) ? rsqrt(nn) : SW_INF;
            const double beta = (nn > 0.0) ? nn * rsb : 0.0;
            tnorm = fmax(tnorm, fabs(alpha) + beta + bjm1);
            J = j + 1;
            const bool exhausted = (J == md) || !(beta > 1e-15 * tnorm);
            const double qn = (rowok && beta > 0.0) ? wr * rsb : 0.0;
            if (tid == 0) {
                sm[Lo.oAl + j] = alpha;
                sm[Lo.oBe + j] = beta;
                sm[Lo.oB2 + j] = nn;
                sm[Lo.oRbe + j] = rsb;
            }
            if (owner && !exhausted) {
                sm[oXn + tid] = qn;
                Qg[(size_t)(j + 1) * ld + tid] = qn;
            }
            qj = qn;
            bjm1 = beta;
            was_full = full;
            if (P.prof && full && tid == 0) atomicAdd(&P.prof[29], 1ull);
            __syncthreads();
            if (exhausted || J >= next_check) {
                lanczos_check(tid, Lo.oAl, Lo.oBe, Lo.oB2, Lo.oRbe, J, beta, tnorm, need_bot, exhausted, md,
                              Lo.oShd, P.prof);
                __syncthreads();
                if (sm[Lo.oShd + CK_DONE] != 0.0) break;
                next_check = (int)sm[Lo.oShd + CK_NEXT];
            }
        }
        const double theta_max = sm[Lo.oShd + CK_TTOP];
        const double theta_min = sm[Lo.oShd + CK_TBOT];
        Team T;
        T.tid = tid; T.nthr = LZT_NT; T.lane = lane; T.warp = warp; T.nwarps = NW;
        int* sh_r = reinterpret_cast<int*>(sm + Lo.oShd + 30);
        tri_twisted_vec(T, sm + Lo.oAl, sm + Lo.oBe, J, theta_max, sm[Lo.oBe + J - 1], sm + Lo.oDp, sm + Lo.oDm,
                        sm + Lo.oSv, sm + Lo.oRed, sh_r);
        if (P.jlast && tid == 0) P.jlast[slot] = J;
        if (P.jsum && tid == 0) {
            atomicAdd(&P.jsum[0], (unsigned long long)J);
            atomicAdd(&P.jsum[1], 1ull);
        }
        if (tid == LZT_NT - 1) {
            const double th2 = theta_max - 1e-12 * fabs(theta_max);
            const int c = sturm_below(sm + Lo.oAl, sm + Lo.oBe, J, th2);
            sh_deg = (md >= 2 && J >= 2 && c <= J - 2) ? 1 : 0;
        }
        // z = Q s (rows of Q: the normalised Lanczos vectors, global): two threads per row
        double* zg = S + S_VEC + 3 * vl;
        if (theta_max > 0.0 || P.zall) {
            const int e = tid & 255, hz = tid >> 8;
            double s0 = 0.0, s1 = 0.0;
            if (e < mdp) {
                int i = hz;
                for (; i + 2 < J; i += 4) {
                    s0 = fma(sm[Lo.oSv + i], Qg[(size_t)i * ld + e], s0);
                    s1 = fma(sm[Lo.oSv + i + 2], Qg[(size_t)(i + 2) * ld + e], s1);
                }
                if (i < J) s0 = fma(sm[Lo.oSv + i], Qg[(size_t)i * ld + e], s0);
            }
            const double zp = s0 + s1;
            if (hz == 1 && e < mdp) sm[Lo.oW + e] = zp;
            __syncthreads();
            if (hz == 0 && e < mdp) zg[e] = zp + sm[Lo.oW + e];
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

}  // namespace sw
