// lanczos_cl.cuh -- K2b for 104 < m <= 208 (configs[4], m = 200) on a PAIR of SMs: a 2-CTA
// thread-block cluster holds the Cholesky-transformed pencil M = -L^{-1} A(v) L^{-T}
// in the two CTAs' shared memory -- CTA h owns rows [104 h, 104 h + 104) --
// and runs Lanczos on it with the vectors exchanged through distributed shared memory
// (north_star item 2: "one CTA or cluster per chain with tiles in shared or distributed shared
// memory").  Replaces the global-scratch variant's Lanczos, which re-read M (320 KB) from
// L2 / HBM every iteration (11.5k cycles per matvec, 210 GB of DRAM traffic per launch).
//
// Per iteration (partial reorthogonalisation as lanczos2.cuh; SW_PRO_TAU):
//   A: each CTA y = M_own q_j (8-row groups x 8 column lanes, 13 LDS.128 of q_j and 104 of M per
//      thread, transposing butterfly); y' = y - beta q_{j-1}; partial sums of q_j.y' and |y'|^2,
//      written to BOTH CTAs' shared memory; warps 4..7 run the omega recurrence (both CTAs, same
//      values).  cluster barrier.
//   B: alpha, beta^2 = |y'|^2 - alpha^2 from the two CTAs' partials in rank order (identical on
//      both); an exact |w|^2 round (cluster barrier) on cancellation or a due Gram-Schmidt pass
//      (dots against the global basis Q per own rows, partial h vectors exchanged); q_{j+1} rows
//      to both CTAs' x buffers and to global Q.  cluster barrier.
// Both CTAs run the convergence checks and the Ritz recurrences redundantly (same inputs, same
// results); each forms its rows of z = Q s; CTA 0 writes the scalars.
#pragma once
#include <cooperative_groups.h>
#include "lanczos2.cuh"

namespace sw {
namespace cg = cooperative_groups;

constexpr int LCL_NT = 256;
constexpr int LCL_ROWS = 104;  // rows per CTA (13 groups of 8)
struct LclLayout {
    int oM, oX, oW, oPart, oH, oAl, oBe, oB2, oRbe, oOm, oDp, oDm, oSv, oRed, oShd, total;
    __host__ __device__ LclLayout(int mp, int ld) {
        const int vl = mp + 8;
        oM = 0;
        oX = oM + LCL_ROWS * ld;  // q_j ping-pong, full length (2 vl)
        oW = oX + 2 * vl;         // w rows (own) for the reorthogonalisation dots
        oPart = oW + vl;          // 64: [0,8) alpha / |y'|^2 partials per CTA, [16,24) |w|^2, flags 40/41
        oH = oPart + 64;          // h = Q^T w: own partials [0, vl), the peer's [vl, 2 vl)
        oAl = oH + 2 * vl;
        oBe = oAl + vl;
        oB2 = oBe + vl;
        oRbe = oB2 + vl;
        oOm = oRbe + vl;          // omega rows, ring of 3
        oDp = oOm + 3 * vl;
        oDm = oDp + vl;
        oSv = oDm + vl;
        oRed = oSv + vl;          // 64
        oShd = oRed + 64;         // check state (CK_*) + thetas
        total = oShd + 40;
    }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(LCL_NT, 1) lanczos_cl_kernel(ChordParams P) {
    extern __shared__ __align__(16) double sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int h = (int)cluster.block_rank();
    double* peer = cluster.map_shared_rank(sm, h ^ 1);  // the other CTA's dynamic shared memory
    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    const LclLayout Lo(mp, ld);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = LCL_NT / 32;
    const int rg = tid >> 3, g = tid & 7;
    const int row0 = h * LCL_ROWS;
    __shared__ int sh_deg;
    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    const int ncl = gridDim.x >> 1, cl = blockIdx.x >> 1;
    for (int rr = cl; rr < count; rr += ncl) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        if (P.mode == 0 && (P.flags[slot] & CF_DONE)) continue;
        double* S = P.wS + (size_t)slot * P.w_sstride;
        const int status = (int)S[S_ST];
        const int md = (int)S[S_MD];
        cluster.sync();  // the peer finished the previous chain (its shared memory is free)
        if ((status & (ST_OUTWARD | ST_FAILED)) || md < 1) {
            if (h == 0 && tid == 0) {
                S[S_TMAX] = -SW_INF;
                S[S_TMIN] = SW_INF;
                S[S_DEG] = 0.0;
            }
            continue;
        }
        const int mdp = (md + 7) & ~7;
        const int nrows = max(0, min(LCL_ROWS, mdp - row0));  // own rows (multiple of 8)
        const int ngroups = nrows >> 3;
        double* Qg = P.wM + (size_t)slot * P.w_mstride;  // M on entry; the Lanczos basis afterwards
        // ---- own rows of M into shared memory
        const int half = mdp >> 1;
        for (int e2 = tid; e2 < nrows * half; e2 += LCL_NT) {
            const int i = e2 / half, c = 2 * (e2 - i * half);
            cp_async16(sm + Lo.oM + i * ld + c, Qg + (size_t)(row0 + i) * ld + c);
        }
        const int r = row0 + tid;                 // global row of an owner thread
        const bool owner = tid < nrows;
        const bool rowok = owner && r < md;
        double ur = 0.0;
        if (rowok) {
            const double f = (double)r * 0.6180339887498949;
            ur = 0.5 + (f - floor(f));
        }
        const double p0 = warp_sum(ur * ur);
        if (lane == 0) sm[Lo.oPart + warp] = p0;
        if (tid == 0) {
            sm[Lo.oShd + CK_INTOP] = -SW_INF;
            sm[Lo.oShd + CK_INBOT] = SW_INF;
            sm[Lo.oShd + CK_JPREV] = 0.0;
            sm[Lo.oShd + CK_LRES] = 0.0;
            sm[Lo.oShd + CK_TTOP] = -SW_INF;
            sm[Lo.oShd + CK_TBOT] = SW_INF;
            sm[Lo.oShd + CK_HINTED] = 0.0;
            sm[Lo.oOm] = 1.0;
            sm[Lo.oPart + 40] = 0.0;
            sm[Lo.oPart + 41] = 0.0;
        }
        cp_async_wait_all();
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += sm[Lo.oPart + w];
            sm[Lo.oPart + 8 + h] = s;
            peer[Lo.oPart + 8 + h] = s;
        }
        cluster.sync();  // both CTAs loaded their M rows (Q may overwrite wM now); |u_0|^2 parts
        const double nn0 = sm[Lo.oPart + 8] + sm[Lo.oPart + 9];
        double qj = rowok ? ur / sqrt(nn0) : 0.0;
        if (owner) {
            sm[Lo.oX + r] = qj;
            peer[Lo.oX + r] = qj;
            Qg[r] = qj;
        }
        double qprev = 0.0, bjm1 = 0.0, tnorm = 0.0;
        int reorth_left = 0;
        bool was_full = true;
        const double eps1 = 2.220446049250313e-16 * sqrt((double)md);
        int next_check = max(12, (md * SW_FIRST_CHECK_PCT_GLOBAL) / 100);
        const bool need_bot = P.need_tmin != 0;
        int J = 0;
        cluster.sync();
        for (int j = 0; j < md; ++j) {
            const int oXj = Lo.oX + (j & 1) * vl, oXn = Lo.oX + ((j + 1) & 1) * vl;
            // ---- A: own rows of y = M q_j (warps 0..3), omega recurrence (warps 4..7)
            double ypr = 0.0;
            if (warp < 4) {
                double acc[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = 0.0;
                const int oMr = Lo.oM + (rg * 8) * ld;
#pragma unroll
                for (int k = 0; k < 13; ++k) {
                    const int c = 2 * g + 16 * k;
                    if (rg < ngroups && c < mdp) {
                        const double2 x2 = *reinterpret_cast<const double2*>(sm + oXj + c);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const double2 m2 = *reinterpret_cast<const double2*>(sm + oMr + i * ld + c);
                            acc[i] = fma(m2.x, x2.x, acc[i]);
                            acc[i] = fma(m2.y, x2.y, acc[i]);
                        }
                    }
                }
                const double y = lz2_butterfly(acc, g);  // own row tid
                ypr = rowok ? y - bjm1 * qprev : 0.0;
                const double pa = warp_sum(qj * ypr), pn = warp_sum(ypr * ypr);
                if (lane == 0) {
                    sm[Lo.oPart + warp] = pa;
                    sm[Lo.oPart + 4 + warp] = pn;
                }
            } else if (j >= 1) {
                const int oRj = Lo.oOm + (j % 3) * vl, oR1 = Lo.oOm + ((j + 2) % 3) * vl,
                          oR2 = Lo.oOm + ((j + 1) % 3) * vl;
                const double sj = sm[Lo.oRbe + j - 1];
                for (int k = tid - 128; k <= j; k += 128) {
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
                        if (fabs(v) > SW_PRO_TAU) sm[Lo.oPart + 40 + (j & 1)] = 1.0;
                    }
                    sm[oRj + k] = v;
                }
            }
            __syncthreads();
            if (tid == 0) {  // this CTA's sums to both CTAs (slots 8 + h: alpha, 10 + h: |y'|^2)
                const double a = (sm[Lo.oPart + 0] + sm[Lo.oPart + 1]) + (sm[Lo.oPart + 2] + sm[Lo.oPart + 3]);
                const double b = (sm[Lo.oPart + 4] + sm[Lo.oPart + 5]) + (sm[Lo.oPart + 6] + sm[Lo.oPart + 7]);
                sm[Lo.oPart + 8 + h] = a;
                sm[Lo.oPart + 10 + h] = b;
                peer[Lo.oPart + 8 + h] = a;
                peer[Lo.oPart + 10 + h] = b;
            }
            cluster.sync();
            // ---- B: alpha, beta; q_{j+1}
            const double alpha0 = sm[Lo.oPart + 8] + sm[Lo.oPart + 9];
            const double nny = sm[Lo.oPart + 10] + sm[Lo.oPart + 11];
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
            double nn = nny - alpha0 * alpha0;
            bool full = false;
            if (reorth || !(nn >= 0.25 * nny)) {
                if (!(nn >= 1e-12 * nny)) reorth = true;  // severe cancellation: a Gram-Schmidt pass (lanczos2)
                full = reorth;
                if (reorth) {
                    if (owner) sm[Lo.oW + tid] = wr;  // own rows, local index
                    __syncthreads();
                    // partial h_i = q_i[own rows] . w[own rows], i <= j: 8 threads per dot
                    for (int i0 = 0; i0 <= j; i0 += LCL_NT / 8) {
                        const int i = i0 + (tid >> 3), sub = tid & 7;
                        double s0 = 0.0, s1 = 0.0;
                        if (i <= j) {
                            const double* qi = Qg + (size_t)i * ld + row0;
                            double2 q2[7];
#pragma unroll
                            for (int k = 0; k < 7; ++k) {
                                const int c = 2 * sub + 16 * k;
                                q2[k] = (c < nrows) ? *reinterpret_cast<const double2*>(qi + c) : make_double2(0.0, 0.0);
                            }
#pragma unroll
                            for (int k = 0; k < 7; ++k) {
                                const int c = 2 * sub + 16 * k;
                                if (c < nrows) {
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
                        if (sub == 0 && i <= j) {
                            sm[Lo.oH + h * vl + i] = sd;
                            peer[Lo.oH + h * vl + i] = sd;
                        }
                    }
                    cluster.sync();
                    // w -= Q h on own rows (h_i = part_0 + part_1 in rank order)
                    double qa[4] = {0.0, 0.0, 0.0, 0.0};
                    if (rowok) {
                        for (int i = 0; i <= j; i += 8) {
                            double qv[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) qv[u] = (i + u <= j) ? Qg[(size_t)(i + u) * ld + r] : 0.0;
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                if (i + u <= j) {
                                    const double hi = sm[Lo.oH + i + u] + sm[Lo.oH + vl + i + u];
                                    qa[u & 3] = fma(hi, qv[u], qa[u & 3]);
                                }
                        }
                    }
                    wr = rowok ? wr - ((qa[0] + qa[1]) + (qa[2] + qa[3])) : 0.0;
                    alpha += sm[Lo.oH + j] + sm[Lo.oH + vl + j];
                }
                if (tid == 0) sm[Lo.oPart + 40 + ((j + 1) & 1)] = 0.0;
                const double pn = warp_sum(wr * wr);
                if (lane == 0) sm[Lo.oPart + 16 + warp] = pn;
                __syncthreads();
                if (tid == 0) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < NW; ++w) s += sm[Lo.oPart + 16 + w];
                    sm[Lo.oPart + 12 + h] = s;
                    peer[Lo.oPart + 12 + h] = s;
                }
                cluster.sync();
                nn = sm[Lo.oPart + 12] + sm[Lo.oPart + 13];
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
                sm[oXn + r] = qn;
                peer[oXn + r] = qn;
                Qg[(size_t)(j + 1) * ld + r] = qn;
            }
            qprev = qj;
            qj = qn;
            bjm1 = beta;
            was_full = full;
            if (P.prof && full && tid == 0 && h == 0) atomicAdd(&P.prof[29], 1ull);
            cluster.sync();  // q_{j+1} complete in both CTAs
            if (exhausted || J >= next_check) {
                lanczos_check(tid, Lo.oAl, Lo.oBe, Lo.oB2, Lo.oRbe, J, beta, tnorm, need_bot, exhausted, md, Lo.oShd,
                              P.prof);
                __syncthreads();
                if (sm[Lo.oShd + CK_DONE] != 0.0) break;
                next_check = (int)sm[Lo.oShd + CK_NEXT];
            }
        }
        const double theta_max = sm[Lo.oShd + CK_TTOP];
        const double theta_min = sm[Lo.oShd + CK_TBOT];
        Team T;
        T.tid = tid; T.nthr = LCL_NT; T.lane = lane; T.warp = warp; T.nwarps = NW;
        int* sh_r = reinterpret_cast<int*>(sm + Lo.oShd + 30);
        tri_twisted_vec(T, sm + Lo.oAl, sm + Lo.oBe, J, theta_max, sm[Lo.oBe + J - 1], sm + Lo.oDp, sm + Lo.oDm,
                        sm + Lo.oSv, sm + Lo.oRed, sh_r);
        if (h == 0 && tid == LCL_NT - 1) {
            const double th2 = theta_max - 1e-12 * fabs(theta_max);
            const int c = sturm_below(sm + Lo.oAl, sm + Lo.oBe, J, th2);
            sh_deg = (md >= 2 && J >= 2 && c <= J - 2) ? 1 : 0;
        }
        // own rows of z = Q s
        double* zg = S + S_VEC + 3 * vl;
        if (theta_max > 0.0 || P.zall) {
            for (int e = tid; e < nrows; e += LCL_NT) {
                double s0 = 0.0, s1 = 0.0;
                int i = 0;
                for (; i + 1 < J; i += 2) {
                    s0 = fma(sm[Lo.oSv + i], Qg[(size_t)i * ld + row0 + e], s0);
                    s1 = fma(sm[Lo.oSv + i + 1], Qg[(size_t)(i + 1) * ld + row0 + e], s1);
                }
                if (i < J) s0 = fma(sm[Lo.oSv + i], Qg[(size_t)i * ld + row0 + e], s0);
                zg[row0 + e] = s0 + s1;
            }
        }
        __syncthreads();
        if (h == 0 && tid == 0) {
            S[S_TMAX] = theta_max;
            S[S_TMIN] = theta_min;
            S[S_DEG] = (double)sh_deg;
            S[S_J] = (double)J;
            if (P.jlast) P.jlast[slot] = J;
            if (P.jsum) {
                atomicAdd(&P.jsum[0], (unsigned long long)J);
                atomicAdd(&P.jsum[1], 1ull);
            }
            if (P.prof) atomicAdd(&P.prof[10], (unsigned long long)J);
        }
    }
    cluster.sync();  // no CTA exits while its peer may still write into its shared memory
}

}  // namespace sw
