// lanczos2.cuh -- K2b with TWO chains resident per SM (m <= 104): the largest eigenvalue
// theta_max of the Cholesky-transformed pencil M = -L^{-1} A(v) L^{-T} (Lemma 3
// P:587-598) by Lanczos with partial reorthogonalisation, M in SHARED memory, the Lanczos basis
// Q in the chain's global work slot (the wM rows the factor kernel wrote M into: M is read
// into shared memory first), 256 threads, 2 CTAs per SM.
//
// Why: the register-resident lanczos_kernel<512, 13> holds one chain per SM (M in 52 registers
// of 512 threads fills the register file) and is bound by per-stage latency (ncu: issue slots
// 32% busy, FP64 pipe 15%, barrier + short-scoreboard stalls).  Here each CTA needs 100 KB of
// shared memory and <= 128 registers per thread, so two chains share an SM and one CTA's
// barrier waits and convergence checks overlap the other's matvecs.
//
// Per iteration (Simon's partial reorthogonalisation, as lanczos_reg's PRO):
//   A: y = M q_j by warps 0..3 (thread = 8-row group x 8 column lanes: 7 LDS.128 of q_j and
//      56 of M, 112 DFMA, a 7-shuffle transposing butterfly leaves lane g with row 8 rg + g);
//      y' = y - beta_{j-1} q_{j-1}; partial sums of q_j.y' and |y'|^2.  Warps 4..7 run the omega
//      recurrence of row j (a Gram-Schmidt pass is due when an estimate exceeds SW_PRO_TAU).
//   B: alpha, beta^2 = |y'|^2 - alpha^2 (one reduction stage; an exact |w|^2 stage when it
//      cancels more than 1/4, or when the pass is due: h = Q^T w from global Q, w -= Q h);
//      q_{j+1} = w / beta to shared memory and to global Q.
// Two barriers per iteration on the plain path.  Convergence checks (lanczos_check, warp 0)
// and the Ritz vector (tri_twisted_vec, z = Q s) as lanczos_reg.
#pragma once
#include "chord3.cuh"

#ifndef SW_FIRST_CHECK_PCT2
#define SW_FIRST_CHECK_PCT2 26  // lanczos2, md > 84: first check at 26% of md (30%: -2.5% at m = 100; r2p)
#endif
#ifndef SW_LZ2_HMC_FULL
#define SW_LZ2_HMC_FULL 1
#endif
#ifndef SW_PRO_TAU2
#define SW_PRO_TAU2 SW_PRO_TAU  // lanczos2's partial-reorthogonalisation threshold
#endif

namespace sw {

constexpr int LZ2_NT = 256;
// dynamic shared memory layout (doubles) of lanczos2_kernel for mp, ld
struct Lz2Layout {
    int oM, oX, oW, oPart, oAl, oBe, oB2, oRbe, oOm, oDp, oDm, oSv, oRed, oShd, total;
    __host__ __device__ Lz2Layout(int mp, int ld) {
        const int vl = mp + 8;
        oM = 0;
        oX = oM + mp * ld;   // q_j ping-pong (2 vl)
        oW = oX + 2 * vl;    // w (exact / reorthogonalisation paths)
        oPart = oW + vl;     // 64: warp partials, h dots
        oAl = oPart + 64 + vl;  // h (Q^T w) lives at oPart + 64
        oBe = oAl + vl;
        oB2 = oBe + vl;
        oRbe = oB2 + vl;
        oOm = oRbe + vl;     // omega rows, ring of 3
        oDp = oOm + 3 * vl;
        oDm = oDp + vl;
        oSv = oDm + vl;
        oRed = oSv + vl;     // 64
        oShd = oRed + 64;    // check state (CK_*) + thetas
        total = oShd + 40;
    }
};

// rows of the 8-row group of this thread summed over the 8 column lanes of its quarter-warp:
// a transposing butterfly (xor 4, 2, 1): lane g ends with the sum of row g
__device__ __forceinline__ double lz2_butterfly(const double (&a)[8], int g) {
    const bool b2 = (g & 4) != 0, b1 = (g & 2) != 0, b0 = (g & 1) != 0;
    double v[4], w[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double send = b2 ? a[i] : a[i + 4];
        const double keep = b2 ? a[i + 4] : a[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = b1 ? v[i] : v[i + 2];
        const double keep = b1 ? v[i + 2] : v[i];
        w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    const double send = b0 ? w[0] : w[1];
    const double keep = b0 ? w[1] : w[0];
    return keep + __shfl_xor_sync(0xffffffffu, send, 1);
}

__global__ void __launch_bounds__(LZ2_NT, 2) lanczos2_kernel(ChordParams P) {
    extern __shared__ __align__(16) double sm[];
    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const int vl = mp + 8;
    const Lz2Layout Lo(mp, ld);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = LZ2_NT / 32;
    const int rg = tid >> 3, g = tid & 7;  // matvec: row group, column lane
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
        double* Qg = P.wM + (size_t)slot * P.w_mstride;  // M on entry; the Lanczos basis afterwards
        // ---- M (md x mdp, zero padded) into shared memory
        for (int e2 = tid; e2 < mdp * (mdp >> 1); e2 += LZ2_NT) {
            const int i = e2 / (mdp >> 1), c = 2 * (e2 - i * (mdp >> 1));
            cp_async16(sm + Lo.oM + i * ld + c, Qg + (size_t)i * ld + c);
        }
        // start vector u_0 (as lanczos_reg), |u_0|^2 partials
        const bool owner = tid < mdp;
        const bool rowok = tid < md;
        double ur = 0.0;
        if (rowok) {
            const double f = (double)tid * 0.6180339887498949;
            ur = 0.5 + (f - floor(f));
        }
        double p0 = warp_sum(ur * ur);
        if (lane == 0) sm[Lo.oPart + warp] = p0;
        if (tid == 0) {
            sm[Lo.oShd + CK_INTOP] = -SW_INF;
            sm[Lo.oShd + CK_INBOT] = SW_INF;
            sm[Lo.oShd + CK_JPREV] = 0.0;
            sm[Lo.oShd + CK_LRES] = 0.0;
            sm[Lo.oShd + CK_TTOP] = -SW_INF;
            sm[Lo.oShd + CK_TBOT] = SW_INF;
            sm[Lo.oShd + CK_HINTED] = 0.0;
            sm[Lo.oOm] = 1.0;  // omega_{0,0}
            sm[Lo.oPart + 40] = 0.0;
            sm[Lo.oPart + 41] = 0.0;
        }
        cp_async_wait_all();
        __syncthreads();
        double nn0 = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) nn0 += sm[Lo.oPart + w];
        double qj = rowok ? ur / sqrt(nn0) : 0.0;  // q_j[r] (owners)
        __syncthreads();  // M loaded everywhere before Q overwrites the global rows
        if (owner) {
            sm[Lo.oX + tid] = qj;
            Qg[tid] = qj;
        }
        double qprev = 0.0, bjm1 = 0.0, tnorm = 0.0;
        int reorth_left = 0;
        bool was_full = true;
        const double eps1 = 2.220446049250313e-16 * sqrt((double)md);
        int next_check = (md <= SW_FIRST_CHECK_FULL_MD) ? md
                       : (md <= SW_FIRST_CHECK_SMALL_MD) ? (md * SW_FIRST_CHECK_PCT_SMALL) / 100
                       : (md <= 64) ? (md * SW_FIRST_CHECK_PCT_MID) / 100
                       : (md <= 84) ? max(12, (md * SW_FIRST_CHECK_PCT) / 100) : max(12, (md * SW_FIRST_CHECK_PCT2) / 100);
        // HMC-r's lambda_min(N_1) solves (P.zall): their own first-check rule (lanczos_kernel's)
        if (P.zall && md > SW_FIRST_PCT_MIN_MD) next_check = max(12, (md * SW_FIRST_CHECK_PCT_HMC) / 100);
        const bool need_bot = P.need_tmin && !P.zall;
        int J = 0;
        const int ngroups = mdp >> 3;
        __syncthreads();
        for (int j = 0; j < md; ++j) {
            const int oXj = Lo.oX + (j & 1) * vl, oXn = Lo.oX + ((j + 1) & 1) * vl;
            // ---- A: y = M q_j (warps 0..3), omega recurrence (warps 4..7)
            double ypr = 0.0;
            if (warp < 4) {  // whole warps: the butterfly shuffles need every lane
                double acc[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = 0.0;
                const int oMr = Lo.oM + (rg * 8) * ld;
#pragma unroll
                for (int k = 0; k < 7; ++k) {
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
                const double y = lz2_butterfly(acc, g);  // row tid
                ypr = rowok ? y - bjm1 * qprev : 0.0;
            }
            if (warp < 4) {
                const double pa = warp_sum(qj * ypr), pn = warp_sum(ypr * ypr);
                if (lane == 0) {
                    sm[Lo.oPart + warp] = pa;
                    sm[Lo.oPart + 8 + warp] = pn;
                }
            } else if (j >= 1) {
                // omega_{j,k} = q_j . q_k estimates (Simon 1984): rows j-1, j-2 of the ring, or the
                // rounding level after a full orthogonalisation of w_{j-1}; flag > SW_PRO_TAU
                const int oRj = Lo.oOm + (j % 3) * vl, oR1 = Lo.oOm + ((j + 2) % 3) * vl,
                          oR2 = Lo.oOm + ((j + 1) % 3) * vl;
                const double sj = sm[Lo.oRbe + j - 1];  // 1 / beta_{j-1}
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
                        if (fabs(v) > SW_PRO_TAU2) sm[Lo.oPart + 40 + (j & 1)] = 1.0;
                    }
                    sm[oRj + k] = v;
                }
            }
            __syncthreads();
            // ---- B: alpha, beta; q_{j+1}
            const double alpha0 = (sm[Lo.oPart + 0] + sm[Lo.oPart + 1]) + (sm[Lo.oPart + 2] + sm[Lo.oPart + 3]);
            const double nny = (sm[Lo.oPart + 8] + sm[Lo.oPart + 9]) + (sm[Lo.oPart + 10] + sm[Lo.oPart + 11]);
            // w_0 against q_0 exactly (no recurrence history); HMC-r's -N_1 solves (P.zall) take a full
            // Gram-Schmidt pass every iteration (their Ritz vector is the hit's kernel vector)
            bool reorth = (j == 0) || (P.zall && SW_LZ2_HMC_FULL);
            if (reorth_left > 0) {
                reorth = true;
                --reorth_left;
            } else if (j >= 1 && sm[Lo.oPart + 40 + (j & 1)] != 0.0) {
                reorth = true;
                reorth_left = 1;
            }
            double alpha = alpha0;
            double wr = rowok ? ypr - alpha * qj : 0.0;
            double nn = nny - alpha0 * alpha0;  // |w|^2 by Pythagoras (q_j unit, w = y' - alpha q_j)
            bool full = false;
            if (reorth || !(nn >= 0.25 * nny)) {
                // exact |w|^2 when the three-term step cancelled more than 3/4 of |y'|^2; one
                // Gram-Schmidt pass of w against q_0..q_j when due, and whenever it cancelled all
                // but 1e-6 of |y'| (the residual is then mostly rounding and has lost orthogonality,
                // as at an invariant subspace of a low-rank M: lanczos_run's criterion)
                if (!(nn >= 1e-12 * nny)) reorth = true;
                full = reorth;
                if (reorth) {
                    if (owner) sm[Lo.oW + tid] = wr;
                    if (tid == 0) sm[Lo.oPart + 40 + ((j + 1) & 1)] = 0.0;
                    __syncthreads();
                    // h_i = q_i . w, i <= j (Q rows from global / L2): 8 threads per dot, 32 dots per
                    // pass, each thread's 7 double2 loads issued together
                    for (int i0 = 0; i0 <= j; i0 += LZ2_NT / 8) {
                        const int i = i0 + (tid >> 3), sub = tid & 7;
                        double s0 = 0.0, s1 = 0.0;
                        if (i <= j) {
                            const double* qi = Qg + (size_t)i * ld;
                            double2 q2[7];
#pragma unroll
                            for (int k = 0; k < 7; ++k) {
                                const int c = 2 * sub + 16 * k;
                                q2[k] = (c < mdp) ? *reinterpret_cast<const double2*>(qi + c) : make_double2(0.0, 0.0);
                            }
#pragma unroll
                            for (int k = 0; k < 7; ++k) {
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
                    // w -= Q h: row r = tid & 127, the two thread halves take alternate rows of Q
                    // (8 loads in flight each), the upper half's partial through shared memory
                    const int rq = tid & 127, hq = tid >> 7;
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
                    const double qh0 = qpart, qh1 = (rowok && tid < 128) ? sm[Lo.oW + tid] : 0.0;
                    wr = rowok ? wr - (qh0 + qh1) : 0.0;
                    alpha += sm[Lo.oPart + 64 + j];
                }
                if (tid == 0) sm[Lo.oPart + 40 + ((j + 1) & 1)] = 0.0;
                const double pn = warp_sum(wr * wr);
                if (lane == 0) sm[Lo.oPart + 16 + warp] = pn;
                __syncthreads();
                nn = 0.0;
#pragma unroll
                for (int w = 0; w < NW; ++w) nn += sm[Lo.oPart + 16 + w];
                // nothing but rounding left after the pass: the Krylov space is invariant (beta = 0)
                if (nn < 1e-28 * nny) nn = 0.0;
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
            qprev = qj;
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
        T.tid = tid; T.nthr = LZ2_NT; T.lane = lane; T.warp = warp; T.nwarps = NW;
        int* sh_r = reinterpret_cast<int*>(sm + Lo.oShd + 30);
        tri_twisted_vec(T, sm + Lo.oAl, sm + Lo.oBe, J, theta_max, sm[Lo.oBe + J - 1], sm + Lo.oDp, sm + Lo.oDm,
                        sm + Lo.oSv, sm + Lo.oRed, sh_r);
        if (P.jlast && tid == 0) P.jlast[slot] = J;
        if (P.jsum && tid == 0) {
            atomicAdd(&P.jsum[0], (unsigned long long)J);
            atomicAdd(&P.jsum[1], 1ull);
        }
        if (tid == LZ2_NT - 1) {
            const double th2 = theta_max - 1e-12 * fabs(theta_max);
            const int c = sturm_below(sm + Lo.oAl, sm + Lo.oBe, J, th2);
            sh_deg = (md >= 2 && J >= 2 && c <= J - 2) ? 1 : 0;
        }
        // z = Q s (rows of Q: the normalised Lanczos vectors, global)
        double* zg = S + S_VEC + 3 * vl;
        if (theta_max > 0.0 || P.zall) {
            for (int e = tid; e < mdp; e += LZ2_NT) {
                double s0 = 0.0, s1 = 0.0;
                int i = 0;
                for (; i + 1 < J; i += 2) {
                    s0 = fma(sm[Lo.oSv + i], Qg[(size_t)i * ld + e], s0);
                    s1 = fma(sm[Lo.oSv + i + 1], Qg[(size_t)(i + 1) * ld + e], s1);
                }
                if (i < J) s0 = fma(sm[Lo.oSv + i], Qg[(size_t)i * ld + e], s0);
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

}  // namespace sw
