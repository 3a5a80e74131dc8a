// chord2.cuh -- K2 v2: the per-chain boundary oracle, blocked and tensor-core based.
//
// Same mathematics as PAPER.md Alg. 2 / Lemma 3 and the
// Cholesky-transformed pencil of P:1207-1215, reorganised for sm_100a:
//   L L^T = A(x)              blocked right-looking Cholesky, nb = 8; the trailing
//                             SYRK updates are DMMA m8n8k4 tiles
//   M = -L^{-1} A(v) L^{-T}   two blocked TRSMs (natural and transposed view),
//                             updates on DMMA tiles
//   theta_max = lambda_max(M) Lanczos with full (CGS2) reorthogonalisation, M
//                             register-resident across the CTA; convergence
//                             checked on T_J by Sturm multisection plus the
//                             residual beta_J |s_J| of the top Ritz pair
//   y = L^{-T} Q s            the PEP eigenvector; t+ = 1/theta_max
// Boundary starts (after a reflection) are Schur-deflated by the known kernel
// vector (R6) and shifted to an aligned (m-1) problem.
#pragma once
#include "chord.cuh"

namespace sw {

constexpr int NVEC2 = 20;
#ifndef SW_GLOBAL_LL
#define SW_GLOBAL_LL 1  // global-scratch variant (m > 112): left-looking congruence
#endif
#ifndef SW_PRO_RUN
#define SW_PRO_RUN 1
#endif
#ifndef SW_PRO_TAU
#define SW_PRO_TAU 1e-13  // reorthogonalise once an omega estimate exceeds this: at 1e-10 the Ritz
                          // vector (the normal) carried errors up to 4e-9 at m = 200 and 13 of 64
                          // configs[4] trajectories left 1e-8 by reflection 20 (profiles/r2c_*); -1.2%
#endif
#ifndef SW_CHECK_STEP0
#define SW_CHECK_STEP0 4    // iterations from the first check to the second (no rate known yet; measured)
#endif
#ifndef SW_CHECK_STEPMAX
#define SW_CHECK_STEPMAX 8  // cap on the rate-predicted distance to the next check
#endif
#ifndef SW_FIRST_CHECK_PCT
#define SW_FIRST_CHECK_PCT 30  // m > 64 (measured: 25-30% of md ~+7% over 40% at m = 100)
#endif
#ifndef SW_FIRST_CHECK_FULL_MD
#define SW_FIRST_CHECK_FULL_MD 36  // up to here the first check is at J = md (the whole space: ~+50% at m = 30)
#endif
#ifndef SW_FIRST_CHECK_PCT_HMC
#define SW_FIRST_CHECK_PCT_HMC 10  // lambda_min(N_1) solves of HMC-r (lanczos_kernel with zall), m > 64 (measured)
#endif
#ifndef SW_FIRST_PCT_MIN_MD
#define SW_FIRST_PCT_MIN_MD 12  // the caller's first-check rule applies above this md (HMC-r: measured +5..35% at m = 16..60)
#endif
#ifndef SW_FIRST_CHECK_PCT_GLOBAL
#define SW_FIRST_CHECK_PCT_GLOBAL 15  // global-scratch variant (m > 112): costlier iterations, cheap checks (measured)
#endif
#ifndef SW_FIRST_CHECK_PCT_SMALL
#define SW_FIRST_CHECK_PCT_SMALL 88  // SW_FIRST_CHECK_FULL_MD < m <= SW_FIRST_CHECK_SMALL_MD (measured)
#endif
#ifndef SW_FIRST_CHECK_SMALL_MD
#define SW_FIRST_CHECK_SMALL_MD 48
#endif
#ifndef SW_FIRST_CHECK_PCT_MID
#define SW_FIRST_CHECK_PCT_MID 50  // SW_FIRST_CHECK_SMALL_MD < m <= 64
#endif
#ifndef SW_LANCZOS_TOL
// Lanczos convergence: residual of the top Ritz pair <= SW_LANCZOS_TOL |T_J|.  The Ritz value
// error is ~res^2 / gap; the Ritz vector (the kernel vector y, the normal) error ~res / gap.
#define SW_LANCZOS_TOL 1e-13
#endif
#ifndef SW_PROF_LANCZOS
#define SW_PROF_LANCZOS 0  // per-stage clock64 counters of lanczos_reg (build with -DSW_PROF_LANCZOS=1)
#endif

__device__ __forceinline__ void dmma_t(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// Conflict-free access to the DMMA accumulator pair C[r][2q], C[r][2q+1] (rows of an even
// leading dimension ld = 4 or 12 mod 16): odd rows touch their two elements in the opposite
// order, so each of the two 8-byte accesses of a half-warp hits 16 distinct bank slots (in
// order, rows r and r+1 collide: 2-way conflicts on every tile load / store, ncu r2fs).
__device__ __forceinline__ void acc_ld(double (&acc)[2], const double* C, int ld, int r, int q) {
    const int sw = r & 1;
    const double v0 = C[r * ld + 2 * q + sw];
    const double v1 = C[r * ld + 2 * q + 1 - sw];
    acc[0] = sw ? v1 : v0;
    acc[1] = sw ? v0 : v1;
}
__device__ __forceinline__ void acc_st(const double (&acc)[2], double* C, int ld, int r, int q) {
    const int sw = r & 1;
    C[r * ld + 2 * q + sw] = sw ? acc[1] : acc[0];
    C[r * ld + 2 * q + 1 - sw] = sw ? acc[0] : acc[1];
}

// acc(8x8) -= A(8 x K) * B(K x 8).  A row-major (lda).  B element (k, c) at
// Bp[k*ldb + c] (BNK = false) or Bp[c*ldb + k] (BNK = true).
template <bool BNK>
__device__ __forceinline__ void tile_msub(double (&acc)[2], const double* A, int lda, const double* Bp, int ldb,
                                          int K, int lane) {
    const int r = lane >> 2, q = lane & 3;
#pragma unroll 2
    for (int k0 = 0; k0 < K; k0 += 4) {
        double a = -A[r * lda + k0 + q];
        double b = BNK ? Bp[r * ldb + k0 + q] : Bp[(k0 + q) * ldb + r];
        dmma_t(acc, a, b);
    }
}

// X <- H X H and Y <- H Y H together (H = I - beta h h^T, X, Y symmetric m x m)
// apply = false: only the rank-2 vectors p (X <- X - h p^T - p h^T is left to the caller, who may
// fuse it into its next pass over the matrices)
__device__ void householder_congruence2(const Team& T, double* X, double* Y, int m, int ld, const double* h,
                                        double beta, double* px, double* py, double* red, bool apply = true) {
    for (int i = T.warp; i < m; i += T.nwarps) {
        double sx = 0.0, sy = 0.0;
        for (int j = T.lane; j < m; j += 32) {
            const double hj = h[j];
            sx += X[i * ld + j] * hj;
            sy += Y[i * ld + j] * hj;
        }
        sx = warp_sum(sx);
        sy = warp_sum(sy);
        if (T.lane == 0) {
            px[i] = beta * sx;
            py[i] = beta * sy;
        }
    }
    __syncthreads();
    double hx = 0.0, hy = 0.0;
    for (int i = T.tid; i < m; i += T.nthr) {
        hx += h[i] * px[i];
        hy += h[i] * py[i];
    }
    hx = warp_sum(hx);
    hy = warp_sum(hy);
    if (T.lane == 0) {
        red[T.warp] = hx;
        red[32 + T.warp] = hy;
    }
    __syncthreads();
    double Kx = 0.0, Ky = 0.0;
    for (int w = 0; w < T.nwarps; ++w) {
        Kx += red[w];
        Ky += red[32 + w];
    }
    Kx *= 0.5 * beta;
    Ky *= 0.5 * beta;
    __syncthreads();
    for (int i = T.tid; i < m; i += T.nthr) {
        px[i] -= Kx * h[i];
        py[i] -= Ky * h[i];
    }
    __syncthreads();
    if (!apply) return;
    for (int i = T.warp; i < m; i += T.nwarps) {
        const double hi = h[i], pxi = px[i], pyi = py[i];
        for (int j = T.lane; j < m; j += 32) {
            const double hj = h[j];
            X[i * ld + j] -= hi * px[j] + pxi * hj;
            Y[i * ld + j] -= hi * py[j] + pyi * hj;
        }
    }
    __syncthreads();
}

// blocked right-looking Cholesky of the lower triangle of G (n = multiple of 8)
__device__ bool cholesky_blocked(const Team& T, double* G, int n, int ld, double* rdiag, int* flag) {
    const int TB = n >> 3;
    for (int kb = 0; kb < TB; ++kb) {
        const int k0 = kb * 8;
        double* D = G + k0 * ld + k0;
        if (T.warp == 0) {
            // 8x8 diagonal block in registers: lane r < 8 holds row r (lower part)
            double a[8];
            const int r = T.lane;
#pragma unroll
            for (int c = 0; c < 8; ++c) a[c] = (r < 8 && c <= r) ? D[r * ld + c] : 0.0;
            bool ok = true;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const double d = __shfl_sync(0xffffffffu, a[c], c);
                if (!(d > 0.0)) ok = false;
                const double l = sqrt(fmax(d, 1e-300));
                const double il = 1.0 / l;
                if (r == c) a[c] = l;
                else if (r > c) a[c] *= il;
#pragma unroll
                for (int k = c + 1; k < 8; ++k) {
                    const double lkc = __shfl_sync(0xffffffffu, a[c], k);
                    if (r >= k) a[k] -= a[c] * lkc;
                }
            }
            if (r < 8) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c <= r) D[r * ld + c] = a[c];
                double dg = a[0];
#pragma unroll
                for (int c = 1; c < 8; ++c)
                    if (c == r) dg = a[c];
                rdiag[k0 + r] = 1.0 / dg;
            }
            if (T.lane == 0) *flag = ok ? 0 : 1;
        }
        __syncthreads();
        if (*flag) return false;
        // panel TRSM: rows below the diagonal block, P = G_ib,kb L_kk^{-T}
        for (int i = k0 + 8 + T.tid; i < n; i += T.nthr) {
            double x[8];
            double* row = G + i * ld + k0;
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = row[c];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                double s = x[c];
#pragma unroll
                for (int cp = 0; cp < c; ++cp) s -= x[cp] * D[c * ld + cp];
                x[c] = s * rdiag[k0 + c];
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) row[c] = x[c];
        }
        __syncthreads();
        // trailing SYRK on DMMA tiles: G_ij -= P_i P_j^T, kb < j <= i
        const int Tr = TB - kb - 1;
        const int ntile = Tr * (Tr + 1) / 2;
        for (int t = T.warp; t < ntile; t += T.nwarps) {
            int ii = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
            while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
            while (ii * (ii + 1) / 2 > t) --ii;
            int jj = t - ii * (ii + 1) / 2;
            int ib = kb + 1 + ii, jb = kb + 1 + jj;
            double* C = G + ib * 8 * ld + jb * 8;
            const int r = T.lane >> 2, q = T.lane & 3;
            double acc[2] = {C[r * ld + 2 * q], C[r * ld + 2 * q + 1]};
            tile_msub<true>(acc, G + ib * 8 * ld + k0, ld, G + jb * 8 * ld + k0, ld, 8, T.lane);
            C[r * ld + 2 * q] = acc[0];
            C[r * ld + 2 * q + 1] = acc[1];
        }
        __syncthreads();
    }
    return true;
}

// B <- L^{-1} B on all n columns.  TR = true works on the transposed view
// W(r, c) = B[c*ld + r].  Blocked right-looking, DMMA tile updates.
template <bool TR>
__device__ void trsm_blocked(const Team& T, const double* G, double* B, int n, int ld, const double* rdiag) {
    const int TB = n >> 3;
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int kb = 0; kb < TB; ++kb) {
        const int k0 = kb * 8;
        const double* D = G + k0 * ld + k0;
        for (int c = T.tid; c < n; c += T.nthr) {
            double x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = TR ? B[c * ld + k0 + i] : B[(k0 + i) * ld + c];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double s = x[i];
#pragma unroll
                for (int ip = 0; ip < i; ++ip) s -= D[i * ld + ip] * x[ip];
                x[i] = s * rdiag[k0 + i];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (TR) B[c * ld + k0 + i] = x[i];
                else B[(k0 + i) * ld + c] = x[i];
            }
        }
        __syncthreads();
        const int nt = (TB - kb - 1) * TB;
        for (int t = T.warp; t < nt; t += T.nwarps) {
            int ib = kb + 1 + t / TB, cb = t % TB;
            const double* A = G + ib * 8 * ld + k0;
            double acc[2];
            if (!TR) {
                double* C = B + ib * 8 * ld + cb * 8;
                acc[0] = C[r * ld + 2 * q];
                acc[1] = C[r * ld + 2 * q + 1];
                tile_msub<false>(acc, A, ld, B + k0 * ld + cb * 8, ld, 8, T.lane);
                C[r * ld + 2 * q] = acc[0];
                C[r * ld + 2 * q + 1] = acc[1];
            } else {
                double* Ct = B + cb * 8 * ld + ib * 8;  // W tile (ib, cb), element (r, c) at Ct[c*ld + r]
                acc[0] = Ct[(2 * q) * ld + r];
                acc[1] = Ct[(2 * q + 1) * ld + r];
                tile_msub<true>(acc, A, ld, B + cb * 8 * ld + k0, ld, 8, T.lane);
                Ct[(2 * q) * ld + r] = acc[0];
                Ct[(2 * q + 1) * ld + r] = acc[1];
            }
        }
        __syncthreads();
    }
}

// Extreme eigenvalue of the symmetric tridiagonal (al, be) of size J by
// Laguerre's method on p(x) = det(x I - T) (all roots real): started above the
// spectrum (top) it decreases monotonically to lambda_max, started below it
// increases monotonically to lambda_min; cubic convergence.  p, p', p'' by the
// three-term recurrence with exact power-of-two rescaling.  One thread.
__device__ double tri_laguerre(const double* al, const double* be, int J, double x) {
    const double eps = 2.220446049250313e-16;
    if (J == 1) return al[0];
    const double n = (double)J;
    for (int it = 0; it < 40; ++it) {
        double p0 = 1.0, d0 = 0.0, s0 = 0.0;          // p_{i-1}, p'_{i-1}, p''_{i-1}
        double p1 = x - al[0], d1 = 1.0, s1 = 0.0;   // p_i ...
        for (int i = 1; i < J; ++i) {
            const double t = x - al[i], b2 = be[i - 1] * be[i - 1];
            const double p2 = t * p1 - b2 * p0;
            const double d2 = p1 + t * d1 - b2 * d0;
            const double s2 = 2.0 * d1 + t * s1 - b2 * s0;
            p0 = p1; d0 = d1; s0 = s1;
            p1 = p2; d1 = d2; s1 = s2;
            const double ap = fmax(fabs(p1), fmax(fabs(d1), fabs(s1)));
            if (ap > 0x1p+400) {
                p0 *= 0x1p-400; d0 *= 0x1p-400; s0 *= 0x1p-400;
                p1 *= 0x1p-400; d1 *= 0x1p-400; s1 *= 0x1p-400;
            } else if (ap < 0x1p-400) {
                p0 *= 0x1p+400; d0 *= 0x1p+400; s0 *= 0x1p+400;
                p1 *= 0x1p+400; d1 *= 0x1p+400; s1 *= 0x1p+400;
            }
        }
        if (p1 == 0.0) return x;
        const double G = d1 / p1;
        const double H = G * G - s1 / p1;
        const double disc = fmax((n - 1.0) * (n * H - G * G), 0.0);
        const double den = G + copysign(sqrt(disc), G);
        if (den == 0.0) return x;
        const double step = n / den;
        x -= step;
        if (fabs(step) <= 2.0 * eps * fabs(x)) break;
    }
    return x;
}

// Eigenvector s of the tridiagonal T_J (al, be) for the eigenvalue theta by a
// twisted factorisation (Parlett-Dhillon): forward pivots D+ and backward
// pivots D- of (T - theta I), twist index r = argmin |gamma_r|,
// gamma_r = D+_r + D-_r - (al_r - theta); s_r = 1 and the two product sweeps
// s_i = -(be_i / D+_i) s_{i+1} (i < r), s_i = -(be_{i-1} / D-_i) s_{i-1} (i > r).
// Returns (to every thread) the Lanczos residual |beta_last| |s_{J-1}| / |s|;
// s is normalised.  CTA-cooperative; dp, dm scratch of length J.
__device__ __noinline__ double tri_twisted_vec(const Team& T, const double* al, const double* be, int J, double theta,
                                  double beta_last, double* dp, double* dm, double* s, double* red, int* sh_r) {
    const double tiny = 1e-290;
    if (T.tid == 0) {
        double d = al[0] - theta;
        dp[0] = d;
        for (int i = 1; i < J; ++i) {
            double prev = dp[i - 1];
            if (fabs(prev) < tiny) prev = (prev < 0.0 ? -tiny : tiny);
            d = (al[i] - theta) - be[i - 1] * be[i - 1] / prev;
            dp[i] = d;
        }
    } else if (T.tid == 32 || (T.nthr <= 32 && T.tid == 1)) {
        double d = al[J - 1] - theta;
        dm[J - 1] = d;
        for (int i = J - 2; i >= 0; --i) {
            double nxt = dm[i + 1];
            if (fabs(nxt) < tiny) nxt = (nxt < 0.0 ? -tiny : tiny);
            d = (al[i] - theta) - be[i] * be[i] / nxt;
            dm[i] = d;
        }
    }
    __syncthreads();
    if (T.warp == 0) {
        double bg = SW_INF;
        int br = 0;
        for (int i = T.lane; i < J; i += 32) {
            double g = fabs(dp[i] + dm[i] - (al[i] - theta));
            if (g < bg) { bg = g; br = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            double og = __shfl_xor_sync(0xffffffffu, bg, o);
            int orr = __shfl_xor_sync(0xffffffffu, br, o);
            if (og < bg || (og == bg && orr < br)) { bg = og; br = orr; }
        }
        if (T.lane == 0) *sh_r = br;
    }
    __syncthreads();
    const int r = *sh_r;
    // the quotients of the two eigenvector recurrences do not depend on the recurrence:
    // all threads form them first (one division each), the chains are then multiplications
    for (int i = T.tid; i < J; i += T.nthr) {
        if (i == r) continue;
        double piv = (i < r) ? dp[i] : dm[i];
        if (fabs(piv) < tiny) piv = (piv < 0.0 ? -tiny : tiny);
        s[i] = ((i < r) ? be[i] : be[i - 1]) / piv;
    }
    __syncthreads();
    if (T.tid == 0) {
        s[r] = 1.0;
        double prev = 1.0;
        for (int i = r - 1; i >= 0; --i) {
            double v = -s[i] * prev;
            if (fabs(v) > 1e200) v = copysign(1e200, v);
            s[i] = v;
            prev = v;
        }
    } else if (T.tid == 32 || (T.nthr <= 32 && T.tid == 1)) {
        double prev = 1.0;
        for (int i = r + 1; i < J; ++i) {
            double v = -s[i] * prev;
            if (fabs(v) > 1e200) v = copysign(1e200, v);
            s[i] = v;
            prev = v;
        }
    }
    __syncthreads();
    double nn = 0.0, mx = 0.0;
    for (int i = T.tid; i < J; i += T.nthr) mx = fmax(mx, fabs(s[i]));
    mx = block_max(T, mx, red);
    double sc = 1.0 / mx;
    for (int i = T.tid; i < J; i += T.nthr) {
        double v = s[i] * sc;
        nn += v * v;
    }
    nn = block_sum(T, nn, red);
    double inv = sc / sqrt(nn);
    for (int i = T.tid; i < J; i += T.nthr) s[i] *= inv;
    __syncthreads();
    return fabs(beta_last) * fabs(s[J - 1]);
}


// |s_J| / |s| for the eigenvector s of the tridiagonal T_J (al, be) at the
// eigenvalue th, by the backward recurrence from s_J = 1 (the top Ritz vector
// grows towards the first Lanczos indices, so this direction is stable);
// rbe = 1 / be.  One thread.  The Lanczos residual is be[J-1] times this.
__device__ double tri_back_lastcomp(const double* al, const double* be, const double* rbe, int J, double th) {
    if (J <= 1) return 1.0;
    double sJ = 1.0, s1 = 1.0;
    double s0 = (th - al[J - 1]) * rbe[J - 2];
    double nn = 1.0 + s0 * s0;
    for (int i = J - 2; i >= 1; --i) {
        const double sm = ((th - al[i]) * s0 - be[i] * s1) * rbe[i - 1];
        s1 = s0;
        s0 = sm;
        nn += sm * sm;
        if (nn > 0x1p+600) {
            s0 *= 0x1p-300; s1 *= 0x1p-300; sJ *= 0x1p-300; nn *= 0x1p-600;
        }
    }
    return sJ / sqrt(nn);
}

// |s_J| / |s| of the eigenvector of T_J at the eigenvalue th (backward
// recurrence from s_J = 1, as tri_back_lastcomp) on shared-memory arrays.
__device__ double tri_back_lastcomp_sm(const int oA, const int oB, const int oRB, const int J, const double th) {
    extern __shared__ __align__(16) double sm[];
    if (J <= 1) return 1.0;
    double sJ = 1.0, s1 = 1.0;
    double s0 = (th - sm[oA + J - 1]) * sm[oRB + J - 2];
    double nn = 1.0 + s0 * s0;
    // i = J-2 .. 1 in groups of 4: the coefficients of a group (loads, products)
    // are formed before its chain, so the chain itself is one FMA per step; full
    // groups run without per-step predicates
    auto step = [&](const double c, const double d) {
        const double sm_ = fma(c, s0, d * s1);
        s1 = s0;
        s0 = sm_;
        nn = fma(sm_, sm_, nn);
    };
    int i0 = J - 2;
    for (; i0 - 3 >= 1; i0 -= 4) {
        double c[4], d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int ii = i0 - u;
            const double rb = sm[oRB + ii - 1];
            c[u] = (th - sm[oA + ii]) * rb;
            d[u] = -sm[oB + ii] * rb;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) step(c[u], d[u]);
        if (nn > 0x1p+600) {
            s0 *= 0x1p-300; s1 *= 0x1p-300; sJ *= 0x1p-300; nn *= 0x1p-600;
        }
    }
    if (i0 >= 1) {  // the last, partial group (1..3 steps)
        for (int ii = i0; ii >= 1; --ii) {
            const double rb = sm[oRB + ii - 1];
            step((th - sm[oA + ii]) * rb, -sm[oB + ii] * rb);
        }
        if (nn > 0x1p+600) {
            s0 *= 0x1p-300; s1 *= 0x1p-300; sJ *= 0x1p-300; nn *= 0x1p-600;
        }
    }
    return sJ / sqrt(nn);
}

// p_J(x), p_J'(x), p_J''(x) of T_J by the three-term recurrence (one lane, its own x), in
// groups of 4 steps with a 2^+-400 rescale after each group; SIGNS also tracks whether every
// p_i has the sign of "x outside the spectrum" (Sturm: above all for top, below all for bottom).
// Full groups run without per-step predicates (no divergence bookkeeping in the chain).
template <bool SIGNS>
__device__ __forceinline__ bool tri_charpoly3(const int oA, const int oB2, const int J, const double x, const bool top,
                                              double& p1, double& d1, double& s1) {
    extern __shared__ __align__(16) double sm[];
    double p0 = 1.0, d0 = 0.0, s0 = 0.0;
    p1 = x - sm[oA];
    d1 = 1.0;
    s1 = 0.0;
    bool outside = top ? (p1 > 0.0) : (p1 < 0.0);
    auto step = [&](const double a, const double b2, const int i) {
        const double t = x - a;
        const double qp = -b2 * p0, qd = fma(-b2, d0, p1), qs = fma(-b2, s0, 2.0 * d1);
        p0 = p1; d0 = d1; s0 = s1;
        p1 = fma(t, p0, qp);
        d1 = fma(t, d0, qd);
        s1 = fma(t, s0, qs);
        if (SIGNS) outside = outside && (top ? (p1 > 0.0) : ((i & 1) ? (p1 > 0.0) : (p1 < 0.0)));
    };
    auto rescale = [&]() {
        const double ap = fmax(fabs(p1), fmax(fabs(d1), fabs(s1)));
        if (ap > 0x1p+400) {
            p0 *= 0x1p-400; d0 *= 0x1p-400; s0 *= 0x1p-400;
            p1 *= 0x1p-400; d1 *= 0x1p-400; s1 *= 0x1p-400;
        } else if (ap < 0x1p-400) {
            p0 *= 0x1p+400; d0 *= 0x1p+400; s0 *= 0x1p+400;
            p1 *= 0x1p+400; d1 *= 0x1p+400; s1 *= 0x1p+400;
        }
    };
    int i0 = 1;
    double an[4], bn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { an[u] = sm[oA + 1 + u]; bn[u] = sm[oB2 + u]; }
    for (; i0 + 3 < J; i0 += 4) {  // full groups (reads up to 7 slots past J: values unused)
        double ac[4], bc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { ac[u] = an[u]; bc[u] = bn[u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u) { an[u] = sm[oA + i0 + 4 + u]; bn[u] = sm[oB2 + i0 + 3 + u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u) step(ac[u], bc[u], i0 + u);
        rescale();
    }
    if (i0 < J) {  // the last, partial group
        step(an[0], bn[0], i0);
        if (i0 + 1 < J) step(an[1], bn[1], i0 + 1);
        if (i0 + 2 < J) step(an[2], bn[2], i0 + 2);
        rescale();
    }
    return outside;
}

// Warp-parallel extreme Ritz value of T_J: every lane runs Laguerre (one
// recurrence sweep per iteration) from its own start x_l = lo + (hi - lo) 2^(-l/2)
// (top; mirrored for the bottom).  A start is valid if its first sweep shows it
// outside the spectrum (all Sturm signs positive, resp. alternating): from there
// Laguerre is monotone to the extreme root.  The lanes stop together once the
// valid lane with the closest start has converged (2 eps |x| or a direction
// flip); its value is returned to all lanes.  lo must be an inner bound (a Ritz
// value of a smaller T or max/min alpha), hi an outer (Gershgorin) bound.
__device__ double tri_laguerre_warp(const int oA, const int oB2, const int J, const double lo, const double hi,
                                    const bool top, const int lane, int* it_out = nullptr,
                                    const double hsafe = 0.0) {
    extern __shared__ __align__(16) double sm[];
    const double eps = 2.220446049250313e-16;
    if (J == 1) return sm[oA];
    const double n = (double)J;
    double x = lo + (hi - lo) * exp2(-0.5 * (double)lane);
    if (lane == 0) x = hi;
    bool valid = true, done = false, has_step = false, restarted = (hsafe == 0.0);
    double last_step = 0.0;
    for (int it = 0; it < 40; ++it) {
        double p1, d1, s1;
        bool outside = false;
        if (it == 0) outside = tri_charpoly3<true>(oA, oB2, J, x, top, p1, d1, s1);
        else tri_charpoly3<false>(oA, oB2, J, x, top, p1, d1, s1);
        if (it == 0) valid = outside;
        if (!done) {
            if (p1 == 0.0) {
                done = true;
            } else {
                const double G = d1 / p1;
                const double H = G * G - s1 / p1;
                const double disc = fmax((n - 1.0) * (n * H - G * G), 0.0);
                const double den = G + copysign(sqrt(disc), G);
                if (den == 0.0) {
                    done = true;
                } else {
                    const double step = n / den;
                    if (has_step && (step > 0.0) != (last_step > 0.0)) {
                        done = true;
                    } else {
                        x -= step;
                        last_step = step;
                        has_step = true;
                        if (fabs(step) <= 2.0 * eps * fabs(x)) done = true;
                    }
                }
            }
        }
        // the valid lane with the innermost start converges first and is the answer
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        const int best = top ? 31 - __clz(vmask) : 31 - __clz(vmask);  // highest lane = innermost start
        if (vmask == 0u) {
            if (restarted) break;
            // the (warm) outer bound was inside the spectrum: restart from the safe bound
            restarted = true;
            x = lo + (hsafe - lo) * exp2(-0.5 * (double)lane);
            if (lane == 0) x = hsafe;
            valid = true; done = false; has_step = false; last_step = 0.0;
            it = -1;
            continue;
        }
        const bool bdone = __shfl_sync(0xffffffffu, done ? 1 : 0, best) != 0;
        if (it_out) *it_out = it + 1;
        if (bdone) return __shfl_sync(0xffffffffu, x, best);
    }
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    const int best = vmask ? 31 - __clz(vmask) : 0;
    return __shfl_sync(0xffffffffu, x, best);
}

// Lanczos check state in shared memory (offsets from oShd): results, the
// bookkeeping of lanczos_reg kept out of registers, and the decision.
enum : int { CK_TTOP = 0, CK_RTOP = 1, CK_TBOT = 2, CK_RBOT = 3, CK_TNORM = 10 /* 2 slots (parity) */,
             CK_GHI = 12, CK_GLO = 13, CK_INTOP = 14, CK_INBOT = 15, CK_LRES = 16, CK_JPREV = 17, CK_NEXT = 18,
             CK_DONE = 19, CK_HINTED = 20 };

// Lanczos convergence check, run by warp 0 (lane 0 does the bookkeeping): Ritz
// value(s) by the warp-parallel Laguerre between the inner bound (previous Ritz
// value or max/min alpha) and Gershgorin, residual be[J-1] |s_J| by the
// backward recurrence; converged when <= 1e-14 |T_J| (or exhausted); else the
// next check is predicted from the observed linear rate (<= 8 iterations on).
// Out of line: one warp works while the CTA waits.
__device__ __noinline__ void lanczos_check(const int tid, const int oAl, const int oBe, const int oB2, const int oRbe,
                                           const int J, const double beta, const double tnorm, const bool need_bot,
                                           const bool exhausted, const int md, const int oShd,
                                           unsigned long long* prof = nullptr) {
    extern __shared__ __align__(16) double sm[];
    if ((tid >> 5) != 0) return;
    const int lane = tid & 31;
    long long ck0 = clock64();
    // Gershgorin bounds (outer) and max / min alpha (inner: Rayleigh quotients of T_J)
    double ghi = -SW_INF, glo = SW_INF, ahi = -SW_INF, alo = SW_INF;
    for (int i = lane; i < J; i += 32) {
        const double a = sm[oAl + i];
        const double rs = (i > 0 ? sm[oBe + i - 1] : 0.0) + (i + 1 < J ? sm[oBe + i] : beta);
        ghi = fmax(ghi, a + rs);
        glo = fmin(glo, a - rs);
        ahi = fmax(ahi, a);
        alo = fmin(alo, a);
    }
    ghi = warp_max(ghi);
    glo = warp_min(glo);
    ahi = warp_max(ahi);
    alo = warp_min(alo);
    const double in_top = fmax(ahi, sm[oShd + CK_INTOP]), in_bot = fmin(alo, sm[oShd + CK_INBOT]);
    // outer start: Gershgorin, or -- after a first check -- the previous Ritz value plus its
    // residual (an eigenvalue of M lies within the residual of a Ritz value; the top one when
    // the residual is below the gap).  tri_laguerre_warp restarts at Gershgorin if the Sturm
    // signs show the bound is inside the spectrum.
    const double th_prev = sm[oShd + CK_TTOP];
    double hi_top = ghi + 1e-13 * tnorm;
    if (th_prev > -SW_INF) hi_top = fmin(hi_top, th_prev + 1.01 * sm[oShd + CK_RTOP] + 1e-13 * tnorm);
    long long ck1 = clock64();
    int lits = 0;
    const double th = tri_laguerre_warp(oAl, oB2, J, fmin(in_top, hi_top), hi_top, true, lane, &lits,
                                        ghi + 1e-13 * tnorm);
    double thb = SW_INF;
    if (need_bot) thb = tri_laguerre_warp(oAl, oB2, J, in_bot, glo - 1e-13 * tnorm, false, lane);
    long long ck2 = clock64();
    if (lane != 0) return;
    const double res = beta * tri_back_lastcomp_sm(oAl, oBe, oRbe, J, th);
#if SW_PROF_LANCZOS
    if (prof) {
        long long ck3 = clock64();
        const bool first = !(sm[oShd + CK_INTOP] > -SW_INF);
        atomicAdd(&prof[first ? 20 : 24], 1ull);
        atomicAdd(&prof[first ? 21 : 25], (unsigned long long)lits);
        atomicAdd(&prof[first ? 22 : 26], (unsigned long long)(ck2 - ck1));
        atomicAdd(&prof[23], (unsigned long long)(ck3 - ck2));
        atomicAdd(&prof[27], (unsigned long long)(ck1 - ck0));
    }
#else
    (void)ck0; (void)ck1; (void)ck2; (void)prof;
#endif
    const double resb = need_bot ? beta * tri_back_lastcomp_sm(oAl, oBe, oRbe, J, thb) : 0.0;
    sm[oShd + CK_TTOP] = th;
    sm[oShd + CK_RTOP] = res;
    sm[oShd + CK_TBOT] = thb;
    sm[oShd + CK_RBOT] = resb;
    // both ends requested (t- and t+: oracle mode, Hit-and-Run): each residual relative to its
    // own Ritz value (floored at 1e-6 |T|): near a face |T| is set by the near end, and a
    // tolerance on |T| alone would leave the far end's t inaccurate (R30)
    const double tol = SW_LANCZOS_TOL * tnorm;
    const double tol_t = need_bot ? SW_LANCZOS_TOL * fmax(fabs(th), 1e-6 * tnorm) : tol;
    const double tol_b = need_bot ? SW_LANCZOS_TOL * fmax(fabs(thb), 1e-6 * tnorm) : tol;
    const bool done = exhausted || (res <= tol_t && resb <= tol_b);
    sm[oShd + CK_DONE] = done ? 1.0 : 0.0;
    if (done) return;
    // Ritz values of T_J are inner bounds for those of every larger T
    sm[oShd + CK_INTOP] = fmax(sm[oShd + CK_INTOP], th);
    if (need_bot) sm[oShd + CK_INBOT] = fmin(sm[oShd + CK_INBOT], thb);
    const double lres = log(fmax(res, resb));
    const int jprev = (int)sm[oShd + CK_JPREV];
    const double lres_prev = sm[oShd + CK_LRES];
    int step = (sm[oShd + CK_HINTED] != 0.0) ? 2 : SW_CHECK_STEP0;  // a hinted first check is close to convergence
    if (jprev > 0 && lres < lres_prev) {
        const double rate = (lres_prev - lres) / (double)(J - jprev);
        step = (int)ceil((lres - log(tol)) / rate);
        step = max(1, min(SW_CHECK_STEPMAX, step));
    }
    sm[oShd + CK_JPREV] = (double)J;
    sm[oShd + CK_LRES] = lres;
    sm[oShd + CK_NEXT] = (double)min(md, J + step);
}

// Lanczos (CGS with a DGKS second pass) on the symmetric md x md matrix M
// (shared or global memory, leading dimension ld, zero padded to mdp).  Q holds
// the orthonormal basis (rows of length ld).  Per iteration: (A) w' = M (w / beta)
// (ping-pong buffers, q_j stored on the fly), (B) dots with q_0..q_j and |w'|^2,
// (C) w' -= Q h with per-warp partial norms; a second pass (D, E) only when the
// first cancelled more than half of |w'|^2.  3 barriers per iteration (5 with
// the second pass).  Convergence: residual beta_J |s_J| <= 1e-14 |T| for the
// requested extreme Ritz pair(s) (top: sv, bottom: sv2), checked from J =
// 0.45 md on, every 8 steps; Ritz values by Laguerre, vectors by a twisted
// factorisation.  wv must hold 2 (mdp + 8) doubles.  Returns J.
__device__ int lanczos_run(const Team& T, const double* M, double* Q, int md, int mdp, int ld, bool need_top,
                           bool need_bot, double* wv, double* hb, double* al, double* be, double* sv, double* sv2,
                           double* dp, double* dm, double* red, int* sh_r, double* shd,
                           unsigned long long* prof, double* theta_top, double* theta_bot,
                           double* om = nullptr, double* part = nullptr, double* b2 = nullptr,
                           double* rbe = nullptr, int oShd = -1) {
    const int lrow = T.tid >> 2, lg = T.tid & 3;
    const int NT = T.nthr;
    double* red2 = red + 16;  // per-warp partial norms (NT <= 512)
    *theta_top = -SW_INF;
    *theta_bot = SW_INF;
    double* win = wv;
    double* wout = wv + (mdp + 8);
    // start vector: fixed pseudo-random, zero padding (w_{-1} = q_0, beta_{-1} = 1)
    double s0 = 0.0;
    for (int e = T.tid; e < mdp; e += T.nthr) {
        double val = 0.0;
        if (e < md) {
            double f = (double)e * 0.6180339887498949;
            val = 0.5 + (f - floor(f));
        }
        win[e] = val;
        s0 += val * val;
    }
    s0 = block_sum(T, s0, red);
    double invb = 1.0 / sqrt(s0);
    // oShd >= 0 (al, be, b2, rbe and the check state in dynamic shared memory): lanczos_reg's
    // warp-parallel checks (Laguerre warm-started from the previous Ritz value, residual by the
    // backward recurrence, the next check from the observed rate) and its first-check rule
    const bool fastck = (oShd >= 0);
    extern __shared__ __align__(16) double sm[];
    const int jfirst = fastck ? ((md <= SW_FIRST_CHECK_FULL_MD) ? md
                                 : (md <= SW_FIRST_CHECK_SMALL_MD) ? (md * SW_FIRST_CHECK_PCT_SMALL) / 100
                                 : (md <= 64) ? (md * SW_FIRST_CHECK_PCT_MID) / 100
                                              : max(12, (md * SW_FIRST_CHECK_PCT_GLOBAL) / 100))
                              : max(min(md, 12), (md * 9) / 20);
    int next_check = jfirst;
    if (fastck && T.tid == 0) {
        sm[oShd + CK_INTOP] = -SW_INF;
        sm[oShd + CK_INBOT] = SW_INF;
        sm[oShd + CK_JPREV] = 0.0;
        sm[oShd + CK_LRES] = 0.0;
        sm[oShd + CK_TTOP] = -SW_INF;
        sm[oShd + CK_TBOT] = SW_INF;
        sm[oShd + CK_HINTED] = 0.0;
    }
    double tnorm = 0.0;
    double th_prev = -SW_INF, res_prev = SW_INF;
    int J = 0;
    // partial reorthogonalisation (as lanczos_reg's SW_PRO, here where Q and M live in global
    // scratch and the Gram-Schmidt dots / updates read O(j m) from L2 every iteration): the
    // three-term step w = y' - alpha q_j always, one Gram-Schmidt pass on w only when Simon's
    // omega estimates (3 rows in `om`) cross tau, for two consecutive vectors.
    const bool pro = SW_PRO_RUN && (om != nullptr);
    const int ovl = mdp + 8;
    const double eps1 = 2.220446049250313e-16 * sqrt((double)md);
    double bjm1 = 0.0, invb_prev = 0.0;
    int reorth_left = 0;
    bool was_full = true;
    if (pro && T.tid == 0) {
        om[0] = 1.0;
        part[40] = 0.0;
        part[41] = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < md; ++j) {
        double* qj = Q + (size_t)j * ld;
        long long tl0 = clock64();
        // ---- (A) q_j = w / beta stored; w' = M q_j: 4 threads per row, double2 columns
        for (int e = T.tid; e < mdp; e += T.nthr) qj[e] = win[e] * invb;
        double apl = 0.0;  // PRO: this thread's part of alpha = q_j . y'
        if (pro) {
            // omega_{j,k} estimates for k = tid <= j (rows j-1, j-2 of the ring); flag > tau
            if (T.tid == 0) part[40 + ((j + 1) & 1)] = 0.0;
            const int k = T.tid;
            if (j >= 1 && k <= j) {
                double v;
                if (k == j) v = 1.0;
                else if (k == j - 1) v = eps1 * tnorm * invb;
                else if (was_full) v = eps1;
                else {
                    const double* P1 = om + ((j - 1) % 3) * ovl;
                    const double* P2 = om + ((j - 2) % 3) * ovl;
                    const double bk = be[k], bkm = (k > 0) ? be[k - 1] : 0.0;
                    double num = bk * P1[k + 1] + (al[k] - al[j - 1]) * P1[k] + ((k > 0) ? bkm * P1[k - 1] : 0.0) -
                                 be[j - 2] * P2[k];
                    num += copysign(eps1 * (bk + bjm1), num);
                    v = num * invb;
                    if (fabs(v) > SW_PRO_TAU) part[40 + (j & 1)] = 1.0;
                }
                om[(j % 3) * ovl + k] = v;
            }
        }
        if (mdp <= 128) {
            // fast path: 16 double2 loads per thread issued up front, 4 accumulators
            for (int r0 = 0; r0 < mdp; r0 += (NT >> 2)) {
                const int rw = r0 + lrow;
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                if (rw < mdp) {
                    const double* Mr = M + (size_t)rw * ld;
                    double2 mv[16], wq[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const int c = 2 * lg + 8 * k;
                        mv[k] = (c < mdp) ? *reinterpret_cast<const double2*>(Mr + c) : make_double2(0.0, 0.0);
                        wq[k] = (c < mdp) ? *reinterpret_cast<const double2*>(win + c) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        acc[k & 3] += mv[k].x * wq[k].x;
                        acc[k & 3] += mv[k].y * wq[k].y;
                    }
                }
                double a0 = (acc[0] + acc[1]) + (acc[2] + acc[3]);
                a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
                a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
                if (lg == 0 && rw < mdp) {
                    double yv = a0 * invb;
                    if (pro) {  // y' = M q_j - beta_{j-1} q_{j-1}; alpha partial q_j . y'
                        if (j > 0) yv -= bjm1 * (wout[rw] * invb_prev);  // q_{j-1} (u_{j-1} still in wout)
                        apl += (win[rw] * invb) * yv;
                    }
                    wout[rw] = yv;
                }
            }
        } else {
            for (int r0 = 0; r0 < mdp; r0 += (NT >> 2)) {
                const int rw = r0 + lrow;
                double a0 = 0.0, a1 = 0.0;
                if (rw < mdp) {
                    const double* Mr = M + (size_t)rw * ld;
                    for (int c = 2 * lg; c < mdp; c += 8) {
                        double2 mv = *reinterpret_cast<const double2*>(Mr + c);
                        double2 wq = *reinterpret_cast<const double2*>(win + c);
                        a0 += mv.x * wq.x;
                        a1 += mv.y * wq.y;
                    }
                }
                a0 += a1;
                a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
                a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
                if (lg == 0 && rw < mdp) {
                    double yv = a0 * invb;
                    if (pro) {
                        if (j > 0) yv -= bjm1 * (wout[rw] * invb_prev);  // q_{j-1} (u_{j-1} still in wout)
                        apl += (win[rw] * invb) * yv;
                    }
                    wout[rw] = yv;
                }
            }
        }
        if (pro) {  // alpha partials: the owner lanes (lg == 0)
            apl += __shfl_xor_sync(0xffffffffu, apl, 16);
            apl += __shfl_xor_sync(0xffffffffu, apl, 8);
            apl += __shfl_xor_sync(0xffffffffu, apl, 4);
            if (T.lane == 0) part[T.warp] = apl;
        }
        __syncthreads();
        long long tl1 = clock64();
        long long tl2 = tl1, tl3 = tl1;
        // ---- (B..E) classical Gram-Schmidt against q_0..q_j
        double alpha = 0.0, nn = 0.0, nn_before = 0.0;
        int pass0 = 0;
        bool full = true;
        if (pro) {
            bool reorth;
            if (reorth_left > 0) { reorth = true; --reorth_left; }
            else if (part[40 + (j & 1)] != 0.0) { reorth = true; reorth_left = 1; }
            else reorth = false;
            for (int w = 0; w < T.nwarps; ++w) alpha += part[w];
            double nloc = 0.0;
            for (int e = T.tid; e < mdp; e += T.nthr) {
                const double wn = (e < md) ? wout[e] - alpha * (win[e] * invb) : 0.0;  // q_j from shared memory
                wout[e] = wn;
                nloc += wn * wn;
            }
            nloc = warp_sum(nloc);
            if (T.lane == 0) red2[T.warp] = nloc;
            __syncthreads();
            for (int w = 0; w < T.nwarps; ++w) nn += red2[w];
            nn_before = alpha * alpha + nn;  // |y'|^2
            if (!reorth && nn >= 1e-12 * nn_before) {
                pass0 = 2;
                full = false;
            } else {
                pass0 = 1;  // one Gram-Schmidt pass on w
            }
        }
        for (int pass = pass0; pass < 2; ++pass) {
            const int nrows = (pass == 0) ? j + 2 : j + 1;  // row j+1 = w'.w'
            if (mdp <= 128) {
                double2 w0 = make_double2(0.0, 0.0), w1 = make_double2(0.0, 0.0);
                const int i0 = 2 * T.lane, i1 = 64 + 2 * T.lane;
                if (i0 < mdp) w0 = *reinterpret_cast<const double2*>(wout + i0);
                if (i1 < mdp) w1 = *reinterpret_cast<const double2*>(wout + i1);
                const int NW = T.nwarps;
                for (int ib = T.warp; ib < nrows; ib += 4 * NW) {
                    double sacc[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = ib + u * NW;
                        const double* qi = (i <= j) ? Q + (size_t)i * ld : wout;
                        double sa = 0.0;
                        if (i < nrows) {
                            if (i0 < mdp) {
                                double2 q0 = *reinterpret_cast<const double2*>(qi + i0);
                                sa += q0.x * w0.x + q0.y * w0.y;
                            }
                            if (i1 < mdp) {
                                double2 q1 = *reinterpret_cast<const double2*>(qi + i1);
                                sa += q1.x * w1.x + q1.y * w1.y;
                            }
                        }
                        sacc[u] = sa;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                        for (int u = 0; u < 4; ++u) sacc[u] += __shfl_xor_sync(0xffffffffu, sacc[u], o);
                    if (T.lane == 0) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (ib + u * NW < nrows) hb[ib + u * NW] = sacc[u];
                    }
                }
            } else {
                for (int i = T.warp; i < nrows; i += T.nwarps) {
                    const double* qi = (i <= j) ? Q + (size_t)i * ld : wout;
                    double sacc = 0.0;
                    for (int c = T.lane; c < mdp; c += 32) sacc += qi[c] * wout[c];
                    sacc = warp_sum(sacc);
                    if (T.lane == 0) hb[i] = sacc;
                }
            }
            __syncthreads();
            if (pass == 0) tl2 = clock64();
            alpha += hb[j];
            if (pass == 0) nn_before = hb[j + 1];
            {
                const int g = T.tid & 3, egrp = T.nthr >> 2;
                double nloc = 0.0;
                for (int e0 = 0; e0 < mdp; e0 += egrp) {
                    const int e = e0 + (T.tid >> 2);
                    double sa = 0.0, sb = 0.0;
                    if (e < mdp) {
                        for (int ibase = 0; ibase <= j; ibase += 64) {
                            double acc4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                const int i = ibase + g + 4 * k;
                                if (i <= j) acc4[k & 3] += hb[i] * Q[(size_t)i * ld + e];
                            }
                            sa += (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
                        }
                    }
                    sa += sb;
                    sa += __shfl_xor_sync(0xffffffffu, sa, 1);
                    sa += __shfl_xor_sync(0xffffffffu, sa, 2);
                    if (e < mdp) {
                        double wn = wout[e] - sa;
                        __syncwarp();
                        if (g == 0) wout[e] = wn;
                        nloc += (g == 0) ? wn * wn : 0.0;
                    }
                }
                // partial norms live in the g == 0 lanes: reduce over lanes 4, 8, 16 apart
                nloc += __shfl_xor_sync(0xffffffffu, nloc, 4);
                nloc += __shfl_xor_sync(0xffffffffu, nloc, 8);
                nloc += __shfl_xor_sync(0xffffffffu, nloc, 16);
                if (T.lane == 0) red2[T.warp] = nloc;
            }
            __syncthreads();
            nn = 0.0;
            for (int w = 0; w < T.nwarps; ++w) nn += red2[w];
            if (pass == 0) tl3 = clock64();
            if (prof && T.tid == 0 && pass == 1) atomicAdd(&prof[15], 1ull);
            // second (DGKS) pass only on severe cancellation, as in lanczos_reg (one CGS pass
            // keeps theta_max within ~20 eps |M|; the 0.5 criterion fired on 2/3 of the iterations)
            if (!(nn < 1e-12 * nn_before)) break;
        }
        // only rounding left after the Gram-Schmidt pass(es): the Krylov space is invariant
        // (low-rank pencils, e.g. the ball); continuing would orthogonalise noise once and breed
        // ghost Ritz values
        if (nn < 1e-28 * nn_before) nn = 0.0;
        const double beta = sqrt(nn);
        if (T.tid == 0) {
            al[j] = alpha;
            be[j] = beta;
            if (fastck) {
                b2[j] = nn;
                rbe[j] = 1.0 / beta;
            }
        }
        if (pro) {
            bjm1 = beta;
            was_full = full;
            invb_prev = invb;  // 1 / beta_{j-1}, the scale of u_j held in win (q_j = u_j * invb)
        }
        tnorm = fmax(tnorm, fabs(alpha) + beta + (j > 0 ? be[j - 1] : 0.0));
        J = j + 1;
        const bool exhausted = (J == md) || !(beta > 1e-15 * tnorm);
        if (prof && T.tid == 0) {
            long long tl4 = clock64();
            atomicAdd(&prof[12], (unsigned long long)(tl1 - tl0));
            atomicAdd(&prof[13], (unsigned long long)(tl2 - tl1));
            atomicAdd(&prof[14], (unsigned long long)(tl3 - tl2));
            atomicAdd(&prof[16], (unsigned long long)(tl4 - tl3));
        }
        // next iteration uses q_{j+1} = w' / beta
        double* tmp = win;
        win = wout;
        wout = tmp;
        invb = 1.0 / beta;
        if (fastck && (exhausted || J >= next_check)) {
            __syncthreads();  // al / be / b2 / rbe of this step visible
            lanczos_check(T.tid, (int)(al - sm), (int)(be - sm), (int)(b2 - sm), (int)(rbe - sm), J, beta, tnorm,
                          need_bot, exhausted, md, oShd, prof);
            __syncthreads();
            if (sm[oShd + CK_DONE] != 0.0) break;
            next_check = (int)sm[oShd + CK_NEXT];
        } else if (exhausted || J >= next_check) {
            __syncthreads();  // al/be of this step visible
            long long tc0 = clock64();
            double glo = SW_INF, ghi = -SW_INF;
            for (int i = T.tid; i < J; i += T.nthr) {
                double rsum = (i > 0 ? fabs(be[i - 1]) : 0.0) + (i + 1 < J ? fabs(be[i]) : 0.0);
                glo = fmin(glo, al[i] - rsum);
                ghi = fmax(ghi, al[i] + rsum);
            }
            ghi = block_max(T, ghi, red);
            if (need_bot) glo = block_min(T, glo, red);
            if (T.tid == 0) shd[0] = tri_laguerre(al, be, J, ghi + 1e-13 * tnorm);
            if (need_bot && T.tid == 32) shd[1] = tri_laguerre(al, be, J, glo - 1e-13 * tnorm);
            __syncthreads();
            const double th = shd[0];
            double res = tri_twisted_vec(T, al, be, J, th, be[J - 1], dp, dm, sv, red, sh_r);
            double thmin = SW_INF, resmin = 0.0;
            if (need_bot) {
                thmin = shd[1];
                resmin = tri_twisted_vec(T, al, be, J, thmin, be[J - 1], dp, dm, sv2, red, sh_r);
            }
            th_prev = th;
            res_prev = res;
            *theta_top = th;
            *theta_bot = thmin;
            if (prof && T.tid == 0) {
                atomicAdd(&prof[9], (unsigned long long)(clock64() - tc0));
                atomicAdd(&prof[11], 1ull);
            }
            const double tol = 1e-14 * tnorm;
            if (exhausted || ((!need_top || res <= tol) && (!need_bot || resmin <= tol))) break;
            next_check = min(md, J + 8);
        }
    }
    (void)th_prev;
    (void)res_prev;
    __syncthreads();
    if (fastck) {  // the converged Ritz values and their vectors of T_J
        const double th = sm[oShd + CK_TTOP];
        *theta_top = th;
        tri_twisted_vec(T, al, be, J, th, be[J - 1], dp, dm, sv, red, sh_r);
        if (need_bot) {
            const double thb = sm[oShd + CK_TBOT];
            *theta_bot = thb;
            tri_twisted_vec(T, al, be, J, thb, be[J - 1], dp, dm, sv2, red, sh_r);
        }
    }
    return J;
}

// K2 vector slots (length vl = mp + 8 each) in the shared vector area
enum : int { V_UU = 0, V_HH = 1, V_PW = 2, V_RDIAG = 3, V_RBE = 4, V_HB = 5, V_AL = 6, V_BE = 7, V_SV = 8, V_ZZ = 9,
             V_YY = 10, V_DP = 11, V_BV = 12, V_SV2 = 13, V_B2 = 13, V_DM = 14, V_WV = 15, V_LZ = 17 };

#ifndef SW_RSQRT_BETA
#define SW_RSQRT_BETA 1
#endif
// sum over the row-owner lanes (g = lane & 3 == 0) of a warp: the other lanes hold zeros, so
// the xor-1 / xor-2 levels of a full warp_sum add exact zeros and can be skipped (same value)
__device__ __forceinline__ double owner_sum(double v) {
    v += __shfl_xor_sync(0xffffffffu, v, 16);  // warp_sum's order
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    return v;
}
// balanced pairwise sum of the N per-warp partials (depth log2 N instead of N)
template <int N>
__device__ __forceinline__ double tree_sum(const double* p) {
    if constexpr (N == 1) return p[0];
    else return tree_sum<N / 2>(p) + tree_sum<N - N / 2>(p + N / 2);
}
template <int NT, int KC, bool GM = false, bool USEQT = true>
__device__ __forceinline__ int lanczos_reg(const int oM, const int oQ, const int md, const int mdp, const int ld,
                                           const bool need_bot, const int oVec, const int vl, const int oRed,
                                           const int first_pct, unsigned long long* prof, const double* __restrict__ Mg = nullptr,
                                           int oQTin = -1) {
    // everything addressed as offsets into the dynamic shared memory (32-bit LDS/STS)
    extern __shared__ __align__(16) double sm[];
    static_assert(KC <= NT / 32, "M row segment of a thread: 8 KC columns <= NT / 4 rows");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    constexpr int NWC = NW;  // compute warps
    const int oAl = oVec + V_AL * vl, oBe = oVec + V_BE * vl, oRbe = oVec + V_RBE * vl, oHb = oVec + V_HB * vl;
    const int oB2 = oVec + V_B2 * vl;
    const int oWu = oVec + V_LZ * vl;  // wu0, wu1 (ping-pong), wp: 3 x (mdp + 8)
    const int oWp = oWu + 2 * (mdp + 8);
    const int oRB = oRed + 16;         // per-warp partial norms
    const int oShd = oRed + 32;        // check results (4) and thetas (2)
    auto csync = [&]() { __syncthreads(); };
    // transposed basis: in M's shared space once M is in registers, or a given region
    const int oQT = (oQTin >= 0) ? oQTin : oM;
    const int r = tid >> 2, g = tid & 3;
    const bool rowok = r < md;
    const bool owner = (g == 0) && (r < mdp);
    double2 mr[KC];
    if (GM) {  // M rows straight from global memory (K2b): all loads of a thread in flight at once
        const double* Mr = Mg + (size_t)(r < mdp ? r : 0) * ld;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const int c = 2 * g + 8 * k;
            mr[k] = (r < mdp && c < mdp) ? __ldg(reinterpret_cast<const double2*>(Mr + c)) : make_double2(0.0, 0.0);
        }
    } else {
        const int oMr = oM + (r < mdp ? r : 0) * ld;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const int c = 2 * g + 8 * k;
            mr[k] = (r < mdp && c < mdp) ? *reinterpret_cast<const double2*>(sm + oMr + c) : make_double2(0.0, 0.0);
        }
    }
    // dots: 8 lanes per dot (lane = 8 u + s), element pairs 2 s + 16 t, t < tcnt
    const int du = lane >> 3, ds = lane & 7;
    const int tcnt = (mdp - 2 * ds + 15) >> 4;
    // start vector u_0 (fixed, zero padded)
    double wr = 0.0;
    if (rowok) {
        double f = (double)r * 0.6180339887498949;
        wr = 0.5 + (f - floor(f));
    }
    if (owner) sm[oWu + r] = wr;
    double p0 = (g == 0) ? wr * wr : 0.0;
    p0 = owner_sum(p0);
    if (lane == 0) sm[oRB + warp] = p0;
    if (tid == 0) {  // bookkeeping of the checks lives in shared memory (register pressure)
        sm[oShd + CK_INTOP] = -SW_INF;
        sm[oShd + CK_INBOT] = SW_INF;
        sm[oShd + CK_JPREV] = 0.0;
        sm[oShd + CK_LRES] = 0.0;
        sm[oShd + CK_TTOP] = -SW_INF;
        sm[oShd + CK_TBOT] = SW_INF;
        sm[oShd + CK_HINTED] = 0.0;
    }
    __syncthreads();  // also: every thread has its M row in registers (QT may overwrite M)
    double nn0 = 0.0;
    nn0 = tree_sum<NW>(sm + oRB);
    double sj = 1.0 / sqrt(nn0);  // q_j = u_j * sj
    double bjm1 = 0.0;
    // first check: 2 before the chain's previous iteration count (consecutive calls
    // of a chain need similar J), else at 40% of md; later checks from the observed rate
    // (a per-chain hint from the previous call was measured to RAISE J: consecutive calls of a
    // chain differ too much; the first check stays at 40% of md)

    // first check by size: small problems need nearly the full dimension (m = 40: J ~ 0.85 md;
    // m <= 24: J = md), larger ones about half (m = 100: J ~ 0.5 md)
    int next_check = (md <= SW_FIRST_CHECK_FULL_MD) ? md
                   : (md <= SW_FIRST_CHECK_SMALL_MD) ? (md * SW_FIRST_CHECK_PCT_SMALL) / 100
                   : (md <= 64) ? (md * SW_FIRST_CHECK_PCT_MID) / 100 : max(12, (md * SW_FIRST_CHECK_PCT) / 100);
    if (first_pct > 0 && md > SW_FIRST_PCT_MIN_MD) next_check = max(12, (md * first_pct) / 100);  // caller's rule (HMC-r)
    int J = 0;
    double tnorm = 0.0;
    {
#if SW_PROF_LANCZOS
    long long c_mv = 0, c_dot = 0, c_upd = 0, c_chk = 0, c_t = clock64();
#define SW_LZ_STAMP(acc) if (prof) { long long c = clock64(); acc += c - c_t; c_t = c; }
#else
#define SW_LZ_STAMP(acc)
#endif
    for (int j = 0; j < md; ++j) {
        const int oU = oWu + (j & 1) * (mdp + 8);
        const int oUn = oWu + ((j + 1) & 1) * (mdp + 8);
        // ---- (1) w' = M q_j
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k0 = 0; k0 < KC; k0 += 4) {
            double2 wq[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = 2 * g + 8 * (k0 + k);
                wq[k] = (k0 + k < KC && c < mdp) ? *reinterpret_cast<const double2*>(sm + oU + c)
                                                 : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k0 + k < KC) {
                    a4[k] = fma(mr[k0 + k].x, wq[k].x, a4[k]);
                    a4[k] = fma(mr[k0 + k].y, wq[k].y, a4[k]);
                }
            }
        }
        double y = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        y += __shfl_xor_sync(0xffffffffu, y, 1);
        y += __shfl_xor_sync(0xffffffffu, y, 2);
        const double wpr = rowok ? y * sj : 0.0;
        const double qj = rowok ? wr * sj : 0.0;  // q_j[r] (all 4 lanes of the row)
        if (owner) {
            const double q = qj;  // q_j (wr = u_j[r])
            sm[oQ + j * ld + r] = q;
            if (USEQT) {
                sm[oQT + r * ld + j] = q;
                sm[oQT + r * ld + j + 1] = 0.0;  // the update reads pairs (i, i + 1): never stale (NaN) data
            }
            sm[oWp + r] = wpr;
        }
        csync();
        SW_LZ_STAMP(c_mv)
        // ---- (2)+(3) classical Gram-Schmidt of w' against q_0..q_j; a second pass
        // (DGKS) only on severe cancellation (|w| < 1e-6 |w'|, e.g. an invariant subspace).
        double wcur = wpr, alpha = 0.0, nnb = 0.0, nn = 0.0;
        const int pass0 = 0;
        for (int pass = pass0; pass < 2; ++pass) {
            // (2) h_i = q_i . w for i <= j, and |w|^2 (slot j + 1): 8 lanes per dot, 4 dots per warp
            for (int ib = 4 * warp; ib <= j + 1; ib += 4 * NWC) {
                const int i = ib + du;
                double sacc = 0.0;
                if (i <= j + 1) {
                    const int oQi = (i <= j ? oQ + i * ld : oWp) + 2 * ds;
                    const int oW = oWp + 2 * ds;
                    double s2 = 0.0;
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        if (t < tcnt) {
                            const double2 q2 = *reinterpret_cast<const double2*>(sm + oQi + 16 * t);
                            const double2 w2 = *reinterpret_cast<const double2*>(sm + oW + 16 * t);
                            if (t & 1) { s2 = fma(q2.x, w2.x, s2); s2 = fma(q2.y, w2.y, s2); }
                            else { sacc = fma(q2.x, w2.x, sacc); sacc = fma(q2.y, w2.y, sacc); }
                        }
                    }
                    sacc += s2;
                }
                sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
                sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
                sacc += __shfl_xor_sync(0xffffffffu, sacc, 4);
                if (ds == 0 && i <= j + 1) {
                    sm[oHb + i] = (i <= j) ? sacc : 0.0;  // hb[j + 1] = 0 pads the last pair
                    if (i == j + 1) sm[oShd + 8] = sacc;
                }
            }
            csync();
            SW_LZ_STAMP(c_dot)
            // (3) w -= Q h (row r: lane g takes the pairs i = 2 g + 8 k)
            double acc0 = 0.0, acc1 = 0.0;
            if (r < mdp) {
                if (USEQT) {
                    const int oQr = oQT + r * ld;
                    for (int i = 2 * g; i <= j; i += 8) {
                        const double2 h2 = *reinterpret_cast<const double2*>(sm + oHb + i);
                        const double2 q2 = *reinterpret_cast<const double2*>(sm + oQr + i);
                        acc0 = fma(h2.x, q2.x, acc0);
                        acc1 = fma(h2.y, q2.y, acc1);
                    }
                } else {  // column access of the row-major basis (lane g takes i = g mod 4)
                    int i = g;
                    for (; i + 4 <= j; i += 8) {
                        acc0 = fma(sm[oHb + i], sm[oQ + i * ld + r], acc0);
                        acc1 = fma(sm[oHb + i + 4], sm[oQ + (i + 4) * ld + r], acc1);
                    }
                    if (i <= j) acc0 = fma(sm[oHb + i], sm[oQ + i * ld + r], acc0);
                }
            }
            double qh = acc0 + acc1;
            qh += __shfl_xor_sync(0xffffffffu, qh, 1);
            qh += __shfl_xor_sync(0xffffffffu, qh, 2);
            wcur = rowok ? wcur - qh : 0.0;
            alpha += sm[oHb + j];
            if (pass == 0) nnb = sm[oShd + 8];
            double pb = (g == 0) ? wcur * wcur : 0.0;
            pb = owner_sum(pb);
            if (lane == 0) sm[oRB + warp] = pb;
            if (owner) sm[oUn + r] = wcur;
            csync();
            nn = 0.0;
            nn = tree_sum<NWC>(sm + oRB);
            if (nn >= 1e-12 * nnb) break;
            if (owner) sm[oWp + r] = wcur;  // second pass on w
            csync();
        }
        wr = wcur;
#if SW_RSQRT_BETA
        // 1/beta by the hardware reciprocal square root (+ Newton, ~1 ulp) and beta = nn / beta:
        // no correctly-rounded sqrt and division sequences on the iteration's critical path
        const double rsb = (nn > 0.0) ? rsqrt(nn) : SW_INF;
        const double beta = (nn > 0.0) ? nn * rsb : 0.0;
#else
        const double beta = sqrt(nn);
        const double rsb = 1.0 / beta;
#endif
        if (tid == 0) {
            sm[oAl + j] = alpha;
            sm[oBe + j] = beta;
            sm[oB2 + j] = nn;
            sm[oRbe + j] = rsb;
        }
        tnorm = fmax(tnorm, fabs(alpha) + beta + bjm1);
        bjm1 = beta;
        sj = rsb;
        J = j + 1;
        const bool exhausted = (J == md) || !(beta > 1e-15 * tnorm);
        SW_LZ_STAMP(c_upd)
        if (exhausted || J >= next_check) {
            __syncthreads();  // al / be / b2 / rbe and the bookkeeping of this step visible
            lanczos_check(tid, oAl, oBe, oB2, oRbe, J, beta, tnorm, need_bot, exhausted, md, oShd, prof);
            __syncthreads();
            SW_LZ_STAMP(c_chk)
            if (sm[oShd + CK_DONE] != 0.0) break;
            next_check = (int)sm[oShd + CK_NEXT];
        }
    }
#if SW_PROF_LANCZOS
    if (prof && tid == 0) {
        atomicAdd(&prof[12], (unsigned long long)c_mv);
        atomicAdd(&prof[13], (unsigned long long)c_dot);
        atomicAdd(&prof[14], (unsigned long long)c_upd);
        atomicAdd(&prof[9], (unsigned long long)c_chk);
    }
#endif
    }  // compute warps
#undef SW_LZ_STAMP
    (void)prof;
    __syncthreads();
    const double th_top = sm[oShd + CK_TTOP];
    if (tid == 0) {
        sm[oShd + 4] = th_top;
        sm[oShd + 5] = sm[oShd + CK_TBOT];
    }
    // top Ritz vector of T_J (z = Q sv, Q orthonormal)
    Team T;
    T.tid = tid; T.nthr = NT; T.lane = lane; T.warp = warp; T.nwarps = NW;
    int* sh_r = reinterpret_cast<int*>(sm + oShd + 6);
    tri_twisted_vec(T, sm + oAl, sm + oBe, J, th_top, sm[oBe + J - 1], sm + oVec + V_DP * vl, sm + oVec + V_DM * vl,
                    sm + oVec + V_SV * vl, sm + oRed, sh_r);
    return J;
}

}  // namespace sw
#include "chol_inv.cuh"
namespace sw {

// resident CTAs per SM the fused kernels are compiled for (the register cap follows)
#ifndef SW_MINB128
#define SW_MINB128 4
#endif
#ifndef SW_MINB192
#define SW_MINB192 4  // m = 33..48: 4 CTAs/SM at 80 registers (some spills) measured +3% (m = 40) over 3;
                      // the 128- and 256-thread variants lost 32% / 9% at their caps (profiles/r2m_minb)
#endif
#ifndef SW_MINB256
#define SW_MINB256 2
#endif
template <int NT, bool SMEM, int KC>
__global__ void __launch_bounds__(NT, (NT <= 128) ? SW_MINB128 : (NT <= 192) ? SW_MINB192 : (NT <= 256) ? SW_MINB256 : 1) chord_kernel2(ChordParams P) {
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

    const int m = P.m, n = P.n, ld = P.ld;
    const int mp = (m + 7) & ~7;
    double* base = SMEM ? smem_dyn : (P.scratch + (size_t)blockIdx.x * P.scratch_stride);
    double* G = base;
    double* B = base + (size_t)(mp + 1) * ld;  // one spare row each: in-place deflation (below)
    double* Qm = G;  // Lanczos basis reuses L's space while L is parked in P.lsave
    // the vector area (+ inverse diagonal blocks) in shared memory on both variants; the global
    // variant keeps only G, B (the Lanczos basis, M) in its scratch slice
    double* vec = SMEM ? B + (size_t)(mp + 1) * ld + 2 : smem_dyn;
    double* Lsave = P.lsave + (size_t)blockIdx.x * P.lsave_stride;
    const int vl = mp + 8;
    double* uu = vec + 0 * vl;
    double* hh = vec + 1 * vl;
    double* pw = vec + 2 * vl;
    double* rdiag = vec + 3 * vl;
    double* wv = vec + 15 * vl;  // 2 slots (ping-pong)
    double* hb = vec + 5 * vl;
    double* al = vec + 6 * vl;
    double* be = vec + 7 * vl;
    double* sv = vec + 8 * vl;
    double* zz = vec + 9 * vl;
    double* yy = vec + 10 * vl;
    double* dp = vec + 11 * vl;
    double* bv = vec + 12 * vl;
    double* sv2 = vec + 13 * vl;
    double* dm = vec + 14 * vl;

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
        __syncthreads();
        long long t_prof = clock64();

        // ---- 1. unpack A(x) -> G, A(v) -> B0 (full symmetric), zero padding.  A boundary start
        // puts B one double further (B0 = B + 1) so that its deflated trailing block
        // B0 + ld + 1 -- M for the Lanczos double2 loads -- is 16-byte aligned
        const bool defl = (bnd == 0);
        double* B0 = B + (defl ? 1 : 0);
        unpack_sym(T, ax, G, m, ld);
        unpack_sym(T, av, B0, m, ld);
        if (defl)
            for (int i = T.tid; i < m; i += T.nthr) uu[i] = P.U[(size_t)slot * m + i];
        __syncthreads();
        PROF_MARK(0);
        int md = m;
        double a_schur = 0.0, beta_h = 0.0;
        bool outward = false;
        double* Gd = G;  // the matrices of the (possibly deflated) pencil
        double* Bd = B0;
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
            // the rank-2 congruence fused with the Schur complement on the trailing block, in
            // place (as factor_kernel): the deflated pencil is (G + ld + 1, B + ld + 1)
            householder_congruence2(T, G, B0, m, ld, hh, beta_h, pw, yy, red, false);
            a_schur = B0[0] - (hh[0] * yy[0] + yy[0] * hh[0]);
            outward = !(a_schur > 0.0);
            for (int i = T.tid; i + 1 < m; i += T.nthr) bv[i] = B0[(i + 1) * ld] - (hh[i + 1] * yy[0] + yy[i + 1] * hh[0]);
            __syncthreads();
            md = m - 1;
            for (int i = 1 + T.warp; i < m; i += T.nwarps) {
                const double hi = hh[i], pxi = pw[i], pyi = yy[i], bi = bv[i - 1];
                for (int jx = 1 + T.lane; jx < m; jx += 32) {
                    const double hj = hh[jx];
                    G[i * ld + jx] -= hi * pw[jx] + pxi * hj;
                    const double bij = B0[i * ld + jx] - (hi * yy[jx] + pyi * hj);
                    B0[i * ld + jx] = outward ? 0.0 : bij - bi * bv[jx - 1] / a_schur;
                }
            }
            Gd = G + ld + 1;
            Bd = B0 + ld + 1;
        }
        const int mdp = (md + 7) & ~7;
        // padding rows/cols [md, mdp): G = I, B = 0
        for (int i = md + T.warp; i < mdp; i += T.nwarps)
            for (int j = T.lane; j < mdp; j += 32) {
                Gd[i * ld + j] = (i == j) ? 1.0 : 0.0;
                Gd[j * ld + i] = (i == j) ? 1.0 : 0.0;
                Bd[i * ld + j] = 0.0;
                Bd[j * ld + i] = 0.0;
            }
        __syncthreads();
        PROF_MARK(1);

        if (!SMEM && P.gsplit) {
            // ---- factor phase of the m > 112 split (as factor_kernel): Cholesky, congruence,
            // M and packed L to the slot's work buffers, the deflation data to its small area;
            // lanczos_cl_kernel and tail_kernel finish the call
            int status = (defl ? ST_DEFL : 0) | (outward ? ST_OUTWARD : 0);
            if (!outward && md >= 1) {
                double* Lv = vec + NVEC2 * vl + 64;
                const bool okc = cholesky_inv_blocked(T, Gd, mdp, ld, rdiag, Lv, &sh_i[2]);
                PROF_MARK(2);
                if (!okc) {
                    status |= ST_FAILED;
                } else {
                    congruence_inv(T, Gd, Lv, Bd, mdp, ld);
                    PROF_MARK(3);
                    double* Mw = P.wM + (size_t)slot * P.w_mstride;
                    double* Lw = P.wL + (size_t)slot * P.w_mstride;
                    if (P.gsplit == 2) {
                        // M as the lower 8 x 8 tiles lanczos_t_kernel holds: tile (I, J), I >= J, at
                        // 64 (I (I + 1) / 2 + J), row-major; L packed by rows
                        const int nbk = mdp >> 3;
                        for (int I = T.warp; I < nbk; I += T.nwarps)
                            for (int J = 0; J <= I; ++J) {
                                double* Mt = Mw + 64 * (I * (I + 1) / 2 + J);
#pragma unroll
                                for (int h2 = 0; h2 < 2; ++h2) {
                                    const int e = T.lane + 32 * h2, gi = 8 * I + (e >> 3), gj = 8 * J + (e & 7);
                                    Mt[e] = -0.5 * (Bd[gi * ld + gj] + Bd[gj * ld + gi]);
                                }
                            }
                        for (int i = T.warp; i < mdp; i += T.nwarps)
                            for (int jx = T.lane; jx <= i; jx += 32) Lw[pk(i, jx)] = Gd[i * ld + jx];
                    } else {
                        for (int i = T.warp; i < mdp; i += T.nwarps)
                            for (int jx = T.lane; jx < mdp; jx += 32) {
                                Mw[i * ld + jx] = -0.5 * (Bd[i * ld + jx] + Bd[jx * ld + i]);
                                if (jx <= i) Lw[pk(i, jx)] = Gd[i * ld + jx];
                            }
                    }
                }
            }
            double* S = P.wS + (size_t)slot * P.w_sstride;
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
            continue;
        }

        // ---- 2. dense chord
        double theta_max = -SW_INF, theta_min = SW_INF;
        bool degenerate = false, failed = false;
        int lanczos_J = 0;
        if (!outward && md >= 1) {
            // global-scratch variant (m > 128): the inverse-diagonal-block DMMA factorisations
            // (measured +1% there; the shared-memory variants keep the substitution versions)
            // (the shared-memory variants with cholesky_inv_blocked_la + the left-looking
            // congruence were measured 3-7% slower at m = 10..60)
            double* Lv = vec + NVEC2 * vl + 64;
            bool okc = SMEM ? cholesky_blocked(T, Gd, mdp, ld, rdiag, &sh_i[2])
                            : cholesky_inv_blocked(T, Gd, mdp, ld, rdiag, Lv, &sh_i[2]);
            PROF_MARK(2);
            if (!okc) {
                failed = true;
            } else {
                if (!SMEM && SW_GLOBAL_LL) {  // m > 112: +11% at m = 200
                    congruence_inv(T, Gd, Lv, Bd, mdp, ld);
                } else if (SMEM) {
                    trsm_blocked<false>(T, Gd, Bd, mdp, ld, rdiag);
                    trsm_blocked<true>(T, Gd, Bd, mdp, ld, rdiag);
                } else {
                    trsm_inv_blocked<false>(T, Gd, Lv, Bd, mdp, ld);
                    trsm_inv_blocked<true>(T, Gd, Lv, Bd, mdp, ld);
                }
                PROF_MARK(3);
                // ---- M = -(B + B^T)/2 in place; park L (lower, with rdiag) in global
                // scratch so that the Lanczos basis can use its shared memory.
                for (int i = T.warp; i < mdp; i += T.nwarps) {
                    for (int jx = T.lane; jx <= i; jx += 32) {
                        double sv_ = -0.5 * (Bd[i * ld + jx] + Bd[jx * ld + i]);
                        Bd[i * ld + jx] = sv_;
                        Bd[jx * ld + i] = sv_;
                        Lsave[i * ld + jx] = Gd[i * ld + jx];
                    }
                }
                __syncthreads();
                int J;
                if (SMEM)
                {
                    // vector area + 64 slack doubles: [0,32) partial sums, [32,40) check results
                    const int oVec = (int)(vec - smem_dyn), oRed = oVec + NVEC2 * vl;
                    J = lanczos_reg<NT, KC>((int)(Bd - smem_dyn), (int)(Qm - smem_dyn), md, mdp, ld, P.need_tmin != 0, oVec,
                                            vl, oRed, 0, P.prof);
                    if (P.jlast && T.tid == 0) P.jlast[slot] = J;
                    theta_max = smem_dyn[oRed + 32 + 4];
                    theta_min = smem_dyn[oRed + 32 + 5];
                }
                else
                    J = lanczos_run(T, Bd, Qm, md, mdp, ld, true, P.need_tmin != 0, wv, hb, al, be, sv, sv2, dp, dm, red,
                                    &sh_i[3], &sh_d[4], P.prof, &theta_max, &theta_min, vec + 17 * vl, vec,
                                    vec + 4 * vl, vec + 9 * vl, (int)(vec - smem_dyn) + 48);
                lanczos_J = J;
                if (P.jsum && T.tid == 0) {
                    atomicAdd(&P.jsum[0], (unsigned long long)J);
                    atomicAdd(&P.jsum[1], 1ull);
                }
                if (P.prof && T.tid == 0) atomicAdd(&P.prof[10], (unsigned long long)J);
                PROF_MARK(4);
                if (T.tid == 0) {
                    double th2 = theta_max - 1e-12 * fabs(theta_max);
                    int c = sturm_below(al, be, J, th2);
                    sh_i[0] = (md >= 2 && J >= 2 && c <= J - 2) ? 1 : 0;
                }
                __syncthreads();
                degenerate = sh_i[0] != 0;
                PROF_MARK(5);
                if (theta_max > 0.0) {
                    // z = Q s
                    for (int e = T.tid; e < mdp; e += T.nthr) {
                        double s = 0.0;
                        for (int i = 0; i < J; ++i) s += sv[i] * Qm[(size_t)i * ld + e];
                        zz[e] = s;
                    }
                    __syncthreads();
                    for (int i = T.warp; i < md; i += T.nwarps)
                        for (int jx = T.lane; jx < i; jx += 32) Gd[i * ld + jx] = Lsave[i * ld + jx];
                    __syncthreads();
                    PROF_MARK(6);
                    // y = L^{-T} z, blocked backwards over 8-row blocks: warp 0 solves the
                    // 8x8 transposed diagonal block, all threads update the rows above
                    for (int kb = (mdp >> 3) - 1; kb >= 0; --kb) {
                        const int k0 = kb * 8;
                        if (T.warp == 0) {
                            const int r = T.lane;
                            double zr = (r < 8) ? zz[k0 + r] : 0.0;
#pragma unroll
                            for (int c = 7; c >= 0; --c) {
                                // y_c = z_c / L_cc; then z_r -= L_cr y_c for r < c
                                const double yc = __shfl_sync(0xffffffffu, zr, c) * rdiag[k0 + c];
                                if (r == c) zr = yc;
                                else if (r < c) zr -= Gd[(k0 + c) * ld + k0 + r] * yc;
                            }
                            if (r < 8) yy[k0 + r] = zr;
                        }
                        __syncthreads();
                        for (int i = T.tid; i < k0; i += T.nthr) {
                            double acc = zz[i];
#pragma unroll
                            for (int c = 0; c < 8; ++c) acc -= Gd[(k0 + c) * ld + i] * yy[k0 + c];
                            zz[i] = acc;
                        }
                        __syncthreads();
                    }
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
                }
                __syncthreads();
            }
        }
        PROF_MARK(7);
        (void)lanczos_J;

#include "chord_tail.inc"
    }
}

}  // namespace sw
