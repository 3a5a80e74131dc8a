// chord.cuh -- K2: the per-chain boundary oracle on the line pencil, fused with
// the closed-form cube / ball constraints, the advance and the step logic.
//
// One CTA per chain (persistent grid-stride over the active-chain list).  The
// dense block is solved as in PAPER.md Alg. 2 through Lemma 3
// and the "special structure" of P:1207-1215:
//   L L^T = A(x)                      (Cholesky, right-looking)
//   M = -L^{-1} A(v) L^{-T}           (two column/row-parallel substitutions)
//   T = Q^T M Q                       (Householder tridiagonalisation)
//   theta_max = lambda_max(T)         (parallel multisection on Sturm counts)
//   z = Q s, (T - theta) s ~ 0        (inverse iteration, pivoted tridiag LU)
//   y = L^{-T} z, t+ = 1/theta_max    (the PEP eigenvector)
// A segment that starts on the dense boundary (after a reflection) is
// deflated by the known kernel vector u (Householder + Schur complement,
// DESIGN.md R6).  Matrices live in shared memory (m <= SW_SMEM_MMAX) or in a
// per-CTA global scratch slice (larger m).
#pragma once
#include "common.cuh"

namespace sw {

constexpr int NVEC = 16;  // vector scratch slots of length m

struct ChordParams {
    int n, np, m, mt, mtp, ld;
    int mode;  // 0 = billiard walk, 1 = boundary_oracle batch
    const double* AV;
    double* AX;
    double* AXs;
    double* Yh;
    double* X;
    double* Xs;
    double* V;
    double* U;
    double* ell;
    int* steps_done;
    int* refl;
    int* bound;
    int* flags;
    long long* calls;
    long long* nrefl;
    int* nrej;
    int* ndeg;
    const double* lo;
    const double* hi;
    const double* ball_c;
    double ball_r;
    int has_ball;
    // walk parameters
    int steps_total;
    double Lpar;
    long long rho;
    unsigned long long seed;
    unsigned tag;
    long long chain_base;
    const long long* gid;  // optional global ids per slot (trace)
    // lists
    const int* list;
    const int* count_dev;
    int count_host;
    int* nlist;
    int* ncount;
    // oracle outputs (mode 1)
    double* o_tminus;
    double* o_tplus;
    double* o_kernel;
    int* o_binding;
    int* o_status;
    // trace (optional)
    int max_trace;
    int* tr_cnt;
    double* tr_hit;
    double* tr_t;
    double* tr_w;
    double* tr_v;
    int* tr_bind;
    // scratch
    double* scratch;
    long long scratch_stride;
    unsigned long long* prof;  // optional per-phase cycle counters (SPECWALK_PROF=1)
    double* lsave;             // per-CTA global slice where L is parked during Lanczos
    long long lsave_stride;
    // HMC-r (K5)
    const double* Ac;  // packed A(c) = sum c_i A_i
    const double* cvec;
    double Temp;
    double* tlast;  // t+ of the last hit (velocity at the hit = v - (c/T) t+)
    int* jlast;     // Lanczos iterations of the chain's previous call (first-check hint)
    // K2 split into factor / Lanczos / tail kernels: per-slot work buffers
    double* wM;     // M = -L^{-1} A(v) L^{-T} (mdp x mdp rows, leading dimension ld)
    double* wL;     // L (lower incl. diagonal, rows of leading dimension ld)
    double* wS;     // scalars + vectors (chord3.cuh: S_*)
    long long w_mstride, w_sstride;
    // K5 split (hmc2.cuh): per-slot Weyl-stepping state, Householder rank-2 vectors
    double* wH;       // H_* scalars per slot
    double* wQ;       // q_0, q_1, q_2 (3 x (mp + 8) per slot)
    int* nxt_list;    // slots still stepping after this iteration
    int* nxt_count;
    int zall;         // lanczos_kernel: z = Q s whatever the sign of theta_max
};

// ---------------------------------------------------------------- team helpers
struct Team {
    int tid, nthr, lane, warp, nwarps;
};

__device__ __forceinline__ double block_sum(const Team& T, double v, double* red) {
    v = warp_sum(v);
    if (T.lane == 0) red[T.warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < T.nwarps; ++w) s += red[w];
    __syncthreads();
    return s;
}
__device__ __forceinline__ double block_max(const Team& T, double v, double* red) {
    v = warp_max(v);
    if (T.lane == 0) red[T.warp] = v;
    __syncthreads();
    double s = -SW_INF;
    for (int w = 0; w < T.nwarps; ++w) s = fmax(s, red[w]);
    __syncthreads();
    return s;
}
__device__ __forceinline__ double block_min(const Team& T, double v, double* red) {
    v = warp_min(v);
    if (T.lane == 0) red[T.warp] = v;
    __syncthreads();
    double s = SW_INF;
    for (int w = 0; w < T.nwarps; ++w) s = fmin(s, red[w]);
    __syncthreads();
    return s;
}

// ---------------------------------------------------------------- dense LA on a CTA
// unpack packed-lower P into full symmetric M (leading dimension ld)
// (all loads of a thread are issued before its stores: one global round trip)
__device__ __forceinline__ void unpack_sym(const Team& T, const double* __restrict__ P, double* M, int m, int ld) {
    const int mt = m * (m + 1) / 2;
    constexpr int K = 16;
    for (int e0 = 0; e0 < mt; e0 += K * T.nthr) {
        double val[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            int e = e0 + k * T.nthr + T.tid;
            val[k] = (e < mt) ? __ldg(P + e) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            int e = e0 + k * T.nthr + T.tid;
            if (e < mt) {
                int i = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
                if (pk(i + 1, 0) <= e) ++i;
                if (pk(i, 0) > e) --i;
                int j = e - pk(i, 0);
                M[i * ld + j] = val[k];
                M[j * ld + i] = val[k];
            }
        }
    }
}

// ax += th * av over the packed vector, loads issued before stores
__device__ __forceinline__ void packed_axpy(const Team& T, double* ax, const double* __restrict__ av, double th,
                                            int mt) {
    constexpr int K = 20;  // m = 100: 5050 / 256 threads -> every load of a thread in flight at once
    for (int e0 = 0; e0 < mt; e0 += K * T.nthr) {
        double a[K], b[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            int e = e0 + k * T.nthr + T.tid;
            a[k] = (e < mt) ? ax[e] : 0.0;
            b[k] = (e < mt) ? __ldg(av + e) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            int e = e0 + k * T.nthr + T.tid;
            if (e < mt) ax[e] = a[k] + th * b[k];
        }
    }
}

// symmetric X <- H X H with H = I - beta h h^T  (X full, m x m)
__device__ void householder_congruence(const Team& T, double* X, int m, int ld, const double* h, double beta,
                                       double* p, double* red) {
    for (int i = T.warp; i < m; i += T.nwarps) {
        double s = 0.0;
        for (int j = T.lane; j < m; j += 32) s += X[i * ld + j] * h[j];
        s = warp_sum(s);
        if (T.lane == 0) p[i] = beta * s;
    }
    __syncthreads();
    double hp = 0.0;
    for (int i = T.tid; i < m; i += T.nthr) hp += h[i] * p[i];
    double K = 0.5 * beta * block_sum(T, hp, red);
    for (int i = T.tid; i < m; i += T.nthr) p[i] = p[i] - K * h[i];  // q
    __syncthreads();
    for (int i = T.warp; i < m; i += T.nwarps) {
        const double hi = h[i], pi = p[i];
        for (int j = T.lane; j < m; j += 32) X[i * ld + j] -= hi * p[j] + pi * h[j];
    }
    __syncthreads();
}

// right-looking Cholesky of the lower triangle of G (md x md); returns false on a
// non-positive pivot (uniform across the CTA).
__device__ bool cholesky_cta(const Team& T, double* G, int md, int ld, double* colk) {
    for (int k = 0; k < md; ++k) {
        double d = G[k * ld + k];
        if (!(d > 0.0)) return false;
        double s = sqrt(d);
        double inv = 1.0 / s;
        for (int i = k + 1 + T.tid; i < md; i += T.nthr) colk[i] = G[i * ld + k] * inv;
        __syncthreads();
        if (T.tid == 0) G[k * ld + k] = s;
        for (int i = k + 1 + T.warp; i < md; i += T.nwarps) {
            double li = colk[i];
            double* row = G + i * ld;
            if (T.lane == 0) row[k] = li;
            for (int j = k + 1 + T.lane; j <= i; j += 32) row[j] -= li * colk[j];
        }
        __syncthreads();
    }
    return true;
}

// B <- -L^{-1} B L^{-T} (B symmetric full md x md, L lower in G); result symmetrised.
__device__ void congruence_cta(const Team& T, const double* G, double* B, int md, int ld) {
    // X = L^{-1} B : thread j owns column j
    for (int j = T.tid; j < md; j += T.nthr) {
        for (int i = 0; i < md; ++i) {
            const double* Li = G + i * ld;
            double s0 = B[i * ld + j], s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int k = 0;
            for (; k + 3 < i; k += 4) {
                s0 -= Li[k] * B[k * ld + j];
                s1 -= Li[k + 1] * B[(k + 1) * ld + j];
                s2 -= Li[k + 2] * B[(k + 2) * ld + j];
                s3 -= Li[k + 3] * B[(k + 3) * ld + j];
            }
            for (; k < i; ++k) s0 -= Li[k] * B[k * ld + j];
            B[i * ld + j] = ((s0 + s1) + (s2 + s3)) / Li[i];
        }
    }
    __syncthreads();
    // row j of M = -(L^{-1} X[j,:]^T)^T : thread j owns row j
    for (int j = T.tid; j < md; j += T.nthr) {
        double* Bj = B + j * ld;
        for (int i = 0; i < md; ++i) {
            const double* Li = G + i * ld;
            double s0 = Bj[i], s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int k = 0;
            for (; k + 3 < i; k += 4) {
                s0 -= Li[k] * Bj[k];
                s1 -= Li[k + 1] * Bj[k + 1];
                s2 -= Li[k + 2] * Bj[k + 2];
                s3 -= Li[k + 3] * Bj[k + 3];
            }
            for (; k < i; ++k) s0 -= Li[k] * Bj[k];
            Bj[i] = ((s0 + s1) + (s2 + s3)) / Li[i];
        }
        for (int i = 0; i < md; ++i) Bj[i] = -Bj[i];
    }
    __syncthreads();
    for (int e = T.tid; e < md * md; e += T.nthr) {
        int i = e / md, j = e - i * md;
        if (j < i) {
            double s = 0.5 * (B[i * ld + j] + B[j * ld + i]);
            B[i * ld + j] = s;
            B[j * ld + i] = s;
        }
    }
    __syncthreads();
}

// Householder tridiagonalisation of symmetric M (md x md, full storage), LAPACK
// dsytd2 conventions: H_k = I - tau_k v v^T, v = [1, M[k+2.., k]].
// d (diag), e (offdiag), tau written; reflector tails stored in column k.
__device__ void tridiag_cta(const Team& T, double* M, int md, int ld, double* d, double* e, double* tau,
                            double* vb, double* pw, double* red) {
    for (int k = 0; k + 2 < md; ++k) {
        const int L = md - k - 1;
        double* x = M + (k + 1) * ld + k;  // x[i*ld], i in [0, L)
        double sig = 0.0;
        for (int i = 1 + T.tid; i < L; i += T.nthr) sig += x[i * ld] * x[i * ld];
        sig = block_sum(T, sig, red);
        double alpha = x[0];
        double tk = 0.0, beta = alpha, scale = 0.0;
        if (sig != 0.0) {
            double nrm = sqrt(alpha * alpha + sig);
            beta = (alpha >= 0.0) ? -nrm : nrm;
            tk = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        if (T.tid == 0) {
            e[k] = beta;
            tau[k] = tk;
            vb[0] = 1.0;
        }
        for (int i = 1 + T.tid; i < L; i += T.nthr) {
            double vi = x[i * ld] * scale;
            vb[i] = vi;
            x[i * ld] = vi;  // store the reflector tail for the back-transform
        }
        __syncthreads();
        if (tk == 0.0) continue;
        double* A22 = M + (k + 1) * ld + (k + 1);
        for (int i = T.warp; i < L; i += T.nwarps) {
            const double* row = A22 + i * ld;
            double s = 0.0;
            for (int j = T.lane; j < L; j += 32) s += row[j] * vb[j];
            s = warp_sum(s);
            if (T.lane == 0) pw[i] = tk * s;
        }
        __syncthreads();
        double pv = 0.0;
        for (int i = T.tid; i < L; i += T.nthr) pv += pw[i] * vb[i];
        double K = 0.5 * tk * block_sum(T, pv, red);
        for (int i = T.tid; i < L; i += T.nthr) pw[i] -= K * vb[i];
        __syncthreads();
        for (int q = T.tid; q < L * L; q += T.nthr) {
            int i = q / L, j = q - i * L;
            A22[i * ld + j] -= vb[i] * pw[j] + pw[i] * vb[j];
        }
        __syncthreads();
    }
    for (int i = T.tid; i < md; i += T.nthr) d[i] = M[i * ld + i];
    if (T.tid == 0 && md >= 2) e[md - 2] = M[(md - 1) * ld + (md - 2)];
    __syncthreads();
}

// number of eigenvalues of T (d, e) strictly below sigma: sign changes of the
// leading principal minors p_i = det(T_i - sigma I) (three-term recurrence with
// exact power-of-two rescaling; a zero minor counts as a sign change).
__device__ __forceinline__ int sturm_below(const double* d, const double* e, int md, double sigma) {
    double pp = 1.0, p = d[0] - sigma;
    int cnt = (p <= 0.0) ? 1 : 0;
    bool neg = (p < 0.0) || (p == 0.0);  // sign of p (zero -> opposite of p_0 = +)
    if (p == 0.0) p = -1e-300;
    for (int i = 1; i < md; ++i) {
        double e2 = e[i - 1] * e[i - 1];
        double pn = (d[i] - sigma) * p - e2 * pp;
        bool nneg;
        if (pn == 0.0) {
            nneg = !neg;
            pn = neg ? 1e-300 : -1e-300;
        } else {
            nneg = pn < 0.0;
        }
        cnt += (nneg != neg) ? 1 : 0;
        neg = nneg;
        pp = p;
        p = pn;
        double ap = fabs(p);
        if (ap > 0x1p+500) {
            p *= 0x1p-500;
            pp *= 0x1p-500;
        } else if (ap < 0x1p-500 && fabs(pp) < 0x1p-500) {
            p *= 0x1p+500;
            pp *= 0x1p+500;
        }
    }
    return cnt;
}

// largest (top=true) or smallest eigenvalue of the tridiagonal by CTA-wide
// multisection: every thread evaluates one Sturm count per round.
__device__ double tri_extreme(const Team& T, const double* d, const double* e, int md, bool top, double* red) {
    double gl = SW_INF, gh = -SW_INF, dmax = -SW_INF, dmin = SW_INF;
    for (int i = T.tid; i < md; i += T.nthr) {
        double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < md ? fabs(e[i]) : 0.0);
        gl = fmin(gl, d[i] - r);
        gh = fmax(gh, d[i] + r);
        dmax = fmax(dmax, d[i]);
        dmin = fmin(dmin, d[i]);
    }
    double lo, hi;
    if (top) {
        lo = block_max(T, dmax, red);  // a Rayleigh quotient: lambda_max >= lo
        hi = block_max(T, gh, red);
    } else {
        lo = block_min(T, gl, red);
        hi = block_min(T, dmin, red);  // lambda_min <= hi
    }
    if (md == 1) return d[0];
    const double eps = 2.220446049250313e-16;
    for (int it = 0; it < 24; ++it) {
        if (!(hi - lo > 2.0 * eps * fmax(fabs(lo), fabs(hi))) || !(hi > lo)) break;
        double sig = lo + (hi - lo) * ((double)(T.tid + 1) / (double)(T.nthr + 1));
        int c = sturm_below(d, e, md, sig);
        double cand_hi, cand_lo;
        if (top) {  // c == md  <=> lambda_max < sig
            cand_hi = (c == md) ? sig : SW_INF;
            cand_lo = (c < md) ? sig : -SW_INF;
        } else {    // c >= 1   <=> lambda_min < sig
            cand_hi = (c >= 1) ? sig : SW_INF;
            cand_lo = (c == 0) ? sig : -SW_INF;
        }
        double nh = block_min(T, cand_hi, red);
        double nl = block_max(T, cand_lo, red);
        hi = fmin(hi, nh);
        lo = fmax(lo, nl);
    }
    return 0.5 * (lo + hi);
}

// eigenvector of the tridiagonal for eigenvalue theta: inverse iteration with a
// partially pivoted LU of (T - theta I) (LAPACK dgttrf/dgttrs pattern); one thread.
__device__ void tri_eigvec(const double* d, const double* e, int md, double theta, double* x, double* a,
                           double* b, double* c, double* u2, double* piv) {
    double tnorm = 0.0;
    for (int i = 0; i < md; ++i) tnorm = fmax(tnorm, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) +
                                                        (i + 1 < md ? fabs(e[i]) : 0.0));
    double tiny = 2.220446049250313e-16 * fmax(tnorm, 1e-300);
    for (int i = 0; i < md; ++i) {
        a[i] = d[i] - theta;
        if (i + 1 < md) {
            b[i] = e[i];
            c[i] = e[i];
        }
        u2[i] = 0.0;
    }
    for (int i = 0; i + 1 < md; ++i) {
        if (fabs(a[i]) >= fabs(c[i])) {
            if (a[i] == 0.0) a[i] = tiny;
            double l = c[i] / a[i];
            c[i] = l;
            a[i + 1] -= l * b[i];
            piv[i] = 0.0;
        } else {
            double l = a[i] / c[i];
            a[i] = c[i];
            double tmp = a[i + 1];
            a[i + 1] = b[i] - l * tmp;
            if (i + 2 < md) {
                u2[i] = b[i + 1];
                b[i + 1] = -l * b[i + 1];
            }
            b[i] = tmp;
            c[i] = l;
            piv[i] = 1.0;
        }
    }
    if (a[md - 1] == 0.0) a[md - 1] = tiny;
    for (int i = 0; i < md; ++i) x[i] = 1.0 / (1.0 + 0.6180339887498949 * (double)i);
    for (int sweep = 0; sweep < 2; ++sweep) {
        for (int i = 0; i + 1 < md; ++i) {
            if (piv[i] == 0.0) {
                x[i + 1] -= c[i] * x[i];
            } else {
                double t = x[i];
                x[i] = x[i + 1];
                x[i + 1] = t - c[i] * x[i];
            }
        }
        x[md - 1] /= a[md - 1];
        if (md >= 2) x[md - 2] = (x[md - 2] - b[md - 2] * x[md - 1]) / a[md - 2];
        for (int i = md - 3; i >= 0; --i) x[i] = (x[i] - b[i] * x[i + 1] - u2[i] * x[i + 2]) / a[i];
        double nn = 0.0;
        for (int i = 0; i < md; ++i) nn = fmax(nn, fabs(x[i]));
        double s = 1.0 / nn;
        for (int i = 0; i < md; ++i) x[i] *= s;
    }
}

// ---------------------------------------------------------------- step bookkeeping
// Draw the next step (Alg. 5 lines 1-2: l = -tau ln eta, v ~ U(sphere)) for one
// chain with a CTA (or a warp when CTA == false).
template <bool CTA>
__device__ void step_start(const Team& T, int slot, long long gidv, int step, int n, int np, int mt, int mtp,
                           double* V, double* X, double* Xs, const double* AX, double* AXs, double* ell,
                           double Lpar, unsigned long long seed, unsigned tag, int kind, double* red) {
    const int nb = (n + 1) / 2;
    double* v = V + (size_t)slot * np;
    uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const double two_pi = 6.283185307179586476925286766559;
    double ss = 0.0;
    double eta_local = 0.0;
    for (int j = T.tid; j <= nb; j += T.nthr) {
        uint4 w = philox4x32_10(make_uint4((uint32_t)j, (uint32_t)step, (uint32_t)gidv, tag), key);
        if (j < nb) {
            double u0 = u01(w.x, w.y), u1 = u01(w.z, w.w);
            double r = sqrt(-2.0 * log(u0));
            double a = two_pi * u1;
            double g0 = r * cos(a);
            v[2 * j] = g0;
            ss += g0 * g0;
            if (2 * j + 1 < n) {
                double g1 = r * sin(a);
                v[2 * j + 1] = g1;
                ss += g1 * g1;
            }
        } else {
            eta_local = u01(w.x, w.y);
        }
    }
    double eta;
    if (CTA) {
        if (T.tid == nb % T.nthr) red[40] = eta_local;
        ss = block_sum(T, ss, red);
        eta = red[40];
    } else {
        ss = warp_sum(ss);
        eta = __shfl_sync(0xffffffffu, eta_local, nb % 32);
    }
    if (kind == 0) {
        double inv = 1.0 / sqrt(ss);
        for (int i = T.tid; i < n; i += T.nthr) v[i] *= inv;
    }
    const double* x = X + (size_t)slot * np;
    double* xs = Xs + (size_t)slot * np;
    for (int i = T.tid; i < n; i += T.nthr) xs[i] = x[i];
    const double* ax = AX + (size_t)slot * mtp;
    double* axs = AXs + (size_t)slot * mtp;
    for (int i = T.tid; i < mt; i += T.nthr) axs[i] = ax[i];
    if (T.tid == 0) ell[slot] = (kind == 0) ? -Lpar * log(eta) : Lpar * eta;
    if (CTA) __syncthreads(); else __syncwarp();
}

// ---------------------------------------------------------------- K2
#define PROF_MARK(ph)                                                        \
    if (P.prof) {                                                            \
        __syncthreads();                                                     \
        long long t_ = clock64();                                            \
        if (T.tid == 0) atomicAdd(&P.prof[ph], (unsigned long long)(t_ - t_prof)); \
        t_prof = t_;                                                         \
    }

template <bool SMEM>
__global__ void __launch_bounds__(256) chord_kernel(ChordParams P) {
    extern __shared__ __align__(16) double smem_dyn[];
    Team T;
    T.tid = threadIdx.x;
    T.nthr = blockDim.x;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = T.nthr >> 5;
    __shared__ double red[64];
    __shared__ int sh_i[8];
    __shared__ double sh_d[16];

    const int m = P.m, n = P.n, ld = P.ld;
    double* base = SMEM ? smem_dyn : (P.scratch + (size_t)blockIdx.x * P.scratch_stride);
    double* G = base;
    double* B = base + (size_t)m * ld;
    double* vec = B + (size_t)m * ld;
    double* uu = vec + 0 * m;   // unit kernel vector (boundary start)
    double* hh = vec + 1 * m;   // Householder vector
    double* dd = vec + 2 * m;
    double* ee = vec + 3 * m;
    double* ta = vec + 4 * m;
    double* vb = vec + 5 * m;
    double* pw = vec + 6 * m;
    double* zz = vec + 7 * m;
    double* yy = vec + 8 * m;
    double* t_a = vec + 9 * m;
    double* t_b = vec + 10 * m;
    double* t_c = vec + 11 * m;
    double* t_u = vec + 12 * m;
    double* t_p = vec + 13 * m;
    double* colk = vec + 14 * m;

    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int r = blockIdx.x; r < count; r += gridDim.x) {
        const int slot = P.list ? P.list[r] : r;
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

        // ---- 1. A(x), A(v) into shared memory
        unpack_sym(T, ax, G, m, ld);
        unpack_sym(T, av, B, m, ld);
        const bool defl = (bnd == 0) && (m >= 1);
        if (defl) {
            for (int i = T.tid; i < m; i += T.nthr) uu[i] = P.U[(size_t)slot * m + i];
        }
        __syncthreads();
        PROF_MARK(0);
        int md = m;
        double* Gw = G;
        double* Bw = B;
        double a_schur = 0.0, beta_h = 0.0;
        bool outward = false;
        if (defl) {
            double nu = 0.0;
            for (int i = T.tid; i < m; i += T.nthr) nu += uu[i] * uu[i];
            nu = sqrt(block_sum(T, nu, red));
            for (int i = T.tid; i < m; i += T.nthr) {
                double ui = uu[i] / nu;
                hh[i] = ui;
            }
            __syncthreads();
            if (T.tid == 0) hh[0] += (hh[0] >= 0.0 ? 1.0 : -1.0);
            __syncthreads();
            double h2 = 0.0;
            for (int i = T.tid; i < m; i += T.nthr) h2 += hh[i] * hh[i];
            beta_h = 2.0 / block_sum(T, h2, red);
            householder_congruence(T, G, m, ld, hh, beta_h, pw, red);
            householder_congruence(T, B, m, ld, hh, beta_h, pw, red);
            a_schur = B[0];
            outward = !(a_schur > 0.0);
            if (!outward) {
                for (int e2 = T.tid; e2 < (m - 1) * (m - 1); e2 += T.nthr) {
                    int i = 1 + e2 / (m - 1), j = 1 + e2 % (m - 1);
                    B[i * ld + j] -= B[i * ld] * B[j] / a_schur;
                }
            }
            __syncthreads();
            md = m - 1;
            Gw = G + ld + 1;
            Bw = B + ld + 1;
        }
        PROF_MARK(1);

        // ---- 2. dense chord
        double theta_max = -SW_INF, theta_min = SW_INF;
        bool degenerate = false, failed = false;
        if (!outward && md >= 1) {
            bool okc = cholesky_cta(T, Gw, md, ld, colk);
            PROF_MARK(2);
            if (!okc) {
                failed = true;
            } else {
                congruence_cta(T, Gw, Bw, md, ld);
                PROF_MARK(3);
                tridiag_cta(T, Bw, md, ld, dd, ee, ta, vb, pw, red);
                PROF_MARK(4);
                theta_max = tri_extreme(T, dd, ee, md, true, red);
                if (P.mode == 1) theta_min = tri_extreme(T, dd, ee, md, false, red);
                PROF_MARK(5);
                if (T.tid == 0) {
                    double th2 = theta_max - 1e-12 * fabs(theta_max);
                    int c = sturm_below(dd, ee, md, th2);
                    sh_i[0] = (md >= 2 && c <= md - 2) ? 1 : 0;
                    if (theta_max > 0.0) tri_eigvec(dd, ee, md, theta_max, zz, t_a, t_b, t_c, t_u, t_p);
                }
                __syncthreads();
                PROF_MARK(6);
                degenerate = sh_i[0] != 0;
                if (theta_max > 0.0) {
                    // back-transform z <- Q s (warp 0), then y = L^{-T} z
                    if (T.warp == 0) {
                        for (int k = md - 3; k >= 0; --k) {
                            double tk = ta[k];
                            if (tk == 0.0) continue;
                            const int L = md - k - 1;
                            const double* vcol = Bw + (k + 1) * ld + k;
                            double s = 0.0;
                            for (int i = T.lane; i < L; i += 32) s += (i == 0 ? 1.0 : vcol[i * ld]) * zz[k + 1 + i];
                            s = warp_sum(s) * tk;
                            for (int i = T.lane; i < L; i += 32) zz[k + 1 + i] -= s * (i == 0 ? 1.0 : vcol[i * ld]);
                            __syncwarp();
                        }
                        for (int i = md - 1; i >= 0; --i) {
                            double yi = zz[i] / Gw[i * ld + i];
                            __syncwarp();
                            if (T.lane == 0) yy[i] = yi;
                            for (int k = T.lane; k < i; k += 32) zz[k] -= Gw[i * ld + k] * yi;
                            __syncwarp();
                        }
                        if (defl) {  // y = H [ -b^T yh / a ; yh ]
                            double s = 0.0;
                            for (int i = T.lane; i < md; i += 32) s += B[(i + 1) * ld] * yy[i];
                            s = warp_sum(s);
                            double alpha = -s / a_schur;
                            __syncwarp();
                            // shift yh into positions 1..m-1 (descending to avoid overlap)
                            for (int base_i = md - 1; base_i >= 0; base_i -= 32) {
                                int i = base_i - T.lane;
                                double val = (i >= 0) ? yy[i] : 0.0;
                                __syncwarp();
                                if (i >= 0) yy[i + 1] = val;
                                __syncwarp();
                            }
                            if (T.lane == 0) yy[0] = alpha;
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
#include "chord_tail.inc"
    }
}

}  // namespace sw
