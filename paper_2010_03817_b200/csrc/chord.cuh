// chord.cuh -- shared K2 infrastructure: the per-call parameter block (ChordParams),
// CTA team helpers (block reductions), packed-symmetric unpack / axpy, the Householder
// congruence of a boundary start (R6), the Sturm count of a tridiagonal, the
// per-step bookkeeping (Philox draws, Alg. 5 P:1033-1034 / Alg. 6) and the
// profiling mark.  The chord kernels themselves are in chord2.cuh (fused) and chord3.cuh
// (split); the dense block is solved as in PAPER.md Alg. 2 through Lemma 3
// and the Cholesky-transformed pencil of P:1207-1215.
#pragma once
#include "common.cuh"

namespace sw {

// per-slot scalar/vector area (doubles), vl = mp + 8
enum : int { S_A = 0, S_BH = 1, S_MD = 2, S_ST = 3, S_TMAX = 4, S_TMIN = 5, S_DEG = 6, S_J = 7, S_VEC = 8 };
enum : int { ST_OUTWARD = 1, ST_FAILED = 2, ST_DEFL = 4 };
__host__ __device__ __forceinline__ long long s_stride(int mp) { return S_VEC + 4LL * (mp + 8); }


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
    int* ncap;  // HMC-r steps rejected because Weyl stepping hit its iteration cap
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
    unsigned long long* jsum;  // [0] sum of Lanczos iterations J, [1] Lanczos solves (measured flop model)
    int wkind;      // walk kind (SPEC_WALK_*): 2 = Hit-and-Run, 3 = coordinate Hit-and-Run
    int need_tmin;  // the chord must return t- as well (oracle mode, Hit-and-Run walks)
    int hnr_boltz;  // Hit-and-Run for exp(-c^T x / Temp) instead of the uniform law
    int gsplit;     // global-scratch chord_kernel2 as the factor phase only (m > 112 split): 1 = M as full rows
                    // (lanczos_cl.cuh), 2 = M as lower 8 x 8 tiles (lanczos_t.cuh)
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
    double eta_local = 0.0, u2_local = 0.0;
    // kind 3 (W-CHnR) needs no normals: only block nb (eta and the coordinate draw)
    for (int j = T.tid; j <= nb; j += T.nthr) {
        if (kind == 3 && j < nb) continue;
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
            u2_local = u01(w.z, w.w);
        }
    }
    double eta, u2;
    if (CTA) {
        if (T.tid == nb % T.nthr) {
            red[40] = eta_local;
            red[41] = u2_local;
        }
        ss = block_sum(T, ss, red);
        eta = red[40];
        u2 = red[41];
    } else {
        ss = warp_sum(ss);
        eta = __shfl_sync(0xffffffffu, eta_local, nb % 32);
        u2 = __shfl_sync(0xffffffffu, u2_local, nb % 32);
    }
    if (kind == 0 || kind == 2) {  // v ~ U(sphere): billiard (Alg. 5) and W-HnR (Alg. 4)
        double inv = 1.0 / sqrt(ss);
        for (int i = T.tid; i < n; i += T.nthr) v[i] *= inv;
    } else if (kind == 3) {  // v = e_j, j = floor(u2 n) (R29)
        const int jc = min(n - 1, (int)(u2 * (double)n));
        for (int i = T.tid; i < n; i += T.nthr) v[i] = (i == jc) ? 1.0 : 0.0;
    }
    const double* x = X + (size_t)slot * np;
    double* xs = Xs + (size_t)slot * np;
    for (int i = T.tid; i < n; i += T.nthr) xs[i] = x[i];
    const double* ax = AX + (size_t)slot * mtp;
    double* axs = AXs + (size_t)slot * mtp;
    for (int i = T.tid; i < mt; i += T.nthr) axs[i] = ax[i];
    // ell: billiard -L ln eta, HMC / collocation HMC L eta (Alg. 5 / Alg. 6 line 1); Hit-and-Run keeps eta (the
    // position of the next point on the chord)
    if (T.tid == 0) ell[slot] = (kind == 0) ? -Lpar * log(eta) : ((kind == 1 || kind == 4) ? Lpar * eta : eta);
    if (CTA) __syncthreads(); else __syncwarp();
}

// A point of the chord [tm, tp] from the restriction of exp(-c^T x / T) to the line x + t v,
// a = c^T v / T (W-HnR for the Boltzmann law, sec:optimization P:1408-1424): truncated
// exponential by its inverse CDF from the end of largest density (log1p / expm1 form);
// |a| (tp - tm) < 1e-12: the uniform point.  s is kept in [2^-26 d, (1 - 2^-26) d] (DESIGN.md
// R30: near a face the chord ends carry relative errors up to ~eps |M| / |theta|, and a point
// drawn closer than that would land on or outside the boundary).
__device__ __forceinline__ double boltz_chord_point(double tm, double tp, double a, double eta) {
    const double d = tp - tm, b = fabs(a) * d;
    double s = (b < 1e-12) ? eta * d : -log1p(eta * expm1(-b)) / fabs(a);
    s = fmin(fmax(s, 0x1p-26 * d), (1.0 - 0x1p-26) * d);
    return a >= 0.0 ? tm + s : tp - s;
}

// ---------------------------------------------------------------- K2
#define PROF_MARK(ph)                                                        \
    if (P.prof) {                                                            \
        __syncthreads();                                                     \
        long long t_ = clock64();                                            \
        if (T.tid == 0) atomicAdd(&P.prof[ph], (unsigned long long)(t_ - t_prof)); \
        t_prof = t_;                                                         \
    }

}  // namespace sw
