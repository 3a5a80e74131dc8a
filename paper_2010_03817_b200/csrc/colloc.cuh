// colloc.cuh -- K7: reflective HMC on collocation polynomials for a log-concave density
// exp(-f) (PAPER.md sec:hmcr P:1116-1158, Alg. 6; R33).
//
// One boundary-oracle call = one trajectory segment of length h' = min(h, l_left):
//   K7a chmc_poly_kernel   warp per chain: Picard iteration for the node forces g_j =
//                          -grad f(p(s_j h')) at the q Chebyshev nodes, then the monomial
//                          coefficients c_1 = v, c_(k+2) = sum_j l_jk g_j / (h'^k (k+1)(k+2))
//                          of the degree-d = q+1 curve p(t) (c_0 = x); the rows c_1..c_d and
//                          the GEMM row list slot*d + k
//   K1  gemm_f64_dmma      B_k = A(c_k) = sum_i c_ki A_i for all d rows of every chain (one
//                          batched DMMA contraction)
//   K7b chmc_chord_kernel  CTA per chain, matrices in a per-CTA global scratch slice: the
//                          first root in (0, h'] of det(A(x) + sum_k t^k B_k) by monotone Weyl
//                          stepping (as K5, hmc.cuh) on the degree-d pencil -- after a dense
//                          reflection on the sqrt(t)-deflated degree-2d pencil in the
//                          Householder basis of the kernel vector (SURVEY V14 generalised:
//                          with t = s^2 and row/column 0 scaled by 1/s, coefficient 2k carries
//                          the inner block of B_k and entry (0,0) of B_(k+1), coefficient
//                          2k-1 the border of B_k); the cube faces by the same Weyl stepping
//                          on each coordinate polynomial; then the advance x = p(t^),
//                          A(x) += sum_k t^k B_k, v = p'(t^) and the reflection bookkeeping.
//   K3/K4 (walk.cuh)       normal and reflection of p'(t+) at a dense hit (kind 4 reflects v
//                          as stored by K7b).
#pragma once
#include "hmc.cuh"

namespace sw {

constexpr int CH_MAXQ = 6;               // collocation nodes (trajectory degree <= 7)
constexpr int CH_MAXD = CH_MAXQ + 1;
constexpr int CH_MAXIT = 64;              // Picard iterations (R33)
constexpr int CH_SCALAR_MAXIT = 400;      // Weyl iterations of one cube-face polynomial
// scratch matrices per CTA: B_0..B_d, the 2d+1 deflated coefficients, K, N, the Lanczos basis, the
// (up to 2d) congruenced coefficients
__host__ __device__ constexpr int chmc_nmat(int d) { return (d + 1) + (2 * d + 1) + 3 + 2 * d; }

enum : int { POT_LINEAR = 0, POT_GAUSS = 1, POT_LOGCOSH = 2 };

// binomial coefficients binom(k, j), k, j < 16 (Taylor coefficients of the shifted pencil)
__device__ const double c_binom[16][16] = {
    {1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 2.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 3.0, 3.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 4.0, 6.0, 4.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 5.0, 10.0, 10.0, 5.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 6.0, 15.0, 20.0, 15.0, 6.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 7.0, 21.0, 35.0, 35.0, 21.0, 7.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 8.0, 28.0, 56.0, 70.0, 56.0, 28.0, 8.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 9.0, 36.0, 84.0, 126.0, 126.0, 84.0, 36.0, 9.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 10.0, 45.0, 120.0, 210.0, 252.0, 210.0, 120.0, 45.0, 10.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 11.0, 55.0, 165.0, 330.0, 462.0, 462.0, 330.0, 165.0, 55.0, 11.0, 1.0, 0.0, 0.0, 0.0, 0.0},
    {1.0, 12.0, 66.0, 220.0, 495.0, 792.0, 924.0, 792.0, 495.0, 220.0, 66.0, 12.0, 1.0, 0.0, 0.0, 0.0},
    {1.0, 13.0, 78.0, 286.0, 715.0, 1287.0, 1716.0, 1716.0, 1287.0, 715.0, 286.0, 78.0, 13.0, 1.0, 0.0, 0.0},
    {1.0, 14.0, 91.0, 364.0, 1001.0, 2002.0, 3003.0, 3432.0, 3003.0, 2002.0, 1001.0, 364.0, 91.0, 14.0, 1.0, 0.0},
    {1.0, 15.0, 105.0, 455.0, 1365.0, 3003.0, 5005.0, 6435.0, 6435.0, 5005.0, 3003.0, 1365.0, 455.0, 105.0, 15.0, 1.0}};

struct ChmcParams {
    double* CF;        // per slot d rows of np: c_1 .. c_d
    double* CB;        // per slot d rows of mtp: packed A(c_k)
    double* GW;        // per slot q rows of np: Picard node forces
    double* hseg;      // per slot: h' of the current segment
    int* elist;        // GEMM rows: list index r, k -> slot*d + k (-1: skipped)
    int q, d;
    double h;
    int pot;
    const double* mu;  // n (GAUSS, LOGCOSH)
    double scale;      // T (LINEAR) or sigma
    const double* cvec;
    double nodes[CH_MAXQ];
    double lcoef[CH_MAXQ * CH_MAXQ];  // lcoef[j*q + k]: s^k coefficient of the Lagrange polynomial l_j
    unsigned long long* picard;       // optional [0] sum of Picard iterations, [1] segments, [2] unconverged,
                                      // [3] congruences N_j = K^-1 D_j K^-T of the Weyl iterations
};

__device__ __forceinline__ double pot_grad(const ChmcParams& H, int i, double x) {
    if (H.pot == POT_LINEAR) return H.cvec[i] / H.scale;
    const double u = x - (H.mu ? H.mu[i] : 0.0);
    if (H.pot == POT_GAUSS) return u / (H.scale * H.scale);
    return tanh(u / H.scale) / H.scale;
}

// coefficients c_2..c_(q+1) of one coordinate from its node forces g[0..q-1]
__device__ __forceinline__ void colloc_coef1(const ChmcParams& H, const double* g, double hs, double* c) {
    double hk = 1.0;
    for (int k = 0; k < H.q; ++k) {
        double s = 0.0;
        for (int j = 0; j < H.q; ++j) s += H.lcoef[j * H.q + k] * g[j];
        c[k] = s / (hk * (double)(k + 1) * (double)(k + 2));
        hk *= hs;
    }
}

// ---------------------------------------------------------------- K7a
__global__ void __launch_bounds__(256) chmc_poly_kernel(ChordParams P, ChmcParams H) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    const int n = P.n, np = P.np, q = H.q, d = H.d;
    for (int rr = blockIdx.x * wpb + (threadIdx.x >> 5); rr < count; rr += gridDim.x * wpb) {
        const int slot = P.list ? P.list[rr] : rr;
        const bool skip = slot < 0 || (P.mode == 0 && (P.flags[slot] & CF_DONE));
        if (lane < d) H.elist[(size_t)rr * d + lane] = skip ? -1 : slot * d + lane;
        if (skip) continue;
        const double* x = P.X + (size_t)slot * np;
        const double* v = P.V + (size_t)slot * np;
        double hs = H.h;
        if (P.mode == 0) {
            const double el = P.ell[slot];
            hs = (el <= H.h) ? el : H.h;
        }
        if (lane == 0) H.hseg[slot] = hs;
        double* G = H.GW + (size_t)slot * q * np;
        for (int i = lane; i < n; i += 32) {
            const double g = -pot_grad(H, i, x[i]);
            for (int j = 0; j < q; ++j) G[j * np + i] = g;
        }
        int used = -1;
        for (int it = 0; it < CH_MAXIT; ++it) {
            double delta = 0.0, gmax = 0.0;
            for (int i = lane; i < n; i += 32) {
                double g[CH_MAXQ], c[CH_MAXQ];
                for (int j = 0; j < q; ++j) g[j] = G[j * np + i];
                colloc_coef1(H, g, hs, c);
                for (int j = 0; j < q; ++j) {
                    const double t = H.nodes[j] * hs;
                    double a = c[q - 1];
                    for (int k = q - 2; k >= 0; --k) a = a * t + c[k];
                    a = (a * t + v[i]) * t + x[i];
                    const double gn = -pot_grad(H, i, a);
                    delta = fmax(delta, fabs(gn - g[j]));
                    gmax = fmax(gmax, fabs(gn));
                    G[j * np + i] = gn;
                }
            }
            delta = warp_max(delta);
            gmax = warp_max(gmax);
            if (delta <= 1e-14 * (1.0 + gmax)) {
                used = it + 1;
                break;
            }
        }
        double* cf = H.CF + (size_t)slot * d * np;
        for (int i = lane; i < n; i += 32) {
            double g[CH_MAXQ], c[CH_MAXQ];
            for (int j = 0; j < q; ++j) g[j] = G[j * np + i];
            colloc_coef1(H, g, hs, c);
            cf[i] = v[i];
            for (int k = 0; k < q; ++k) cf[(size_t)(k + 1) * np + i] = c[k];
        }
        if (H.picard && lane == 0) {
            atomicAdd(&H.picard[0], (unsigned long long)(used > 0 ? used : CH_MAXIT));
            atomicAdd(&H.picard[1], 1ull);
            if (used < 0) atomicAdd(&H.picard[2], 1ull);
        }
    }
}

// smallest positive root of 1 + a h - sum_{j=2..D} c_j h^j (c_j >= 0): weyl_step for any degree
__device__ double weyl_step_n(double a, const double* c, int D) {
    auto f = [&](double h) {
        double v = 1.0 + a * h, hp = h;
        for (int j = 2; j <= D; ++j) {
            hp *= h;
            v -= c[j] * hp;
        }
        return v;
    };
    bool anyc = false;
    for (int j = 2; j <= D; ++j) anyc = anyc || (c[j] > 0.0);
    if (a >= 0.0 && !anyc) return SW_INF;
    double hi = (a < 0.0) ? -1.0 / a : 1.0;
    int guard = 0;
    while (f(hi) >= 0.0) {
        hi *= 2.0;
        if (++guard > 2000 || hi > 1e300) return SW_INF;
    }
    double lo = 0.0;
    for (int it = 0; it < 200; ++it) {
        double mid = 0.5 * (lo + hi);
        if (!(mid > lo && mid < hi)) break;
        if (f(mid) >= 0.0) lo = mid;
        else hi = mid;
    }
    return lo;
}

// First root in (0, tmax] of the scalar polynomial g (degree D, g[0] > 0) by Weyl stepping;
// on_face: g[0] is the face just left (treated as exactly 0) and the root t = 0 is divided
// out.  Returns SW_INF (no root in range), or -1 when an on-face start moves outward.
__device__ double scalar_first_root(const double* g0, int D, double tmax, bool on_face) {
    double g[2 * CH_MAXD + 2];
    int De = D;
    if (on_face) {
        for (int k = 1; k <= D; ++k) g[k - 1] = g0[k];
        De = D - 1;
        if (!(g[0] > 0.0)) return -1.0;
    } else {
        for (int k = 0; k <= D; ++k) g[k] = g0[k];
    }
    double s = 0.0;
    for (int it = 0; it < CH_SCALAR_MAXIT; ++it) {
        double e[2 * CH_MAXD + 2];
        for (int j = 0; j <= De; ++j) {
            double acc = 0.0;
            for (int k = De; k >= j; --k) acc = acc * s + c_binom[k][j] * g[k];
            e[j] = acc;
        }
        if (!(e[0] > 0.0)) return s;  // rounding past the root: the last safe point
        double c[2 * CH_MAXD + 2];
        for (int j = 2; j <= De; ++j) c[j] = fabs(e[j]) / e[0];
        const double h = weyl_step_n(De >= 1 ? e[1] / e[0] : 0.0, c, De);
        if (!(s + h < tmax)) return SW_INF;
        s += h;
        if (h <= 1e-15 * s) return s;
    }
    return s;
}

// ---------------------------------------------------------------- K7b
template <int NT>
__global__ void __launch_bounds__(NT, (NT <= 256) ? 2 : 1) chmc_chord_kernel(ChordParams P, ChmcParams H) {
    Team T;
    T.tid = threadIdx.x;
    T.nthr = NT;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = NT >> 5;
    __shared__ double red[64];
    __shared__ int sh_i[8];
    __shared__ double sh_d[16];
    extern __shared__ __align__(16) double smem_dyn[];

    const int m = P.m, ld = P.ld, n = P.n, np = P.np, d = H.d;
    const int mp = (m + 7) & ~7;
    const size_t MS = (size_t)mp * ld;
    double* base = P.scratch + (size_t)blockIdx.x * P.scratch_stride;
    double* Cm = base;                      // d+1 raw coefficient matrices B_0..B_d
    double* Ct = base + (size_t)(d + 1) * MS;  // 2d+1 deflated coefficients (boundary start)
    double* Kf = Ct + (size_t)(2 * d + 1) * MS;
    double* Nw = Kf + MS;
    double* Qb = Nw + MS;
    double* NK = Qb + MS;  // D congruenced coefficients N~_k
    const int vl = mp + 8;
    double* vec = smem_dyn;
    double* hh = vec + 0 * vl;
    double* pw = vec + 1 * vl;
    double* rdiag = vec + 2 * vl;
    double* hb = vec + 4 * vl;
    double* al = vec + 5 * vl;
    double* be = vec + 6 * vl;
    double* sv = vec + 7 * vl;
    double* sv2 = vec + 8 * vl;
    double* dp = vec + 9 * vl;
    double* dm = vec + 10 * vl;
    double* zz = vec + 11 * vl;
    double* yy = vec + 12 * vl;
    double* yk = vec + 13 * vl;
    double* wv = vec + 14 * vl;  // 2 slots (ping-pong)
    double* pq = vec + 16 * vl;  // p = K^-1 e_0 and q_k = K^-1 b_k (d + 1 vectors)

    const int count = P.count_dev ? min(*P.count_dev, P.count_host) : P.count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = P.list ? P.list[rr] : rr;
        if (slot < 0) continue;
        if (P.mode == 0 && (P.flags[slot] & CF_DONE)) continue;
        const long long gidv = P.gid ? P.gid[slot] : P.chain_base + slot;
        double* x = P.X + (size_t)slot * np;
        double* v = P.V + (size_t)slot * np;
        double* ax = P.AX + (size_t)slot * P.mtp;
        const double* cf = H.CF + (size_t)slot * d * np;
        const double* cb = H.CB + (size_t)slot * d * P.mtp;
        const double hs = H.hseg[slot];
        const int bnd = P.bound[slot];
        __syncthreads();

        // ---- B_0 = A(x), B_k = A(c_k), padded (identity on the padding of B_0)
        unpack_sym(T, ax, Cm, m, ld);
        for (int k = 1; k <= d; ++k) unpack_sym(T, cb + (size_t)(k - 1) * P.mtp, Cm + k * MS, m, ld);
        __syncthreads();
        for (int k = 0; k <= d; ++k)
            for (int i = T.warp; i < mp; i += T.nwarps)
                for (int j = T.lane; j < mp; j += 32)
                    if (i >= m || j >= m) Cm[k * MS + i * ld + j] = (k == 0 && i == j) ? 1.0 : 0.0;
        __syncthreads();
        const bool defl = (bnd == 0);
        int D = d;
        double* Cs = Cm;  // the stepping pencil: Cm (interior) or Ct (deflated)
        double beta_h = 0.0;
        bool outward = false;
        if (defl) {
            double nu = 0.0;
            for (int i = T.tid; i < m; i += T.nthr) {
                hh[i] = P.U[(size_t)slot * m + i];
                nu += hh[i] * hh[i];
            }
            nu = sqrt(block_sum(T, nu, red));
            for (int i = T.tid; i < m; i += T.nthr) hh[i] /= nu;
            __syncthreads();
            if (T.tid == 0) hh[0] += (hh[0] >= 0.0 ? 1.0 : -1.0);
            __syncthreads();
            double h2 = 0.0;
            for (int i = T.tid; i < m; i += T.nthr) h2 += hh[i] * hh[i];
            beta_h = 2.0 / block_sum(T, h2, red);
            for (int k = 0; k <= d; ++k) householder_congruence(T, Cm + k * MS, m, ld, hh, beta_h, pw, red);
            outward = !(Cm[MS] > 0.0);  // u^T B_1 u: the reflected velocity must point inward
            // t = s^2, row/column 0 scaled by 1/s: Ct_2k = [B_(k+1)(0,0) | inner B_k],
            // Ct_(2k-1) = border of B_k
            D = 2 * d;
            for (int e = 0; e <= D; ++e) {
                double* C = Ct + e * MS;
                for (int i = T.warp; i < mp; i += T.nwarps)
                    for (int j = T.lane; j < mp; j += 32) {
                        const bool bi = (i == 0), bj = (j == 0);
                        double val = 0.0;
                        if (i < m && j < m) {
                            if (e & 1) {
                                const int k = (e + 1) >> 1;
                                if (bi != bj) val = Cm[k * MS + i * ld + j];
                            } else {
                                const int k = e >> 1;
                                if (bi && bj) val = (k + 1 <= d) ? Cm[(k + 1) * MS] : 0.0;
                                else if (!bi && !bj) val = Cm[k * MS + i * ld + j];
                            }
                        } else if (e == 0 && i == j) {
                            val = 1.0;
                        }
                        C[i * ld + j] = val;
                    }
            }
            __syncthreads();
            Cs = Ct;
        }
        const double s_end = defl ? sqrt(hs) : hs;

        // ---- monotone Weyl stepping on sum_e s^e Cs_e over (0, s_end]
        double s = 0.0;
        bool failed = false, hit = false, capped = false;
        if (!outward) {
            bool ended = false;
            for (int it = 0; it < HMC_MAX_IT; ++it) {
                for (int i = T.warp; i < mp; i += T.nwarps)
                    for (int j = T.lane; j < mp; j += 32) {
                        double acc = Cs[D * MS + i * ld + j];
                        for (int k = D - 1; k >= 0; --k) acc = acc * s + Cs[k * MS + i * ld + j];
                        Kf[i * ld + j] = acc;
                    }
                __syncthreads();
                bool ok = cholesky_blocked(T, Kf, mp, ld, rdiag, &sh_i[2]);
                if (!ok) {
                    if (it == 0) failed = true;  // start not interior
                    else hit = true;             // rounding past the root: s is the last safe point
                    ended = true;
                    break;
                }
                double cj[2 * CH_MAXD + 2];
                for (int j = 0; j <= D; ++j) cj[j] = 0.0;
                double a_min = 0.0;
                // each coefficient congruenced once: N~_k = K^-1 Cs_k K^-T (dense), or -- the border
                // coefficients of a deflated start (odd k: e_0 b^T + b e_0^T) -- p q_k^T + q_k p^T with
                // p = K^-1 e_0, q_k = K^-1 b_k (vector solves); then N_j = sum_k binom(k, j) s^(k-j) N~_k
                int ncong = 0;
                for (int k = 1; k <= D; ++k) {
                    if (defl && (k & 1)) continue;
                    double* Nk = NK + (size_t)(k - 1) * MS;
                    for (int i = T.warp; i < mp; i += T.nwarps)
                        for (int jx = T.lane; jx < mp; jx += 32) Nk[i * ld + jx] = Cs[k * MS + i * ld + jx];
                    __syncthreads();
                    trsm_blocked<false>(T, Kf, Nk, mp, ld, rdiag);
                    trsm_blocked<true>(T, Kf, Nk, mp, ld, rdiag);
                    ++ncong;
                }
                if (defl) {
                    // warp w: vector w (0: e_0, k = 2w - 1: column 0 of Cs_k), forward substitution
                    for (int w = T.warp; w <= d; w += T.nwarps) {
                        double* xv = pq + (size_t)w * vl;
                        for (int i = T.lane; i < mp; i += 32)
                            xv[i] = (w == 0) ? (i == 0 ? 1.0 : 0.0) : (i == 0 ? 0.0 : Cs[(2 * w - 1) * MS + i * ld]);
                        __syncwarp();
                        for (int i = 0; i < mp; ++i) {
                            double acc = 0.0;
                            for (int k = T.lane; k < i; k += 32) acc += Kf[i * ld + k] * xv[k];
                            acc = warp_sum(acc);
                            if (T.lane == 0) xv[i] = (xv[i] - acc) * rdiag[i];
                            __syncwarp();
                        }
                    }
                    __syncthreads();
                }
                for (int j = 1; j <= D; ++j) {
                    for (int i = T.warp; i < mp; i += T.nwarps)
                        for (int jx = T.lane; jx < mp; jx += 32) {
                            double acc = 0.0;
                            for (int k = D; k >= j; --k) {
                                double nk;
                                if (defl && (k & 1)) {
                                    const double* qk = pq + (size_t)((k + 1) >> 1) * vl;
                                    nk = pq[i] * qk[jx] + qk[i] * pq[jx];
                                } else {
                                    nk = NK[(size_t)(k - 1) * MS + i * ld + jx];
                                }
                                acc = acc * s + c_binom[k][j] * nk;
                            }
                            Nw[i * ld + jx] = acc;
                        }
                    __syncthreads();
                    double fro = 0.0;
                    for (int i = T.warp; i < mp; i += T.nwarps)
                        for (int jx = T.lane; jx <= i; jx += 32) {
                            double sym = 0.5 * (Nw[i * ld + jx] + Nw[jx * ld + i]);
                            Nw[i * ld + jx] = sym;
                            Nw[jx * ld + i] = sym;
                            fro += (jx == i ? 1.0 : 2.0) * sym * sym;
                        }
                    fro = block_sum(T, fro, red);
                    if (j == 1) {
                        double th_top, th_bot;
                        int J = lanczos_run(T, Nw, Qb, m, mp, ld, false, true, wv, hb, al, be, sv, sv2, dp, dm, red,
                                            &sh_i[3], &sh_d[4], nullptr, &th_top, &th_bot);
                        if (P.jsum && T.tid == 0) {
                            atomicAdd(&P.jsum[0], (unsigned long long)J);
                            atomicAdd(&P.jsum[1], 1ull);
                        }
                        a_min = th_bot;
                        for (int e = T.tid; e < mp; e += T.nthr) {
                            double acc = 0.0;
                            for (int i = 0; i < J; ++i) acc += sv2[i] * Qb[(size_t)i * ld + e];
                            zz[e] = acc;
                        }
                        __syncthreads();
                        if (T.warp == 0) {
                            for (int i = m - 1; i >= 0; --i) {
                                double yi = zz[i] * rdiag[i];
                                __syncwarp();
                                if (T.lane == 0) yk[i] = yi;
                                for (int k = T.lane; k < i; k += 32) zz[k] -= Kf[i * ld + k] * yi;
                                __syncwarp();
                            }
                        }
                        __syncthreads();
                    } else {
                        cj[j] = sqrt(fro);
                    }
                }
                if (T.tid == 0) {
                    sh_d[6] = weyl_step_n(a_min, cj, D);
                    if (H.picard) atomicAdd(&H.picard[3], (unsigned long long)ncong);  // dense congruences (flop model)
                }
                __syncthreads();
                const double h = sh_d[6];
                for (int i = T.tid; i < m; i += T.nthr) yy[i] = yk[i];
                __syncthreads();
                if (!(s + h < s_end)) {  // no root before the end of the segment
                    ended = true;
                    break;
                }
                s += h;
                if (h <= 1e-15 * s) {
                    hit = true;
                    ended = true;
                    break;
                }
            }
            capped = !ended;
            if (capped) hit = true;  // s only bounds the root from below: reported / rejected below
        }
        if (hit && T.warp == 0) {
            if (defl) {
                if (T.lane == 0) yy[0] /= s;
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
        const double t_dense = outward ? 0.0 : (hit ? (defl ? s * s : s) : SW_INF);

        // ---- cube faces: first root in (0, h'] of hi_i - p_i(t) and p_i(t) - lo_i (warp 0)
        if (T.warp == 0) {
            double tpl = t_dense;
            int bind = (tpl < SW_INF) ? 0 : SW_BIND_NONE_DEV;
            bool cube_out = false;
            if (P.lo && !outward) {
                double bt = SW_INF;
                int bi = 0x7fffffff, bcode = 0;
                for (int i = T.lane; i < n; i += 32) {
                    double gu[CH_MAXD + 1], gl[CH_MAXD + 1];
                    gu[0] = P.hi[i] - x[i];
                    gl[0] = x[i] - P.lo[i];
                    for (int k = 1; k <= d; ++k) {
                        const double ck = cf[(size_t)(k - 1) * np + i];
                        gu[k] = -ck;
                        gl[k] = ck;
                    }
                    const double tu = scalar_first_root(gu, d, hs, bnd == 1 + 2 * i);
                    const double tl = scalar_first_root(gl, d, hs, bnd == 2 + 2 * i);
                    if (tu < 0.0 || tl < 0.0) cube_out = true;
                    if (tu >= 0.0 && tu < bt) { bt = tu; bi = i; bcode = 1 + 2 * i; }
                    if (tl >= 0.0 && tl < bt) { bt = tl; bi = i; bcode = 2 + 2 * i; }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    double ot = __shfl_xor_sync(0xffffffffu, bt, o);
                    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    int oc = __shfl_xor_sync(0xffffffffu, bcode, o);
                    if (ot < bt || (ot == bt && oi < bi)) { bt = ot; bi = oi; bcode = oc; }
                }
                cube_out = __any_sync(0xffffffffu, cube_out);
                if (bt < tpl) { tpl = bt; bind = bcode; }
            }
            if (T.lane == 0) {
                sh_d[0] = tpl;
                sh_i[1] = bind;
                sh_i[5] = (outward || cube_out) ? 1 : 0;
            }
        }
        __syncthreads();
        const double tplus = sh_d[0];
        const int bind = sh_i[1];
        const bool out_any = sh_i[5] != 0;
        if (P.mode == 1) {
            const bool cap_hit = capped && bind == 0;
            if (T.tid == 0) {
                const double nan = __longlong_as_double(0x7ff8000000000000LL);
                P.o_tplus[slot] = cap_hit ? nan : (out_any ? 0.0 : tplus);
                P.o_tminus[slot] = 0.0;
                P.o_binding[slot] = cap_hit ? SW_BIND_NONE_DEV : bind;
                P.o_status[slot] = failed ? 2 : (cap_hit ? 3 : (out_any ? 4 : 0));
                P.flags[slot] = (bind == 0 && !failed && !cap_hit && !out_any) ? CF_NEED_NORMAL : 0;
            }
            if (P.o_kernel)
                for (int i = T.tid; i < m; i += T.nthr) P.o_kernel[(size_t)slot * m + i] = (bind == 0) ? yy[i] : 0.0;
            if (bind == 0 && !failed) {
                double* yh = P.Yh + (size_t)slot * P.mtp;
                for (int i = T.warp; i < m; i += T.nwarps)
                    for (int j = T.lane; j <= i; j += 32) yh[pk(i, j)] = (i == j ? 1.0 : 2.0) * yy[i] * yy[j];
            }
            continue;
        }
        if (failed) {
            if (T.tid == 0) {
                P.flags[slot] |= CF_DONE | CF_FAILED;
                P.calls[slot] += 1;
            }
            continue;
        }
        const int refl0 = P.refl[slot];
        const int sdone0 = P.steps_done[slot];
        const int trk0 = (P.max_trace > 0) ? P.tr_cnt[slot] : 0;
        const double el = P.ell[slot];
        const bool last = (el <= H.h);
        const bool nohit = (hs <= tplus);  // reading R4: a tie ends the segment
        const double th = nohit ? hs : tplus;
        __syncthreads();
        // x <- p(t^), v <- p'(t^), A(x) <- A(x) + sum_k t^k A(c_k)
        if (!out_any) {
            for (int i = T.tid; i < n; i += T.nthr) {
                double a = cf[(size_t)(d - 1) * np + i];
                double b = (double)d * a;
                for (int k = d - 1; k >= 1; --k) {
                    const double ck = cf[(size_t)(k - 1) * np + i];
                    a = a * th + ck;
                    b = b * th + (double)k * ck;
                }
                x[i] = a * th + x[i];
                v[i] = b;
            }
            for (int e = T.tid; e < P.mt; e += T.nthr) {
                double a = cb[(size_t)(d - 1) * P.mtp + e];
                for (int k = d - 1; k >= 1; --k) a = a * th + cb[(size_t)(k - 1) * P.mtp + e];
                ax[e] += th * a;
            }
        }
        __syncthreads();
        bool end_step = false, reject = false;
        if (out_any) {
            reject = end_step = true;
            if (T.tid == 0) P.ndeg[slot] += 1;
        } else if (nohit) {
            if (last) end_step = true;
            else if (T.tid == 0) {
                P.ell[slot] = el - hs;
                P.bound[slot] = SW_BIND_NONE_DEV;
            }
        } else {
            const int rf = refl0 + 1;
            if (T.tid == 0) {
                P.refl[slot] = rf;
                P.ell[slot] = el - th;
                P.nrefl[slot] += 1;
                P.tlast[slot] = th;
            }
            if (rf > P.rho) {
                reject = end_step = true;
                if (T.tid == 0) P.nrej[slot] += 1;
            } else if (bind == 0) {
                if (capped) {
                    reject = end_step = true;
                    if (T.tid == 0) P.ncap[slot] += 1;
                } else {
                    double* yh = P.Yh + (size_t)slot * P.mtp;
                    for (int i = T.warp; i < m; i += T.nwarps)
                        for (int j = T.lane; j <= i; j += 32) yh[pk(i, j)] = (i == j ? 1.0 : 2.0) * yy[i] * yy[j];
                    for (int i = T.tid; i < m; i += T.nthr) P.U[(size_t)slot * m + i] = yy[i];
                    if (T.tid == 0) {
                        P.bound[slot] = 0;
                        P.flags[slot] |= CF_NEED_NORMAL;
                        int qn = atomicAdd(P.ncount, 1);
                        P.nlist[qn] = slot;
                    }
                }
            } else if (bind > 0) {
                const int f = (bind - 1) >> 1;
                if (T.tid == 0) {
                    v[f] = -v[f];
                    P.bound[slot] = bind;
                }
            }
            if (P.max_trace > 0 && !reject) {
                __syncthreads();
                int k = trk0;
                if (k < P.max_trace) {
                    size_t o = ((size_t)slot * P.max_trace + k);
                    for (int i = T.tid; i < n; i += T.nthr) {
                        P.tr_hit[o * n + i] = x[i];
                        if (bind > 0) {
                            P.tr_v[o * n + i] = v[i];
                            P.tr_w[o * n + i] = (i == ((bind - 1) >> 1)) ? ((bind & 1) ? 1.0 : -1.0) : 0.0;
                        }
                    }
                    if (T.tid == 0) {
                        P.tr_t[o] = th;
                        P.tr_bind[o] = bind;
                        P.tr_cnt[slot] = k + 1;
                        if (k + 1 >= P.max_trace && bind != 0) P.flags[slot] |= CF_DONE;
                    }
                }
            }
        }
        if (T.tid == 0) P.calls[slot] += 1;
        __syncthreads();
        if (end_step) {
            if (reject) {
                const double* xs = P.Xs + (size_t)slot * np;
                const double* axs = P.AXs + (size_t)slot * P.mtp;
                for (int i = T.tid; i < n; i += T.nthr) x[i] = xs[i];
                for (int i = T.tid; i < P.mt; i += T.nthr) ax[i] = axs[i];
            }
            __syncthreads();
            const int sd = sdone0 + 1;
            if (T.tid == 0) {
                P.steps_done[slot] = sd;
                P.refl[slot] = 0;
                P.bound[slot] = SW_BIND_NONE_DEV;
            }
            if (sd >= P.steps_total) {
                if (T.tid == 0) P.flags[slot] |= CF_DONE;
            } else {
                step_start<true>(T, slot, gidv, sd, n, np, P.mt, P.mtp, P.V, P.X, P.Xs, P.AX, P.AXs, P.ell, P.Lpar,
                                 P.seed, P.tag, 4, red);
            }
        }
    }
}

}  // namespace sw
