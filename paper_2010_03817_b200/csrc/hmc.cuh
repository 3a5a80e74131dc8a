// hmc.cuh -- K5: the reflective-HMC boundary oracle for the Boltzmann density
// exp(-c^T x / T) (Alg. 6, eq:boltz_ode P:1440-1446).
//
// The trajectory p(t) = p + v t - (c / 2T) t^2 is a degree-2 curve, so the chord
// is the first positive root of the quadratic pencil (Lemma 3)
//     G(t) = A(p) + t A(v) - t^2 A(c) / (2T).
// Interior start: G(0) > 0; after a dense reflection G(0) is singular with known
// kernel u and, in the Householder basis of u, the congruence diag(1/sqrt t, I)
// with t = s^2 turns det G into det of a SYMMETRIC quartic in s with G~(0) > 0
// (SURVEY a-10 / V14).  Either way we solve "first s > 0 with G~(s) singular"
// by monotone Weyl stepping: at s_k with K K^T = G~(s_k),
//     lambda_min(I + h N1 + ... + h^d Nd) >= 1 + h lambda_min(N1) - sum_j h^j |Nj|_F,
// N_j = K^{-1} (d^j G~ / j! ds^j)(s_k) K^{-T}; the smallest positive root h of the
// scalar bound is a safe step (never past the root), and the iteration converges
// quadratically because the N1 term dominates near the root.  lambda_min(N1) by
// Lanczos (bottom Ritz pair); its Ritz vector gives the kernel vector at the hit.
// Matrices live in a per-CTA global scratch slice (L2 resident).
#pragma once
#include "chord2.cuh"

namespace sw {

// Weyl-stepping iteration cap of one HMC-r chord (V6: ~4 iterations; reaching it is counted
// in spec_walk_stats.capped and the step is rejected)
constexpr int HMC_MAX_IT = 60;

// smallest positive root of alpha + beta t + gamma t^2 (alpha >= 0); on_face:
// alpha is exactly 0 (the face just left), the root t = 0 is excluded.
__device__ __forceinline__ double first_pos_root2(double alpha, double beta, double gamma, bool on_face) {
    if (on_face) {
        if (gamma != 0.0) {
            double r = -beta / gamma;
            return r > 0.0 ? r : SW_INF;
        }
        return SW_INF;
    }
    if (gamma == 0.0) return (beta < 0.0) ? -alpha / beta : SW_INF;
    double disc = beta * beta - 4.0 * alpha * gamma;
    if (disc < 0.0) return SW_INF;
    double sq = sqrt(disc);
    double q = -0.5 * (beta + (beta >= 0.0 ? sq : -sq));
    double r1 = (q != 0.0) ? alpha / q : SW_INF;
    double r2 = q / gamma;
    double best = SW_INF;
    if (r1 > 0.0) best = r1;
    if (r2 > 0.0 && r2 < best) best = r2;
    return best;
}

// smallest positive root of 1 + a h - sum_{j=2..d} c_j h^j (c_j >= 0, concave):
// largest h with a non-negative value, by bisection.  +inf if none.
__device__ double weyl_step(double a, const double* c, int d) {
    auto f = [&](double h) {
        double v = 1.0 + a * h, hp = h;
        for (int j = 2; j <= d; ++j) {
            hp *= h;
            v -= c[j] * hp;
        }
        return v;
    };
    bool anyc = false;
    for (int j = 2; j <= d; ++j) anyc = anyc || (c[j] > 0.0);
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

// Cube faces, selection, the oracle outputs (mode 1) or the HMC advance, reflection
// and step logic (Alg. 6) for one slot, given the dense chord t_dense and the unit
// kernel vector yy (shared memory) -- shared by hmc_kernel and the split tail.
__device__ __forceinline__ void hmc_finish(const Team& T, const ChordParams& P, int slot, long long gidv, double* x,
                                           double* v, const double* av, double* ax, int bnd, const double* yy,
                                           double t_dense, bool failed, bool outward, bool capped, double* red,
                                           double* sh_d, int* sh_i) {
    const int m = P.m, n = P.n;
    const double Tinv = 1.0 / P.Temp;
    {

        // ---- cube faces: per-coordinate quadratic x_i(t) = x_i + v_i t - c_i t^2 / 2T
        if (T.warp == 0) {
            double tpl = t_dense;
            int bind = (tpl < SW_INF) ? 0 : SW_BIND_NONE_DEV;
            if (P.lo) {
                double bt = SW_INF;
                int bi = 0x7fffffff, bcode = 0;
                for (int i = T.lane; i < n; i += 32) {
                    const double g = 0.5 * P.cvec[i] * Tinv;
                    double tu = first_pos_root2(P.hi[i] - x[i], -v[i], g, bnd == 1 + 2 * i);
                    double tl = first_pos_root2(x[i] - P.lo[i], v[i], -g, bnd == 2 + 2 * i);
                    if (tu < bt) { bt = tu; bi = i; bcode = 1 + 2 * i; }
                    if (tl < bt) { bt = tl; bi = i; bcode = 2 + 2 * i; }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    double ot = __shfl_xor_sync(0xffffffffu, bt, o);
                    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    int oc = __shfl_xor_sync(0xffffffffu, bcode, o);
                    if (ot < bt || (ot == bt && oi < bi)) { bt = ot; bi = oi; bcode = oc; }
                }
                if (bt < tpl) { tpl = bt; bind = bcode; }
            }
            if (T.lane == 0) {
                sh_d[0] = tpl;
                sh_i[1] = bind;
            }
        }
        __syncthreads();
        const double tplus = sh_d[0];
        const int bind = sh_i[1];
        if (P.mode == 1) {
            // a dense hit found with the Weyl iteration cap reached is only a lower bound on
            // the crossing time: reported as status 3, t+ = NaN, binding none (never silent)
            const bool cap_hit = capped && bind == 0;
            if (T.tid == 0) {
                P.o_tplus[slot] = cap_hit ? __longlong_as_double(0x7ff8000000000000LL) : tplus;
                P.o_tminus[slot] = 0.0;
                P.o_binding[slot] = cap_hit ? SW_BIND_NONE_DEV : bind;
                P.o_status[slot] = failed ? 2 : (cap_hit ? 3 : 0);
                P.flags[slot] = (bind == 0 && !failed && !cap_hit) ? CF_NEED_NORMAL : 0;
            }
            if (P.o_kernel)
                for (int i = T.tid; i < m; i += T.nthr) P.o_kernel[(size_t)slot * m + i] = (bind == 0) ? yy[i] : 0.0;
            if (bind == 0 && !failed) {
                double* yh = P.Yh + (size_t)slot * P.mtp;
                for (int i = T.warp; i < m; i += T.nwarps)
                    for (int j = T.lane; j <= i; j += 32) yh[pk(i, j)] = (i == j ? 1.0 : 2.0) * yy[i] * yy[j];
            }
            return;
        }
        // ---- HMC advance (Alg. 6): p <- p(t^), A(p) <- A(p) + t^ A(v) + t^2 C2
        if (failed) {
            if (T.tid == 0) {
                P.flags[slot] |= CF_DONE | CF_FAILED;
                P.calls[slot] += 1;
            }
            return;
        }
        // per-chain counters read by every thread BEFORE thread 0 updates them below
        // (a read after the update would give threads different values: a race)
        const int refl0 = P.refl[slot];
        const int sdone0 = P.steps_done[slot];
        const int trk0 = (P.max_trace > 0) ? P.tr_cnt[slot] : 0;
        const double el = P.ell[slot];
        const bool accept = (el <= tplus);
        const double th = accept ? el : tplus;
        const double qa = -0.5 * th * th * Tinv;
        for (int i = T.tid; i < n; i += T.nthr) x[i] += th * v[i] + qa * P.cvec[i];
        for (int i = T.tid; i < P.mt; i += T.nthr) ax[i] += th * av[i] + qa * P.Ac[i];
        __syncthreads();
        bool end_step = accept, reject = false;
        if (!accept) {
            int rf = refl0 + 1;
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
                if (outward) {
                    reject = end_step = true;
                    if (T.tid == 0) P.ndeg[slot] += 1;
                } else if (capped) {
                    // Weyl stepping hit HMC_MAX_IT: s is a lower bound on the root only,
                    // so the segment cannot be advanced to a boundary point: reject the step
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
                        int q = atomicAdd(P.ncount, 1);
                        P.nlist[q] = slot;
                    }
                }
            } else if (bind > 0) {
                // velocity at the hit u = v - (c/T) t, reflected at the face (w = +-e_i)
                const int f = (bind - 1) >> 1;
                for (int i = T.tid; i < n; i += T.nthr) {
                    double u = v[i] - P.cvec[i] * Tinv * th;
                    v[i] = (i == f) ? -u : u;
                }
                if (T.tid == 0) P.bound[slot] = bind;
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
                const double* xs = P.Xs + (size_t)slot * P.np;
                const double* axs = P.AXs + (size_t)slot * P.mtp;
                for (int i = T.tid; i < n; i += T.nthr) x[i] = xs[i];
                for (int i = T.tid; i < P.mt; i += T.nthr) ax[i] = axs[i];
            }
            __syncthreads();
            int sd = sdone0 + 1;
            if (T.tid == 0) {
                P.steps_done[slot] = sd;
                P.refl[slot] = 0;
                P.bound[slot] = SW_BIND_NONE_DEV;
            }
            if (sd >= P.steps_total) {
                if (T.tid == 0) P.flags[slot] |= CF_DONE;
            } else {
                step_start<true>(T, slot, gidv, sd, n, P.np, P.mt, P.mtp, P.V, P.X, P.Xs, P.AX, P.AXs, P.ell, P.Lpar,
                                 P.seed, P.tag, 1, red);
            }
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) hmc_kernel(ChordParams P) {
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

    const int m = P.m, ld = P.ld;
    const int mp = (m + 7) & ~7;
    const size_t MS = (size_t)mp * ld;
    double* base = P.scratch + (size_t)blockIdx.x * P.scratch_stride;
    double* Cm[5] = {base, base + MS, base + 2 * MS, base + 3 * MS, base + 4 * MS};
    double* Kf = base + 5 * MS;  // Cholesky factor of G~(s_k)
    double* Nw = base + 6 * MS;  // congruence / Lanczos operand
    double* Qb = base + 7 * MS;  // Lanczos basis
    const int vl = mp + 8;
    double* vec = smem_dyn;
    double* hh = vec + 0 * vl;
    double* pw = vec + 1 * vl;
    double* rdiag = vec + 2 * vl;
    double* wv = vec + 14 * vl;  // 2 slots (ping-pong)
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
    const double Tinv = 1.0 / P.Temp;

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

        // ---- coefficient matrices C0 = A(p), C1 = A(v), C2 = -A(c)/(2T), padded
        unpack_sym(T, ax, Cm[0], m, ld);
        unpack_sym(T, av, Cm[1], m, ld);
        unpack_sym(T, P.Ac, Cm[2], m, ld);
        __syncthreads();
        const double c2s = -0.5 * Tinv;
        for (int i = T.warp; i < m; i += T.nwarps)
            for (int j = T.lane; j < m; j += 32) Cm[2][i * ld + j] *= c2s;
        for (int k = 0; k < 5; ++k)
            for (int i = T.warp; i < mp; i += T.nwarps)
                for (int j = T.lane; j < mp; j += 32)
                    if (i >= m || j >= m) Cm[k][i * ld + j] = (k == 0 && i == j) ? 1.0 : 0.0;
        __syncthreads();
        const bool defl = (bnd == 0);
        int d = 2;
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
            for (int k = 0; k < 3; ++k) householder_congruence(T, Cm[k], m, ld, hh, beta_h, pw, red);
            const double a1 = Cm[1][0], a2 = Cm[2][0];
            outward = !(a1 > 0.0);
            // quartic in s = sqrt(t): C3 = border(b2), C4 = inner(V2), C2 = [a2 | inner V1],
            // C1 = border(b1), C0 = [a1 | inner G0^]
            for (int i = T.warp; i < m; i += T.nwarps)
                for (int j = T.lane; j < m; j += 32) {
                    const bool bi = (i == 0), bj = (j == 0);
                    double g2 = Cm[2][i * ld + j];
                    Cm[3][i * ld + j] = (bi != bj) ? g2 : 0.0;
                    Cm[4][i * ld + j] = (!bi && !bj) ? g2 : 0.0;
                }
            __syncthreads();
            for (int i = T.warp; i < m; i += T.nwarps)
                for (int j = T.lane; j < m; j += 32) {
                    const bool bi = (i == 0), bj = (j == 0);
                    double g1 = Cm[1][i * ld + j];
                    Cm[2][i * ld + j] = (!bi && !bj) ? g1 : ((bi && bj) ? a2 : 0.0);
                    Cm[1][i * ld + j] = (bi != bj) ? g1 : 0.0;
                    if (bi || bj) Cm[0][i * ld + j] = (bi && bj) ? a1 : 0.0;
                }
            __syncthreads();
            d = 4;
        }
        PROF_MARK(0);

        // ---- monotone Weyl stepping on G~(s)
        double s = 0.0;
        bool failed = false, hit = false, capped = false;
        int iters = 0;
        if (!outward) {
            bool ended = false;  // converged, Cholesky breakdown, or no root
            for (int it = 0; it < HMC_MAX_IT; ++it) {
                ++iters;
                // Kf = G~(s) (Horner), Cholesky
                for (int i = T.warp; i < mp; i += T.nwarps)
                    for (int j = T.lane; j < mp; j += 32) {
                        double acc = Cm[d][i * ld + j];
                        for (int k = d - 1; k >= 0; --k) acc = acc * s + Cm[k][i * ld + j];
                        Kf[i * ld + j] = acc;
                    }
                __syncthreads();
                bool ok = cholesky_blocked(T, Kf, mp, ld, rdiag, &sh_i[2]);
                if (!ok) {
                    if (it == 0) failed = true;  // start not interior
                    ended = true;
                    break;                       // rounding past the root: keep s (the last safe point)
                }
                // N1 = K^{-1} G~'(s) K^{-T}
                double cj[5] = {0, 0, 0, 0, 0};
                double a_min = 0.0;
                for (int j = 1; j <= d; ++j) {
                    for (int i = T.warp; i < mp; i += T.nwarps)
                        for (int jx = T.lane; jx < mp; jx += 32) {
                            // D_j = sum_{k>=j} binom(k, j) s^{k-j} C_k
                            double acc = 0.0;
                            for (int k = d; k >= j; --k) {
                                double bin = 1.0;
                                for (int q = 0; q < j; ++q) bin = bin * (double)(k - q) / (double)(q + 1);
                                acc = acc * s + bin * Cm[k][i * ld + jx];
                            }
                            Nw[i * ld + jx] = acc;
                        }
                    __syncthreads();
                    trsm_blocked<false>(T, Kf, Nw, mp, ld, rdiag);
                    trsm_blocked<true>(T, Kf, Nw, mp, ld, rdiag);
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
                                            &sh_i[3], &sh_d[4], P.prof, &th_top, &th_bot);
                        if (P.jsum && T.tid == 0) {
                            atomicAdd(&P.jsum[0], (unsigned long long)J);
                            atomicAdd(&P.jsum[1], 1ull);
                        }
                        a_min = th_bot;
                        // z = Q s (bottom Ritz vector), y_k = K^{-T} z
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
                if (T.tid == 0) sh_d[6] = weyl_step(a_min, cj, d);
                __syncthreads();
                double h = sh_d[6];
                for (int i = T.tid; i < m; i += T.nthr) yy[i] = yk[i];
                __syncthreads();
                if (!(h < SW_INF)) {
                    s = SW_INF;
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
            if (s < SW_INF) hit = true;
            capped = !ended;
        }
        if (P.prof && T.tid == 0) atomicAdd(&P.prof[17], (unsigned long long)iters);
        PROF_MARK(4);
        // kernel vector of G(t+): boundary start maps back y = H D y~, D = diag(1/s, I)
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
        double t_dense = outward ? 0.0 : (hit ? (d == 4 ? s * s : s) : SW_INF);
        hmc_finish(T, P, slot, gidv, x, v, av, ax, bnd, yy, t_dense, failed, outward, capped, red, sh_d, sh_i);
        PROF_MARK(8);
    }
}

}  // namespace sw
