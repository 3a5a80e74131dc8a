// walk.cuh -- K4 (normal finalisation + reflection), step-start, list
// compaction and the deterministic end-point reductions.
#pragma once
#include "chord.cuh"

namespace sw {

struct NormalParams {
    int n, np, m, mt, mtp;
    int mode;  // 0 walk, 1 oracle
    const double* Gn;  // [slot*np] g_i = y^T A_i y
    double* V;
    double* X;
    const double* Xs;
    double* AX;
    double* AXs;
    double* ell;
    int* steps_done;
    int* refl;
    int* bound;
    int* flags;
    int* ndeg;
    double amax;
    const int* nlist;
    const int* ncount;
    int count_host;
    // walk parameters
    int steps_total;
    double Lpar;
    unsigned long long seed;
    unsigned tag;
    long long chain_base;
    const long long* gid;
    // oracle mode
    const int* o_binding;
    const double* o_tplus;
    const double* Vin;  // oracle: directions
    double* o_normal;
    const double* ball_c;
    double ball_r;
    // trace
    int max_trace;
    int* tr_cnt;
    double* tr_w;
    double* tr_v;
    // HMC-r: velocity at the hit u = v - (c/T) t+ before the reflection
    int kind;
    const double* cvec;
    double Tinv;
    const double* tlast;
};

// One warp per chain.  Walk: w = -g/|g| (outward, lemma:gradient P:752-764,
// c dropped P:784-788), v <- v - 2<v,w>w (eq:reflection P:737-747); a
// degenerate normal (|g| < 1e-12 max|A_i|, rank <= m-2 P:763) rejects the step.
__global__ void __launch_bounds__(256) normal_reflect_kernel(NormalParams P) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int count = P.ncount ? min(*P.ncount, P.count_host) : P.count_host;
    __shared__ double red_s[8][64];
    double* red = red_s[threadIdx.x >> 5];
    Team T;
    T.tid = lane;
    T.nthr = 32;
    T.lane = lane;
    T.warp = 0;
    T.nwarps = 1;
    for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < count; r += gridDim.x * wpb) {
        const int slot = P.nlist ? P.nlist[r] : r;
        const double* g = P.Gn + (size_t)slot * P.np;
        if (P.mode == 1) {
            double* out = P.o_normal + (size_t)slot * P.n;
            int b = P.o_binding[slot];
            if (b == 0) {
                double s = 0.0;
                for (int i = lane; i < P.n; i += 32) s += g[i] * g[i];
                s = sqrt(warp_sum(s));
                bool deg = !(s >= 1e-12 * P.amax) || s == 0.0;
                for (int i = lane; i < P.n; i += 32) out[i] = deg ? __longlong_as_double(0x7ff8000000000000LL) : -g[i] / s;
            } else if (b > 0) {
                int f = (b - 1) >> 1;
                for (int i = lane; i < P.n; i += 32) out[i] = (i == f) ? ((b & 1) ? 1.0 : -1.0) : 0.0;
            } else if (b == SW_BIND_BALL_DEV) {
                const double* x = P.X + (size_t)slot * P.np;
                const double* v = P.Vin + (size_t)slot * P.np;
                double tp = P.o_tplus[slot];
                double s = 0.0;
                for (int i = lane; i < P.n; i += 32) {
                    double di = x[i] + tp * v[i] - P.ball_c[i];
                    s += di * di;
                }
                s = sqrt(warp_sum(s));
                for (int i = lane; i < P.n; i += 32) out[i] = (x[i] + tp * v[i] - P.ball_c[i]) / s;
            } else {
                for (int i = lane; i < P.n; i += 32) out[i] = __longlong_as_double(0x7ff8000000000000LL);
            }
            continue;
        }
        double* v = P.V + (size_t)slot * P.np;
        double gg = 0.0, gv = 0.0;
        for (int i = lane; i < P.n; i += 32) {
            gg += g[i] * g[i];
            gv += g[i] * v[i];
        }
        gg = warp_sum(gg);
        gv = warp_sum(gv);
        double gn = sqrt(gg);
        if (lane == 0) P.flags[slot] &= ~CF_NEED_NORMAL;
        if (!(gn >= 1e-12 * P.amax) || gn == 0.0) {
            // degenerate: reject the step (x <- x_i, A(x) <- A(x_i))
            double* x = P.X + (size_t)slot * P.np;
            const double* xs = P.Xs + (size_t)slot * P.np;
            double* ax = P.AX + (size_t)slot * P.mtp;
            const double* axs = P.AXs + (size_t)slot * P.mtp;
            for (int i = lane; i < P.n; i += 32) x[i] = xs[i];
            for (int i = lane; i < P.mt; i += 32) ax[i] = axs[i];
            if (P.max_trace > 0 && lane == 0) {
                int k = P.tr_cnt[slot];
                if (k > 0) P.tr_cnt[slot] = k - 1;  // the hit recorded by K2 did not reflect
            }
            int sd = P.steps_done[slot] + 1;
            __syncwarp();
            if (lane == 0) {
                P.ndeg[slot] += 1;
                P.steps_done[slot] = sd;
                P.refl[slot] = 0;
                P.bound[slot] = SW_BIND_NONE_DEV;
                if (sd >= P.steps_total) P.flags[slot] |= CF_DONE;
            }
            if (sd < P.steps_total) {
                long long gidv = P.gid ? P.gid[slot] : P.chain_base + slot;
                step_start<false>(T, slot, gidv, sd, P.n, P.np, P.mt, P.mtp, P.V, P.X, (double*)P.Xs, P.AX, P.AXs,
                                  P.ell, P.Lpar, P.seed, P.tag, P.kind, red);
            }
            continue;
        }
        if (P.kind == 1) {  // HMC: reflect the velocity at the hit, u = v - (c/T) t+
            const double tl = P.tlast[slot];
            gv = 0.0;
            for (int i = lane; i < P.n; i += 32) {
                double u = v[i] - P.cvec[i] * P.Tinv * tl;
                v[i] = u;
                gv += g[i] * u;
            }
            gv = warp_sum(gv);
        }
        // w = -g/|g|; v <- v - 2 <v,w> w = v - 2 (g.v / |g|^2) g
        double f = 2.0 * gv / gg;
        for (int i = lane; i < P.n; i += 32) v[i] -= f * g[i];
        if (P.max_trace > 0) {
            __syncwarp();
            int k = P.tr_cnt[slot] - 1;
            if (k >= 0 && k < P.max_trace) {
                size_t o = (size_t)slot * P.max_trace + k;
                for (int i = lane; i < P.n; i += 32) {
                    P.tr_w[o * P.n + i] = -g[i] / gn;
                    P.tr_v[o * P.n + i] = v[i];
                }
                if (lane == 0 && k + 1 >= P.max_trace) P.flags[slot] |= CF_DONE;
            }
        }
    }
}

// Walk start: every chain draws its step-0 direction and length and saves x_0.
__global__ void __launch_bounds__(256) walk_start_kernel(int count, int n, int np, int mt, int mtp, double* V,
                                                         double* X, double* Xs, const double* AX, double* AXs,
                                                         double* ell, double Lpar, unsigned long long seed,
                                                         unsigned tag, int kind, long long chain_base,
                                                         const long long* gid) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    __shared__ double red_s[8][64];
    double* red = red_s[threadIdx.x >> 5];
    Team T;
    T.tid = lane;
    T.nthr = 32;
    T.lane = lane;
    T.warp = 0;
    T.nwarps = 1;
    for (int slot = blockIdx.x * wpb + (threadIdx.x >> 5); slot < count; slot += gridDim.x * wpb) {
        long long gidv = gid ? gid[slot] : chain_base + slot;
        step_start<false>(T, slot, gidv, 0, n, np, mt, mtp, V, X, Xs, AX, AXs, ell, Lpar, seed, tag, kind, red);
    }
}

__global__ void compact_kernel(const int* list, const int* count_dev, int count_host, const int* flags, int* out,
                               int* out_count) {
    int count = min(*count_dev, count_host);
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < count; r += gridDim.x * blockDim.x) {
        int slot = list[r];
        if (!(flags[slot] & CF_DONE)) {
            int q = atomicAdd(out_count, 1);
            out[q] = slot;
        }
    }
}

// Deterministic end-point moments: thread per output entry, chains summed in
// slot order (sum_x: n entries, sum_xx: n(n+1)/2 packed lower).
__global__ void moments_kernel(const double* X, int np, int n, int chains, double* sum_x, double* sum_xx) {
    int nx = n, nxx = n * (n + 1) / 2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nx + nxx; e += gridDim.x * blockDim.x) {
        if (e < nx) {
            double s = 0.0;
            for (int c = 0; c < chains; ++c) s += X[(size_t)c * np + e];
            sum_x[e] = s;
        } else {
            int q = e - nx;
            int i = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
            while (pk(i + 1, 0) <= q) ++i;
            while (pk(i, 0) > q) --i;
            int j = q - pk(i, 0);
            double s = 0.0;
            for (int c = 0; c < chains; ++c) s += X[(size_t)c * np + i] * X[(size_t)c * np + j];
            sum_xx[q] = s;
        }
    }
}

__global__ void stats_kernel(int chains, const long long* calls, const long long* nrefl, const int* nrej,
                             const int* ndeg, const int* ncap, const int* flags, const int* steps_done,
                             long long* out) {
    __shared__ long long acc[7];
    if (threadIdx.x < 7) acc[threadIdx.x] = 0;
    __syncthreads();
    long long a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < chains; c += gridDim.x * blockDim.x) {
        a0 += calls[c];
        a1 += nrefl[c];
        a2 += nrej[c];
        a3 += ndeg[c];
        a4 += (flags[c] & CF_FAILED) ? 1 : 0;
        a5 += steps_done[c];
        a6 += ncap[c];
    }
    atomicAdd((unsigned long long*)&acc[0], (unsigned long long)a0);
    atomicAdd((unsigned long long*)&acc[1], (unsigned long long)a1);
    atomicAdd((unsigned long long*)&acc[2], (unsigned long long)a2);
    atomicAdd((unsigned long long*)&acc[3], (unsigned long long)a3);
    atomicAdd((unsigned long long*)&acc[4], (unsigned long long)a4);
    atomicAdd((unsigned long long*)&acc[5], (unsigned long long)a5);
    atomicAdd((unsigned long long*)&acc[6], (unsigned long long)a6);
    __syncthreads();
    if (threadIdx.x < 7) atomicAdd((unsigned long long*)&out[threadIdx.x], (unsigned long long)acc[threadIdx.x]);
}

// W-CHnR direction contraction: v = e_j, so A(v) = A_j is row j of Ahat -- a
// copy instead of the K1 GEMM (the O(m^2) construction of the pencil).  One CTA per chain.
__global__ void __launch_bounds__(256) coord_dir_kernel(const int* list, const int* count_dev, int count_host,
                                                        const double* V, int np, int n, const double* Ahat,
                                                        int mtp, double* AV) {
    __shared__ int jj;
    const int count = count_dev ? min(*count_dev, count_host) : count_host;
    for (int rr = blockIdx.x; rr < count; rr += gridDim.x) {
        const int slot = list ? list[rr] : rr;
        if (slot < 0) continue;
        if (threadIdx.x == 0) jj = 0;
        __syncthreads();
        const double* v = V + (size_t)slot * np;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            if (v[i] != 0.0) jj = i;  // exactly one non-zero entry
        __syncthreads();
        const double2* src = (const double2*)(Ahat + (size_t)jj * mtp);
        double2* dst = (double2*)(AV + (size_t)slot * mtp);
        for (int e = threadIdx.x; e < (mtp >> 1); e += blockDim.x) dst[e] = src[e];
        __syncthreads();
    }
}

__global__ void iota_kernel(int* list, int count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) list[i] = i;
}

// copy rows of a dense (count x n) buffer into the padded (count x np) layout
__global__ void pad_rows_kernel(const double* src, int src_stride, int rows, int n, double* dst, int np) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)rows * np;
         e += (long long)gridDim.x * blockDim.x) {
        int r = (int)(e / np), i = (int)(e % np);
        dst[e] = (i < n) ? src[(size_t)r * src_stride + i] : 0.0;
    }
}
__global__ void unpad_rows_kernel(const double* src, int np, int rows, int n, double* dst) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)rows * n;
         e += (long long)gridDim.x * blockDim.x) {
        int r = (int)(e / n), i = (int)(e % n);
        dst[e] = src[(size_t)r * np + i];
    }
}

}  // namespace sw
