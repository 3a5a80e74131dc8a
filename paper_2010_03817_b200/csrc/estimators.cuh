// estimators.cuh -- K6 (exact ball sampling + batched membership, PAPER.md
// Alg. 1) and K7 (deterministic f-value / moment reductions) used by
// the volume (eq:mmc_vol P:1291-1300) and expectation estimators.
#pragma once
#include "chord2.cuh"

namespace sw {

// x_j = c0 + r eta^(1/n) g/|g| for sample ids begin..begin+count-1 (same Philox
// layout as the step draws: g from blocks 0..ceil(n/2)-1, eta from block
// ceil(n/2), counter (block, 0, sample id, tag)).  One warp per sample.
__global__ void __launch_bounds__(256) ball_sample_kernel(int count, long long begin, int n, int np,
                                                          unsigned long long seed, unsigned tag,
                                                          const double* c0, double r, double* X) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int nb = (n + 1) / 2;
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const double two_pi = 6.283185307179586476925286766559;
    for (int s = blockIdx.x * wpb + (threadIdx.x >> 5); s < count; s += gridDim.x * wpb) {
        double* x = X + (size_t)s * np;
        const uint32_t id = (uint32_t)(begin + s);
        double ss = 0.0, eta = 0.0;
        for (int j = lane; j <= nb; j += 32) {
            uint4 w = philox4x32_10(make_uint4((uint32_t)j, 0u, id, tag), key);
            if (j < nb) {
                double u0 = u01(w.x, w.y), u1 = u01(w.z, w.w);
                double rr = sqrt(-2.0 * log(u0));
                double a = two_pi * u1;
                double g0 = rr * cos(a);
                x[2 * j] = g0;
                ss += g0 * g0;
                if (2 * j + 1 < n) {
                    double g1 = rr * sin(a);
                    x[2 * j + 1] = g1;
                    ss += g1 * g1;
                }
            } else {
                eta = u01(w.x, w.y);
            }
        }
        ss = warp_sum(ss);
        eta = __shfl_sync(0xffffffffu, eta, nb % 32);
        const double sc = r * pow(eta, 1.0 / (double)n) / sqrt(ss);
        __syncwarp();
        for (int i = lane; i < np; i += 32) x[i] = (i < n) ? c0[i] + sc * x[i] : 0.0;
    }
}

// Membership of x_j: cube lo < x < hi and every Cholesky pivot of A(x_j) above
// 1e-10 |A(x_j)|_max (the oracle's O6 threshold).  One CTA per sample.
template <int NT>
__global__ void __launch_bounds__(NT) membership_kernel(int count, int n, int np, int m, int mt, int mtp, int ld,
                                                        const double* X, const double* AX, const double* lo,
                                                        const double* hi, int* inside, double* gscr,
                                                        long long gstride) {
    extern __shared__ __align__(16) double smem_dyn[];
    Team T;
    T.tid = threadIdx.x;
    T.nthr = NT;
    T.lane = T.tid & 31;
    T.warp = T.tid >> 5;
    T.nwarps = NT >> 5;
    __shared__ double red[64];
    __shared__ int flag;
    const int mp = (m + 7) & ~7;
    // A(x_j) in shared memory, or (large m, gscr != NULL) in this CTA's global scratch slice
    double* G = gscr ? gscr + (size_t)blockIdx.x * gstride : smem_dyn;
    double* rdiag = gscr ? smem_dyn : G + (size_t)mp * ld;
    for (int s = blockIdx.x; s < count; s += gridDim.x) {
        const double* x = X + (size_t)s * np;
        bool ok = true;
        if (lo) {
            bool in = true;
            for (int i = T.tid; i < n; i += NT) in = in && (x[i] > lo[i]) && (x[i] < hi[i]);
            double v = in ? 0.0 : 1.0;
            ok = block_max(T, v, red) == 0.0;
        }
        __syncthreads();
        if (ok) {
            unpack_sym(T, AX + (size_t)s * mtp, G, m, ld);
            for (int i = T.warp; i < mp; i += T.nwarps)
                for (int j = T.lane; j < mp; j += 32)
                    if (i >= m || j >= m) G[i * ld + j] = (i == j) ? 1.0 : 0.0;
            double fmx = 0.0;
            const double* P = AX + (size_t)s * mtp;
            for (int e = T.tid; e < mt; e += NT) fmx = fmax(fmx, fabs(P[e]));
            fmx = block_max(T, fmx, red);
            bool chol = cholesky_blocked(T, G, mp, ld, rdiag, &flag);
            if (chol) {
                double mn = SW_INF;
                for (int i = T.tid; i < m; i += NT) mn = fmin(mn, G[i * ld + i] * G[i * ld + i]);
                mn = block_min(T, mn, red);
                ok = mn > 1e-10 * fmx;
            } else {
                ok = false;
            }
        }
        if (T.tid == 0) inside[s] = ok ? 1 : 0;
        __syncthreads();
    }
}

// f values over end points: 0 = c.x, 1 = |x|^2, 2 = 1(c.x <= b1 or c.x >= b2).
__global__ void fvalue_kernel(int count, int n, int np, const double* X, const double* c, int f_id, double b1,
                              double b2, double* out) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int s = blockIdx.x * wpb + (threadIdx.x >> 5); s < count; s += gridDim.x * wpb) {
        const double* x = X + (size_t)s * np;
        double a = 0.0;
        for (int i = lane; i < n; i += 32) a += (f_id == 1) ? x[i] * x[i] : c[i] * x[i];
        a = warp_sum(a);
        if (lane == 0) out[s] = (f_id == 2) ? ((a <= b1 || a >= b2) ? 1.0 : 0.0) : a;
    }
}

// Chunked end-point moments: chunk k sums chains [k*CH, (k+1)*CH) in order.
// out[k*(n + n(n+1)/2) ...] = (sum x, packed sum x x^T).  Chunk boundaries are
// global-chain aligned, so the partials do not depend on the GPU count.
__global__ void moments_chunk_kernel(const double* X, int np, int n, int chains, int CH, double* out) {
    const int nx = n, nxx = n * (n + 1) / 2, stride = nx + nxx;
    const int nchunk = (chains + CH - 1) / CH;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)nchunk * stride;
         e += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(e / stride), q = (int)(e % stride);
        const int c0 = k * CH, c1 = min(chains, c0 + CH);
        double s = 0.0;
        if (q < nx) {
            for (int c = c0; c < c1; ++c) s += X[(size_t)c * np + q];
        } else {
            int qq = q - nx;
            int i = (int)((sqrt(8.0 * qq + 1.0) - 1.0) * 0.5);
            while (pk(i + 1, 0) <= qq) ++i;
            while (pk(i, 0) > qq) --i;
            int j = qq - pk(i, 0);
            for (int c = c0; c < c1; ++c) s += X[(size_t)c * np + i] * X[(size_t)c * np + j];
        }
        out[e] = s;
    }
}

}  // namespace sw
