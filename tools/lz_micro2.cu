// Lanczos matvec-stage variants in isolation: cycles per iteration (1 CTA x 512 threads, M in registers)
#include <cstdio>
__device__ __forceinline__ double bfly8(const double (&p)[8], const int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    double a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { const double s = b4 ? p[i] : p[i + 4], k = b4 ? p[i + 4] : p[i]; a[i] = k + __shfl_xor_sync(0xffffffffu, s, 16); }
    double b[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) { const double s = b3 ? a[i] : a[i + 2], k = b3 ? a[i + 2] : a[i]; b[i] = k + __shfl_xor_sync(0xffffffffu, s, 8); }
    double c; { const double s = b2 ? b[0] : b[1], k = b2 ? b[1] : b[0]; c = k + __shfl_xor_sync(0xffffffffu, s, 4); }
    c += __shfl_xor_sync(0xffffffffu, c, 2); c += __shfl_xor_sync(0xffffffffu, c, 1);
    return c;
}
// MODE 0: 4 lanes/row, LDS.128 u (current)   MODE 1: row blocks + butterfly, LDS.64 u
// MODE 2: 4 lanes/row, LDS.64 u               MODE 3: MODE 1 without the barrier
// MODE 4: MODE 0 without barrier  MODE 5: only barrier + owner store
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, int iters, int mdp) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = tid >> 2, g = tid & 3, rb = 8 * warp;
    for (int i = tid; i < 4096; i += 512) sm[i] = 1.0 / (1 + i);
    __syncthreads();
    double mr[26], mreg[8][4];
    if (MODE == 0 || MODE == 2 || MODE == 4)
        for (int k = 0; k < 26; ++k) mr[k] = 0.001 * (r + k);
    if (MODE == 1 || MODE == 3)
        for (int q = 0; q < 8; ++q) for (int k = 0; k < 4; ++k) mreg[q][k] = (lane + 32 * k < mdp && rb + q < mdp) ? 0.001 * (q + k) : 0.0;
    double wr = 0.5, acc = 0.0;
    long long c0 = clock64();
    for (int j = 0; j < iters; ++j) {
        const int oU = (j & 1) * 256;
        double y = 0.0;
        if (MODE == 0 || MODE == 4) {
            double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < 13; ++k) {
                const int c = 2 * g + 8 * k;
                double2 w = (c < mdp) ? *reinterpret_cast<const double2*>(sm + oU + c) : make_double2(0.0, 0.0);
                a8[(2 * k) & 7] = fma(mr[2 * k], w.x, a8[(2 * k) & 7]);
                a8[(2 * k + 1) & 7] = fma(mr[2 * k + 1], w.y, a8[(2 * k + 1) & 7]);
            }
            y = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
            y += __shfl_xor_sync(0xffffffffu, y, 1);
            y += __shfl_xor_sync(0xffffffffu, y, 2);
        } else if (MODE == 2) {
            double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < 26; ++k) {
                const int c = g + 4 * k;
                double w = (c < mdp) ? sm[oU + c] : 0.0;
                a8[k & 7] = fma(mr[k], w, a8[k & 7]);
            }
            y = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
            y += __shfl_xor_sync(0xffffffffu, y, 1);
            y += __shfl_xor_sync(0xffffffffu, y, 2);
        } else if (MODE == 1 || MODE == 3) {
            if (rb < mdp) {
                double uk[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) { const int col = lane + 32 * k; uk[k] = (col < mdp) ? sm[oU + col] : 0.0; }
                double p[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) { double a = mreg[q][0] * uk[0];
#pragma unroll
                    for (int k = 1; k < 4; ++k) a = fma(mreg[q][k], uk[k], a); p[q] = a; }
                y = bfly8(p, lane);
            }
        }
        y = y * 1e-3 + wr;
        if (g == 0 && r < mdp) sm[256 * ((j + 1) & 1) + r] = y;
        acc += y;
        if (MODE != 3 && MODE != 4) __syncthreads();
    }
    long long c1 = clock64();
    out[tid] = acc + wr;
    if (tid == 0) cyc[0] = c1 - c0;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8 * 512); cudaMallocManaged(&c, 8 * 8);
    const int it = 2000;
    auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        kern<<<1, 512, 200 * 1024>>>(o, c, it, 104); cudaDeviceSynchronize();
        kern<<<1, 512, 200 * 1024>>>(o, c, it, 104); cudaDeviceSynchronize();
        printf("%-45s %.0f cycles/iter  err=%s\n", name, c[0] / (double)it, cudaGetErrorString(cudaGetLastError()));
    };
    run(k<0>, "4 lanes/row, LDS.128 u, barrier");
    run(k<4>, "4 lanes/row, LDS.128 u, no barrier");
    run(k<2>, "4 lanes/row, LDS.64 u, barrier");
    run(k<1>, "row blocks + butterfly, LDS.64 u, barrier");
    run(k<3>, "row blocks + butterfly, no barrier");
    run(k<5>, "store + barrier only");
}
