// Microbenchmark of the Lanczos convergence check pieces (cycles), one CTA of 512 threads.
#include <cstdio>
#include "../paper_2010_03817_b200/csrc/chord2.cuh"
using namespace sw;
__global__ void __launch_bounds__(512, 1) k(long long* cyc, int J, int reps) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x;
    // tridiagonal of a Wigner-like matrix: al ~ small, be ~ 1 (deterministic)
    const int oAl = 0, oBe = 256, oB2 = 512, oRbe = 768, oShd = 1024;
    for (int i = tid; i < 256; i += 512) {
        double f = i * 0.6180339887498949; f -= floor(f);
        sm[oAl + i] = 0.3 * (f - 0.5);
        sm[oBe + i] = 0.8 + 0.4 * f;
        sm[oB2 + i] = sm[oBe + i] * sm[oBe + i];
        sm[oRbe + i] = 1.0 / sm[oBe + i];
    }
    for (int i = tid; i < 64; i += 512) sm[oShd + i] = 0.0;
    if (tid == 0) { sm[oShd + CK_INTOP] = -SW_INF; sm[oShd + CK_INBOT] = SW_INF; }
    __syncthreads();
    long long c0 = clock64();
    double th = 0;
    for (int r = 0; r < reps; ++r) th += tri_laguerre_warp(oAl, oB2, J, 0.0, 3.0, true, tid & 31);
    long long c1 = clock64();
    double b = 0;
    for (int r = 0; r < reps; ++r) b += tri_back_lastcomp_sm(oAl, oBe, oRbe, J, th / reps + r * 1e-9);
    long long c2 = clock64();
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        lanczos_check(tid, oAl, oBe, oB2, oRbe, J, 1e-3, 3.0, false, false, 200, oShd);
        __syncthreads();
    }
    long long c3 = clock64();
    if (tid == 0) { cyc[0] = (c1 - c0) / reps; cyc[1] = (c2 - c1) / reps; cyc[2] = (c3 - c2) / reps; cyc[3] = (long long)(th + b); }
}
int main() {
    long long* c; cudaMallocManaged(&c, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int J : {20, 50, 100}) {
        k<<<1, 512, 64 * 1024>>>(c, J, 20); cudaDeviceSynchronize();
        printf("J=%d laguerre_warp %lld  back_lastcomp %lld  full check %lld cycles  (%s)\n", J, c[0], c[1], c[2],
               cudaGetErrorString(cudaGetLastError()));
    }
}
