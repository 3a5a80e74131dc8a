// latency microbenchmarks (cycles): dependent DFMA, DADD, SHFL(double), LDS, __syncthreads(512)
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b) {
    __shared__ double sm[1024];
    int t = threadIdx.x;
    sm[t] = t * 0.5; sm[t + 512] = 1.0;
    __syncthreads();
    double x = a + t;
    long long c0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < 1000; ++i) x = fma(x, b, a);
    long long c1 = clock64();
    #pragma unroll 1
    for (int i = 0; i < 1000; ++i) x = x + b;
    long long c2 = clock64();
    #pragma unroll 1
    for (int i = 0; i < 1000; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
    long long c3 = clock64();
    int idx = t;
    #pragma unroll 1
    for (int i = 0; i < 1000; ++i) { idx = (int)sm[idx & 511] & 511; }
    long long c4 = clock64();
    #pragma unroll 1
    for (int i = 0; i < 1000; ++i) __syncthreads();
    long long c5 = clock64();
    double y = x;
    #pragma unroll 1
    for (int i = 0; i < 1000; ++i) y = 1.0 / (y + 1.0);
    long long c6 = clock64();
    #pragma unroll 1
    for (int i = 0; i < 1000; ++i) y = sqrt(y + 1.0);
    long long c7 = clock64();
    out[t] = x + idx + y;
    if (t == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4; cyc[5] = c6 - c5; cyc[6] = c7 - c6; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 512); cudaMallocManaged(&c, 8 * 8);
    k<<<1, 512>>>(o, c, 1.0, 0.999); cudaDeviceSynchronize();
    k<<<1, 512>>>(o, c, 1.0, 0.999); cudaDeviceSynchronize();
    printf("per-op latency (cycles): dfma %.1f dadd %.1f shfl+dadd %.1f lds(dep) %.1f syncthreads(512) %.1f ddiv %.1f dsqrt %.1f\n",
           c[0] / 1000.0, c[1] / 1000.0, c[2] / 1000.0, c[3] / 1000.0, c[4] / 1000.0, c[5] / 1000.0, c[6] / 1000.0);
    k<<<1, 32>>>(o, c, 1.0, 0.999); cudaDeviceSynchronize();
    printf("1 warp: dfma %.1f dadd %.1f shfl+dadd %.1f lds(dep) %.1f syncthreads(32) %.1f ddiv %.1f dsqrt %.1f\n",
           c[0] / 1000.0, c[1] / 1000.0, c[2] / 1000.0, c[3] / 1000.0, c[4] / 1000.0, c[5] / 1000.0, c[6] / 1000.0);
}
