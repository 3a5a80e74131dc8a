// Microbenchmark of the K2 Lanczos stages in isolation (cycles per iteration, 1 CTA of 512 threads)
#include <cstdio>
template <int KC, int MODE>
__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, int iters, int mdp) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = tid >> 2, g = tid & 3;
    for (int i = tid; i < 4096; i += 512) sm[i] = 1.0 / (1 + i);
    __syncthreads();
    double2 mr[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) mr[k] = make_double2(0.001 * (r + k), 0.002 * (g + k));
    double wr = 0.5, acc = 0.0;
    long long c0 = clock64();
    for (int j = 0; j < iters; ++j) {
        const int oU = (j & 1) * 256;
        double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k0 = 0; k0 < KC; k0 += 4) {
            double2 wq[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = 2 * g + 8 * (k0 + k);
                wq[k] = (k0 + k < KC && c < mdp) ? *reinterpret_cast<const double2*>(sm + oU + c) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k0 + k < KC) {
                    a8[2 * k] = fma(mr[k0 + k].x, wq[k].x, a8[2 * k]);
                    a8[2 * k + 1] = fma(mr[k0 + k].y, wq[k].y, a8[2 * k + 1]);
                }
        }
        double y = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
        y += __shfl_xor_sync(0xffffffffu, y, 1);
        y += __shfl_xor_sync(0xffffffffu, y, 2);
        if (MODE >= 1) {
            y *= 1e-3;
        }
        if (g == 0 && r < mdp) sm[256 * ((j + 1) & 1) + r] = y + wr;
        acc += y;
        __syncthreads();
        if (MODE >= 2) {
            // a second barrier stage with a rows_sum8 + tree of 16
            double v = y * y;
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (lane == 0) sm[1024 + 32 * (j & 1) + warp] = v;
            __syncthreads();
            double t[16];
#pragma unroll
            for (int w = 0; w < 16; ++w) t[w] = sm[1024 + 32 * (j & 1) + w];
#pragma unroll
            for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
                for (int w = 0; w < h; ++w) t[w] += t[w + h];
            wr = 1.0 / sqrt(t[0] + 1.0);
        }
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
        long long one = c[0];
        kern<<<148, 512, 200 * 1024>>>(o, c, it, 104); cudaDeviceSynchronize();
        printf("%-40s %.0f cycles/iter (1 CTA)  %.0f (148 CTAs)  err=%s\n", name, one / (double)it, c[0] / (double)it,
               cudaGetErrorString(cudaGetLastError()));
    };
    run(k<13, 0>, "matvec+barrier");
    run(k<13, 1>, "matvec+scale+barrier");
    run(k<13, 2>, "matvec+barrier+reduce+barrier");
    run(k<16, 2>, "KC16 matvec+barrier+reduce+barrier");
}
