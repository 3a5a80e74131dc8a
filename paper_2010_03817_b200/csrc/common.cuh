// common.cuh -- shared device helpers for the specwalk kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define SW_INF (__longlong_as_double(0x7ff0000000000000LL))

// packed lower-triangular index (row-major packing of the lower triangle)
__host__ __device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }

#define SW_BIND_NONE_DEV (-2)
#define SW_BIND_BALL_DEV (-1)

// chain flag bits
enum : int {
    CF_DONE = 1,         // all steps done
    CF_NEED_NORMAL = 2,  // dense-block hit: K3/K4 must build the normal and reflect
    CF_FAILED = 4,       // start of a segment was not interior (Cholesky failed)
};

// Philox4x32-10 (Salmon et al. SC'11), written for the device independently of
// the oracle; counter = (block j, step, global chain id, tag), key = seed.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += W0;
        k.y += W1;
    }
    return c;
}

// 52-bit uniform in [2^-53, 1 - 2^-53] (reading R7)
__device__ __forceinline__ double u01(uint32_t a, uint32_t b) {
    return ((double)(a >> 6) * 67108864.0 + (double)(b >> 6) + 0.5) * (1.0 / 4503599627370496.0);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
