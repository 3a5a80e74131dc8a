// gemm.cuh -- K1 / K3: batched FP64 contractions on the DMMA tensor pipe.
//
// K1 (direction contraction, "B_k = sum_j p_jk A_j", cost O(dnm^2)
//     P:667):  AV[c, :] = sum_i V[c, i] * Ahat[i, :]        (B stored K x N)
// K0 (A(x0)):  AX[c, :] = a0 + sum_i X[c, i] * Ahat[i, :]   (same kernel + bias)
// K3 (normal contraction, lemma:gradient P:752-764):
//              G[c, i] = sum_j Yhat[c, j] * Ahat[i, j]      (B stored N x K)
// where Ahat row i = packed lower triangle of A_{i+1}, Yhat = packed y y^T with
// the off-diagonal entries doubled, so G[c, i] = y^T A_{i+1} y.
//
// Rows of the A operand (chains) are gathered through a list of chain slots;
// row r >= *count_dev (or list[r] < 0) is zero and not stored.
// Tile 64 x 64 x 16, 4 warps, warp tile 32 x 32 = 4 x 4 DMMA m8n8k4 tiles,
// cp.async double buffering.  K and N must be multiples of 16 / 64 (padded).
#pragma once
#include "common.cuh"

namespace sw {

constexpr int GB_M = 64, GB_N = 64, GB_K = 16;
constexpr int GA_LD = GB_K + 4;  // 20 doubles: conflict-free 8x4 fragment reads
constexpr int GB_LD = GB_N + 4;  // 68 doubles

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int nbytes = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(nbytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <bool B_NK>
__global__ void __launch_bounds__(128) gemm_f64_dmma(const double* __restrict__ A, int lda,
                                                      const int* __restrict__ list,
                                                      const int* __restrict__ count_dev, int count_host,
                                                      const double* __restrict__ B, int ldb,
                                                      double* __restrict__ C, int ldc,
                                                      const double* __restrict__ bias, int K) {
    __shared__ __align__(16) double As[2][GB_M * GA_LD];
    __shared__ __align__(16) double Bs[2][B_NK ? GB_N * GA_LD : GB_K * GB_LD];
    __shared__ int rows[GB_M];

    const int count = count_dev ? min(*count_dev, count_host) : count_host;
    const int m0 = blockIdx.y * GB_M;
    if (m0 >= count) return;
    const int n0 = blockIdx.x * GB_N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < GB_M) {
        int r = m0 + tid;
        rows[tid] = (r < count) ? (list ? list[r] : r) : -1;
    }
    __syncthreads();

    auto load_stage = [&](int st, int k0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // A: 64 rows x 16 doubles = 512 chunks of 2
            int q = tid + i * 128;
            int r = q >> 3, c2 = (q & 7) * 2;
            int slot = rows[r];
            const double* src = A + (size_t)(slot < 0 ? 0 : slot) * lda + k0 + c2;
            cp_async16(&As[st][r * GA_LD + c2], src, slot >= 0);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int q = tid + i * 128;
            if (!B_NK) {  // B: 16 rows (k) x 64 cols (n)
                int kk = q >> 5, c2 = (q & 31) * 2;
                cp_async16(&Bs[st][kk * GB_LD + c2], B + (size_t)(k0 + kk) * ldb + n0 + c2, true);
            } else {      // B: 64 rows (n) x 16 cols (k)
                int nn = q >> 3, c2 = (q & 7) * 2;
                cp_async16(&Bs[st][nn * GA_LD + c2], B + (size_t)(n0 + nn) * ldb + k0 + c2, true);
            }
        }
        cp_async_commit();
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int wm = warp >> 1, wn = warp & 1;
    const int fr = lane >> 2, fc = lane & 3;
    const int KT = K / GB_K;
    load_stage(0, 0);
    for (int kt = 0; kt < KT; ++kt) {
        if (kt + 1 < KT) {
            load_stage((kt + 1) & 1, (kt + 1) * GB_K);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* as = As[kt & 1];
        const double* bs = Bs[kt & 1];
#pragma unroll
        for (int kk = 0; kk < GB_K; kk += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = as[(wm * 32 + mi * 8 + fr) * GA_LD + kk + fc];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
                b[ni] = B_NK ? bs[(wn * 32 + ni * 8 + fr) * GA_LD + kk + fc]
                             : bs[(kk + fc) * GB_LD + wn * 32 + ni * 8 + fr];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni], a[mi], b[ni]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
        int r = wm * 32 + mi * 8 + fr;
        int slot = rows[r];
        if (slot < 0) continue;
        double* crow = C + (size_t)slot * ldc;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            int col = n0 + wn * 32 + ni * 8 + fc * 2;
            double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            if (bias) {
                v.x += bias[col];
                v.y += bias[col + 1];
            }
            *reinterpret_cast<double2*>(crow + col) = v;
        }
    }
}

}  // namespace sw
