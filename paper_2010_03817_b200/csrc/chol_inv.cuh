// chol_inv.cuh -- blocked Cholesky that also keeps the inverses of its 8 x 8
// diagonal blocks, and the two triangular solves of the congruence
// M = -L^{-1} A(v) L^{-T} built on them, so that every
// block operation is an FP64 tensor-core (DMMA m8n8k4) product:
//   panel      L_ik   = A_ik L_kk^{-T}            (was: 8 x 8 substitution per row,
//                                                  a 36-deep chain of 24-cycle FMAs)
//   TRSM step  B_k    = L_kk^{-1} B_k             (was: 8 x 8 substitution per column)
//   updates    A_ij  -= L_ik L_jk^T, B_i -= L_ik B_k  (DMMA, unchanged)
// Warp 0 computes the 8 x 8 diagonal factor (rsqrt: no division) and its
// inverse in registers, with a one-block lookahead over the trailing update.
// (All warps factoring it redundantly, to drop a barrier, was measured slower:
// 16x the shuffles.)
// Same arithmetic as the substitution (up to rounding order) -- results agree
// with the oracle's unblocked Cholesky and substitutions to ~1e-15.
#pragma once
#include "chord2.cuh"

namespace sw {

// Inverse diagonal blocks (Lv, 64 doubles each) are stored row-major with the column index
// XOR-swizzled by bit 1 of the row, so that the DMMA fragment loads W[r][q], W[r][4+q] of a
// half-warp (rows 0..3 or 4..7) hit 16 distinct 8-byte bank slots (an unswizzled 8-wide row
// puts rows r and r+2 on the same banks: 2-way conflicts, ncu r2fs).
__device__ __forceinline__ int lv_idx(int r, int c) { return r * 8 + (c ^ ((r & 2) << 1)); }

// acc(8x8) = A(8x8, row-major lda) * W^T, W 8x8 row-major (ldw): C[r][c] = sum_k A[r][k] W[c][k]
__device__ __forceinline__ void tile_mul_wt(double (&acc)[2], const double* A, int lda, const double* W, int ldw,
                                            int lane) {
    const int r = lane >> 2, q = lane & 3;
    const double a0 = A[r * lda + q], a1 = A[r * lda + 4 + q];
    const double b0 = W[lv_idx(r, q)], b1 = W[lv_idx(r, 4 + q)];  // W: an Lv block (ldw = 8, swizzled)
    acc[0] = 0.0;
    acc[1] = 0.0;
    dmma_t(acc, a0, b0);
    dmma_t(acc, a1, b1);
}

// acc(8x8) = W(8x8 row-major, ldw) * B(8x8 at Bp, row-major ldb): C[r][c] = sum_k W[r][k] B[k][c]
__device__ __forceinline__ void tile_mul_w(double (&acc)[2], const double* W, int ldw, const double* Bp, int ldb,
                                           int lane) {
    const int r = lane >> 2, q = lane & 3;
    const double a0 = W[lv_idx(r, q)], a1 = W[lv_idx(r, 4 + q)];  // W: an Lv block (ldw = 8, swizzled)
    const double b0 = Bp[q * ldb + r], b1 = Bp[(4 + q) * ldb + r];
    acc[0] = 0.0;
    acc[1] = 0.0;
    dmma_t(acc, a0, b0);
    dmma_t(acc, a1, b1);
}

// Blocked right-looking Cholesky of the lower triangle of G (n = multiple of 8),
// rdiag = 1 / diag(L), Lv = the inverses of the 8 x 8 diagonal blocks (row-major,
// 64 doubles per block).  Returns false on a non-positive pivot (CTA-uniform).
// 8 x 8 diagonal factor of D (lower, leading dimension ld) and its inverse, by one
// warp in registers (lane r < 8 holds row r; rsqrt: no division; the inverse is the
// forward substitution L X = I).  Stores L_kk into D, 1/diag into rd8, X into V (row-major
// 8 x 8).  Returns the pivot test (warp-uniform).
__device__ __forceinline__ bool diag_factor_inv(double* D, int ld, double* rd8, double* V, int lane) {
    const int r = lane;
    double a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = (r < 8 && c <= r) ? D[r * ld + c] : 0.0;
    bool ok = true;
    double rd = 1.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double d = __shfl_sync(0xffffffffu, a[c], c);
        if (!(d > 0.0)) ok = false;
        const double il = rsqrt(fmax(d, 1e-300));
        if (r == c) { a[c] = d * il; rd = il; }
        else if (r > c) a[c] *= il;
#pragma unroll
        for (int k = c + 1; k < 8; ++k) {
            const double lkc = __shfl_sync(0xffffffffu, a[c], k);
            if (r >= k) a[k] = fma(-a[c], lkc, a[k]);
        }
    }
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (r == k) {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = ((c == k ? 1.0 : 0.0) - x[c]) * rd;
        }
#pragma unroll
        for (int c = 0; c <= k; ++c) {
            const double xkc = __shfl_sync(0xffffffffu, x[c], k);
            if (r > k && r < 8) x[c] = fma(a[k], xkc, x[c]);
        }
    }
    if (r < 8) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c <= r) D[r * ld + c] = a[c];
            V[lv_idx(r, c)] = (c <= r) ? x[c] : 0.0;
        }
        rd8[r] = rd;
    }
    return ok;
}

// The same factor and inverse with the whole 8 x 8 block in every lane's registers (36
// broadcast loads): the column steps need no shuffles (rsqrt -> scale -> update is the whole
// chain), and lane c < 8 forms column c of the inverse by its own forward substitution.  Same
// operations in the same order as diag_factor_inv (bit-identical L, 1/diag and inverse).
__device__ __forceinline__ bool diag_factor_inv_reg(double* D, int ld, double* rd8, double* V, int lane) {
    double a[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) a[r][c] = D[r * ld + c];
    bool ok = true;
    double rd[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double d = a[c][c];
        if (!(d > 0.0)) ok = false;
        const double il = rsqrt(fmax(d, 1e-300));
        a[c][c] = d * il;
        rd[c] = il;
#pragma unroll
        for (int r = c + 1; r < 8; ++r) a[r][c] *= il;
#pragma unroll
        for (int k = c + 1; k < 8; ++k)
#pragma unroll
            for (int r = k; r < 8; ++r) a[r][k] = fma(-a[r][c], a[k][c], a[r][k]);
    }
    // column `lane` of X = L^{-1}: X[r][c] = (delta_rc - sum_{k<r} L[r][k] X[k][c]) / L[r][r]
    const int c = lane & 7;
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < r; ++k) acc = fma(a[r][k], x[k], acc);
        x[r] = ((r == c ? 1.0 : 0.0) - acc) * rd[r];
    }
    __syncwarp();  // every lane has read D
    if (lane < 8) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            V[lv_idx(r, c)] = (r >= c) ? x[r] : 0.0;
            if (r == lane) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k <= r) D[r * ld + k] = a[r][k];
                rd8[r] = rd[r];
            }
        }
    }
    return ok;
}
#ifndef SW_DIAG_REG
#define SW_DIAG_REG 1
#endif
#if SW_DIAG_REG
#define SW_DIAG_FACTOR diag_factor_inv_reg
#else
#define SW_DIAG_FACTOR diag_factor_inv
#endif

// Blocked right-looking Cholesky of the lower triangle of G (n = multiple of 8),
// rdiag = 1 / diag(L), Lv = the inverses of the 8 x 8 diagonal blocks (row-major,
// 64 doubles per block).  Returns false on a non-positive pivot (CTA-uniform).
// Lookahead: in step kb warp 0 updates tile (kb+1, kb+1) first and factors it
// right away, while the other warps do the rest of the trailing update, so the
// diagonal factor (the critical path) overlaps the SYRK; two barriers per step.
__device__ bool cholesky_inv_blocked_la(const Team& T, double* G, int n, int ld, double* rdiag, double* Lv,
                                        int* flag) {
    const int TB = n >> 3;
    const int rr = T.lane >> 2, q = T.lane & 3;
    if (T.warp == 0) {
        const bool ok = SW_DIAG_FACTOR(G, ld, rdiag, Lv, T.lane);
        if (T.lane == 0) *flag = ok ? 0 : 1;
    }
    __syncthreads();
    if (*flag) return false;
    for (int kb = 0; kb < TB; ++kb) {
        const int k0 = kb * 8;
        const double* Vk = Lv + kb * 64;
        // panel: L_ib,kb = A_ib,kb L_kk^{-T}, one 8 x 8 tile per warp (DMMA)
        for (int ib = kb + 1 + T.warp; ib < TB; ib += T.nwarps) {
            double* Ct = G + ib * 8 * ld + k0;
            double acc[2];
            tile_mul_wt(acc, Ct, ld, Vk, 8, T.lane);
            __syncwarp();
            acc_st(acc, Ct, ld, rr, q);
        }
        __syncthreads();
        const int Tr = TB - kb - 1;
        if (Tr == 0) break;
        if (T.warp == 0) {
            // tile (kb+1, kb+1) of the trailing update, then its factor and inverse
            double* C = G + (kb + 1) * 8 * ld + (kb + 1) * 8;
            double acc[2];
            acc_ld(acc, C, ld, rr, q);
            tile_msub<true>(acc, G + (kb + 1) * 8 * ld + k0, ld, G + (kb + 1) * 8 * ld + k0, ld, 8, T.lane);
            acc_st(acc, C, ld, rr, q);
            __syncwarp();
            const bool ok = SW_DIAG_FACTOR(C, ld, rdiag + (kb + 1) * 8, Lv + (kb + 1) * 64, T.lane);
            if (T.lane == 0) *flag = ok ? 0 : 1;
        } else {
            // the rest of the trailing SYRK: G_ij -= P_i P_j^T, kb < j <= i, (i, j) != (kb+1, kb+1),
            // tiles walked incrementally over the warps 1..nwarps-1
            int ii = 0, jj = 0, t = T.warp;  // tile 0 = (0, 0) belongs to warp 0
            while (ii < Tr && jj + t > ii) { t -= ii + 1 - jj; jj = 0; ++ii; }
            jj += t;
            while (ii < Tr) {
                const int ib = kb + 1 + ii, jb = kb + 1 + jj;
                double* C = G + ib * 8 * ld + jb * 8;
                double acc[2];
            acc_ld(acc, C, ld, rr, q);
                tile_msub<true>(acc, G + ib * 8 * ld + k0, ld, G + jb * 8 * ld + k0, ld, 8, T.lane);
                acc_st(acc, C, ld, rr, q);
                jj += T.nwarps - 1;
                while (ii < Tr && jj > ii) { jj -= ii + 1; ++ii; }
            }
        }
        __syncthreads();
        if (*flag) return false;
    }
    return true;
}

// Without lookahead (three barriers per step): used on the global-scratch variant (m > 128),
// where the lookahead was measured 3% slower.
__device__ bool cholesky_inv_blocked(const Team& T, double* G, int n, int ld, double* rdiag, double* Lv,
                                     int* flag) {
    const int TB = n >> 3;
    for (int kb = 0; kb < TB; ++kb) {
        const int k0 = kb * 8;
        double* D = G + k0 * ld + k0;
        double* Vk = Lv + kb * 64;
        if (T.warp == 0) {
            const int r = T.lane;
            double a[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) a[c] = (r < 8 && c <= r) ? D[r * ld + c] : 0.0;
            bool ok = true;
            double rd = 1.0;  // 1 / L_rr of this lane's row
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const double d = __shfl_sync(0xffffffffu, a[c], c);
                if (!(d > 0.0)) ok = false;
                const double il = rsqrt(fmax(d, 1e-300));
                if (r == c) { a[c] = d * il; rd = il; }
                else if (r > c) a[c] *= il;
#pragma unroll
                for (int k = c + 1; k < 8; ++k) {
                    const double lkc = __shfl_sync(0xffffffffu, a[c], k);
                    if (r >= k) a[k] = fma(-a[c], lkc, a[k]);
                }
            }
            // X = L_kk^{-1}: forward substitution on L X = I, lane r owns row r of X
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (r == k) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) x[c] = ((c == k ? 1.0 : 0.0) - x[c]) * rd;
                }
#pragma unroll
                for (int c = 0; c <= k; ++c) {
                    const double xkc = __shfl_sync(0xffffffffu, x[c], k);
                    if (r > k && r < 8) x[c] = fma(a[k], xkc, x[c]);
                }
            }
            if (r < 8) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (c <= r) D[r * ld + c] = a[c];
                    Vk[lv_idx(r, c)] = (c <= r) ? x[c] : 0.0;
                }
                rdiag[k0 + r] = rd;
            }
            if (T.lane == 0) *flag = ok ? 0 : 1;
        }
        __syncthreads();
        if (*flag) return false;
        // panel: L_ib,kb = A_ib,kb L_kk^{-T}, one 8 x 8 tile per warp (DMMA)
        for (int ib = kb + 1 + T.warp; ib < TB; ib += T.nwarps) {
            double* Ct = G + ib * 8 * ld + k0;
            double acc[2];
            tile_mul_wt(acc, Ct, ld, Vk, 8, T.lane);
            __syncwarp();
            const int r = T.lane >> 2, q = T.lane & 3;
            acc_st(acc, Ct, ld, r, q);
        }
        __syncthreads();
        // trailing SYRK on DMMA tiles: G_ij -= P_i P_j^T, kb < j <= i (tile index walked
        // incrementally: no divisions / square roots)
        const int Tr = TB - kb - 1;
        int ii = 0, jj = T.warp;
        while (ii < Tr && jj > ii) { jj -= ii + 1; ++ii; }
        while (ii < Tr) {
            const int ib = kb + 1 + ii, jb = kb + 1 + jj;
            double* C = G + ib * 8 * ld + jb * 8;
            const int rr = T.lane >> 2, q = T.lane & 3;
            double acc[2];
            acc_ld(acc, C, ld, rr, q);
            tile_msub<true>(acc, G + ib * 8 * ld + k0, ld, G + jb * 8 * ld + k0, ld, 8, T.lane);
            acc_st(acc, C, ld, rr, q);
            jj += T.nwarps;
            while (ii < Tr && jj > ii) { jj -= ii + 1; ++ii; }
        }
        __syncthreads();
    }
    return true;
}

// B <- L^{-1} B on all n columns, with the inverse diagonal blocks Lv.  TR =
// true works on the transposed view W(r, c) = B[c*ld + r] (i.e. B <- B L^{-T}).
template <bool TR>
__device__ void trsm_inv_blocked(const Team& T, const double* G, const double* Lv, double* B, int n, int ld) {
    const int TB = n >> 3;
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int kb = 0; kb < TB; ++kb) {
        const int k0 = kb * 8;
        const double* Vk = Lv + kb * 64;
        // block row kb: W_kb = L_kk^{-1} W_kb (one tile per warp)
        for (int cb = T.warp; cb < TB; cb += T.nwarps) {
            double acc[2];
            if (!TR) {
                double* Bt = B + k0 * ld + cb * 8;  // W tile (kb, cb) = B rows k0.., cols cb*8..
                tile_mul_w(acc, Vk, 8, Bt, ld, T.lane);
                __syncwarp();
                acc_st(acc, Bt, ld, r, q);
            } else {
                double* Bt = B + cb * 8 * ld + k0;  // W tile (kb, cb) = (B rows cb*8.., cols k0..)^T
                tile_mul_wt(acc, Bt, ld, Vk, 8, T.lane);
                __syncwarp();
                acc_st(acc, Bt, ld, r, q);
            }
        }
        __syncthreads();
        int ib = kb + 1, cb = T.warp;
        while (cb >= TB) { cb -= TB; ++ib; }
        for (; ib < TB; cb += T.nwarps) {
            while (cb >= TB) { cb -= TB; ++ib; }
            if (ib >= TB) break;
            const double* A = G + ib * 8 * ld + k0;
            double acc[2];
            if (!TR) {
                double* C = B + ib * 8 * ld + cb * 8;
                acc[0] = C[r * ld + 2 * q];
                acc[1] = C[r * ld + 2 * q + 1];
                tile_msub<false>(acc, A, ld, B + k0 * ld + cb * 8, ld, 8, T.lane);
                acc_st(acc, C, ld, r, q);
            } else {
                double* Ct = B + cb * 8 * ld + ib * 8;
                acc[0] = Ct[(2 * q) * ld + r];
                acc[1] = Ct[(2 * q + 1) * ld + r];
                tile_msub<true>(acc, A, ld, B + cb * 8 * ld + k0, ld, 8, T.lane);
                Ct[(2 * q) * ld + r] = acc[0];
                Ct[(2 * q + 1) * ld + r] = acc[1];
            }
        }
        __syncthreads();
    }
}

// As trsm_inv_blocked with a one-row lookahead: the warp that updates a tile of block
// row kb+1 in step kb also multiplies it by L_{kb+1,kb+1}^{-1} right away, so the row
// multiply needs no phase (and barrier) of its own -- one barrier per block step.
template <bool TR>
__device__ void trsm_inv_blocked_la(const Team& T, const double* G, const double* Lv, double* B, int n, int ld) {
    const int TB = n >> 3;
    const int r = T.lane >> 2, q = T.lane & 3;
    // block row 0
    for (int cb = T.warp; cb < TB; cb += T.nwarps) {
        double acc[2];
        if (!TR) {
            double* Bt = B + cb * 8;
            tile_mul_w(acc, Lv, 8, Bt, ld, T.lane);
            __syncwarp();
            acc_st(acc, Bt, ld, r, q);
        } else {
            double* Bt = B + cb * 8 * ld;
            tile_mul_wt(acc, Bt, ld, Lv, 8, T.lane);
            __syncwarp();
            acc_st(acc, Bt, ld, r, q);
        }
    }
    __syncthreads();
    for (int kb = 0; kb + 1 < TB; ++kb) {
        const int k0 = kb * 8;
        const double* Vn = Lv + (kb + 1) * 64;
        int ib = kb + 1, cb = T.warp;
        while (cb >= TB) { cb -= TB; ++ib; }
        for (; ib < TB; cb += T.nwarps) {
            while (cb >= TB) { cb -= TB; ++ib; }
            if (ib >= TB) break;
            const double* A = G + ib * 8 * ld + k0;
            double acc[2];
            if (!TR) {
                double* C = B + ib * 8 * ld + cb * 8;
                acc[0] = C[r * ld + 2 * q];
                acc[1] = C[r * ld + 2 * q + 1];
                tile_msub<false>(acc, A, ld, B + k0 * ld + cb * 8, ld, 8, T.lane);
                acc_st(acc, C, ld, r, q);
                if (ib == kb + 1) {  // finish block row kb+1: W = L^{-1} W for this tile
                    __syncwarp();
                    tile_mul_w(acc, Vn, 8, C, ld, T.lane);
                    __syncwarp();
                    acc_st(acc, C, ld, r, q);
                }
            } else {
                double* Ct = B + cb * 8 * ld + ib * 8;
                acc[0] = Ct[(2 * q) * ld + r];
                acc[1] = Ct[(2 * q + 1) * ld + r];
                tile_msub<true>(acc, A, ld, B + cb * 8 * ld + k0, ld, 8, T.lane);
                Ct[(2 * q) * ld + r] = acc[0];
                Ct[(2 * q + 1) * ld + r] = acc[1];
                if (ib == kb + 1) {
                    __syncwarp();
                    tile_mul_wt(acc, Ct, ld, Vn, 8, T.lane);
                    __syncwarp();
                    acc_st(acc, Ct, ld, r, q);
                }
            }
        }
        __syncthreads();
    }
}

// acc -= A(8 x K) * B(K x 8) as tile_msub, with two accumulator chains (even / odd k-steps)
// so that consecutive DMMAs do not wait on each other.
template <bool BNK>
__device__ __forceinline__ void tile_msub2(double (&acc)[2], const double* A, int lda, const double* Bp, int ldb,
                                           int K, int lane) {
    const int r = lane >> 2, q = lane & 3;
    double acc2[2] = {0.0, 0.0};
    int k0 = 0;
#pragma unroll 2
    for (; k0 + 8 <= K; k0 += 8) {
        const double a0 = -A[r * lda + k0 + q];
        const double a1 = -A[r * lda + k0 + 4 + q];
        const double b0 = BNK ? Bp[r * ldb + k0 + q] : Bp[(k0 + q) * ldb + r];
        const double b1 = BNK ? Bp[r * ldb + k0 + 4 + q] : Bp[(k0 + 4 + q) * ldb + r];
        dmma_t(acc, a0, b0);
        dmma_t(acc2, a1, b1);
    }
    if (k0 < K) {
        const double a0 = -A[r * lda + k0 + q];
        const double b0 = BNK ? Bp[r * ldb + k0 + q] : Bp[(k0 + q) * ldb + r];
        dmma_t(acc, a0, b0);
    }
    acc[0] += acc2[0];
    acc[1] += acc2[1];
}

// B <- L^{-1} B, left-looking with one warp per 8-column block: for each block row i,
// acc = B_ic - L_i,0:i X_0:i,c (one DMMA chain over all earlier blocks, accumulator in
// registers), X_ic = L_ii^{-1} acc.  Column blocks are independent, so there is no CTA
// barrier inside (the right-looking trsm_inv_blocked_la needs one per block step and
// re-loads / stores every trailing tile at each step).  Ends with a barrier.
__device__ void trsm_ll_cols(const Team& T, const double* G, const double* Lv, double* B, int n, int ld) {
    const int TB = n >> 3;
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int cb = T.warp; cb < TB; cb += T.nwarps) {
        double* Bc = B + cb * 8;
        for (int ib = 0; ib < TB; ++ib) {
            double* C = Bc + ib * 8 * ld;
            double acc[2];
            acc_ld(acc, C, ld, r, q);
            if (ib > 0) tile_msub2<false>(acc, G + ib * 8 * ld, ld, Bc, ld, 8 * ib, T.lane);
            acc_st(acc, C, ld, r, q);
            __syncwarp();
            tile_mul_w(acc, Lv + ib * 64, 8, C, ld, T.lane);
            __syncwarp();
            acc_st(acc, C, ld, r, q);
            __syncwarp();
        }
    }
    __syncthreads();
}

// B <- B L^{-T}, left-looking with one warp per 8-row block: M_rj = (B_rj - M_r,0:j L_j,0:j^T)
// L_jj^{-T}, j ascending (each block row only reads itself and L).  Ends with a barrier.
__device__ void trsm_ll_rows(const Team& T, const double* G, const double* Lv, double* B, int n, int ld) {
    const int TB = n >> 3;
    const int r = T.lane >> 2, q = T.lane & 3;
    for (int rb = T.warp; rb < TB; rb += T.nwarps) {
        double* Br = B + rb * 8 * ld;
        for (int jb = 0; jb < TB; ++jb) {
            double* C = Br + jb * 8;
            double acc[2];
            acc_ld(acc, C, ld, r, q);
            if (jb > 0) tile_msub2<true>(acc, Br, ld, G + jb * 8 * ld, ld, 8 * jb, T.lane);
            acc_st(acc, C, ld, r, q);
            __syncwarp();
            tile_mul_wt(acc, C, ld, Lv + jb * 64, 8, T.lane);
            __syncwarp();
            acc_st(acc, C, ld, r, q);
            __syncwarp();
        }
    }
    __syncthreads();
}

// the congruence B <- L^{-1} B L^{-T} of the split factor kernels (SW_TRSM_LL = 0: the
// right-looking pair)
#ifndef SW_TRSM_LL
#define SW_TRSM_LL 1
#endif
__device__ __forceinline__ void congruence_inv(const Team& T, const double* G, const double* Lv, double* B, int n,
                                               int ld) {
#if SW_TRSM_LL
    trsm_ll_cols(T, G, Lv, B, n, ld);
    trsm_ll_rows(T, G, Lv, B, n, ld);
#else
    trsm_inv_blocked_la<false>(T, G, Lv, B, n, ld);
    trsm_inv_blocked_la<true>(T, G, Lv, B, n, ld);
#endif
}

}  // namespace sw
