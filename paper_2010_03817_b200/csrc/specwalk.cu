// specwalk.cu -- host side of the C-ABI (include/specwalk.h): context, device
// memory layout, the round scheduler that drives the kernels, and the
// boundary_oracle / walk_sample / walk_trace entry points.
//
// Device layout (per context / GPU):
//   Ahat   : np x mtp   row i = packed lower(A_{i+1}), zero padded
//   a0     : mtp        packed lower(A0)
//   chains : X, Xs, V (C x np); AX, AXs, AV, Yh (C x mtp); U (C x m); Gn (C x np)
//            scalar SoA: ell, steps_done, refl, bound, flags, counters
// np = roundup(n, 64), mt = m(m+1)/2, mtp = roundup(mt, 64).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/specwalk.h"
#include "gemm.cuh"
#include "walk.cuh"
#include "chord2.cuh"
#include "chord3.cuh"
#include "lanczos2.cuh"
#include "lanczos_cl.cuh"
#include "lanczos_t.cuh"
#include "hmc.cuh"
#include "hmc2.cuh"
#include "colloc.cuh"
#include "factor_t.cuh"
#include "factor_g.cuh"
#include "estimators.cuh"
#include <algorithm>

using namespace sw;

static thread_local std::string g_err;

extern "C" const char* spec_last_error(void) { return g_err.c_str(); }

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(SPEC_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

static int roundup(int a, int b) { return (a + b - 1) / b * b; }

struct spec_ctx;
static bool walk_is_active(spec_ctx* ctx);
#define SW_NOT_DURING_WALK(ctx)                                                                  \
    do {                                                                                        \
        if (walk_is_active(ctx))                                                                \
            return fail(SPEC_EINVAL, "a resumable walk is in progress (call walk_end first)"); \
    } while (0)

struct ChainBuf {
    long long cap = 0;
    double *X = nullptr, *Xs = nullptr, *V = nullptr, *AX = nullptr, *AXs = nullptr, *AV = nullptr, *Yh = nullptr,
           *U = nullptr, *Gn = nullptr, *ell = nullptr, *tlast = nullptr;
    int *steps_done = nullptr, *refl = nullptr, *bound = nullptr, *flags = nullptr, *nrej = nullptr, *ndeg = nullptr,
        *ncap = nullptr;
    int* jlast = nullptr;
    double *wM = nullptr, *wL = nullptr, *wS = nullptr;  // K2 split work buffers
    long long *calls = nullptr, *nrefl = nullptr;
    int *list = nullptr, *list2 = nullptr, *nlist = nullptr;
    int* counters = nullptr;  // [0] count, [1] count2, [2] ncount
    long long* gid = nullptr;
};

struct OracleBuf {
    long long cap = 0;
    int m_cap = 0;
    double *x = nullptr, *v = nullptr, *u = nullptr;            // host-input staging (batch x n, batch x m)
    double *tm = nullptr, *tp = nullptr, *nrm = nullptr, *ker = nullptr;
    int *bind = nullptr, *stat = nullptr;
};
static void free_obuf(OracleBuf& o) {
    void* ps[] = {o.x, o.v, o.u, o.tm, o.tp, o.nrm, o.ker, o.bind, o.stat};
    for (void* p : ps)
        if (p) cudaFree(p);
    o = OracleBuf();
}
// K5 split work buffers (hmc2.cuh), grown with the chain capacity on first HMC use
struct HmcBuf {
    long long cap = 0;
    double *wH = nullptr, *wQ = nullptr;
    double *wM = nullptr, *wL = nullptr, *wS = nullptr;  // own copies when the K2 split is off
    int *il0 = nullptr, *il1 = nullptr, *cnt = nullptr;
};

// K7 (collocation HMC-r, colloc.cuh) per-slot buffers, grown with the chain capacity and d
struct ChmcBuf {
    long long cap = 0;
    int d = 0;
    double *CF = nullptr, *CB = nullptr, *GW = nullptr, *hseg = nullptr;
    int* elist = nullptr;
};
static void free_chmc_bufs(ChmcBuf& h) {
    void* ps[] = {h.CF, h.CB, h.GW, h.hseg, h.elist};
    for (void* p : ps)
        if (p) cudaFree(p);
    h = ChmcBuf();
}

struct spec_ctx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    int n = 0, m = 0, np = 0, mt = 0, mtp = 0, ld = 0;
    double* Ahat = nullptr;
    double* a0 = nullptr;
    double *lo = nullptr, *hi = nullptr;
    int has_cube = 0;
    double* c = nullptr;
    double* Ac = nullptr;
    int has_obj = 0;
    double* hmc_scratch = nullptr;
    long long hmc_stride = 0;
    int hmc_grid = 0;
    size_t hmc_smem = 0;
    int hmc_split = 0;   // K5 as setup / (factor, Lanczos, Weyl)^k / tail (hmc2.cuh), m <= 128
    int hmc_nt = 512, hmc_kc = 13;
    int hf_grid = 0, hl_grid = 0, ht_grid = 0, hs_grid = 0;
    size_t hf_smem = 0, hl_smem = 0, ht_smem = 0;
    HmcBuf hb;
    double* ball_c = nullptr;
    double* c0 = nullptr;  // centre of the exact ball samples of volume() (n doubles)
    double ball_r = 0.0;
    int has_ball = 0;
    double amax = 0.0;
    ChainBuf cb;
    double* scratch = nullptr;
    long long scratch_stride = 0;
    int scratch_ctas = 0;
    bool smem_path = true;
    int k2_variant = 0;
    int k2_split = 0;  // K2 as factor / Lanczos / tail kernels (chord3.cuh)
    int f_grid = 0, l_grid = 0, t_grid = 0;
    int lz2 = 0, l2_grid = 0;  // K2b as lanczos2_kernel (two chains per SM, m <= 104)
    int t512 = 0;              // m > 112 split tail with 512 threads (one CTA per SM)
    int fg = 0, fg_grid = 0;   // m > 112 factor phase as factor_g_kernel<fg> (G/L/W tiles in shared memory, B tiles in L2)
    size_t fg_smem = 0;
    int ft = 0, ft_grid = 0;   // K2a as factor_t_kernel (lower-tile storage, two chains per SM, m <= 104)
    size_t ft_smem = 0;
    // m > 112: factor (global scratch) | lanczos_t_kernel (g_split = 2) or lanczos_cl_kernel (2-CTA
    // cluster, g_split = 1) | tail
    int g_split = 0, cl_grid = 0, lt_grid = 0;
    size_t cl_smem = 0, lt_smem = 0;
    size_t l2_smem = 0;
    size_t f_smem = 0, l_smem = 0, t_smem = 0;
    size_t smem_bytes = 0;
    size_t g_smem = 0;  // global-scratch K2 variant: vector area in shared memory
    int chord_threads = 256;
    int chord_grid_max = 0;
    int num_sms = 0;
    long long* dstats = nullptr;
    unsigned long long* jsum = nullptr;  // Lanczos iteration counters (spec_lanczos_iterations)
    unsigned long long* prof = nullptr;
    double* lsave = nullptr;
    long long lsave_stride = 0;
    long long launches = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    void* walk = nullptr;  // WalkRun*
    spec_comm comm{nullptr, 0, 1, nullptr};
    int has_comm = 0;
    void* obuf = nullptr;  // OracleBuf*
    // collocation HMC-r (K7): potential f of exp(-f) (spec_set_potential) and its buffers
    int pot = -1;
    double pot_scale = 1.0;
    double* pot_mu = nullptr;
    int has_mu = 0;
    ChmcBuf chb;
    double* chmc_scratch = nullptr;
    long long chmc_stride = 0;
    int chmc_grid = 0, chmc_d = 0, chmc_nt = 512;
    size_t chmc_smem = 0;
    unsigned long long* picard = nullptr;  // Picard iterations, segments, unconverged
};

static void free_chains(ChainBuf& b) {
    void* ps[] = {b.X, b.Xs, b.V, b.AX, b.AXs, b.AV, b.Yh, b.U, b.Gn, b.ell, b.tlast, b.steps_done, b.refl, b.bound,
                  b.flags, b.nrej, b.ndeg, b.ncap, b.calls, b.nrefl, b.list, b.list2, b.nlist, b.counters, b.gid, b.jlast, b.wM, b.wL, b.wS};
    for (void* p : ps)
        if (p) cudaFree(p);
    b = ChainBuf();
}

template <typename T>
static cudaError_t zalloc(T** p, size_t count) {
    cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (count ? count : 1));
    if (e == cudaSuccess) e = cudaMemset(*p, 0, sizeof(T) * (count ? count : 1));
    // cudaMemset runs on the legacy default stream, which the library's non-blocking stream
    // does not wait for: without this the zero fill could land after the first kernels
    // writing the buffer (seen as intermittently zeroed chain state)
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    return e;
}

static int ensure_chains(spec_ctx* ctx, long long C) {
    ChainBuf& b = ctx->cb;
    if (C <= b.cap) return SPEC_OK;
    free_chains(b);
    long long cap = C;
    size_t np = ctx->np, mtp = ctx->mtp, m = ctx->m;
    cudaError_t e = cudaSuccess;
#define ZA(ptr, cnt) \
    if (e == cudaSuccess) e = zalloc(&b.ptr, (size_t)(cnt));
    ZA(X, cap * np) ZA(Xs, cap * np) ZA(V, cap * np) ZA(Gn, cap * np) ZA(AX, cap * mtp) ZA(AXs, cap * mtp)
    ZA(AV, cap * mtp) ZA(Yh, cap * mtp) ZA(U, cap * m) ZA(ell, cap) ZA(tlast, cap) ZA(steps_done, cap) ZA(refl, cap)
    ZA(bound, cap) ZA(flags, cap) ZA(nrej, cap) ZA(ndeg, cap) ZA(ncap, cap) ZA(calls, cap) ZA(nrefl, cap) ZA(list, cap)
    ZA(list2, cap) ZA(nlist, cap) ZA(counters, 8) ZA(gid, cap) ZA(jlast, cap)
    if (ctx->k2_split || ctx->g_split) {
        const size_t mp = (size_t)roundup(ctx->m, 8);
        ZA(wM, cap * mp * ctx->ld) ZA(wL, cap * mp * ctx->ld) ZA(wS, cap * (size_t)s_stride((int)mp))
    }
#undef ZA
    if (e != cudaSuccess) {
        free_chains(b);
        cudaGetLastError();
        return fail(SPEC_ENOMEM, std::string("chain buffers: ") + cudaGetErrorString(e));
    }
    b.cap = cap;
    return SPEC_OK;
}

static int create_impl(spec_ctx* ctx, int n, int m, const double* A, const double* cube_lo, const double* cube_hi,
                       int device);
extern "C" int spec_create(int n, int m, const double* A, const double* cube_lo, const double* cube_hi,
                           int device, spec_ctx** out) {
    if (!out) return fail(SPEC_EINVAL, "out is NULL");
    *out = nullptr;
    if (n < 1 || m < 1 || m > SPEC_MAX_M || !A) return fail(SPEC_EINVAL, "bad n/m/A");
    if ((cube_lo == nullptr) != (cube_hi == nullptr)) return fail(SPEC_EINVAL, "cube_lo/cube_hi: both or neither");
    const size_t mm = (size_t)m * m;
    for (size_t e = 0; e < (size_t)(n + 1) * mm; ++e)
        if (!std::isfinite(A[e])) return fail(SPEC_EINVAL, "A has NaN/Inf");
    for (int k = 0; k <= n; ++k)
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < i; ++j) {
                double a = A[k * mm + (size_t)i * m + j], b = A[k * mm + (size_t)j * m + i];
                if (std::fabs(a - b) > 1e-12 * std::fmax(1.0, std::fabs(a)))
                    return fail(SPEC_EINVAL, "A_" + std::to_string(k) + " is not symmetric");
            }
    if (cube_lo)
        for (int i = 0; i < n; ++i)
            if (!(cube_lo[i] < cube_hi[i])) return fail(SPEC_EINVAL, "cube_lo >= cube_hi");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(SPEC_ECUDA, "no CUDA device (the library has no CPU fallback)");
    }
    spec_ctx* ctx = new spec_ctx();
    ctx->obuf = new OracleBuf();
    int rc = create_impl(ctx, n, m, A, cube_lo, cube_hi, device);
    if (rc) {
        std::string msg = g_err;
        spec_destroy(ctx);  // frees whatever was allocated before the failure
        g_err = msg;
        return rc;
    }
    *out = ctx;
    return SPEC_OK;
}

static int create_impl(spec_ctx* ctx, int n, int m, const double* A, const double* cube_lo, const double* cube_hi,
                       int device) {
    const size_t mm = (size_t)m * m;
    if (device < 0) cudaGetDevice(&device);
    ctx->dev = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ctx->e0));
    CK(cudaEventCreate(&ctx->e1));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    ctx->num_sms = prop.multiProcessorCount;
    ctx->n = n;
    ctx->m = m;
    ctx->np = roundup(n, 64);
    ctx->mt = m * (m + 1) / 2;
    ctx->mtp = roundup(ctx->mt, 64);
    // packed, symmetrised, padded coefficient matrix
    std::vector<double> Ah((size_t)ctx->np * ctx->mtp, 0.0), a0((size_t)ctx->mtp, 0.0);
    double amax = 0.0;
    for (int k = 0; k <= n; ++k)
        for (int i = 0; i < m; ++i)
            for (int j = 0; j <= i; ++j) {
                double v = 0.5 * (A[k * mm + (size_t)i * m + j] + A[k * mm + (size_t)j * m + i]);
                if (k == 0) a0[pk(i, j)] = v;
                else {
                    Ah[(size_t)(k - 1) * ctx->mtp + pk(i, j)] = v;
                    amax = std::fmax(amax, std::fabs(v));
                }
            }
    ctx->amax = amax;
    CK(zalloc(&ctx->Ahat, Ah.size()));
    CK(zalloc(&ctx->a0, a0.size()));
    // stream-ordered uploads (a pageable cudaMemcpy may return before its DMA completes, and
    // the library's stream does not wait for the legacy default stream)
    CK(cudaMemcpyAsync(ctx->Ahat, Ah.data(), sizeof(double) * Ah.size(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->a0, a0.data(), sizeof(double) * a0.size(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (cube_lo) {
        CK(zalloc(&ctx->lo, n));
        CK(zalloc(&ctx->hi, n));
        CK(cudaMemcpyAsync(ctx->lo, cube_lo, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->hi, cube_hi, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->has_cube = 1;
    }
    CK(zalloc(&ctx->c, ctx->np));
    CK(zalloc(&ctx->Ac, ctx->mtp));
    CK(zalloc(&ctx->ball_c, ctx->np));
    CK(zalloc(&ctx->c0, ctx->np));
    CK(zalloc(&ctx->dstats, 8));
    CK(zalloc(&ctx->jsum, 2));
    if (getenv("SPECWALK_PROF")) CK(zalloc(&ctx->prof, 32));
    // K2 variant: M register-resident (m <= 128) with matrices in shared memory,
    // else matrices + Lanczos basis in a per-CTA global scratch slice.
    const int mp = roundup(m, 8);
    ctx->ld = mp + 4;
    // K2 variants: 0 = <256, smem, KC 8> (mp <= 64), 1 = <512, smem, KC 13> (mp <= 104),
    // 3 = <512, smem, KC 16> (mp <= 128), 2 = global scratch (larger m).
    // small m: smaller CTAs, more chains resident per SM (4 = <128, KC 4>, 5 = <192, KC 6>)
    if (mp <= 32) {
        ctx->k2_variant = 4;
        ctx->chord_threads = 128;
    } else if (mp <= 48) {
        ctx->k2_variant = 5;
        ctx->chord_threads = 192;
    } else if (mp <= 64) {
        ctx->k2_variant = 0;
        ctx->chord_threads = 256;
    } else if (mp <= 104) {
        ctx->k2_variant = 1;
        ctx->chord_threads = 512;
    } else if (mp <= 128) {
        ctx->k2_variant = 3;
        ctx->chord_threads = 512;
    } else {
        ctx->k2_variant = 2;
        ctx->chord_threads = 512;
    }
    size_t vecs = (size_t)NVEC2 * (mp + 8) + 64;
    // G, B with one spare row each (in-place deflation) and B's alignment shift
    size_t per_cta = (size_t)2 * (mp + 1) * ctx->ld + 2 + vecs;
    ctx->smem_bytes = per_cta * sizeof(double);
    int occ = 0;
    if (ctx->k2_variant != 2 && ctx->smem_bytes <= 227 * 1024) {
        ctx->smem_path = true;
#define SW_K2_SETUP(NT_, KC_)                                                                                   \
    CK(cudaFuncSetAttribute(chord_kernel2<NT_, true, KC_>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                            (int)ctx->smem_bytes));                                                           \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chord_kernel2<NT_, true, KC_>, NT_, ctx->smem_bytes));
        if (ctx->k2_variant == 4) {
            SW_K2_SETUP(128, 4)
        } else if (ctx->k2_variant == 5) {
            SW_K2_SETUP(192, 6)
        } else if (ctx->k2_variant == 0) {
            SW_K2_SETUP(256, 8)
        } else if (ctx->k2_variant == 1) {
            SW_K2_SETUP(512, 13)
        } else {
            SW_K2_SETUP(512, 16)
        }
#undef SW_K2_SETUP
        if (occ < 1) return fail(SPEC_ECUDA, "chord kernel cannot be resident (registers / shared memory)");
        ctx->chord_grid_max = occ * ctx->num_sms;
    } else {
        ctx->smem_path = false;
        ctx->k2_variant = 2;
        // vectors + inverse diagonal blocks in shared memory, matrices in the scratch slice
        ctx->g_smem = sizeof(double) * (vecs + 8 * (size_t)mp);
        CK(cudaFuncSetAttribute(chord_kernel2<512, false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)ctx->g_smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chord_kernel2<512, false, 16>, 512, ctx->g_smem));
        if (occ < 1) occ = 1;
        if (occ > 2) occ = 2;
        if (getenv("SPECWALK_G_CTAS")) occ = std::max(1, std::min(occ, atoi(getenv("SPECWALK_G_CTAS"))));  // A/B
        ctx->chord_grid_max = occ * ctx->num_sms;
        ctx->scratch_stride = (long long)roundup((int)(per_cta + 8 * (size_t)mp), 32);  // + inverse diagonal blocks
        ctx->scratch_ctas = ctx->chord_grid_max;
        CK(zalloc(&ctx->scratch, (size_t)ctx->scratch_stride * ctx->scratch_ctas));
        ctx->smem_bytes = 0;
        // m > 112 split, opt-in (SPECWALK_G_SPLIT=1): the fused kernel as the factor phase, Lanczos
        // on a 2-CTA cluster with M in the pair's shared memory (lanczos_cl.cuh, mp <= 2 x 104), the
        // split tail kernel.  Measured slower than the fused kernel at m = 200 (116.1k vs 123.6k
        // K2 calls/s) and m = 136 (206k vs 250k): one chain per SM pair with three cluster barriers
        // per iteration (~13k cycles) does not beat two L2-bound chains per SM, and the factor
        // phase pays the M / L round trip through HBM (profiles/r2k_m200_split)
        const LclLayout lcl(mp, ctx->ld);
        const size_t t_smem =
            sizeof(double) * ((((size_t)mp * (mp + 1) / 2 + 1) & ~(size_t)1) + 5 * (size_t)(mp + 8) + 64);
        // default for mp <= 208 (SPECWALK_G_SPLIT=0: the fused kernel, =cl: the cluster variant): the
        // same factor phase and tail around lanczos_t_kernel (M as lower 8 x 8 tiles in one CTA's
        // shared memory, lanczos_t.cuh)
        const char* gsenv = getenv("SPECWALK_G_SPLIT");
        const bool gs_off = gsenv && gsenv[0] == '0';
        const bool gs_cl = gsenv && gsenv[0] == 'c';
        const LztLayout lzt(mp);
        if (!gs_off && !gs_cl && mp <= 8 * LZT_NBMAX && sizeof(double) * (size_t)lzt.total <= 227 * 1024 &&
            t_smem <= 227 * 1024) {
            ctx->lt_smem = sizeof(double) * (size_t)lzt.total;
            ctx->t_smem = t_smem;
            CK(cudaFuncSetAttribute(lanczos_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->lt_smem));
            CK(cudaFuncSetAttribute(tail_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->t_smem));
            int ol = 0, ot = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ol, lanczos_t_kernel, LZT_NT, ctx->lt_smem));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ot, tail_kernel<256>, 256, ctx->t_smem));
            if (ol >= 1 && ot >= 1) {
                ctx->g_split = 2;
                ctx->lt_grid = ol * ctx->num_sms;
                ctx->t_grid = ot * ctx->num_sms;
                // one tail CTA per SM (L no longer fits twice, mp > 152): 512 threads (SPECWALK_T512=0: 256)
                if (ot == 1 && !(getenv("SPECWALK_T512") && getenv("SPECWALK_T512")[0] == '0')) {
                    int o5 = 0;
                    CK(cudaFuncSetAttribute(tail_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->t_smem));
                    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o5, tail_kernel<512>, 512, ctx->t_smem));
                    if (o5 >= 1) ctx->t512 = 1;
                }
                // factor phase as factor_g_kernel (factor_g.cuh; SPECWALK_G_FACTOR=0: the global-scratch
                // chord kernel, =256: 256 threads instead of 384)
                const char* fge = getenv("SPECWALK_G_FACTOR");
                const int fnt = (fge && atoi(fge) == 256) ? 256 : 384;
                const size_t fgs = sizeof(double) * fg_smem_doubles(mp, fnt / 32);
                if (!(fge && fge[0] == '0') && mp <= 8 * FG_TBMAX && fgs <= 227 * 1024 &&
                    (long long)fg_scratch_doubles(mp) <= ctx->scratch_stride) {
                    int og = 0;
                    if (fnt == 256) {
                        CK(cudaFuncSetAttribute(factor_g_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fgs));
                        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&og, factor_g_kernel<256>, 256, fgs));
                    } else {
                        CK(cudaFuncSetAttribute(factor_g_kernel<384>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fgs));
                        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&og, factor_g_kernel<384>, 384, fgs));
                    }
                    if (og >= 1) {
                        ctx->fg = fnt;
                        ctx->fg_smem = fgs;
                        ctx->fg_grid = std::min(ctx->num_sms, ctx->scratch_ctas);
                    }
                }
            }
        }
        if (!ctx->g_split && mp <= 2 * LCL_ROWS && sizeof(double) * (size_t)lcl.total <= 227 * 1024 &&
            t_smem <= 227 * 1024 && gs_cl) {
            ctx->cl_smem = sizeof(double) * (size_t)lcl.total;
            ctx->t_smem = t_smem;
            CK(cudaFuncSetAttribute(lanczos_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->cl_smem));
            CK(cudaFuncSetAttribute(tail_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->t_smem));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2 * ctx->num_sms, 1, 1);
            cfg.blockDim = dim3(LCL_NT, 1, 1);
            cfg.dynamicSmemBytes = ctx->cl_smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int ncl = 0, ot = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, lanczos_cl_kernel, &cfg) != cudaSuccess) {
                cudaGetLastError();  // no cluster occupancy: keep the fused kernel
                ncl = 0;
            }
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ot, tail_kernel<256>, 256, ctx->t_smem));
            if (ncl >= 1 && ot >= 1) {
                ctx->g_split = 1;
                ctx->cl_grid = 2 * ncl;
                ctx->t_grid = ot * ctx->num_sms;
            }
        }
    }
    // K2 split (chord3.cuh) for 64 < m <= 128 unless SPECWALK_K2_FUSED is set (for m <= 64 the
    // fused kernel was measured faster: 1.9M vs 1.4M calls/s at m = 40; it does not spill there)
    // (and only where the factor kernel's G, B and inverse diagonal blocks fit: mp <= 104;
    // 104 < mp <= 112 keeps the fused variant 3)
    const size_t f_smem = per_cta * sizeof(double) + sizeof(double) * 8 * (size_t)mp;  // + inverse diagonal blocks
    if ((ctx->k2_variant == 1 || ctx->k2_variant == 3) && f_smem <= 227 * 1024 && !getenv("SPECWALK_K2_FUSED")) {
        ctx->k2_split = 1;
        ctx->f_smem = f_smem;
        ctx->l_smem = sizeof(double) * ((size_t)mp * ctx->ld + (size_t)NVEC2 * (mp + 8) + 64);  // Q + vectors
        ctx->t_smem = sizeof(double) * ((((size_t)mp * (mp + 1) / 2 + 1) & ~(size_t)1) + 5 * (size_t)(mp + 8) + 64);
        int of = 0, ol = 0, ot = 0;
#define SW_SPLIT_SETUP(NT_, KC_)                                                                                     \
    CK(cudaFuncSetAttribute(factor_kernel<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->f_smem));     \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, factor_kernel<NT_>, NT_, ctx->f_smem));                     \
    CK(cudaFuncSetAttribute(lanczos_kernel<NT_, KC_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->l_smem)); \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ol, lanczos_kernel<NT_, KC_>, NT_, ctx->l_smem));
        if (ctx->k2_variant == 0) {
            SW_SPLIT_SETUP(256, 8)
        } else if (ctx->k2_variant == 1) {
            SW_SPLIT_SETUP(512, 13)
        } else {
            SW_SPLIT_SETUP(512, 16)
        }
#undef SW_SPLIT_SETUP
        CK(cudaFuncSetAttribute(tail_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->t_smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ot, tail_kernel<256>, 256, ctx->t_smem));
        if (of < 1 || ol < 1 || ot < 1) return fail(SPEC_ECUDA, "K2 split kernels cannot be resident");
        ctx->f_grid = of * ctx->num_sms;
        ctx->l_grid = ol * ctx->num_sms;
        ctx->t_grid = ot * ctx->num_sms;
        // K2a with both matrices as lower 8 x 8 tiles, two chains per SM (factor_t.cuh): K2a
        // 25.24 -> 20.61 ms per 65536-chain M100 round (profiles/r2ft1); SPECWALK_FACTOR_T=0 keeps
        // factor_kernel<512> (A/B)
        const char* ftenv = getenv("SPECWALK_FACTOR_T");
        if (ctx->k2_variant == 1 && mp <= 8 * FT_TBMAX && !(ftenv && ftenv[0] == '0')) {
            ctx->ft_smem = sizeof(double) * ft_smem_doubles(mp);
            int o2 = 0;
            CK(cudaFuncSetAttribute(factor_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->ft_smem));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, factor_t_kernel, FT_NT, ctx->ft_smem));
            if (o2 >= 1) {
                ctx->ft = 1;
                ctx->ft_grid = o2 * ctx->num_sms;
            }
        }
        // billiard / oracle K2b with two chains per SM (lanczos2.cuh) where M fits half an SM's
        // shared memory; SPECWALK_LZ_OLD=1 keeps the register-resident lanczos_kernel (A/B)
        if (ctx->k2_variant == 1 && !getenv("SPECWALK_LZ_OLD")) {
            const Lz2Layout lo(mp, ctx->ld);
            ctx->l2_smem = sizeof(double) * (size_t)lo.total;
            int o2 = 0;
            CK(cudaFuncSetAttribute(lanczos2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->l2_smem));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, lanczos2_kernel, LZ2_NT, ctx->l2_smem));
            if (o2 >= 1) {
                ctx->lz2 = 1;
                ctx->l2_grid = o2 * ctx->num_sms;
            }
        }
    }
    ctx->lsave_stride = (long long)mp * ctx->ld;
    CK(zalloc(&ctx->lsave, (size_t)ctx->lsave_stride * ctx->chord_grid_max));
    return SPEC_OK;
}

static void free_walk(spec_ctx* ctx);
static void free_hmc_bufs(HmcBuf& h);
extern "C" int spec_destroy(spec_ctx* ctx) {
    if (!ctx) return SPEC_OK;
    free_walk(ctx);
    cudaSetDevice(ctx->dev);
    free_chains(ctx->cb);
    free_hmc_bufs(ctx->hb);
    free_chmc_bufs(ctx->chb);
    if (ctx->obuf) {
        free_obuf(*(OracleBuf*)ctx->obuf);
        delete (OracleBuf*)ctx->obuf;
    }
    void* ps[] = {ctx->Ahat, ctx->a0, ctx->lo, ctx->hi, ctx->c, ctx->ball_c, ctx->c0, ctx->scratch, ctx->dstats, ctx->jsum, ctx->prof, ctx->lsave, ctx->Ac, ctx->hmc_scratch, ctx->pot_mu, ctx->chmc_scratch, ctx->picard};
    for (void* p : ps)
        if (p) cudaFree(p);
    if (ctx->e0) cudaEventDestroy(ctx->e0);
    if (ctx->e1) cudaEventDestroy(ctx->e1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return SPEC_OK;
}

extern "C" int spec_sync(spec_ctx* ctx) {
    CK(cudaStreamSynchronize(ctx->stream));
    return SPEC_OK;
}
extern "C" void* spec_stream(spec_ctx* ctx) { return (void*)ctx->stream; }
extern "C" int64_t spec_kernel_launches(spec_ctx* ctx) { return ctx ? ctx->launches : 0; }

static void launch_gemm_av(spec_ctx* ctx, const double* Arows, const int* list, const int* count_dev,
                           int count_host, double* out, const double* bias);
extern "C" int spec_set_objective(spec_ctx* ctx, const double* c) {
    if (!ctx || !c) return fail(SPEC_EINVAL, "null argument");
    if (walk_is_active(ctx)) return fail(SPEC_EINVAL, "a resumable walk is in progress (call walk_end first)");
    double s = 0.0;
    for (int i = 0; i < ctx->n; ++i) s += c[i] * c[i];
    if (!(s > 0.0) || !std::isfinite(s)) return fail(SPEC_EINVAL, "|c| must be finite and > 0");
    CK(cudaSetDevice(ctx->dev));
    CK(cudaMemcpyAsync(ctx->c, c, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->stream));
    // A(c) = sum_i c_i A_i (packed), the t^2 coefficient of the HMC pencil up to -1/(2T)
    launch_gemm_av(ctx, ctx->c, nullptr, nullptr, 1, ctx->Ac, nullptr);
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->has_obj = 1;
    return SPEC_OK;
}

extern "C" int spec_set_ball(spec_ctx* ctx, const double* center, double radius) {
    if (!ctx) return fail(SPEC_EINVAL, "null ctx");
    if (walk_is_active(ctx)) return fail(SPEC_EINVAL, "a resumable walk is in progress (call walk_end first)");
    CK(cudaSetDevice(ctx->dev));
    if (!(radius > 0.0)) {
        ctx->has_ball = 0;
        return SPEC_OK;
    }
    if (!center) return fail(SPEC_EINVAL, "center is NULL");
    CK(cudaMemcpyAsync(ctx->ball_c, center, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->ball_r = radius;
    ctx->has_ball = 1;
    return SPEC_OK;
}

// ---------------------------------------------------------------- kernel launch helpers
static void launch_gemm_av(spec_ctx* ctx, const double* Arows, const int* list, const int* count_dev,
                           int count_host, double* out, const double* bias) {
    dim3 grid(ctx->mtp / GB_N, (count_host + GB_M - 1) / GB_M);
    gemm_f64_dmma<false><<<grid, 128, 0, ctx->stream>>>(Arows, ctx->np, list, count_dev, count_host, ctx->Ahat,
                                                        ctx->mtp, out, ctx->mtp, bias, ctx->np);
    ctx->launches++;
}
static void launch_gemm_normal(spec_ctx* ctx, const int* list, const int* count_dev, int count_host) {
    dim3 grid(ctx->np / GB_N, (count_host + GB_M - 1) / GB_M);
    gemm_f64_dmma<true><<<grid, 128, 0, ctx->stream>>>(ctx->cb.Yh, ctx->mtp, list, count_dev, count_host,
                                                       ctx->Ahat, ctx->mtp, ctx->cb.Gn, ctx->np, nullptr, ctx->mtp);
    ctx->launches++;
}

static ChordParams chord_params(spec_ctx* ctx, int mode) {
    ChordParams P;
    memset(&P, 0, sizeof(P));
    ChainBuf& b = ctx->cb;
    P.n = ctx->n; P.np = ctx->np; P.m = ctx->m; P.mt = ctx->mt; P.mtp = ctx->mtp; P.ld = ctx->ld;
    P.mode = mode;
    P.AV = b.AV; P.AX = b.AX; P.AXs = b.AXs; P.Yh = b.Yh; P.X = b.X; P.Xs = b.Xs; P.V = b.V; P.U = b.U;
    P.ell = b.ell; P.steps_done = b.steps_done; P.refl = b.refl; P.bound = b.bound; P.flags = b.flags;
    P.calls = b.calls; P.nrefl = b.nrefl; P.nrej = b.nrej; P.ndeg = b.ndeg; P.ncap = b.ncap;
    P.lo = ctx->has_cube ? ctx->lo : nullptr;
    P.hi = ctx->has_cube ? ctx->hi : nullptr;
    P.ball_c = ctx->ball_c; P.ball_r = ctx->ball_r; P.has_ball = ctx->has_ball;
    P.scratch = ctx->scratch; P.scratch_stride = ctx->scratch_stride;
    P.nlist = b.nlist; P.ncount = b.counters + 2;
    P.prof = ctx->prof;
    P.lsave = ctx->lsave;
    P.lsave_stride = ctx->lsave_stride;
    P.Ac = ctx->Ac;
    P.cvec = ctx->c;
    P.tlast = b.tlast;
    P.jlast = b.jlast;
    P.jsum = ctx->jsum;
    P.wM = b.wM;
    P.wL = b.wL;
    P.wS = b.wS;
    P.w_mstride = (long long)roundup(ctx->m, 8) * ctx->ld;
    P.w_sstride = s_stride(roundup(ctx->m, 8));
    P.need_tmin = (mode == 1);
    P.wkind = 0;
    P.hnr_boltz = 0;
    P.gsplit = 0;
    return P;
}

static void launch_chord(spec_ctx* ctx, const ChordParams& P, int count_host, cudaEvent_t* sub = nullptr) {
    if (ctx->g_split) {
        ChordParams Pf = P;
        Pf.gsplit = ctx->g_split;
        int grid = std::max(1, std::min(count_host, ctx->chord_grid_max));
        if (ctx->g_split == 2 && ctx->fg == 384)
            factor_g_kernel<384><<<std::max(1, std::min(count_host, ctx->fg_grid)), 384, ctx->fg_smem, ctx->stream>>>(P);
        else if (ctx->g_split == 2 && ctx->fg == 256)
            factor_g_kernel<256><<<std::max(1, std::min(count_host, ctx->fg_grid)), 256, ctx->fg_smem, ctx->stream>>>(P);
        else
            chord_kernel2<512, false, 16><<<grid, 512, ctx->g_smem, ctx->stream>>>(Pf);
        if (sub) cudaEventRecord(sub[0], ctx->stream);
        // clusters: one per chain (grid rounded to whole clusters)
        if (ctx->g_split == 2) {
            lanczos_t_kernel<<<std::max(1, std::min(count_host, ctx->lt_grid)), LZT_NT, ctx->lt_smem, ctx->stream>>>(P);
        } else {
            const int cg2 = std::max(2, std::min(2 * count_host, ctx->cl_grid));
            lanczos_cl_kernel<<<cg2, LCL_NT, ctx->cl_smem, ctx->stream>>>(P);
        }
        if (sub) cudaEventRecord(sub[1], ctx->stream);
        if (ctx->t512)
            tail_kernel<512><<<std::max(1, std::min(count_host, ctx->t_grid)), 512, ctx->t_smem, ctx->stream>>>(P);
        else
            tail_kernel<256><<<std::max(1, std::min(count_host, ctx->t_grid)), 256, ctx->t_smem, ctx->stream>>>(P);
        ctx->launches += 3;
        return;
    }
    if (ctx->k2_split) {
        auto g = [&](int gmax) { return std::max(1, std::min(count_host, gmax)); };
        if (ctx->k2_variant == 0) {
            factor_kernel<256><<<g(ctx->f_grid), 256, ctx->f_smem, ctx->stream>>>(P);
            if (sub) cudaEventRecord(sub[0], ctx->stream);
            lanczos_kernel<256, 8><<<g(ctx->l_grid), 256, ctx->l_smem, ctx->stream>>>(P);
        } else if (ctx->k2_variant == 1) {
            if (ctx->ft)
                factor_t_kernel<<<g(ctx->ft_grid), FT_NT, ctx->ft_smem, ctx->stream>>>(P);
            else
                factor_kernel<512><<<g(ctx->f_grid), 512, ctx->f_smem, ctx->stream>>>(P);
            if (sub) cudaEventRecord(sub[0], ctx->stream);
            if (ctx->lz2)
                lanczos2_kernel<<<g(ctx->l2_grid), LZ2_NT, ctx->l2_smem, ctx->stream>>>(P);
            else
                lanczos_kernel<512, 13><<<g(ctx->l_grid), 512, ctx->l_smem, ctx->stream>>>(P);
        } else {
            factor_kernel<512><<<g(ctx->f_grid), 512, ctx->f_smem, ctx->stream>>>(P);
            if (sub) cudaEventRecord(sub[0], ctx->stream);
            lanczos_kernel<512, 16><<<g(ctx->l_grid), 512, ctx->l_smem, ctx->stream>>>(P);
        }
        if (sub) cudaEventRecord(sub[1], ctx->stream);
        tail_kernel<256><<<g(ctx->t_grid), 256, ctx->t_smem, ctx->stream>>>(P);
        ctx->launches += 3;
        return;
    }
    int grid = count_host < ctx->chord_grid_max ? count_host : ctx->chord_grid_max;
    if (grid < 1) grid = 1;
    if (ctx->k2_variant == 4)
        chord_kernel2<128, true, 4><<<grid, 128, ctx->smem_bytes, ctx->stream>>>(P);
    else if (ctx->k2_variant == 5)
        chord_kernel2<192, true, 6><<<grid, 192, ctx->smem_bytes, ctx->stream>>>(P);
    else if (ctx->k2_variant == 0)
        chord_kernel2<256, true, 8><<<grid, 256, ctx->smem_bytes, ctx->stream>>>(P);
    else if (ctx->k2_variant == 1)
        chord_kernel2<512, true, 13><<<grid, 512, ctx->smem_bytes, ctx->stream>>>(P);
    else if (ctx->k2_variant == 3)
        chord_kernel2<512, true, 16><<<grid, 512, ctx->smem_bytes, ctx->stream>>>(P);
    else
        chord_kernel2<512, false, 16><<<grid, 512, ctx->g_smem, ctx->stream>>>(P);
    ctx->launches++;
}

// K5 (HMC-r) resources.  G and one operand in shared memory (m <= 112): the split kernels of
// hmc2.cuh (per-slot work buffers, allocated with the chain capacity by ensure_hmc_bufs); larger m: hmc_kernel with
// 8 matrices of mp x ld per CTA in global scratch.
static int ensure_hmc(spec_ctx* ctx) {
    if (ctx->hmc_split || ctx->hmc_scratch) return SPEC_OK;
    const int mp = roundup(ctx->m, 8);
    const size_t hf_smem = sizeof(double) * ((size_t)2 * mp * ctx->ld + (size_t)8 * (mp + 8) + 8 * (size_t)mp);
    if (mp <= 128 && hf_smem <= 227 * 1024 && !getenv("SPECWALK_HMC_FUSED")) {
        const int vl = mp + 8;
        ctx->hmc_nt = (mp <= 64) ? 256 : 512;
        ctx->hmc_kc = (mp <= 64) ? 8 : (mp <= 104) ? 13 : 16;
        ctx->hf_smem = hf_smem;
        ctx->hl_smem = sizeof(double) * ((size_t)mp * ctx->ld + (size_t)NVEC2 * vl + 64);
        ctx->ht_smem = sizeof(double) * ((size_t)mp * ctx->ld + 4 * (size_t)vl);
        int of = 0, ol = 0, ot = 0, os = 0;
#define SW_HMC_SETUP(NT_, KC_)                                                                                     \
    CK(cudaFuncSetAttribute(hmc_factor_kernel<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->hf_smem)); \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, hmc_factor_kernel<NT_>, NT_, ctx->hf_smem));                \
    CK(cudaFuncSetAttribute(lanczos_kernel<NT_, KC_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->hl_smem)); \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ol, lanczos_kernel<NT_, KC_>, NT_, ctx->hl_smem));
        if (ctx->hmc_kc == 8) {
            SW_HMC_SETUP(256, 8)
        } else if (ctx->hmc_kc == 13) {
            SW_HMC_SETUP(512, 13)
        } else {
            SW_HMC_SETUP(512, 16)
        }
#undef SW_HMC_SETUP
        CK(cudaFuncSetAttribute(hmc_tail_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->ht_smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ot, hmc_tail_kernel<256>, 256, ctx->ht_smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&os, hmc_setup_kernel<256>, 256, 0));
        if (of < 1 || ol < 1 || ot < 1 || os < 1) return fail(SPEC_ECUDA, "K5 split kernels cannot be resident");
        ctx->hf_grid = of * ctx->num_sms;
        ctx->hl_grid = ol * ctx->num_sms;
        ctx->ht_grid = ot * ctx->num_sms;
        ctx->hs_grid = os * ctx->num_sms;
        ctx->hmc_split = 1;
        return SPEC_OK;
    }
    ctx->hmc_stride = (long long)8 * mp * ctx->ld;
    ctx->hmc_smem = sizeof(double) * (size_t)16 * (mp + 8);
    CK(cudaFuncSetAttribute(hmc_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->hmc_smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hmc_kernel<512>, 512, ctx->hmc_smem));
    if (occ < 1) return fail(SPEC_ECUDA, "hmc kernel cannot be resident");
    if (occ > 2) occ = 2;
    ctx->hmc_grid = occ * ctx->num_sms;
    CK(zalloc(&ctx->hmc_scratch, (size_t)ctx->hmc_stride * ctx->hmc_grid));
    return SPEC_OK;
}

static void free_hmc_bufs(HmcBuf& h) {
    void* ps[] = {h.wH, h.wQ, h.wM, h.wL, h.wS, h.il0, h.il1, h.cnt};
    for (void* p : ps)
        if (p) cudaFree(p);
    h = HmcBuf();
}

static int ensure_hmc_bufs(spec_ctx* ctx) {
    HmcBuf& h = ctx->hb;
    const long long cap = ctx->cb.cap;
    if (cap <= h.cap) return SPEC_OK;
    free_hmc_bufs(h);
    const size_t mp = (size_t)roundup(ctx->m, 8), vl = mp + 8;
    cudaError_t e = cudaSuccess;
#define ZA(ptr, cnt) \
    if (e == cudaSuccess) e = zalloc(&h.ptr, (size_t)(cnt));
    ZA(wH, cap * H_NS) ZA(wQ, cap * 3 * vl) ZA(il0, cap) ZA(il1, cap) ZA(cnt, 2)
    if (!ctx->k2_split) {
        ZA(wM, cap * mp * ctx->ld) ZA(wL, cap * mp * ctx->ld) ZA(wS, cap * (size_t)s_stride((int)mp))
    }
#undef ZA
    if (e != cudaSuccess) {
        free_hmc_bufs(h);
        cudaGetLastError();
        return fail(SPEC_ENOMEM, std::string("HMC buffers: ") + cudaGetErrorString(e));
    }
    h.cap = cap;
    return SPEC_OK;
}

// One HMC-r boundary-oracle call for every slot of the list (P.list / P.count_dev).
static int launch_hmc(spec_ctx* ctx, ChordParams P, int count_host) {
    if (!ctx->hmc_split) {
        int grid = count_host < ctx->hmc_grid ? count_host : ctx->hmc_grid;
        if (grid < 1) grid = 1;
        P.scratch = ctx->hmc_scratch;
        P.scratch_stride = ctx->hmc_stride;
        hmc_kernel<512><<<grid, 512, ctx->hmc_smem, ctx->stream>>>(P);
        ctx->launches++;
        return SPEC_OK;
    }
    int rc = ensure_hmc_bufs(ctx);
    if (rc) return rc;
    HmcBuf& h = ctx->hb;
    P.wH = h.wH;
    P.wQ = h.wQ;
    if (!ctx->k2_split) {
        P.wM = h.wM;
        P.wL = h.wL;
        P.wS = h.wS;
    }
    P.zall = 1;
    auto g = [&](int gmax) { return std::max(1, std::min(count_host, gmax)); };
    int* il[2] = {h.il0, h.il1};
    CK(cudaMemsetAsync(h.cnt, 0, 2 * sizeof(int), ctx->stream));
    ChordParams Ps = P;
    Ps.nxt_list = il[0];
    Ps.nxt_count = h.cnt;
    hmc_setup_kernel<256><<<g(ctx->hs_grid), 256, 0, ctx->stream>>>(Ps);
    ctx->launches++;
    const int wblocks = std::max(1, std::min((count_host + 255) / 256, 4096));
    for (int k = 0; k < HMC_MAX_IT; ++k) {
        ChordParams Pk = P;
        Pk.list = il[k & 1];
        Pk.count_dev = h.cnt + (k & 1);
        Pk.nxt_list = il[(k + 1) & 1];
        Pk.nxt_count = h.cnt + ((k + 1) & 1);
        CK(cudaMemsetAsync(Pk.nxt_count, 0, sizeof(int), ctx->stream));
        if (ctx->hmc_kc == 8) {
            hmc_factor_kernel<256><<<g(ctx->hf_grid), 256, ctx->hf_smem, ctx->stream>>>(Pk);
            lanczos_kernel<256, 8><<<g(ctx->hl_grid), 256, ctx->hl_smem, ctx->stream>>>(Pk);
        } else if (ctx->hmc_kc == 13) {
            hmc_factor_kernel<512><<<g(ctx->hf_grid), 512, ctx->hf_smem, ctx->stream>>>(Pk);
            // lanczos2_kernel with a full Gram-Schmidt pass every iteration for the -N_1 solves
            // (partially reorthogonalised Ritz vectors near the root missed the HMC parity bound);
            // SPECWALK_HMC_LZ_OLD=1: the register-resident kernel (A/B)
            if (ctx->lz2 && !getenv("SPECWALK_HMC_LZ_OLD"))
                lanczos2_kernel<<<g(ctx->l2_grid), LZ2_NT, ctx->l2_smem, ctx->stream>>>(Pk);
            else
                lanczos_kernel<512, 13><<<g(ctx->hl_grid), 512, ctx->hl_smem, ctx->stream>>>(Pk);
        } else {
            hmc_factor_kernel<512><<<g(ctx->hf_grid), 512, ctx->hf_smem, ctx->stream>>>(Pk);
            lanczos_kernel<512, 16><<<g(ctx->hl_grid), 512, ctx->hl_smem, ctx->stream>>>(Pk);
        }
        hmc_weyl_kernel<<<wblocks, 256, 0, ctx->stream>>>(Pk);
        ctx->launches += 3;
        if ((k & 3) == 3) {  // most chains stop after ~4 steps: look at the list every 4 iterations
            int left = 0;
            CK(cudaMemcpyAsync(&left, Pk.nxt_count, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            if (left == 0) break;
        }
    }
    hmc_tail_kernel<256><<<g(ctx->ht_grid), 256, ctx->ht_smem, ctx->stream>>>(P);
    ctx->launches++;
    return SPEC_OK;
}

// ---------------------------------------------------------------- K7: collocation HMC-r
extern "C" int spec_set_potential(spec_ctx* ctx, int pot, const double* mu, double scale) {
    if (!ctx) return fail(SPEC_EINVAL, "null ctx");
    SW_NOT_DURING_WALK(ctx);
    if (pot != SPEC_POT_LINEAR && pot != SPEC_POT_GAUSS && pot != SPEC_POT_LOGCOSH)
        return fail(SPEC_EINVAL, "unknown potential");
    if (!(scale > 0.0) || !std::isfinite(scale)) return fail(SPEC_EINVAL, "scale must be finite and > 0");
    if (pot == SPEC_POT_LINEAR && !ctx->has_obj) return fail(SPEC_EINVAL, "SPEC_POT_LINEAR needs spec_set_objective");
    CK(cudaSetDevice(ctx->dev));
    if (!ctx->pot_mu) CK(zalloc(&ctx->pot_mu, ctx->n));
    if (mu) {
        for (int i = 0; i < ctx->n; ++i)
            if (!std::isfinite(mu[i])) return fail(SPEC_EINVAL, "mu has NaN/Inf");
        CK(cudaMemcpyAsync(ctx->pot_mu, mu, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->stream));
    } else {
        CK(cudaMemsetAsync(ctx->pot_mu, 0, sizeof(double) * ctx->n, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->pot = pot;
    ctx->pot_scale = scale;
    return SPEC_OK;
}

// Chebyshev nodes of [0, 1] and the monomial coefficients of the Lagrange basis, by expanding
// l_j(s) = prod_{i != j} (s - s_i) / (s_j - s_i) (R33)
static void chmc_basis(int q, double* nodes, double* lcoef) {
    const double pi = 3.14159265358979323846;
    for (int j = 0; j < q; ++j) nodes[j] = 0.5 * (1.0 - std::cos((2.0 * j + 1.0) * pi / (2.0 * q)));
    for (int j = 0; j < q; ++j) {
        double poly[CH_MAXQ + 1] = {1.0};
        int deg = 0;
        for (int i = 0; i < q; ++i) {
            if (i == j) continue;
            const double den = nodes[j] - nodes[i];
            double nxt[CH_MAXQ + 1] = {0.0};
            for (int k = 0; k <= deg; ++k) {
                nxt[k + 1] += poly[k] / den;
                nxt[k] -= poly[k] * nodes[i] / den;
            }
            ++deg;
            for (int k = 0; k <= deg; ++k) poly[k] = nxt[k];
        }
        for (int k = 0; k < q; ++k) lcoef[j * q + k] = poly[k];
    }
}

static int check_chmc(spec_ctx* ctx, int q, double h) {
    if (ctx->pot < 0) return fail(SPEC_EINVAL, "collocation HMC needs spec_set_potential");
    if (q < 1 || q > CH_MAXQ) return fail(SPEC_EINVAL, "collocation nodes q must be in 1..6");
    if (!(h > 0.0) || !std::isfinite(h)) return fail(SPEC_EINVAL, "collocation step h must be finite and > 0");
    if (ctx->has_ball) return fail(SPEC_EINVAL, "collocation HMC with a ball constraint is not supported");
    return SPEC_OK;
}

// per-CTA scratch for the degree d and per-slot buffers for C chains
static int ensure_chmc(spec_ctx* ctx, int q, long long C) {
    const int d = q + 1;
    const int mp = roundup(ctx->m, 8);
    if (d > ctx->chmc_d) {
        if (ctx->chmc_scratch) cudaFree(ctx->chmc_scratch);
        ctx->chmc_scratch = nullptr;
        ctx->chmc_smem = sizeof(double) * (size_t)(16 + CH_MAXD + 1) * (mp + 8);
        // m <= 64: 256 threads and two chains per SM (the per-chain latency chain is short of work
        // for 16 warps); larger m: 512 threads, one chain per SM
        ctx->chmc_nt = (mp <= 128 && !getenv("SPECWALK_CHMC_512")) ? 256 : 512;
        int occ = 0;
        if (ctx->chmc_nt == 256) {
            CK(cudaFuncSetAttribute(chmc_chord_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ctx->chmc_smem));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chmc_chord_kernel<256>, 256, ctx->chmc_smem));
        } else {
            CK(cudaFuncSetAttribute(chmc_chord_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ctx->chmc_smem));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chmc_chord_kernel<512>, 512, ctx->chmc_smem));
        }
        if (occ < 1) return fail(SPEC_ECUDA, "collocation chord kernel cannot be resident");
        ctx->chmc_grid = occ * ctx->num_sms;
        ctx->chmc_stride = (long long)chmc_nmat(d) * mp * ctx->ld;
        cudaError_t e = zalloc(&ctx->chmc_scratch, (size_t)ctx->chmc_stride * ctx->chmc_grid);
        if (e != cudaSuccess) {
            cudaGetLastError();
            ctx->chmc_scratch = nullptr;
            return fail(SPEC_ENOMEM, std::string("collocation scratch: ") + cudaGetErrorString(e));
        }
        ctx->chmc_d = d;
    }
    if (!ctx->picard) CK(zalloc(&ctx->picard, 4));
    ChmcBuf& b = ctx->chb;
    if (C <= b.cap && d <= b.d) return SPEC_OK;
    free_chmc_bufs(b);
    const long long cap = std::max(C, ctx->cb.cap);
    const int dd = std::max(d, ctx->chmc_d);
    cudaError_t e = cudaSuccess;
#define ZA(ptr, cnt) \
    if (e == cudaSuccess) e = zalloc(&b.ptr, (size_t)(cnt));
    ZA(CF, cap * dd * ctx->np) ZA(CB, cap * dd * ctx->mtp) ZA(GW, cap * (dd - 1) * ctx->np) ZA(hseg, cap)
    ZA(elist, cap * dd)
#undef ZA
    if (e != cudaSuccess) {
        free_chmc_bufs(b);
        cudaGetLastError();
        return fail(SPEC_ENOMEM, std::string("collocation buffers: ") + cudaGetErrorString(e));
    }
    b.cap = cap;
    b.d = dd;
    return SPEC_OK;
}

static ChmcParams chmc_params(spec_ctx* ctx, int q, double h) {
    ChmcParams H;
    memset(&H, 0, sizeof(H));
    H.CF = ctx->chb.CF; H.CB = ctx->chb.CB; H.GW = ctx->chb.GW; H.hseg = ctx->chb.hseg; H.elist = ctx->chb.elist;
    H.q = q;
    H.d = q + 1;
    H.h = h;
    H.pot = ctx->pot;
    H.mu = ctx->pot_mu;
    H.scale = ctx->pot_scale;
    H.cvec = ctx->c;
    chmc_basis(q, H.nodes, H.lcoef);
    H.picard = ctx->picard;
    return H;
}

// One collocation-HMC boundary-oracle call (one segment) for every slot of the list:
// K7a (polynomial), the B_k = A(c_k) contraction over d rows per chain, K7b (chord + advance).
static int launch_chmc(spec_ctx* ctx, ChordParams P, const ChmcParams& H, int count_host) {
    const int wblocks = std::min((count_host + 7) / 8, 65535 * 4);
    chmc_poly_kernel<<<std::max(wblocks, 1), 256, 0, ctx->stream>>>(P, H);
    launch_gemm_av(ctx, H.CF, H.elist, nullptr, count_host * H.d, H.CB, nullptr);
    P.scratch = ctx->chmc_scratch;
    P.scratch_stride = ctx->chmc_stride;
    const int grid = std::min(count_host, ctx->chmc_grid);
    if (ctx->chmc_nt == 256)
        chmc_chord_kernel<256><<<std::max(grid, 1), 256, ctx->chmc_smem, ctx->stream>>>(P, H);
    else
        chmc_chord_kernel<512><<<std::max(grid, 1), 512, ctx->chmc_smem, ctx->stream>>>(P, H);
    ctx->launches += 2;
    CK(cudaGetLastError());
    return SPEC_OK;
}

static NormalParams normal_params(spec_ctx* ctx, int mode) {
    NormalParams Q;
    memset(&Q, 0, sizeof(Q));
    ChainBuf& b = ctx->cb;
    Q.n = ctx->n; Q.np = ctx->np; Q.m = ctx->m; Q.mt = ctx->mt; Q.mtp = ctx->mtp; Q.mode = mode;
    Q.Gn = b.Gn; Q.V = b.V; Q.X = b.X; Q.Xs = b.Xs; Q.AX = b.AX; Q.AXs = b.AXs; Q.ell = b.ell;
    Q.steps_done = b.steps_done; Q.refl = b.refl; Q.bound = b.bound; Q.flags = b.flags; Q.ndeg = b.ndeg;
    Q.amax = ctx->amax;
    Q.cvec = ctx->c;
    Q.tlast = b.tlast;
    Q.ball_c = ctx->ball_c; Q.ball_r = ctx->ball_r;
    return Q;
}

// ---------------------------------------------------------------- boundary_oracle
// Device staging of one boundary_oracle / hmc_oracle batch: grown with the batch and kept in the
// context (no cudaMalloc / cudaFree per call); freed by spec_destroy.
static int ensure_obuf(spec_ctx* ctx, long long B) {
    OracleBuf& o = *(OracleBuf*)ctx->obuf;
    if (B <= o.cap) return SPEC_OK;
    free_obuf(o);
    const size_t n = ctx->n, m = ctx->m;
    cudaError_t e = cudaSuccess;
#define ZA(ptr, cnt) \
    if (e == cudaSuccess) e = zalloc(&o.ptr, (size_t)(cnt));
    ZA(x, B * n) ZA(v, B * n) ZA(u, B * m) ZA(tm, B) ZA(tp, B) ZA(nrm, B * n) ZA(ker, B * m) ZA(bind, B) ZA(stat, B)
#undef ZA
    if (e != cudaSuccess) {
        free_obuf(o);
        cudaGetLastError();
        return fail(SPEC_ENOMEM, std::string("oracle buffers: ") + cudaGetErrorString(e));
    }
    o.cap = B;
    return SPEC_OK;
}

static int oracle_impl(spec_ctx* ctx, int64_t batch, const double* dx, const double* dv, const double* du,
                       double* t_minus, double* t_plus, double* normal, double* kernel, int32_t* binding,
                       bool host_out, int* status_out, int* capped_out, double hmcT = 0.0,
                       const ChmcParams* chmc = nullptr, int* outward_out = nullptr) {
    ChainBuf& b = ctx->cb;
    OracleBuf& o = *(OracleBuf*)ctx->obuf;
    const int B = (int)batch;
    const int n = ctx->n, np = ctx->np, m = ctx->m;
    // pad x, v into the chain layout
    int thr = 256, blocks = (int)std::min<long long>(((long long)B * np + thr - 1) / thr, 65535);
    pad_rows_kernel<<<blocks, thr, 0, ctx->stream>>>(dx, n, B, n, b.X, np);
    pad_rows_kernel<<<blocks, thr, 0, ctx->stream>>>(dv, n, B, n, b.V, np);
    ctx->launches += 2;
    std::vector<int> bound_h(B, du ? 0 : SW_BIND_NONE_DEV);
    CK(cudaMemcpyAsync(b.bound, bound_h.data(), sizeof(int) * B, cudaMemcpyHostToDevice, ctx->stream));
    if (du) CK(cudaMemcpyAsync(b.U, du, sizeof(double) * (size_t)B * m, cudaMemcpyDeviceToDevice, ctx->stream));
    // A(x) = a0 + X Ahat ; A(v) = V Ahat  (K0, K1)
    launch_gemm_av(ctx, b.X, nullptr, nullptr, B, b.AX, ctx->a0);
    if (!chmc) launch_gemm_av(ctx, b.V, nullptr, nullptr, B, b.AV, nullptr);
    // K2 in oracle mode
    ChordParams P = chord_params(ctx, 1);
    P.count_host = B;
    P.o_tminus = o.tm; P.o_tplus = o.tp; P.o_kernel = kernel ? o.ker : nullptr; P.o_binding = o.bind;
    P.o_status = o.stat;
    if (chmc) {
        int rc = launch_chmc(ctx, P, *chmc, B);
        if (rc) return rc;
    } else if (hmcT > 0.0) {
        P.Temp = hmcT;
        int rc = launch_hmc(ctx, P, B);
        if (rc) return rc;
    } else {
        launch_chord(ctx, P, B);
    }
    // K3 normal contraction for every line (non-dense rows are ignored by K4)
    launch_gemm_normal(ctx, nullptr, nullptr, B);
    NormalParams Q = normal_params(ctx, 1);
    Q.count_host = B;
    Q.o_binding = o.bind; Q.o_tplus = o.tp; Q.Vin = b.V; Q.o_normal = o.nrm;
    normal_reflect_kernel<<<(B + 7) / 8, 256, 0, ctx->stream>>>(Q);
    ctx->launches++;
    CK(cudaGetLastError());
    cudaMemcpyKind kind = host_out ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    CK(cudaMemcpyAsync(t_minus, o.tm, sizeof(double) * B, kind, ctx->stream));
    CK(cudaMemcpyAsync(t_plus, o.tp, sizeof(double) * B, kind, ctx->stream));
    CK(cudaMemcpyAsync(normal, o.nrm, sizeof(double) * (size_t)B * n, kind, ctx->stream));
    if (kernel) CK(cudaMemcpyAsync(kernel, o.ker, sizeof(double) * (size_t)B * m, kind, ctx->stream));
    CK(cudaMemcpyAsync(binding, o.bind, sizeof(int) * B, kind, ctx->stream));
    std::vector<int> st(B);
    CK(cudaMemcpyAsync(st.data(), o.stat, sizeof(int) * B, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    int worst = 0;
    int ncapped = 0, nout = 0;
    for (int i = 0; i < B; ++i) {
        worst = std::max(worst, st[i] == 2 ? 2 : 0);
        ncapped += st[i] == 3;
        nout += st[i] == 4;
    }
    if (status_out) *status_out = worst;
    if (capped_out) *capped_out = ncapped;
    if (outward_out) *outward_out = nout;
    return SPEC_OK;
}

static int oracle_entry(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u,
                        double* t_minus, double* t_plus, double* normal, double* kernel, int32_t* binding,
                        bool host, double hmcT = 0.0, int chmc_q = 0, double chmc_h = 0.0) {
    if (!ctx) return fail(SPEC_EINVAL, "null ctx");
    if (walk_is_active(ctx)) return fail(SPEC_EINVAL, "a resumable walk is in progress (call walk_end first)");
    if (batch < 0 || batch > (1LL << 30)) return fail(SPEC_EINVAL, "bad batch");
    if (batch == 0) return SPEC_OK;
    if (!x || !v || !t_minus || !t_plus || !normal || !binding) return fail(SPEC_EINVAL, "null buffer");
    if (hmcT > 0.0 && !ctx->has_obj) return fail(SPEC_EINVAL, "hmc_oracle needs spec_set_objective");
    CK(cudaSetDevice(ctx->dev));
    int rc = ensure_chains(ctx, batch);
    if (rc) return rc;
    rc = ensure_obuf(ctx, batch);
    if (rc) return rc;
    if (hmcT > 0.0) {
        rc = ensure_hmc(ctx);
        if (rc) return rc;
    }
    ChmcParams H;
    if (chmc_q > 0) {
        rc = check_chmc(ctx, chmc_q, chmc_h);
        if (rc) return rc;
        rc = ensure_chmc(ctx, chmc_q, batch);
        if (rc) return rc;
        H = chmc_params(ctx, chmc_q, chmc_h);
    }
    OracleBuf& o = *(OracleBuf*)ctx->obuf;
    const int n = ctx->n, m = ctx->m;
    const double *dx = x, *dv = v, *du = u;
    if (host) {
        CK(cudaMemcpyAsync(o.x, x, sizeof(double) * batch * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(o.v, v, sizeof(double) * batch * n, cudaMemcpyHostToDevice, ctx->stream));
        if (u) CK(cudaMemcpyAsync(o.u, u, sizeof(double) * batch * m, cudaMemcpyHostToDevice, ctx->stream));
        dx = o.x; dv = o.v; du = u ? o.u : nullptr;
    }
    int status = 0, capped = 0, outward = 0;
    rc = oracle_impl(ctx, batch, dx, dv, du, t_minus, t_plus, normal, kernel, binding, host, &status, &capped, hmcT,
                     chmc_q > 0 ? &H : nullptr, &outward);
    if (rc) return rc;
    if (status == 2) return fail(SPEC_EPRECOND, "some x is not interior (Cholesky of F(x) failed)");
    if (capped) g_err = std::to_string(capped) + " line(s): Weyl iteration cap reached (t_plus = NaN)";
    if (outward) g_err = std::to_string(outward) + " line(s): boundary start moving outward (t_plus = 0)";
    return SPEC_OK;
}

extern "C" int boundary_oracle(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u,
                               double* t_minus, double* t_plus, double* normal, double* kernel, int32_t* binding) {
    return oracle_entry(ctx, batch, x, v, u, t_minus, t_plus, normal, kernel, binding, true);
}
extern "C" int hmc_oracle(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u,
                          double T, double* t_plus, double* normal, double* kernel, int32_t* binding) {
    if (!(T > 0.0)) return fail(SPEC_EINVAL, "T must be > 0");
    std::vector<double> tm((size_t)(batch > 0 ? batch : 1));
    return oracle_entry(ctx, batch, x, v, u, tm.data(), t_plus, normal, kernel, binding, true, T);
}
// Collocation HMC-r device counters since the last reset: Picard iterations, segments, segments
// whose Picard iteration did not converge, congruences of the Weyl iterations.
extern "C" int spec_chmc_counters(spec_ctx* ctx, int reset, int64_t* out4) {
    if (!ctx || !out4) return fail(SPEC_EINVAL, "null argument");
    CK(cudaSetDevice(ctx->dev));
    if (!ctx->picard) {
        for (int i = 0; i < 4; ++i) out4[i] = 0;
        return SPEC_OK;
    }
    unsigned long long h[4];
    CK(cudaMemcpyAsync(h, ctx->picard, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 4; ++i) out4[i] = (int64_t)h[i];
    if (reset) CK(cudaMemsetAsync(ctx->picard, 0, sizeof(h), ctx->stream));
    return SPEC_OK;
}
extern "C" int chmc_oracle(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u, int q,
                           double h, double* t_plus, double* normal, double* kernel, int32_t* binding) {
    if (q < 1) return fail(SPEC_EINVAL, "collocation nodes q must be in 1..6");
    std::vector<double> tm((size_t)(batch > 0 ? batch : 1));
    return oracle_entry(ctx, batch, x, v, u, tm.data(), t_plus, normal, kernel, binding, true, 0.0, q, h);
}
extern "C" int boundary_oracle_dev(spec_ctx* ctx, int64_t batch, const double* x, const double* v,
                                   const double* u, double* t_minus, double* t_plus, double* normal,
                                   double* kernel, int32_t* binding) {
    return oracle_entry(ctx, batch, x, v, u, t_minus, t_plus, normal, kernel, binding, false);
}

// ---------------------------------------------------------------- walks
struct TraceBufs {
    int max_trace = 0;
    int* cnt = nullptr;
    double *hit = nullptr, *t = nullptr, *w = nullptr, *v = nullptr;
    int* bind = nullptr;
};

// Walk state kept in the context between walk_begin / walk_rounds / walk_end.
struct WalkRun {
    bool active = false;
    spec_walk_params p;
    ChordParams P;
    NormalParams Q;
    int count = 0;  // upper bound of active chains (exact after each compaction)
    int cur = 0;
    long long rounds = 0;
    double ms = 0.0;
    bool timing = false;        // per-kernel CUDA-event timing
    double kms[4] = {0, 0, 0, 0};  // K1, K2, K3, K4
    double k2ms[3] = {0, 0, 0};    // K2 split phases: factor, Lanczos, tail
    long long kcount[4] = {0, 0, 0, 0};
    long long k2_items = 0;        // chain-calls processed by K2 launches (upper bound incl. done)
    ChmcParams H;                  // collocation HMC-r (kind SPEC_WALK_CHMC)
};
static WalkRun& walk_run(spec_ctx* ctx);

// Set up a walk: reset per-chain state, x_0, A(x_0) (K0) and the step-0 draws.
static int walk_setup(spec_ctx* ctx, const spec_walk_params* p, const double* dx0, int x0_per_chain,
                      const long long* dgid, TraceBufs* tr) {
    ChainBuf& b = ctx->cb;
    WalkRun& W = walk_run(ctx);
    const int C = (int)p->chains;
    const int n = ctx->n, np = ctx->np;
    CK(cudaMemsetAsync(b.steps_done, 0, sizeof(int) * C, ctx->stream));
    CK(cudaMemsetAsync(b.refl, 0, sizeof(int) * C, ctx->stream));
    CK(cudaMemsetAsync(b.flags, 0, sizeof(int) * C, ctx->stream));
    CK(cudaMemsetAsync(b.nrej, 0, sizeof(int) * C, ctx->stream));
    CK(cudaMemsetAsync(b.ndeg, 0, sizeof(int) * C, ctx->stream));
    CK(cudaMemsetAsync(b.ncap, 0, sizeof(int) * C, ctx->stream));
    CK(cudaMemsetAsync(b.calls, 0, sizeof(long long) * C, ctx->stream));
    CK(cudaMemsetAsync(b.nrefl, 0, sizeof(long long) * C, ctx->stream));
    CK(cudaMemsetAsync(b.jlast, 0, sizeof(int) * C, ctx->stream));
    {
        std::vector<int> bnd(C, SW_BIND_NONE_DEV);
        CK(cudaMemcpyAsync(b.bound, bnd.data(), sizeof(int) * C, cudaMemcpyHostToDevice, ctx->stream));
    }
    int thr = 256;
    int blocks = (int)std::min<long long>(((long long)C * np + thr - 1) / thr, 65535);
    if (dx0) {
        pad_rows_kernel<<<blocks, thr, 0, ctx->stream>>>(dx0, x0_per_chain ? n : 0, C, n, b.X, np);
        ctx->launches++;
    } else {
        CK(cudaMemsetAsync(b.X, 0, sizeof(double) * (size_t)C * np, ctx->stream));
    }
    iota_kernel<<<(C + 255) / 256, 256, 0, ctx->stream>>>(b.list, C);
    ctx->launches++;
    launch_gemm_av(ctx, b.X, nullptr, nullptr, C, b.AX, ctx->a0);  // K0: A(x_0)
    walk_start_kernel<<<(C + 7) / 8, 256, 0, ctx->stream>>>(C, n, np, ctx->mt, ctx->mtp, b.V, b.X, b.Xs, b.AX,
                                                            b.AXs, b.ell, p->L, p->seed, p->tag, p->kind,
                                                            p->chain_begin, dgid);
    ctx->launches++;
    if (p->kind == SPEC_WALK_CHMC) {
        int rc = ensure_chmc(ctx, p->q, C);
        if (rc) return rc;
        W.H = chmc_params(ctx, p->q, p->h);
    }
    W.p = *p;
    W.count = C;
    W.cur = 0;
    W.rounds = 0;
    W.ms = 0.0;
    for (int i = 0; i < 4; ++i) W.kms[i] = 0.0, W.kcount[i] = 0;
    for (int i = 0; i < 3; ++i) W.k2ms[i] = 0.0;
    W.k2_items = 0;
    CK(cudaMemcpyAsync(b.counters, &W.count, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    ChordParams& P = W.P;
    P = chord_params(ctx, 0);
    P.steps_total = (int)p->steps;
    P.Lpar = p->L;
    P.rho = p->rho;
    P.seed = p->seed;
    P.tag = p->tag;
    P.chain_base = p->chain_begin;
    P.gid = dgid;
    P.Temp = p->T;
    P.wkind = p->kind;
    P.need_tmin = (p->kind == SPEC_WALK_HNR || p->kind == SPEC_WALK_CHNR) ? 1 : 0;
    P.hnr_boltz = (P.need_tmin && p->T > 0.0 && std::isfinite(p->T)) ? 1 : 0;
    NormalParams& Q = W.Q;
    Q = normal_params(ctx, 0);
    Q.steps_total = (int)p->steps;
    Q.Lpar = p->L;
    Q.seed = p->seed;
    Q.tag = p->tag;
    Q.chain_base = p->chain_begin;
    Q.gid = dgid;
    Q.kind = p->kind;
    Q.Tinv = (p->kind == SPEC_WALK_HMC) ? 1.0 / p->T : 0.0;
    if (tr) {
        P.max_trace = tr->max_trace; P.tr_cnt = tr->cnt; P.tr_hit = tr->hit; P.tr_t = tr->t; P.tr_w = tr->w;
        P.tr_v = tr->v; P.tr_bind = tr->bind;
        Q.max_trace = tr->max_trace; Q.tr_cnt = tr->cnt; Q.tr_w = tr->w; Q.tr_v = tr->v;
    }
    W.active = true;
    return SPEC_OK;
}

// Run up to max_rounds scheduler rounds (max_rounds <= 0: until every chain is
// done).  Every round each active chain makes exactly one boundary-oracle call
// (K1 -> K2 -> K3 -> K4); finished chains are compacted out every 8 rounds.
static int walk_do_rounds(spec_ctx* ctx, long long max_rounds) {
    ChainBuf& b = ctx->cb;
    WalkRun& W = walk_run(ctx);
    ChordParams& P = W.P;
    NormalParams& Q = W.Q;
    int* lists[2] = {b.list, b.list2};
    const int check = 8;
    long long done_rounds = 0;
    // per-kernel event pool: 7 events per round (K1 | K2a | K2b | K2c | K3 | K4), read back at each sync
    const int pool = 7 * check;
    std::vector<cudaEvent_t> ev;
    if (W.timing) {
        ev.resize(pool);
        for (int i = 0; i < pool; ++i) CK(cudaEventCreate(&ev[i]));
    }
    CK(cudaEventRecord(ctx->e0, ctx->stream));
    while (W.count > 0 && (max_rounds <= 0 || done_rounds < max_rounds)) {
        int kr = 0;
        for (int k = 0; k < check && W.count > 0 && (max_rounds <= 0 || done_rounds < max_rounds); ++k) {
            int* list = lists[W.cur];
            const int count = W.count;
            cudaEvent_t* e = W.timing ? &ev[7 * k] : nullptr;
            CK(cudaMemsetAsync(b.counters + 2, 0, sizeof(int), ctx->stream));
            if (e) CK(cudaEventRecord(e[0], ctx->stream));
            if (W.p.kind == SPEC_WALK_CHMC) {
                // no K1: the direction is part of the segment polynomial (K7a + its contraction)
            } else if (W.p.kind == SPEC_WALK_CHNR) {  // A(e_j) = A_j: a row copy
                coord_dir_kernel<<<std::min(count, ctx->num_sms * 8), 256, 0, ctx->stream>>>(
                    list, b.counters, count, b.V, ctx->np, ctx->n, ctx->Ahat, ctx->mtp, b.AV);
                ctx->launches++;
            } else {
                launch_gemm_av(ctx, b.V, list, b.counters, count, b.AV, nullptr);  // K1
            }
            if (e) CK(cudaEventRecord(e[1], ctx->stream));
            P.list = list;
            P.count_dev = b.counters;
            P.count_host = count;
            if (W.p.kind == SPEC_WALK_HMC) {  // K5
                int rc = launch_hmc(ctx, P, count);
                if (rc) return rc;
            } else if (W.p.kind == SPEC_WALK_CHMC) {  // K7
                int rc = launch_chmc(ctx, P, W.H, count);
                if (rc) return rc;
            } else launch_chord(ctx, P, count, (e && (ctx->k2_split || ctx->g_split)) ? &e[5] : nullptr);  // K2
            if (e) CK(cudaEventRecord(e[2], ctx->stream));
            if (W.p.kind == SPEC_WALK_BILLIARD || W.p.kind == SPEC_WALK_HMC || W.p.kind == SPEC_WALK_CHMC) {
                // (Hit-and-Run never reflects)
                launch_gemm_normal(ctx, b.nlist, b.counters + 2, count);  // K3
                if (e) CK(cudaEventRecord(e[3], ctx->stream));
                Q.nlist = b.nlist;
                Q.ncount = b.counters + 2;
                Q.count_host = count;
                int nb = (count + 7) / 8;
                if (nb > 65535 * 4) nb = 65535 * 4;
                normal_reflect_kernel<<<nb, 256, 0, ctx->stream>>>(Q);  // K4
                ctx->launches++;
            } else if (e) {
                CK(cudaEventRecord(e[3], ctx->stream));
            }
            if (e) CK(cudaEventRecord(e[4], ctx->stream));
            W.k2_items += count;
            ++W.rounds;
            ++done_rounds;
            ++kr;
        }
        CK(cudaMemsetAsync(b.counters + 1, 0, sizeof(int), ctx->stream));
        compact_kernel<<<std::min((W.count + 255) / 256, 4096), 256, 0, ctx->stream>>>(
            lists[W.cur], b.counters, W.count, b.flags, lists[W.cur ^ 1], b.counters + 1);
        ctx->launches++;
        CK(cudaMemcpyAsync(b.counters, b.counters + 1, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(&W.count, b.counters + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaGetLastError());
        if (W.timing) {
            for (int k = 0; k < kr; ++k) {
                for (int i = 0; i < 4; ++i) {
                    float t = 0.f;
                    CK(cudaEventElapsedTime(&t, ev[7 * k + i], ev[7 * k + i + 1]));
                    W.kms[i] += t;
                    W.kcount[i] += 1;
                }
                if ((ctx->k2_split || ctx->g_split) && W.p.kind != SPEC_WALK_HMC && W.p.kind != SPEC_WALK_CHMC) {
                    float t0 = 0.f, t1 = 0.f, t2 = 0.f;
                    CK(cudaEventElapsedTime(&t0, ev[7 * k + 1], ev[7 * k + 5]));
                    CK(cudaEventElapsedTime(&t1, ev[7 * k + 5], ev[7 * k + 6]));
                    CK(cudaEventElapsedTime(&t2, ev[7 * k + 6], ev[7 * k + 2]));
                    W.k2ms[0] += t0;
                    W.k2ms[1] += t1;
                    W.k2ms[2] += t2;
                }
            }
        }
        W.cur ^= 1;
    }
    CK(cudaEventRecord(ctx->e1, ctx->stream));
    CK(cudaEventSynchronize(ctx->e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->e0, ctx->e1));
    W.ms += ms;
    for (cudaEvent_t x : ev) cudaEventDestroy(x);
    return SPEC_OK;
}

static int walk_collect_stats(spec_ctx* ctx, spec_walk_stats* st) {
    ChainBuf& b = ctx->cb;
    WalkRun& W = walk_run(ctx);
    const int C = (int)W.p.chains;
    CK(cudaMemsetAsync(ctx->dstats, 0, sizeof(long long) * 8, ctx->stream));
    stats_kernel<<<std::min((C + 255) / 256, 1024), 256, 0, ctx->stream>>>(C, b.calls, b.nrefl, b.nrej, b.ndeg,
                                                                           b.ncap, b.flags, b.steps_done, ctx->dstats);
    ctx->launches++;
    long long hs[8];
    CK(cudaMemcpyAsync(hs, ctx->dstats, sizeof(long long) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (st) {
        st->calls = hs[0];
        st->reflections = hs[1];
        st->rejects = hs[2];
        st->degenerates = hs[3];
        st->failures = hs[4];
        st->steps = hs[5];
        st->capped = hs[6];
        st->rounds = W.rounds;
        st->device_ms = W.ms;
    }
    if (ctx->prof) {
        unsigned long long ph[32];
        CK(cudaMemcpy(ph, ctx->prof, sizeof(ph), cudaMemcpyDeviceToHost));
        CK(cudaMemset(ctx->prof, 0, sizeof(ph)));
        CK(cudaStreamSynchronize(0));
        const char* names[] = {"unpack", "deflate", "cholesky", "congruence", "eigen", "extreme", "eigvec",
                               "backtransform+y", "select+advance"};
        double tot = 0;
        for (int i = 0; i < 9; ++i) tot += (double)ph[i];
        fprintf(stderr, "[specwalk prof] m=%d calls=%lld cycles/call:", ctx->m, (long long)hs[0]);
        for (int i = 0; i < 9; ++i) fprintf(stderr, " %s=%.0f", names[i], (double)ph[i] / (double)hs[0]);
        fprintf(stderr, " total=%.0f | lanczos: J/call=%.1f check_cycles/call=%.0f checks/call=%.2f\n",
                tot / (double)hs[0], (double)ph[10] / (double)hs[0], (double)ph[9] / (double)hs[0],
                (double)ph[11] / (double)hs[0]);
        fprintf(stderr, "[specwalk prof] lanczos_reg per iteration: matvec=%.0f dots=%.0f update=%.0f | check/call=%.0f\n",
                (double)ph[12] / fmax((double)ph[10], 1.0), (double)ph[13] / fmax((double)ph[10], 1.0),
                (double)ph[14] / fmax((double)ph[10], 1.0), (double)ph[9] / (double)hs[0]);
        if (ph[20] + ph[24] > 0)
            fprintf(stderr, "[specwalk prof] checks/call: first=%.2f later=%.2f | laguerre its: first=%.2f later=%.2f | "
                            "cycles: laguerre first=%.0f later=%.0f back=%.0f bounds=%.0f (per check)\n",
                    (double)ph[20] / hs[0], (double)ph[24] / hs[0], (double)ph[21] / fmax(1.0, (double)ph[20]),
                    (double)ph[25] / fmax(1.0, (double)ph[24]), (double)ph[22] / fmax(1.0, (double)ph[20]),
                    (double)ph[26] / fmax(1.0, (double)ph[24]), (double)ph[23] / fmax(1.0, (double)(ph[20] + ph[24])),
                    (double)ph[27] / fmax(1.0, (double)(ph[20] + ph[24])));
        if (ph[29] > 0)
            fprintf(stderr, "[specwalk prof] PRO: fully orthogonalised iterations/call=%.2f of %.2f\n",
                    (double)ph[29] / hs[0], (double)ph[10] / hs[0]);
        if (ph[18] > 0)
            fprintf(stderr, "[specwalk prof] async lanczos: iterations run/call=%.2f (J used %.2f) checks/call=%.2f "
                            "check cycles=%.0f\n", (double)ph[18] / hs[0], (double)ph[10] / hs[0],
                    (double)ph[28] / hs[0], (double)ph[19] / fmax(1.0, (double)ph[28]));
        if (ph[17] > 0)
            fprintf(stderr, "[specwalk prof] hmc: Weyl iterations/call=%.2f\n", (double)ph[17] / (double)hs[0]);
        double it = (double)ph[10];
        fprintf(stderr, "[specwalk prof] per lanczos iteration: matvec=%.0f dots=%.0f axpy+norm(+pass2)=%.0f qwrite=%.0f pass2_frac=%.3f\n",
                ph[12] / it, ph[13] / it, ph[14] / it, ph[16] / it, ph[15] / it);
    }
    return SPEC_OK;
}

static int run_walk(spec_ctx* ctx, const spec_walk_params* p, const double* dx0, int x0_per_chain,
                    const long long* dgid, TraceBufs* tr, spec_walk_stats* st) {
    int rc = walk_setup(ctx, p, dx0, x0_per_chain, dgid, tr);
    if (!rc) rc = walk_do_rounds(ctx, 0);
    if (!rc) rc = walk_collect_stats(ctx, st);
    walk_run(ctx).active = false;  // also on failure: the context stays usable
    return rc;
}

static int gather_f64(spec_ctx* ctx, int rc_local, const std::vector<double>& local, std::vector<double>& global);
static int check_walk_params(spec_ctx* ctx, const spec_walk_params* p) {
    if (!ctx || !p) return fail(SPEC_EINVAL, "null argument");
    if (p->kind != SPEC_WALK_BILLIARD && p->kind != SPEC_WALK_HMC && p->kind != SPEC_WALK_HNR &&
        p->kind != SPEC_WALK_CHNR && p->kind != SPEC_WALK_CHMC)
        return fail(SPEC_EINVAL, "unknown walk kind");
    if (p->kind == SPEC_WALK_CHMC) {
        int rc = check_chmc(ctx, p->q, p->h);
        if (rc) return rc;
    }
    if ((p->kind == SPEC_WALK_HNR || p->kind == SPEC_WALK_CHNR) && p->T > 0.0 && std::isfinite(p->T) && !ctx->has_obj)
        return fail(SPEC_EINVAL, "Hit-and-Run for exp(-c^T x / T) needs spec_set_objective (T = inf: uniform)");
    if (p->kind == SPEC_WALK_HMC) {
        if (!ctx->has_obj) return fail(SPEC_EINVAL, "HMC needs spec_set_objective");
        if (!(p->T > 0.0) || !std::isfinite(p->T)) return fail(SPEC_EINVAL, "HMC needs T > 0");
        if (ctx->has_ball) return fail(SPEC_EINVAL, "HMC with a ball constraint is not supported");
        int rc = ensure_hmc(ctx);
        if (rc) return rc;
    }
    if (p->chains < 1 || p->chains > (1LL << 30)) return fail(SPEC_EINVAL, "chains out of range");
    if (p->steps < 0 || p->steps > (1LL << 31) - 1) return fail(SPEC_EINVAL, "steps out of range");
    if (!(p->L > 0.0) || !std::isfinite(p->L)) return fail(SPEC_EINVAL, "L must be > 0");
    if (p->rho < 0) return fail(SPEC_EINVAL, "rho must be >= 0");
    return SPEC_OK;
}

// Scoped device allocation (freed on every return path).
struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 1); }
    template <typename T>
    T* as() const {
        return (T*)p;
    }
};

// The walk itself (no collective): parameters, x0 upload, rounds to completion.
static int walk_local(spec_ctx* ctx, const spec_walk_params* p, const double* x0, int x0_per_chain, bool host,
                      spec_walk_stats* local) {
    int rc = check_walk_params(ctx, p);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->dev));
    rc = ensure_chains(ctx, p->chains);
    if (rc) return rc;
    const int C = (int)p->chains, n = ctx->n;
    DevBuf dx0;
    const double* x0d = x0;
    if (x0 && host) {
        size_t cnt = (size_t)(x0_per_chain ? C : 1) * n;
        CK(dx0.alloc(sizeof(double) * cnt));
        CK(cudaMemcpyAsync(dx0.p, x0, sizeof(double) * cnt, cudaMemcpyHostToDevice, ctx->stream));
        x0d = dx0.as<double>();
    }
    rc = run_walk(ctx, p, x0d, x0_per_chain, nullptr, nullptr, local);
    CK(cudaStreamSynchronize(ctx->stream));  // x0 staging is read by the walk's first kernels
    return rc;
}

// end-point moments of this rank's chains as chunk partials (1024 consecutive global chain ids
// per chunk, chain order), into part (host)
static int local_moment_chunks(spec_ctx* ctx, int C, std::vector<double>& part) {
    const int n = ctx->n, np = ctx->np, nxx = n * (n + 1) / 2;
    const int CH = 1024;
    const int nchunk = (C + CH - 1) / CH;
    const int stride = n + nxx;
    DevBuf dpart;
    CK(dpart.alloc(sizeof(double) * (size_t)nchunk * stride));
    moments_chunk_kernel<<<std::min((nchunk * stride + 255) / 256, 8192), 256, 0, ctx->stream>>>(
        ctx->cb.X, np, n, C, CH, dpart.as<double>());
    ctx->launches++;
    part.assign((size_t)nchunk * stride, 0.0);
    CK(cudaMemcpyAsync(part.data(), dpart.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SPEC_OK;
}

static int walk_entry(spec_ctx* ctx, const spec_walk_params* p, const double* x0, int x0_per_chain,
                      double* sum_x, double* sum_xx, double* final_x, spec_walk_stats* st, bool host) {
    SW_NOT_DURING_WALK(ctx);
    if (!p) return fail(SPEC_EINVAL, "null argument");
    const bool moments = sum_x || sum_xx;
    const int n = ctx->n, np = ctx->np, nxx = n * (n + 1) / 2;
    const int C = (int)p->chains;
    spec_walk_stats local;
    memset(&local, 0, sizeof(local));
    int rc = SPEC_OK;
    if (moments && ctx->has_comm && (C % 1024 || p->chain_begin % 1024))
        rc = fail(SPEC_EINVAL, "multi-rank moments need shards of multiples of 1024 chains");
    if (!rc) rc = walk_local(ctx, p, x0, x0_per_chain, host, &local);
    if (!rc && local.failures > 0)
        rc = fail(SPEC_EPRECOND, std::to_string(local.failures) + " chain(s) started outside int S");
    if (st) *st = local;
    if (moments) {
        // gathered over ranks (every rank reaches the collective, with its status) and summed
        // in global chunk order: identical for any world size
        std::vector<double> part, allp;
        if (!rc) rc = local_moment_chunks(ctx, C, part);
        else part.assign((size_t)((C + 1023) / 1024) * (n + nxx), 0.0);
        rc = gather_f64(ctx, rc, part, allp);
        if (rc) return rc;
        const int stride = n + nxx;
        std::vector<double> acc(allp.begin(), allp.begin() + stride);
        for (size_t k = 1; k < allp.size() / stride; ++k)
            for (int q = 0; q < stride; ++q) acc[q] += allp[k * stride + q];
        cudaMemcpyKind kk = host ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice;
        if (sum_x) CK(cudaMemcpyAsync(sum_x, acc.data(), sizeof(double) * n, kk, ctx->stream));
        if (sum_xx) CK(cudaMemcpyAsync(sum_xx, acc.data() + n, sizeof(double) * nxx, kk, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if (rc) return rc;
    if (final_x) {
        ChainBuf& b = ctx->cb;
        if (host) {
            DevBuf tmp;
            CK(tmp.alloc(sizeof(double) * (size_t)C * n));
            unpad_rows_kernel<<<4096, 256, 0, ctx->stream>>>(b.X, np, C, n, tmp.as<double>());
            CK(cudaMemcpyAsync(final_x, tmp.p, sizeof(double) * (size_t)C * n, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        } else {
            unpad_rows_kernel<<<4096, 256, 0, ctx->stream>>>(b.X, np, C, n, final_x);
        }
        ctx->launches++;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return SPEC_OK;
}

extern "C" int walk_sample(spec_ctx* ctx, const spec_walk_params* p, const double* x0, int x0_per_chain,
                           double* sum_x, double* sum_xx, double* final_x, spec_walk_stats* st) {
    return walk_entry(ctx, p, x0, x0_per_chain, sum_x, sum_xx, final_x, st, true);
}
extern "C" int walk_sample_dev(spec_ctx* ctx, const spec_walk_params* p, const double* x0, int x0_per_chain,
                               double* sum_x, double* sum_xx, double* final_x, spec_walk_stats* st) {
    return walk_entry(ctx, p, x0, x0_per_chain, sum_x, sum_xx, final_x, st, false);
}

extern "C" int walk_trace(spec_ctx* ctx, const spec_walk_params* p, const int64_t* chain_ids, int64_t nchains,
                          int64_t max_refl, double* hit_x, double* t, double* w, double* v_after, int32_t* binding,
                          int64_t* nrec) {
    if (!chain_ids || nchains < 1 || max_refl < 1) return fail(SPEC_EINVAL, "bad trace arguments");
    SW_NOT_DURING_WALK(ctx);
    spec_walk_params q = *p;
    q.chains = nchains;
    int rc = check_walk_params(ctx, &q);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->dev));
    rc = ensure_chains(ctx, nchains);
    if (rc) return rc;
    const int C = (int)nchains, n = ctx->n;
    const int R = (int)max_refl;
    CK(cudaMemcpyAsync(ctx->cb.gid, chain_ids, sizeof(long long) * C, cudaMemcpyHostToDevice, ctx->stream));
    TraceBufs tb;
    tb.max_trace = R;
    CK(zalloc(&tb.cnt, C));
    CK(zalloc(&tb.hit, (size_t)C * R * n));
    CK(zalloc(&tb.t, (size_t)C * R));
    CK(zalloc(&tb.w, (size_t)C * R * n));
    CK(zalloc(&tb.v, (size_t)C * R * n));
    CK(zalloc(&tb.bind, (size_t)C * R));
    spec_walk_stats local;
    rc = run_walk(ctx, &q, nullptr, 0, ctx->cb.gid, &tb, &local);
    if (!rc) {
        std::vector<int> cnt(C);
        CK(cudaMemcpy(cnt.data(), tb.cnt, sizeof(int) * C, cudaMemcpyDeviceToHost));
        for (int i = 0; i < C; ++i) nrec[i] = cnt[i];
        CK(cudaMemcpy(hit_x, tb.hit, sizeof(double) * (size_t)C * R * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(t, tb.t, sizeof(double) * (size_t)C * R, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(w, tb.w, sizeof(double) * (size_t)C * R * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(v_after, tb.v, sizeof(double) * (size_t)C * R * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(binding, tb.bind, sizeof(int) * (size_t)C * R, cudaMemcpyDeviceToHost));
    }
    cudaFree(tb.cnt); cudaFree(tb.hit); cudaFree(tb.t); cudaFree(tb.w); cudaFree(tb.v); cudaFree(tb.bind);
    return rc;
}

static WalkRun& walk_run(spec_ctx* ctx) {
    if (!ctx->walk) ctx->walk = new WalkRun();
    return *(WalkRun*)ctx->walk;
}
// The resumable walk owns the chain buffers between walk_begin and walk_end: every other
// entry point that uses them (oracle, walks, estimators, objective) returns EINVAL meanwhile.
static bool walk_is_active(spec_ctx* ctx) { return ctx && ctx->walk && ((WalkRun*)ctx->walk)->active; }
static void free_walk(spec_ctx* ctx) {
    delete (WalkRun*)ctx->walk;
    ctx->walk = nullptr;
}

// ---------------------------------------------------------------- resumable walk API
extern "C" int walk_begin(spec_ctx* ctx, const spec_walk_params* p, const double* x0_dev, int x0_per_chain) {
    SW_NOT_DURING_WALK(ctx);
    int rc = check_walk_params(ctx, p);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->dev));
    rc = ensure_chains(ctx, p->chains);
    if (rc) return rc;
    return walk_setup(ctx, p, x0_dev, x0_per_chain, nullptr, nullptr);
}

extern "C" int walk_rounds(spec_ctx* ctx, int64_t max_rounds, int64_t* active) {
    if (!ctx || !walk_run(ctx).active) return fail(SPEC_EINVAL, "no walk in progress (call walk_begin)");
    CK(cudaSetDevice(ctx->dev));
    int rc = walk_do_rounds(ctx, max_rounds <= 0 ? 0 : max_rounds);
    if (active) *active = walk_run(ctx).count;
    return rc;
}

extern "C" int walk_end(spec_ctx* ctx, double* sum_x_dev, double* sum_xx_dev, double* final_x_dev,
                        spec_walk_stats* st) {
    if (!ctx || !walk_run(ctx).active) return fail(SPEC_EINVAL, "no walk in progress (call walk_begin)");
    CK(cudaSetDevice(ctx->dev));
    WalkRun& W = walk_run(ctx);
    int rc = walk_collect_stats(ctx, st);
    if (rc) return rc;
    const int C = (int)W.p.chains, n = ctx->n, np = ctx->np;
    if (sum_x_dev || sum_xx_dev) {
        double *dsx = sum_x_dev, *dsxx = sum_xx_dev, *tx = nullptr, *txx = nullptr;
        const int nxx = n * (n + 1) / 2;
        if (!dsx) { CK(cudaMalloc(&tx, sizeof(double) * n)); dsx = tx; }
        if (!dsxx) { CK(cudaMalloc(&txx, sizeof(double) * nxx)); dsxx = txx; }
        moments_kernel<<<std::min((n + nxx + 127) / 128, 4096), 128, 0, ctx->stream>>>(ctx->cb.X, np, n, C, dsx,
                                                                                         dsxx);
        ctx->launches++;
        CK(cudaStreamSynchronize(ctx->stream));
        if (tx) cudaFree(tx);
        if (txx) cudaFree(txx);
    }
    if (final_x_dev) {
        unpad_rows_kernel<<<4096, 256, 0, ctx->stream>>>(ctx->cb.X, np, C, n, final_x_dev);
        ctx->launches++;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    W.active = false;
    return SPEC_OK;
}

extern "C" int spec_kernel_timing(spec_ctx* ctx, int enable) {
    if (!ctx) return fail(SPEC_EINVAL, "null ctx");
    WalkRun& W = walk_run(ctx);
    W.timing = enable != 0;
    for (int i = 0; i < 4; ++i) W.kms[i] = 0.0, W.kcount[i] = 0;
    for (int i = 0; i < 3; ++i) W.k2ms[i] = 0.0;
    W.k2_items = 0;
    return SPEC_OK;
}

extern "C" const char* spec_k2_config(spec_ctx* ctx) {
    static thread_local std::string s;
    if (!ctx) return "";
    char buf[256];
    if (ctx->g_split == 2 && ctx->fg)
        snprintf(buf, sizeof(buf), "split (m > 112): factor_g_kernel<%d> (G/L/W tiles in shared memory, B tiles in L2, %d CTAs) | "
                 "lanczos_t_kernel (M as lower tiles in shared memory, %d CTAs) | tail_kernel<%d> (%d CTAs)",
                 ctx->fg, ctx->fg_grid, ctx->lt_grid, ctx->t512 ? 512 : 256, ctx->t_grid);
    else if (ctx->g_split == 2)
        snprintf(buf, sizeof(buf), "split (m > 112): chord_kernel2<512, global scratch> factor phase (%d CTAs) | "
                 "lanczos_t_kernel (M as lower tiles in shared memory, %d CTAs) | tail_kernel<256> (%d CTAs)",
                 ctx->chord_grid_max, ctx->lt_grid, ctx->t_grid);
    else if (ctx->g_split)
        snprintf(buf, sizeof(buf), "split (m > 112): chord_kernel2<512, global scratch> factor phase (%d CTAs) | "
                 "lanczos_cl_kernel (2-CTA clusters, %d CTAs) | tail_kernel<256> (%d CTAs)",
                 ctx->chord_grid_max, ctx->cl_grid, ctx->t_grid);
    else if (ctx->k2_split)
        snprintf(buf, sizeof(buf), "split: %s (%d CTAs) | %s (%d CTAs) | tail_kernel<256> (%d CTAs)",
                 ctx->ft ? "factor_t_kernel<256 thr, tiles>" : "factor_kernel<512>", ctx->ft ? ctx->ft_grid : ctx->f_grid,
                 ctx->lz2 ? "lanczos2_kernel<256 thr, 2/SM>" : "lanczos_kernel<512>",
                 ctx->lz2 ? ctx->l2_grid : ctx->l_grid, ctx->t_grid);
    else
        snprintf(buf, sizeof(buf), "fused: chord_kernel2<%d, %s> (%d CTAs)", ctx->chord_threads,
                 ctx->smem_path ? "shared" : "global scratch", ctx->chord_grid_max);
    s = buf;
    return s.c_str();
}

extern "C" int spec_lanczos_iterations(spec_ctx* ctx, int reset, double* mean_j, int64_t* solves) {
    if (!ctx) return fail(SPEC_EINVAL, "null ctx");
    CK(cudaSetDevice(ctx->dev));
    unsigned long long h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, ctx->jsum, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    if (reset) CK(cudaMemsetAsync(ctx->jsum, 0, sizeof(h), ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (mean_j) *mean_j = h[1] ? (double)h[0] / (double)h[1] : 0.0;
    if (solves) *solves = (int64_t)h[1];
    return SPEC_OK;
}

extern "C" int spec_k2_phase_times(spec_ctx* ctx, double* ms3) {
    if (!ctx || !ms3) return fail(SPEC_EINVAL, "null argument");
    WalkRun& W = walk_run(ctx);
    for (int i = 0; i < 3; ++i) ms3[i] = W.k2ms[i];
    return SPEC_OK;
}

extern "C" int spec_kernel_times(spec_ctx* ctx, double* ms4, int64_t* launches4, int64_t* k2_items) {
    if (!ctx) return fail(SPEC_EINVAL, "null ctx");
    WalkRun& W = walk_run(ctx);
    for (int i = 0; i < 4; ++i) {
        if (ms4) ms4[i] = W.kms[i];
        if (launches4) launches4[i] = W.kcount[i];
    }
    if (k2_items) *k2_items = W.k2_items;
    return SPEC_OK;
}

extern "C" int spec_walk_stats_now(spec_ctx* ctx, spec_walk_stats* st) {
    if (!ctx || !walk_run(ctx).active) return fail(SPEC_EINVAL, "no walk in progress");
    return walk_collect_stats(ctx, st);
}

// ---------------------------------------------------------------- multi-rank plumbing
extern "C" int spec_set_comm(spec_ctx* ctx, const spec_comm* comm) {
    if (!ctx) return fail(SPEC_EINVAL, "null ctx");
    if (!comm) {
        ctx->has_comm = 0;
        ctx->comm = spec_comm{nullptr, 0, 1, nullptr};
        return SPEC_OK;
    }
    if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world || !comm->allgather_f64)
        return fail(SPEC_EINVAL, "bad spec_comm");
    ctx->comm = *comm;
    ctx->has_comm = comm->world > 1;
    return SPEC_OK;
}

// allgather of equal host shards in rank order (identity on one rank).  rc_local is this
// rank's status so far: it travels with the shard, every rank reaches the collective even
// after a local failure, and all ranks return the first failing rank's code together
// (no rank is left blocked in a collective the others skipped).
static int gather_f64(spec_ctx* ctx, int rc_local, const std::vector<double>& local, std::vector<double>& global) {
    const int W = ctx->has_comm ? ctx->comm.world : 1;
    if (W == 1) {
        if (rc_local) return rc_local;
        global = local;
        return SPEC_OK;
    }
    const size_t nl = local.size();
    std::vector<double> buf(nl + 1, 0.0), all((nl + 1) * (size_t)W, 0.0);
    std::copy(local.begin(), local.end(), buf.begin());
    buf[nl] = (double)rc_local;
    const std::string msg = g_err;
    int rc = ctx->comm.allgather_f64(ctx->comm.user, buf.data(), (int64_t)(nl + 1), all.data());
    if (rc) return fail(SPEC_ECUDA, "allgather callback failed");
    for (int r = 0; r < W; ++r) {
        const int rr = (int)all[(size_t)r * (nl + 1) + nl];
        if (rr) return fail(rr, r == ctx->comm.rank ? msg : "rank " + std::to_string(r) + " failed (code " +
                                                                 std::to_string(rr) + ")");
    }
    global.resize(nl * (size_t)W);
    for (int r = 0; r < W; ++r)
        std::copy(all.begin() + (size_t)r * (nl + 1), all.begin() + (size_t)r * (nl + 1) + nl,
                  global.begin() + (size_t)r * nl);
    return SPEC_OK;
}

// ---------------------------------------------------------------- K6: ball sampling + membership
static int ball_inside_count(spec_ctx* ctx, uint64_t seed, uint32_t tag, long long begin, int count,
                             const double* c0_host, double r, long long* inside_out) {
    ChainBuf& b = ctx->cb;
    int rc = ensure_chains(ctx, count);
    if (rc) return rc;
    const int n = ctx->n, np = ctx->np, m = ctx->m;
    double* dc0 = ctx->c0;
    CK(cudaMemcpyAsync(dc0, c0_host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    ball_sample_kernel<<<(count + 7) / 8, 256, 0, ctx->stream>>>(count, begin, n, np, seed, tag, dc0, r, b.X);
    ctx->launches++;
    launch_gemm_av(ctx, b.X, nullptr, nullptr, count, b.AX, ctx->a0);  // A(x_j)
    const int mp = roundup(m, 8);
    size_t smem = sizeof(double) * ((size_t)mp * ctx->ld + mp + 8);
    const int NT = mp <= 64 ? 128 : 256;
    if (NT == 128) {
        CK(cudaFuncSetAttribute(membership_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        membership_kernel<128><<<std::min(count, ctx->num_sms * 8), 128, smem, ctx->stream>>>(
            count, n, np, m, ctx->mt, ctx->mtp, ctx->ld, b.X, b.AX, ctx->has_cube ? ctx->lo : nullptr, ctx->hi,
            b.steps_done, nullptr, 0);
    } else if (smem <= 227 * 1024 || !ctx->scratch) {
        CK(cudaFuncSetAttribute(membership_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        membership_kernel<256><<<std::min(count, ctx->num_sms * 2), 256, smem, ctx->stream>>>(
            count, n, np, m, ctx->mt, ctx->mtp, ctx->ld, b.X, b.AX, ctx->has_cube ? ctx->lo : nullptr, ctx->hi,
            b.steps_done, nullptr, 0);
    } else {
        // m > ~160: A(x_j) does not fit in shared memory; factor it in the global-scratch slices
        // of the K2 variant (one per CTA, >= mp x ld doubles each)
        smem = sizeof(double) * (mp + 8);
        membership_kernel<256><<<std::min(count, ctx->scratch_ctas), 256, smem, ctx->stream>>>(
            count, n, np, m, ctx->mt, ctx->mtp, ctx->ld, b.X, b.AX, ctx->has_cube ? ctx->lo : nullptr, ctx->hi,
            b.steps_done, ctx->scratch, ctx->scratch_stride);
    }
    ctx->launches++;
    std::vector<int> flags(count);
    CK(cudaMemcpyAsync(flags.data(), b.steps_done, sizeof(int) * count, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    long long cnt = 0;
    for (int v : flags) cnt += v;
    *inside_out = cnt;
    return SPEC_OK;
}

// ---------------------------------------------------------------- volume (ball-phase MMC)
static uint32_t vol_tag(int purpose, int phase, bool ball, int attempt) {
    return ((uint32_t)purpose << 28) | ((uint32_t)attempt << 20) | ((uint32_t)phase << 1) | (ball ? 1u : 0u);
}

static double log_ball_volume(int n, double r) {
    return 0.5 * n * std::log(M_PI) - std::lgamma(0.5 * n + 1.0) + n * std::log(r);
}

extern "C" int volume(spec_ctx* ctx, double eps, uint64_t seed, int64_t chains_per_phase,
                      const spec_volume_opts* o, spec_volume_report* out) {
    if (!ctx || !out) return fail(SPEC_EINVAL, "null argument");
    if (!(eps > 0.0 && eps < 1.0)) return fail(SPEC_EINVAL, "eps must be in (0,1)");
    SW_NOT_DURING_WALK(ctx);
    const int n = ctx->n;
    spec_volume_opts opt;
    opt.walk_len = 10; opt.burn = 20; opt.L = 2.0 * std::sqrt((double)n); opt.rho = 10 * n;  // burn: R25
    opt.rho_star = 0.325; opt.q_stop = 0.25; opt.max_phases = 64; opt.max_growth = 16;
    if (o) {
        if (o->walk_len > 0) opt.walk_len = o->walk_len;
        if (o->burn > 0) opt.burn = o->burn;
        if (o->L > 0) opt.L = o->L;
        if (o->rho > 0) opt.rho = o->rho;
        if (o->rho_star > 0) opt.rho_star = o->rho_star;
        if (o->q_stop > 0) opt.q_stop = o->q_stop;
        if (o->max_phases > 0) opt.max_phases = std::min(o->max_phases, (int)SPEC_MAX_PHASES);
        if (o->max_growth > 0) opt.max_growth = o->max_growth;
    }
    const int W = ctx->has_comm ? ctx->comm.world : 1, R = ctx->has_comm ? ctx->comm.rank : 0;
    const long long N = chains_per_phase;
    if (N < 8 || N % W) return fail(SPEC_EINVAL, "chains_per_phase must be >= 8 and divisible by the world size");
    CK(cudaSetDevice(ctx->dev));
    std::vector<double> c0(n, 0.0);
    long long calls = 0;
    // the phase balls are installed on the context: removed on every return path
    struct BallGuard {
        spec_ctx* c;
        ~BallGuard() { c->has_ball = 0; }
    } ball_guard{ctx};
    struct EventGuard {
        cudaEvent_t e = nullptr;
        ~EventGuard() {
            if (e) cudaEventDestroy(e);
        }
    } g0, g1;
    CK(cudaEventCreate(&g0.e));
    CK(cudaEventCreate(&g1.e));
    cudaEvent_t e0 = g0.e, e1 = g1.e;
    CK(cudaEventRecord(e0, ctx->stream));

    auto walk_phase = [&](double r, const std::vector<double>& X0, long long Nt, long long steps, uint32_t tag,
                          std::vector<double>& X) -> int {
        const long long Cl = Nt / W, begin = (long long)R * Cl;
        X.assign((size_t)Cl * n, 0.0);
        int rc2 = spec_set_ball(ctx, r > 0 ? c0.data() : nullptr, r > 0 ? r : 0.0);
        if (rc2) return rc2;
        spec_walk_params p;
        p.kind = SPEC_WALK_BILLIARD; p.chain_begin = begin; p.chains = Cl; p.steps = steps; p.L = opt.L;
        p.rho = opt.rho; p.seed = seed; p.tag = tag; p.T = 1.0;
        X.assign((size_t)Cl * n, 0.0);
        spec_walk_stats st;
        rc2 = walk_entry(ctx, &p, X0.data(), 1, nullptr, nullptr, X.data(), &st, true);
        if (getenv("SPECWALK_DEBUG_VOLUME"))
            fprintf(stderr, "[volume] walk r=%.6g tag=%08x chains=%lld steps=%lld rc=%d calls=%lld failures=%lld\n", r,
                    tag, Cl, steps, rc2, (long long)st.calls, (long long)st.failures);
        calls += st.calls;
        return rc2;
    };
    auto q_of = [&](double r, uint32_t tag, long long Nt, double* q) -> int {
        const long long Cl = Nt / W, begin = (long long)R * Cl;
        long long cnt = 0;
        int rc2 = ball_inside_count(ctx, seed, tag, begin, (int)Cl, c0.data(), r, &cnt);
        std::vector<double> loc(1, (double)cnt), glob;
        rc2 = gather_f64(ctx, rc2, loc, glob);
        if (rc2) return rc2;
        double tot = 0.0;
        for (double v : glob) tot += v;
        *q = tot / (double)Nt;
        return SPEC_OK;
    };
    auto norm = [&](const double* x) {
        double s2 = 0.0;
        for (int i = 0; i < n; ++i) s2 += (x[i] - c0[i]) * (x[i] - c0[i]);
        return std::sqrt(s2);
    };
    // A warm start re-forms F(x) from x, and a walk end point can lie within
    // rounding of the boundary (a step may end at l = t+ - ulp): contract it
    // towards the interior point c0 by 2^-40 (R24; the oracle does the same).
    auto warm = [&](const double* x, double* out) {
        const double lam = 1.0 - 0x1p-40;
        for (int i = 0; i < n; ++i) out[i] = c0[i] + lam * (x[i] - c0[i]);
    };
    // warm starts of this rank's chains [begin, begin + Cl) from the global points strictly inside B(r)
    auto resample = [&](const std::vector<double>& Xg, double r, long long Nt, std::vector<double>& X0) -> int {
        const long long Cl = Nt / W, begin = (long long)R * Cl;
        std::vector<long long> inside;
        const long long Ng = (long long)(Xg.size() / n);
        for (long long j = 0; j < Ng; ++j)
            if (norm(&Xg[(size_t)j * n]) < r) inside.push_back(j);
        if (inside.empty()) return fail(SPEC_ERUNTIME, "no sample strictly inside the next ball");
        X0.resize((size_t)Cl * n);
        for (long long j = 0; j < Cl; ++j) {
            long long src = inside[(size_t)((begin + j) % (long long)inside.size())];
            warm(&Xg[(size_t)src * n], &X0[(size_t)j * n]);
        }
        return SPEC_OK;
    };

    int rc = SPEC_OK;
    std::vector<double> radii;  // r_1..r_k
    std::vector<double> X, Xg, X0((size_t)(N / W) * n, 0.0), burned_g;
    // ---- pilot
    rc = walk_phase(-1.0, X0, N, opt.burn, vol_tag(3, 0, false, 0), X);
    rc = gather_f64(ctx, rc, X, burned_g);
    if (rc) return rc;
    Xg = burned_g;
    for (int i = 0; i < opt.max_phases; ++i) {
        std::vector<double> d((size_t)N);
        for (long long j = 0; j < N; ++j) d[(size_t)j] = norm(&Xg[(size_t)j * n]);
        std::sort(d.begin(), d.end());
        long long qi = (long long)std::ceil(opt.rho_star * (double)N) - 1;
        if (qi < 0) qi = 0;
        const double r_next = d[(size_t)qi];
        double q = 0.0;
        rc = q_of(r_next, vol_tag(3, i, true, 0), N, &q);
        if (rc) return rc;
        radii.push_back(r_next);
        if (q >= opt.q_stop) break;
        rc = resample(Xg, r_next, N, X0);
        if (rc) return rc;
        rc = walk_phase(r_next, X0, N, opt.walk_len, vol_tag(3, i + 1, false, 0), X);
        rc = gather_f64(ctx, rc, X, Xg);
        if (rc) return rc;
    }
    const int k = (int)radii.size();
    // ---- estimation
    int attempt = 0;
    long long Ne = N;
    std::vector<double> ratios;
    double q = 0.0, sig = 0.0;
    for (;;) {
        const long long Cl = Ne / W, begin = (long long)R * Cl;
        X0.resize((size_t)Cl * n);
        for (long long j = 0; j < Cl; ++j) {
            long long src = (begin + j) % N;
            warm(&burned_g[(size_t)src * n], &X0[(size_t)j * n]);
        }
        ratios.clear();
        for (int i = 0; i < k; ++i) {
            rc = walk_phase(i == 0 ? -1.0 : radii[i - 1], X0, Ne, opt.walk_len, vol_tag(1, i, false, attempt), X);
            rc = gather_f64(ctx, rc, X, Xg);
            if (rc) return rc;
            long long in = 0;
            for (long long j = 0; j < Ne; ++j) in += (norm(&Xg[(size_t)j * n]) <= radii[i]) ? 1 : 0;
            ratios.push_back((double)in / (double)Ne);
            if (in == 0) return fail(SPEC_ERUNTIME, "empty phase ratio");
            rc = resample(Xg, radii[i], Ne, X0);
            if (rc) return rc;
        }
        rc = q_of(radii[k - 1], vol_tag(1, k, true, attempt), Ne, &q);
        if (rc) return rc;
        if (!(q > 0.0)) return fail(SPEC_ERUNTIME, "no ball sample inside S");
        double var = (1.0 - q) / ((double)Ne * q);
        for (double rt : ratios) var += (1.0 - rt) / ((double)Ne * rt);
        sig = std::sqrt(var);
        if (sig <= eps / 2 || Ne >= (long long)opt.max_growth * N) break;
        ++attempt;
        Ne *= 2;
    }
    ctx->has_ball = 0;
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double logv = log_ball_volume(n, radii[k - 1]) + std::log(q);
    for (double rt : ratios) logv -= std::log(rt);
    // calls summed over ranks
    std::vector<double> cl(1, (double)calls), clg;
    rc = gather_f64(ctx, SPEC_OK, cl, clg);
    if (rc) return rc;
    double calls_tot = 0.0;
    for (double v : clg) calls_tot += v;
    memset(out, 0, sizeof(*out));
    out->volume = std::exp(logv);
    out->log_volume = logv;
    out->std_rel = sig;
    out->q = q;
    out->phases = k;
    out->chains = Ne;
    out->calls = (int64_t)calls_tot;
    out->device_ms = ms;
    for (int i = 0; i < k; ++i) {
        out->radii[i] = radii[i];
        out->ratios[i] = ratios[i];
    }
    return SPEC_OK;
}

// ---------------------------------------------------------------- expectation
extern "C" int expectation(spec_ctx* ctx, int f_id, double T, uint64_t seed, const spec_expect_params* ep,
                           double* est, double* stderr_out) {
    if (!ctx || !ep || !est) return fail(SPEC_EINVAL, "null argument");
    SW_NOT_DURING_WALK(ctx);
    if (f_id < 0 || f_id > 2) return fail(SPEC_EINVAL, "unknown f_id");
    if ((f_id == SPEC_F_LINEAR_C || f_id == SPEC_F_HALFSPACE_UNION) && !ctx->has_obj)
        return fail(SPEC_EINVAL, "f needs the objective c (spec_set_objective)");
    if (f_id == SPEC_F_HALFSPACE_UNION && !(ep->b2 > ep->b1)) return fail(SPEC_EINVAL, "need b2 > b1");
    const int W = ctx->has_comm ? ctx->comm.world : 1, R = ctx->has_comm ? ctx->comm.rank : 0;
    if (ep->chains < 2 || ep->chains % W) return fail(SPEC_EINVAL, "chains must be >= 2 and divisible by world");
    const long long Cl = ep->chains / W;
    spec_walk_params p;
    const bool hmc = (T > 0.0) && std::isfinite(T);
    p.kind = hmc ? SPEC_WALK_HMC : SPEC_WALK_BILLIARD;
    p.chain_begin = (long long)R * Cl;
    p.chains = Cl;
    p.steps = ep->steps;
    p.L = ep->L;
    p.rho = ep->rho;
    p.seed = seed;
    p.tag = 0;
    p.T = hmc ? T : 1.0;
    spec_walk_stats st;
    std::vector<double> fl((size_t)Cl, 0.0), fg;
    int rc = walk_entry(ctx, &p, nullptr, 0, nullptr, nullptr, nullptr, &st, true);
    if (!rc) {
        rc = [&]() -> int {
            DevBuf df;
            CK(df.alloc(sizeof(double) * Cl));
            fvalue_kernel<<<(int)std::min<long long>((Cl + 7) / 8, 65535), 256, 0, ctx->stream>>>(
                (int)Cl, ctx->n, ctx->np, ctx->cb.X, ctx->c, f_id, ep->b1, ep->b2, df.as<double>());
            ctx->launches++;
            CK(cudaMemcpyAsync(fl.data(), df.p, sizeof(double) * Cl, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            return SPEC_OK;
        }();
    }
    rc = gather_f64(ctx, rc, fl, fg);
    if (rc) return rc;
    double s = 0.0;
    for (double v : fg) s += v;  // global chain order: identical for any GPU count
    const double Nd = (double)fg.size();
    const double mean = s / Nd;
    double ss = 0.0;
    for (double v : fg) ss += (v - mean) * (v - mean);
    *est = mean;
    if (stderr_out) *stderr_out = std::sqrt(ss / (Nd - 1.0) / Nd);
    return SPEC_OK;
}

// ---------------------------------------------------------------- SDP by simulated annealing (sec:optimization)
// min c^T x over S (eq:sdp P:1406) by sampling exp(-c^T x / T_i) with T_0 ~ R and
// T_{i+1} = T_i (1 - 1/sqrt(n)), warm-starting every chain from its previous
// point, walk length 1 for HMC-r (Fig. hmc_hnr), the first (uniform)
// point by the billiard walk.  chains run independently; the reported point is the
// best c^T x over all chains and temperatures.  Tags: purpose 4, phase = temperature index + 1.
extern "C" int sdp_anneal(spec_ctx* ctx, const spec_sdp_params* sp, double* best_x, double* history,
                          spec_sdp_report* out) {
    if (!ctx || !sp || !out) return fail(SPEC_EINVAL, "null argument");
    SW_NOT_DURING_WALK(ctx);
    if (!ctx->has_obj) return fail(SPEC_EINVAL, "sdp_anneal needs the objective (spec_set_objective)");
    if (sp->kind != SPEC_WALK_HMC && sp->kind != SPEC_WALK_HNR && sp->kind != SPEC_WALK_CHNR)
        return fail(SPEC_EINVAL, "sdp_anneal: kind must be HMC, HNR or CHNR");
    if (sp->iters < 1 || sp->iters > (1 << 27)) return fail(SPEC_EINVAL, "sdp_anneal: iters out of range");
    const int n = ctx->n, np = ctx->np;
    const int W = ctx->has_comm ? ctx->comm.world : 1, R = ctx->has_comm ? ctx->comm.rank : 0;
    if (sp->chains < 1 || sp->chains % W) return fail(SPEC_EINVAL, "chains must be >= 1 and divisible by world");
    const long long Cl = sp->chains / W, begin = (long long)R * Cl;
    const long long walk_len = sp->walk_len > 0 ? sp->walk_len : 1;
    const long long burn = sp->burn > 0 ? sp->burn : 10;
    const long long rho = sp->rho > 0 ? sp->rho : 10LL * n;
    const double eps = sp->eps > 0.0 ? sp->eps : 0.05;
    CK(cudaSetDevice(ctx->dev));
    std::vector<double> hc(n);
    CK(cudaMemcpyAsync(hc.data(), ctx->c, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    struct EventGuard {
        cudaEvent_t e = nullptr;
        ~EventGuard() {
            if (e) cudaEventDestroy(e);
        }
    } g0, g1;
    CK(cudaEventCreate(&g0.e));
    CK(cudaEventCreate(&g1.e));
    CK(cudaEventRecord(g0.e, ctx->stream));
    DevBuf dX, df;
    CK(dX.alloc(sizeof(double) * (size_t)Cl * n));
    CK(df.alloc(sizeof(double) * (size_t)Cl));
    long long calls = 0;
    auto run = [&](int kind, long long steps, double L, double T, uint32_t tag, bool start_origin) -> int {
        spec_walk_params p;
        p.kind = kind; p.chain_begin = begin; p.chains = Cl; p.steps = steps; p.L = L; p.rho = rho;
        p.seed = sp->seed; p.tag = tag; p.T = T;
        spec_walk_stats st;
        int rc2 = walk_entry(ctx, &p, start_origin ? nullptr : dX.as<double>(), 1, nullptr, nullptr, dX.as<double>(),
                             &st, false);
        calls += st.calls;
        return rc2;
    };
    // local best (value, x) of the current end points -> gathered, min in rank order
    double best = HUGE_VAL, fmin_now = HUGE_VAL;
    std::vector<double> bx(n, 0.0);
    auto update_best = [&](int rc_in) -> int {
        std::vector<double> loc(n + 1, 0.0), glob;
        int rc2 = rc_in;
        if (!rc2) {
            rc2 = [&]() -> int {
                fvalue_kernel<<<(int)std::min<long long>((Cl + 7) / 8, 65535), 256, 0, ctx->stream>>>(
                    (int)Cl, n, np, ctx->cb.X, ctx->c, SPEC_F_LINEAR_C, 0.0, 0.0, df.as<double>());
                ctx->launches++;
                std::vector<double> fl((size_t)Cl);
                CK(cudaMemcpyAsync(fl.data(), df.p, sizeof(double) * Cl, cudaMemcpyDeviceToHost, ctx->stream));
                CK(cudaStreamSynchronize(ctx->stream));
                long long a = 0;
                for (long long j = 1; j < Cl; ++j)
                    if (fl[(size_t)j] < fl[(size_t)a]) a = j;
                loc[0] = fl[(size_t)a];
                CK(cudaMemcpyAsync(loc.data() + 1, dX.as<double>() + (size_t)a * n, sizeof(double) * n,
                                   cudaMemcpyDeviceToHost, ctx->stream));
                CK(cudaStreamSynchronize(ctx->stream));
                return SPEC_OK;
            }();
        }
        rc2 = gather_f64(ctx, rc2, loc, glob);
        if (rc2) return rc2;
        int rb = 0;
        for (int r = 1; r < W; ++r)
            if (glob[(size_t)r * (n + 1)] < glob[(size_t)rb * (n + 1)]) rb = r;
        fmin_now = glob[(size_t)rb * (n + 1)];
        if (fmin_now < best) {
            best = fmin_now;
            std::copy(glob.begin() + (size_t)rb * (n + 1) + 1, glob.begin() + (size_t)(rb + 1) * (n + 1), bx.begin());
        }
        return SPEC_OK;
    };
    // 1. uniform starting points (billiard from the origin)
    int rc = run(SPEC_WALK_BILLIARD, burn, 2.0 * std::sqrt((double)n), 1.0, (4u << 28), true);
    // T_0 = R: the largest distance of a burned-in point from the start (S within R B_n)
    double Rn = 0.0;
    {
        std::vector<double> loc(1, 0.0), glob;
        if (!rc) {
            rc = [&]() -> int {
                std::vector<double> X((size_t)Cl * n);
                CK(cudaMemcpyAsync(X.data(), dX.p, sizeof(double) * X.size(), cudaMemcpyDeviceToHost, ctx->stream));
                CK(cudaStreamSynchronize(ctx->stream));
                for (long long j = 0; j < Cl; ++j) {
                    double s2 = 0.0;
                    for (int i = 0; i < n; ++i) s2 += X[(size_t)j * n + i] * X[(size_t)j * n + i];
                    loc[0] = std::fmax(loc[0], std::sqrt(s2));
                }
                return SPEC_OK;
            }();
        }
        rc = gather_f64(ctx, rc, loc, glob);
        if (rc) return rc;
        for (double v : glob) Rn = std::fmax(Rn, v);
    }
    rc = update_best(SPEC_OK);
    if (rc) return rc;
    double T = sp->T0 > 0.0 ? sp->T0 : Rn;
    const double T0v = T;
    const double L = sp->L > 0.0 ? sp->L : Rn;
    const double cool = 1.0 - 1.0 / std::sqrt((double)n);
    long long it = 0;
    const bool have_target = std::isfinite(sp->f_target);
    for (; it < sp->iters; ++it) {
        rc = run(sp->kind, walk_len, L, T, (4u << 28) | (uint32_t)(it + 1), false);
        rc = update_best(rc);
        if (rc) return rc;
        if (history) history[it] = best;
        T = std::fmax(T * cool, T0v * 0x1p-20);  // cooling floor (R30)
        if (have_target && best - sp->f_target <= eps * std::fabs(sp->f_target)) {
            ++it;
            break;
        }
    }
    CK(cudaEventRecord(g1.e, ctx->stream));
    CK(cudaEventSynchronize(g1.e));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, g0.e, g1.e));
    std::vector<double> cl(1, (double)calls), clg;
    rc = gather_f64(ctx, SPEC_OK, cl, clg);
    if (rc) return rc;
    double calls_tot = 0.0;
    for (double v : clg) calls_tot += v;
    memset(out, 0, sizeof(*out));
    out->best = best;
    out->last_min = fmin_now;
    out->T0 = sp->T0 > 0.0 ? sp->T0 : Rn;
    out->T_final = T;
    out->L = L;
    out->iters = it;
    out->calls = (int64_t)calls_tot;
    out->device_ms = ms;
    if (best_x) std::copy(bx.begin(), bx.end(), best_x);
    return SPEC_OK;
}
