/*
 * specwalk.h -- C-ABI of the B200-native spectrahedron boundary oracle and the
 * walks / estimators above it (arXiv 2010.03817, /root/reference/PAPER.md).
 *
 * "P:123" = PAPER.md line 123.  All floating point is IEEE fp64.
 *
 * Conventions for every call
 * --------------------------
 * - Return value: SPEC_OK (0) or one of the SPEC_E* codes below; the message of
 *   the last failure on the calling thread is spec_last_error().
 * - Host pointers ("host") are read/written synchronously: the call returns
 *   after the device work and the copies finished.  "_dev" variants take
 *   DEVICE pointers on the context's GPU and are asynchronous with respect to
 *   the host only where stated.
 * - The library never falls back to the CPU: without a usable CUDA device
 *   spec_create fails with SPEC_ECUDA.
 * - Calls on one context are not re-entrant; distinct contexts are independent.
 * - Between walk_begin and walk_end the resumable walk owns the context's chain
 *   buffers: every other call that uses them (boundary_oracle*, hmc_oracle,
 *   walk_sample*, walk_trace, volume, expectation, spec_set_objective,
 *   spec_set_ball, walk_begin) returns SPEC_EINVAL until walk_end.
 * - Multi-rank (spec_set_comm): a failure on one rank inside volume,
 *   expectation or walk_sample's moment reduction is exchanged through the
 *   allgather, so every rank returns the failing rank's code together.
 * - Layouts are row-major.  n = ambient dimension, m = matrix size of the LMI.
 * - A "boundary-oracle call" (the unit of BASELINE.json's metric) is one chord
 *   solve (Alg. 2) plus, if the segment ends on a dense-block hit,
 *   the normal (lemma:gradient), for one chain on one segment.
 */
#ifndef SPECWALK_H
#define SPECWALK_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SPEC_OK = 0,
    SPEC_EINVAL = 1,     /* bad argument (sizes, NaN, asymmetry, unknown kind) */
    SPEC_EPRECOND = 2,   /* a precondition of the paper fails (start not interior) */
    SPEC_ERUNTIME = 3,   /* numerical failure that is not a counted walk event */
    SPEC_ECUDA = 4,      /* CUDA / NCCL error or no device */
    SPEC_ENOMEM = 5,     /* device allocation failed */
    SPEC_EUNBOUNDED = 6  /* t+ = +inf: S is unbounded along a direction */
};

/* binding ids returned per hit */
#define SPEC_BIND_DENSE 0   /* the dense LMI block A(x) */
#define SPEC_BIND_BALL (-1) /* the ball constraint of a volume phase */
/* cube: 1+2i = upper face x_i = hi_i, 2+2i = lower face x_i = lo_i */
#define SPEC_BIND_NONE (-2)

typedef struct spec_ctx spec_ctx;

const char* spec_last_error(void);

/* spec_create -- upload an LMI F(x) = A0 + sum_i x_i A_i (eq:lmi).
 *  n, m     : ambient dimension (>=1) and matrix size (1..SPEC_MAX_M).
 *  A        : host, (n+1)*m*m doubles, A[0] = A0, A[i] = A_i, each m x m
 *             row-major; symmetrised as (A+A^T)/2 on load.  Copied: the
 *             caller keeps ownership.
 *  cube_lo, cube_hi : host, n doubles each, or both NULL (no cube block).  The
 *             cube is the diagonal part of the LMI (hi_i - x_i >= 0,
 *             x_i - lo_i >= 0) handled in closed form.
 *  device   : CUDA device ordinal (-1 = current device).
 *  out      : receives the context (owns all device memory).
 * Errors: EINVAL for n<1, m<1, m>SPEC_MAX_M, NaN/Inf, |A-A^T| > 1e-12 max(1,|A|),
 *         lo>=hi; ECUDA / ENOMEM. */
#define SPEC_MAX_M 256
int spec_create(int n, int m, const double* A, const double* cube_lo, const double* cube_hi, int device,
                spec_ctx** out);
int spec_destroy(spec_ctx* ctx);

/* Objective c (n doubles, host) for the Boltzmann density exp(-c^T x / T) of
 * HMC-r (eq:boltz_ode).  EINVAL if |c| = 0. */
int spec_set_objective(spec_ctx* ctx, const double* c);

/* Potential f of the density exp(-f) sampled by SPEC_WALK_CHMC / chmc_oracle (sec:hmcr
 * P:1116-1124):
 *   SPEC_POT_LINEAR  f = c^T x / scale        (c from spec_set_objective; the Boltzmann law)
 *   SPEC_POT_GAUSS   f = |x - mu|^2 / (2 scale^2)
 *   SPEC_POT_LOGCOSH f = sum_i log cosh((x_i - mu_i) / scale)
 * mu: host n doubles (NULL = 0; ignored by LINEAR).  EINVAL: unknown pot, scale <= 0 or not
 * finite, NaN in mu, LINEAR without an objective. */
enum { SPEC_POT_LINEAR = 0, SPEC_POT_GAUSS = 1, SPEC_POT_LOGCOSH = 2 };
int spec_set_potential(spec_ctx* ctx, int pot, const double* mu, double scale);

/* Ball constraint |x - center| <= radius added to S (a volume phase S_i of
 * eq:mmc_vol).  radius <= 0 removes it.  center: host n doubles. */
int spec_set_ball(spec_ctx* ctx, const double* center, double radius);

/* boundary_oracle -- the batched INTERSECTION + REFLECTION normal
 * (Alg. 2, Alg. 3) on lines x_b + t v_b.
 *  batch    : number of lines (>=0; 0 is a no-op).
 *  x, v     : host, batch x n.  v need not be unit (t scales with 1/|v|).
 *  u        : host, batch x m, or NULL.  If given, x_b is ON the boundary of
 *             the dense block with unit kernel vector u_b (F(x_b) u_b = 0) and
 *             the chord is solved by Schur deflation (R6); t_minus
 *             is then 0 for that block.
 *  t_minus, t_plus : host, batch doubles (Lemma 3: max negative / min
 *             positive root of det F(x + t v)).  +-inf if unbounded.
 *  normal   : host, batch x n: outward unit normal at x + t_plus v
 *             (-grad det F / |grad det F|, lemma:gradient P:752-764; cube faces
 *             +-e_i; ball (x_hit - c)/r), or NaN if the hit is degenerate.
 *  kernel   : host, batch x m or NULL: unit kernel vector of F(x + t_plus v)
 *             for dense hits (the PEP eigenvector), else zeros.
 *  binding  : host, batch int32: SPEC_BIND_* id of the first strict minimum
 *             (tie order dense, cube i = 0..n-1, ball).
 * Errors: EPRECOND if some x_b is not interior (Cholesky of F(x_b) fails) and
 *         u == NULL; the outputs of the other lines are still written. */
int boundary_oracle(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u,
                    double* t_minus, double* t_plus, double* normal, double* kernel, int32_t* binding);
/* same, all pointers on the device (asynchronous on the context stream until
 * spec_sync; u / kernel may be NULL). */
int boundary_oracle_dev(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u,
                        double* t_minus, double* t_plus, double* normal, double* kernel, int32_t* binding);

/* hmc_oracle -- the reflective-HMC boundary oracle (Alg. 6) for
 * the Boltzmann density exp(-c^T x / T) (c from spec_set_objective): the first
 * positive root t+ of det F(x + t v - t^2 c / (2T)) (eq:boltz_ode P:1440-1446,
 * a degree-2 PEP, eq:PEP P:307-316), by monotone Weyl stepping on the
 * quadratic pencil (interior start) or on the sqrt(t)-deflated symmetric
 * quartic (u != NULL: x on the dense boundary with unit kernel u).
 * Outputs as boundary_oracle (no t_minus); normal is the outward normal at
 * the hit.  A line whose Weyl stepping reaches the iteration cap (60) without
 * converging gets t_plus = NaN, normal NaN, binding SPEC_BIND_NONE (the call
 * still returns SPEC_OK; spec_last_error() names the count).
 * EINVAL without an objective or T <= 0. */
int hmc_oracle(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u, double T,
               double* t_plus, double* normal, double* kernel, int32_t* binding);

/* chmc_oracle -- one collocation-HMC segment per line (sec:hmcr P:1116-1158, Lemma 3 for a
 * degree-(q+1) curve): the polynomial p(t) of p'' = -grad f on [0, h] from (x, v) (f from
 * spec_set_potential), and its first boundary hit in (0, h].  Arguments as hmc_oracle (host
 * pointers; u: batch x m unit kernel vectors of F(x) for lines starting on the dense boundary,
 * or NULL).  t_plus: the hit time, or +inf when p stays inside on (0, h]; binding, normal,
 * kernel: as boundary_oracle.  A line whose start moves outward gets t_plus = 0 and the status
 * text in spec_last_error; one that hits the Weyl iteration cap gets NaN.  EPRECOND: some x is
 * not interior.  EINVAL: no potential, q not in 1..6, h <= 0. */
int chmc_oracle(spec_ctx* ctx, int64_t batch, const double* x, const double* v, const double* u, int q, double h,
                double* t_plus, double* normal, double* kernel, int32_t* binding);
/* Collocation HMC-r device counters since the last reset (out4, host): Picard iterations,
 * segments, segments whose Picard iteration hit its cap (64) without converging, and the
 * congruences K^-1 D_j K^-T of all Weyl iterations (the measured flop model of bench.py). */
int spec_chmc_counters(spec_ctx* ctx, int reset, int64_t* out4);

/* ---- walks ---- */
/* BILLIARD: Alg. 5; HMC: reflective HMC for exp(-c^T x / T), Alg. 6
 * (P:1079-1115); HNR: Hit-and-Run for the uniform law, Alg. 4 -- the next point
 * is uniform on the chord [x + t- v, x + t+ v], v ~ U(sphere); CHNR: coordinate-directions
 * Hit-and-Run, v = e_j with j uniform, A(v) = A_j read from the packed
 * coefficients (no contraction).  Hit-and-Run makes exactly one boundary-oracle call per
 * step and never reflects (L and rho are ignored); with 0 < T < inf it samples the
 * Boltzmann law exp(-c^T x / T) (sec:optimization P:1408-1424; needs the objective): the
 * point on the chord is a truncated exponential; T <= 0 or T = inf: the uniform law. */
enum { SPEC_WALK_BILLIARD = 0, SPEC_WALK_HMC = 1, SPEC_WALK_HNR = 2, SPEC_WALK_CHNR = 3, SPEC_WALK_CHMC = 4 };
/* CHMC: reflective HMC for a log-concave density exp(-f) on collocation polynomials (sec:hmcr
 * P:1116-1158; R33; f from spec_set_potential): l = L eta, v ~ N(0, I); the ODE
 * p'' = -grad f(p) is followed in segments of length h' = min(h, l_left), each the degree-(q+1)
 * polynomial through (x, v) whose second derivative matches -grad f at q Chebyshev nodes (Picard
 * iteration); a segment's chord is the first root of det F(p(t)) in (0, h'] (Lemma 3 for a
 * degree-d curve).  No root: x = p(h'), v = p'(h').  A root t+: p'(t+) is reflected (Alg. 3) and
 * the reflection counts towards rho.  One segment = one boundary-oracle call.  The Picard iteration
 * contracts when h^2 times the largest curvature of f is below ~1 (Gaussian: h < sigma); a segment
 * whose iteration did not converge in 64 steps uses the last iterate and is counted
 * (spec_chmc_counters). */

typedef struct spec_walk_params {
    int kind;            /* SPEC_WALK_BILLIARD (Alg. 5), SPEC_WALK_HMC (Alg. 6, Boltzmann), SPEC_WALK_HNR, SPEC_WALK_CHNR */
    int64_t chain_begin; /* global id of this rank's first chain (keys the RNG) */
    int64_t chains;      /* number of chains run by this call */
    int64_t steps;       /* walk steps per chain (each ends in accept or reject) */
    double L;            /* tau: billiard l = -tau ln eta; HMC l = tau eta */
    int64_t rho;         /* reflection bound (reject the step when #refl > rho) */
    uint64_t seed;       /* Philox4x32-10 key */
    uint32_t tag;        /* counter word 3 (purpose << 28 | phase), 0 for plain walks */
    double T;            /* HMC temperature (>0); Hit-and-Run: 0 < T < inf Boltzmann, else uniform;
                            ignored for billiard */
    int q;               /* CHMC: collocation nodes (1..6), trajectory degree q + 1 */
    double h;            /* CHMC: ODE segment length (> 0) */
} spec_walk_params;

typedef struct spec_walk_stats {
    int64_t calls;       /* boundary-oracle calls (device-counted) */
    int64_t reflections;
    int64_t rejects;     /* steps rejected because #refl > rho */
    int64_t degenerates; /* steps rejected at a rank <= m-2 / corner hit */
    int64_t failures;    /* chains whose start was not interior */
    int64_t steps;
    int64_t rounds;      /* scheduler rounds (one oracle call per active chain) */
    double device_ms;    /* CUDA-event time of the walk on the context stream */
    int64_t capped;      /* HMC-r steps rejected because the Weyl stepping of a chord reached
                            its iteration cap (60) before converging: the crossing time is then
                            only bounded below, so the step is rejected (never silent) */
} spec_walk_stats;

/* walk_sample -- run p->chains independent chains for p->steps steps each
 * from x0 (host: n doubles shared by all chains, or chains x n if
 * x0_per_chain, or NULL = origin).  Outputs (host, may be NULL):
 *  sum_x   : n doubles, sum over chains of the end points;
 *  sum_xx  : n(n+1)/2 doubles, packed lower sum of x x^T over end points;
 *  final_x : chains x n end points.
 * Sums are accumulated in fixed chain order (deterministic). */
int walk_sample(spec_ctx* ctx, const spec_walk_params* p, const double* x0, int x0_per_chain, double* sum_x,
                double* sum_xx, double* final_x, spec_walk_stats* st);
/* device variant: x0 and outputs are device pointers (x0 may be NULL). */
int walk_sample_dev(spec_ctx* ctx, const spec_walk_params* p, const double* x0, int x0_per_chain, double* sum_x,
                    double* sum_xx, double* final_x, spec_walk_stats* st);

/* walk_trace -- the first max_refl reflections of each chain in chain_ids
 * (global ids), for parity.  Outputs host, nchains x max_refl x {n,1,n,n,1};
 * nrec[k] = number recorded for chain k. */
int walk_trace(spec_ctx* ctx, const spec_walk_params* p, const int64_t* chain_ids, int64_t nchains,
               int64_t max_refl, double* hit_x, double* t, double* w, double* v_after, int32_t* binding,
               int64_t* nrec);

/* ---- resumable walk (the scheduler behind walk_sample) ----
 * walk_begin  : set up p->chains chains at x0_dev (DEVICE pointer, n or chains x n
 *               doubles, or NULL = origin), draw step 0.
 * walk_rounds : run up to max_rounds scheduler rounds (<= 0: until all chains
 *               finished); one round = one boundary-oracle call per active
 *               chain.  *active receives the number of unfinished chains.
 * walk_end    : statistics and DEVICE outputs (any may be NULL), as walk_sample.
 * spec_walk_stats_now : statistics of the walk in progress (device counters). */
int walk_begin(spec_ctx* ctx, const spec_walk_params* p, const double* x0_dev, int x0_per_chain);
int walk_rounds(spec_ctx* ctx, int64_t max_rounds, int64_t* active);
int walk_end(spec_ctx* ctx, double* sum_x_dev, double* sum_xx_dev, double* final_x_dev, spec_walk_stats* st);
int spec_walk_stats_now(spec_ctx* ctx, spec_walk_stats* st);

/* Per-kernel CUDA-event timing of the walk scheduler (off by default; adds a
 * host sync per round).  spec_kernel_times returns accumulated ms and launch
 * counts for K1 (A(v) GEMM), K2 (chord), K3 (normal GEMM), K4 (reflect), and the
 * number of chain slots K2 processed (including finished ones not yet compacted). */
int spec_kernel_timing(spec_ctx* ctx, int enable);
int spec_kernel_times(spec_ctx* ctx, double* ms4, int64_t* launches4, int64_t* k2_items);
/* The chord (K2) launch configuration of this context, as text (evidence / logs). */
const char* spec_k2_config(spec_ctx* ctx);
/* Lanczos iterations per extreme-eigenvalue solve, counted on the device since creation or
 * the last reset (every billiard chord makes one solve; an HMC-r chord one per Weyl
 * iteration): *mean_j = sum J / solves.  reset != 0 zeroes the counters after reading.
 * This is the measured k of the flop model 2 k m^2. */
int spec_lanczos_iterations(spec_ctx* ctx, int reset, double* mean_j, int64_t* solves);
/* With timing enabled and K2 split into factor / Lanczos / tail kernels (64 < m <= 128): the
 * accumulated ms of each phase (ms3[0..2], host buffer); zeros for the fused K2 variants. */
int spec_k2_phase_times(spec_ctx* ctx, double* ms3);

/* ---- estimators ----
 * Multi-rank: spec_set_comm installs an allgather of equal HOST shards in rank
 * order (e.g. torch.distributed over NCCL); chains are split into contiguous
 * global-id ranges, every reduction is an ordered sum over global chain ids,
 * so results are identical for any world size.  NULL = single rank. */
typedef struct spec_comm {
    void* user;
    int rank, world;
    int (*allgather_f64)(void* user, const double* in, int64_t n_local, double* out /* world*n_local */);
} spec_comm;
int spec_set_comm(spec_ctx* ctx, const spec_comm* comm);

/* volume -- ball-phase multiphase Monte Carlo (eq:mmc_vol P:1291-1300, the
 * telescoping ratio estimator P:1246-1259, schedule: DESIGN.md R11-R14):
 * c0 = origin (must be interior).  Pilot: burned-in billiard samples of
 * S_0 = S; r_{i+1} = rho_star-quantile of |x - c0| over the samples of
 * S_i = S cap B(c0, r_i); stop when q(r) = P_{U(B(r))}[x in S] >= q_stop
 * (exact ball sampling + MEMBERSHIP, Alg. 1).  Estimation: fresh walks of each
 * S_i warm-started from the previous phase's points inside B(r_i), ratio
 * rho_i = #{|x - c0| <= r_{i+1}} / N, q by N exact ball samples;
 * vol = omega_n r_k^n q / prod rho_i.  N doubles (fresh randomness) until the
 * binomial sigma_rel <= eps / 2 or N = max_growth * chains_per_phase.
 * chains_per_phase: global N (divisible by the world size).  opts may be NULL
 * (defaults in brackets).  EINVAL: eps outside (0,1); ERUNTIME: an empty phase. */
#define SPEC_MAX_PHASES 64
typedef struct spec_volume_opts {
    int64_t walk_len; /* billiard steps per phase [10] */
    int64_t burn;     /* phase-0 burn-in steps from c0 [20] (R25) */
    double L;         /* billiard tau [2 sqrt(n)] */
    int64_t rho;      /* reflection bound [10 n] */
    double rho_star;  /* pilot quantile level [0.325] */
    double q_stop;    /* stop threshold on q(r) [0.25] */
    int max_phases;   /* [64] */
    int max_growth;   /* [16] */
} spec_volume_opts;
typedef struct spec_volume_report {
    double volume, log_volume, std_rel, q;
    int phases;
    int64_t chains; /* N of the accepted estimation round */
    int64_t calls;  /* boundary-oracle calls of all walks (all ranks) */
    double device_ms;
    double radii[SPEC_MAX_PHASES];
    double ratios[SPEC_MAX_PHASES];
} spec_volume_report;
int volume(spec_ctx* ctx, double eps, uint64_t seed, int64_t chains_per_phase, const spec_volume_opts* opts,
           spec_volume_report* out);

/* expectation -- E[f] over the end points of p->chains independent chains
 * (P:1326-1334): uniform law by the billiard walk if T <= 0 or T = +inf, the
 * Boltzmann law exp(-c^T x / T) by HMC-r otherwise.  f: SPEC_F_LINEAR_C c^T x,
 * SPEC_F_SQNORM |x|^2, SPEC_F_HALFSPACE_UNION 1(c^T x <= b1 or c^T x >= b2)
 * (P:1355-1358).  est = mean, stderr = sample sd / sqrt(chains). */
enum { SPEC_F_LINEAR_C = 0, SPEC_F_SQNORM = 1, SPEC_F_HALFSPACE_UNION = 2 };
typedef struct spec_expect_params {
    int64_t chains, steps;
    double L;
    int64_t rho;
    double b1, b2;
} spec_expect_params;
int expectation(spec_ctx* ctx, int f_id, double T, uint64_t seed, const spec_expect_params* p, double* est,
                double* stderr_out);

/* sdp_anneal -- approximate min c^T x over S (eq:sdp P:1406, c from spec_set_objective) by
 * simulated annealing (sec:optimization P:1408-1434, after Kalai-Vempala): sample
 * pi_i ~ exp(-c^T x / T_i) with T_0 ~ R (S within the ball of radius R around the start) and
 * T_{i+1} = max(T_i (1 - 1/sqrt(n)), 2^-20 T_0) (the floor: DESIGN.md R30), every chain
 * warm-started from its previous point, the first
 * (uniform) point from the billiard walk, the walk length 1 for HMC-r.
 * p->chains independent chains (global, divisible by the world size; global ids key the
 * RNG, tags purpose 4 / temperature index) -- the batched form of the paper's single chain.
 *  best_x  : host, n doubles (may be NULL): the point of the smallest c^T x seen (end points of
 *            every temperature, all chains).
 *  history : host, p->iters doubles (may be NULL): that best value after each temperature.
 * Stops after p->iters temperatures, or -- with a finite f_target -- once
 * best - f_target <= eps |f_target| (the paper's protocol for Table tab:hmc_hnr).
 * EINVAL: no objective, kind not HMC / HNR / CHNR, chains or iters out of range. */
typedef struct spec_sdp_params {
    int kind;          /* SPEC_WALK_HMC (the paper's W-HMC-r), SPEC_WALK_HNR or SPEC_WALK_CHNR */
    int64_t chains;    /* independent annealing chains (global) */
    int64_t iters;     /* number of temperatures (maximum) */
    int64_t walk_len;  /* walk steps per temperature [1] */
    int64_t burn;      /* billiard steps for the uniform start [10] */
    double T0;         /* initial temperature [<= 0: R = max |x| over the start points] */
    double L;          /* HMC-r trajectory length tau [<= 0: R] (ignored by Hit-and-Run) */
    int64_t rho;       /* reflection bound [10 n] */
    uint64_t seed;
    double f_target;   /* known optimum, or NaN / inf for none */
    double eps;        /* relative stop tolerance with f_target [0.05] */
} spec_sdp_params;
typedef struct spec_sdp_report {
    double best;       /* smallest c^T x seen */
    double last_min;   /* smallest c^T x among the last temperature's points */
    double T0, T_final, L; /* T_final: the temperature after the last one run */
    int64_t iters;     /* temperatures run */
    int64_t calls;     /* boundary-oracle calls (all ranks) */
    double device_ms;
} spec_sdp_report;
int sdp_anneal(spec_ctx* ctx, const spec_sdp_params* p, double* best_x, double* history, spec_sdp_report* out);

/* Make the host wait for all work queued on the context stream. */
int spec_sync(spec_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) for callers timing with events. */
void* spec_stream(spec_ctx* ctx);
/* Number of kernels this context launched since creation (evidence counter). */
int64_t spec_kernel_launches(spec_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
