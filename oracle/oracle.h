/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the spectrahedron
 * boundary oracle and the walks/estimators above it.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code with paper_2010_03817_b200/ (the CUDA product path).
 *
 * Paper = /root/reference/PAPER.md (arXiv 2010.03817).  "P:123" = line 123.
 * fp64 everywhere, compiled with -O2 -ffp-contract=off -fno-fast-math.
 */
#ifndef SPEC_ORACLE_H
#define SPEC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The LMI as a list of diagonal blocks.  Block b has size
 * mb[b] and coefficient matrices C[b][k] (k = 0..n), row-major mb x mb, so
 * F_b(x) = C_b0 + sum_k x_k C_bk  (eq:lmi).
 * Block order: 0 = dense block, then for each coordinate i the cube blocks
 * (hi_i - x_i) [1+2i] and (x_i - lo_i) [2+2i], then the ball arrow block. */
typedef struct orc_lmi {
    int n;
    int nblocks;
    int has_cube;
    int has_ball;
    int* mb;
    double** C; /* C[b] has (n+1)*mb[b]*mb[b] doubles */
} orc_lmi;

/* literal != 0 assembles every block into ONE block of size m+2n(+n+1)
 * (literal vs split blocks).  lo/hi may be NULL (no cube),
 * ball_c may be NULL (no ball). */
orc_lmi* orc_lmi_create(int n, int m, const double* A, const double* lo, const double* hi,
                        const double* ball_c, double ball_r, int literal);
void orc_lmi_destroy(orc_lmi* L);
int orc_lmi_nblocks(const orc_lmi* L);
int orc_lmi_block_size(const orc_lmi* L, int b);

/* F_b(x) and F1_b(v) = sum_k v_k C_bk  (B_0, B_1 of Lemma 3). */
void orc_eval_block(const orc_lmi* L, int b, const double* x, double* out);
void orc_dir_block(const orc_lmi* L, int b, const double* v, double* out);

/* ---- dense linear algebra (no BLAS) ---- */
int orc_cholesky(int m, const double* A, double* Lw);          /* 0 ok, 1 not PD */
int orc_jacobi(int m, const double* A, double* evals, double* evecs /* columns */);
int orc_sym_eig(int m, const double* A, double* evals, double* evecs); /* = jacobi */

/* ---- Philox4x32-10 ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double orc_u01(uint32_t a, uint32_t b);
/* per-(chain, step) draws: g (n normals, Box-Muller) and eta in (0,1). */
void orc_step_draws(uint64_t seed, uint32_t tag, uint32_t chain, uint32_t step, int n,
                    double* g, double* eta);
/* the two doubles of block ceil(n/2) of a step: eta and u2 (W-CHnR coordinate j = floor(u2 n)) */
void orc_step_uniforms(uint64_t seed, uint32_t tag, uint32_t chain, uint32_t step, int n, double* eta,
                       double* u2);

/* ---- the boundary oracle ---- */
typedef struct orc_chord_res {
    double t_plus, t_minus;
    int binding;        /* block index of the first strict minimum */
    int degenerate;     /* top-two theta of the binding block equal (rank <= m-2) */
    int outward;        /* boundary start with u^T F1 u <= 0 */
    double theta_max, theta_2;
    int ylen;
    double y[1024 + 8]; /* kernel vector of the binding block (mb <= 1024) */
} orc_chord_res;

/* chord on the line x + t v (Algorithm 2, Lemma 3).
 * F0: carried dense block F_0(x) (NULL = evaluate from x).  F1_0: dense block
 * direction matrix (NULL = compute).  bound >= 0 with unit kernel u: the
 * segment starts on the boundary of block `bound` (Schur deflation O1').
 * Returns 0, or 2 (EPRECOND: x not interior for a non-bound block). */
int orc_chord(const orc_lmi* L, const double* x, const double* F0, const double* F1_0,
              const double* v, int bound, const double* u, orc_chord_res* r);

/* outward unit normal at the hit (lemma:gradient P:752-764):
 * g_k = u^T C_bk u, w = -g/|g|.  Returns 1 if degenerate. */
int orc_normal(const orc_lmi* L, int b, const double* y, int ylen, double* w);

/* s = u - 2<u,w>w  (eq:reflection P:737-747) */
void orc_reflect(int n, const double* u, const double* w, double* s);

/* membership (Algorithm 1): 1 if every block is PD with pivots
 * above 1e-10 * |F_b|_max. */
int orc_membership(const orc_lmi* L, const double* x);

/* ---- walks ---- */
enum { ORC_BILLIARD = 0, ORC_HMC = 1, ORC_HNR = 2, ORC_CHNR = 3, ORC_CHMC = 4 }; /* HnR: Alg. 4; CHnR: P:985-996;
                                                                    CHMC: HMC-r on collocation polynomials P:1146-1158 */
enum { ORC_POT_LINEAR = 0, ORC_POT_GAUSS = 1, ORC_POT_LOGCOSH = 2 };
typedef struct orc_stats {
    int64_t calls, reflections, rejects, degenerates, steps, failures;
} orc_stats;

typedef struct orc_walk_params {
    int kind;
    uint64_t seed;
    uint32_t tag;
    int64_t steps;
    double L;      /* tau of Alg. 5 / Alg. 6 */
    int64_t rho;
    double T;      /* HMC temperature */
    const double* c; /* HMC objective (n) */
    /* ORC_CHMC only (collocation HMC-r for exp(-f), sec:hmcr P:1116-1158): */
    int pot;          /* ORC_POT_*: f = c^T x / T (LINEAR), |x - mu|^2 / (2 sigma^2) (GAUSS),
                         sum_i log cosh((x_i - mu_i) / sigma) (LOGCOSH) */
    const double* mu; /* n (GAUSS, LOGCOSH) */
    double sigma;
    int q;            /* collocation nodes (1..6): trajectory degree d = q + 1 */
    double h;         /* ODE step: one polynomial covers at most [0, h] */
} orc_walk_params;

/* Run chains [chain_begin, chain_end) for p->steps steps from x0 (stride 0:
 * shared start, stride n: per-chain rows).  final_x: (chain_end-chain_begin) x n. */
int orc_walk(const orc_lmi* L, const orc_walk_params* p, int64_t chain_begin, int64_t chain_end,
             const double* x0, int x0_stride, double* final_x, orc_stats* st, int nthreads);

/* State of one chain after exactly max_calls chord calls (parity entry for the
 * GPU round scheduler: one call per active chain per round). */
int orc_replay(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0, int64_t max_calls,
               double* x_out, int64_t* calls_out);

/* Record the first max_refl reflections of one chain (parity entry). */
int orc_trace(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0,
              int64_t max_refl, double* hit_x, double* t, double* w, double* v_after,
              int32_t* binding, int64_t* nrec);
int orc_trace_stats(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0,
                    int64_t max_refl, double* hit_x, double* t, double* w, double* v_after,
                    int32_t* binding, int64_t* nrec, orc_stats* st_out);

/* HMC-r first positive root of det(F(p) + t F1(v) - t^2 F1(c)/(2T)) for one block
 * via the mu-companion + Hessenberg + Francis QR. */
int orc_qep_root(int mb, const double* B0, const double* B1, const double* B2, int bound,
                 const double* u, double* t_plus, double* y);
int orc_hmc_chord(const orc_lmi* L, const double* x, const double* F0, const double* v,
                  const double* c, double T, int bound, const double* u, orc_chord_res* r);

/* ---- collocation HMC-r (sec:hmcr P:1116-1158; Lemma 3 P:587-651 for degree d) ----
 * Collocation ([Lee18]): on [0, h] the trajectory of p'' = -grad f(p),
 * p(0) = x0, p'(0) = v0 is the degree-(q+1) polynomial whose second derivative
 * interpolates -grad f(p(h s_j)) at the q Chebyshev nodes s_j = (1 - cos((2j+1) pi / 2q)) / 2
 * of [0, 1]; the node values come from Picard (fixed-point) iteration.  DESIGN.md R33.
 * orc_colloc_basis: nodes[q] and lcoef[q*q], lcoef[j*q + k] = coefficient of s^k in the
 * Lagrange basis polynomial l_j (Vandermonde solve by Gaussian elimination).
 * orc_colloc_poly: coef[(q+2)*n], coef[k*n + i] = coefficient of t^k of p_i(t); returns
 * the Picard iterations used (stop when the node forces move by <= 1e-14 (1 + max|g|)),
 * or -(ORC_COLLOC_MAXIT) if that never happened (the last iterate is returned). */
#define ORC_COLLOC_MAXIT 64
int orc_colloc_basis(int q, double* nodes, double* lcoef);
int orc_colloc_poly(int n, const orc_walk_params* p, const double* x0, const double* v0, double h,
                    double* coef);
/* First root in (0, tmax] of det(B_0 + t B_1 + ... + t^d B_d) for one block (Lemma 3 with a
 * degree-d curve; PEP by the mu = 1/t companion linearisation of P:320-354 + Francis QR).
 * B: (d+1) row-major mb x mb matrices.  Boundary start (bound != 0, B_0 u = 0): Householder
 * basis of u and the first row of the pencil divided by t (as orc_qep_root).  t_plus = +inf
 * if no root in (0, tmax].  Returns 0, 2 (B_0 not PD), 3 (outward: u^T B_1 u <= 0). */
int orc_pep_root(int mb, int d, const double* B, int bound, const double* u, double tmax, double* t_plus,
                 double* y);
/* chord of the curve p(t) = sum_k coef_k t^k (coef as orc_colloc_poly, degree d) over every
 * block, t in (0, tmax]; F0 = carried dense block F_0(coef_0) (NULL: evaluate). */
int orc_colloc_chord(const orc_lmi* L, const double* F0, const double* coef, int d, double tmax, int bound,
                     const double* u, orc_chord_res* r);

#ifdef __cplusplus
}
#endif
#endif
