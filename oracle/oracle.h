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
enum { ORC_BILLIARD = 0, ORC_HMC = 1, ORC_HNR = 2, ORC_CHNR = 3 }; /* HnR: Alg. 4; CHnR: P:985-996 */
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

#ifdef __cplusplus
}
#endif
#endif
