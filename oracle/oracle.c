/*
 * oracle.c -- plain CPU oracle for arXiv 2010.03817.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Every routine follows the paper
 * step by step with the free choices fixed in SURVEY.md 8(c) / DESIGN.md
 * "Readings".  No blocking, fusion or reordering beyond the definitions:
 *   - Cholesky: column-oriented, unpivoted ("Cholesky").
 *   - symmetric eigen: cyclic Jacobi (north_star: "Jacobi dense symmetric
 *     eigensolver on the Cholesky-transformed pencil").
 *   - QEP: mu-companion + Householder-Hessenberg + Francis QR.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define IDX(i, j, ld) ((size_t)(i) * (size_t)(ld) + (size_t)(j))

static void* xmalloc(size_t nbytes) {
    void* p = malloc(nbytes ? nbytes : 8);
    if (!p) abort();
    return p;
}
static double* dalloc(size_t n) { return (double*)calloc(n ? n : 1, sizeof(double)); }

/* ------------------------------------------------------------------------ */
/* LMI as diagonal blocks (eq:lmi P:70-75)                         */
/* ------------------------------------------------------------------------ */

orc_lmi* orc_lmi_create(int n, int m, const double* A, const double* lo, const double* hi,
                        const double* ball_c, double ball_r, int literal) {
    orc_lmi* L = (orc_lmi*)xmalloc(sizeof(orc_lmi));
    L->n = n;
    L->has_cube = (lo != NULL && hi != NULL);
    L->has_ball = (ball_c != NULL);
    int nb = 1 + (L->has_cube ? 2 * n : 0) + (L->has_ball ? 1 : 0);
    /* sizes of the split blocks */
    int* mbs = (int*)xmalloc(sizeof(int) * nb);
    mbs[0] = m;
    for (int b = 1; b < nb; ++b) mbs[b] = 1;
    if (L->has_ball) mbs[nb - 1] = n + 1;
    double** Cs = (double**)xmalloc(sizeof(double*) * nb);
    for (int b = 0; b < nb; ++b) Cs[b] = dalloc((size_t)(n + 1) * mbs[b] * mbs[b]);
    /* dense block: the A_k (symmetrised (A+A^T)/2 on load) */
    for (int k = 0; k <= n; ++k)
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j)
                Cs[0][(size_t)k * m * m + IDX(i, j, m)] =
                    0.5 * (A[(size_t)k * m * m + IDX(i, j, m)] + A[(size_t)k * m * m + IDX(j, i, m)]);
    if (L->has_cube) {
        for (int i = 0; i < n; ++i) {
            double* up = Cs[1 + 2 * i]; /* hi_i - x_i */
            double* dn = Cs[2 + 2 * i]; /* x_i - lo_i */
            up[0] = hi[i];
            up[i + 1] = -1.0;
            dn[0] = -lo[i];
            dn[i + 1] = 1.0;
        }
    }
    if (L->has_ball) {
        int mb = n + 1;
        double* B = Cs[nb - 1];
        /* [[r I, x - c], [(x - c)^T, r]] */
        for (int i = 0; i < n; ++i) B[IDX(i, i, mb)] = ball_r;
        B[IDX(n, n, mb)] = ball_r;
        for (int i = 0; i < n; ++i) {
            B[IDX(i, n, mb)] = -ball_c[i];
            B[IDX(n, i, mb)] = -ball_c[i];
        }
        for (int k = 1; k <= n; ++k) {
            double* Bk = B + (size_t)k * mb * mb;
            Bk[IDX(k - 1, n, mb)] = 1.0;
            Bk[IDX(n, k - 1, mb)] = 1.0;
        }
    }
    if (!literal) {
        L->nblocks = nb;
        L->mb = mbs;
        L->C = Cs;
        return L;
    }
    /* literal: one block-diagonal matrix of size sum(mb) */
    int tot = 0;
    for (int b = 0; b < nb; ++b) tot += mbs[b];
    double* C = dalloc((size_t)(n + 1) * tot * tot);
    int off = 0;
    for (int b = 0; b < nb; ++b) {
        int s = mbs[b];
        for (int k = 0; k <= n; ++k)
            for (int i = 0; i < s; ++i)
                for (int j = 0; j < s; ++j)
                    C[(size_t)k * tot * tot + IDX(off + i, off + j, tot)] =
                        Cs[b][(size_t)k * s * s + IDX(i, j, s)];
        off += s;
        free(Cs[b]);
    }
    free(Cs);
    free(mbs);
    L->nblocks = 1;
    L->mb = (int*)xmalloc(sizeof(int));
    L->mb[0] = tot;
    L->C = (double**)xmalloc(sizeof(double*));
    L->C[0] = C;
    return L;
}

void orc_lmi_destroy(orc_lmi* L) {
    if (!L) return;
    for (int b = 0; b < L->nblocks; ++b) free(L->C[b]);
    free(L->C);
    free(L->mb);
    free(L);
}
int orc_lmi_nblocks(const orc_lmi* L) { return L->nblocks; }
int orc_lmi_block_size(const orc_lmi* L, int b) { return L->mb[b]; }

void orc_eval_block(const orc_lmi* L, int b, const double* x, double* out) {
    int s = L->mb[b];
    size_t ss = (size_t)s * s;
    const double* C = L->C[b];
    for (size_t e = 0; e < ss; ++e) out[e] = C[e];
    for (int k = 1; k <= L->n; ++k) {
        double xk = x[k - 1];
        const double* Ck = C + (size_t)k * ss;
        for (size_t e = 0; e < ss; ++e) out[e] += xk * Ck[e];
    }
}

void orc_dir_block(const orc_lmi* L, int b, const double* v, double* out) {
    int s = L->mb[b];
    size_t ss = (size_t)s * s;
    const double* C = L->C[b];
    for (size_t e = 0; e < ss; ++e) out[e] = 0.0;
    for (int k = 1; k <= L->n; ++k) {
        double vk = v[k - 1];
        const double* Ck = C + (size_t)k * ss;
        for (size_t e = 0; e < ss; ++e) out[e] += vk * Ck[e];
    }
}

/* ------------------------------------------------------------------------ */
/* Dense linear algebra                                                       */
/* ------------------------------------------------------------------------ */

/* Unpivoted column-oriented Cholesky A = L L^T; Lw row-major lower. */
int orc_cholesky(int m, const double* A, double* Lw) {
    for (size_t e = 0; e < (size_t)m * m; ++e) Lw[e] = 0.0;
    for (int j = 0; j < m; ++j) {
        double d = A[IDX(j, j, m)];
        for (int k = 0; k < j; ++k) d -= Lw[IDX(j, k, m)] * Lw[IDX(j, k, m)];
        if (!(d > 0.0)) return 1;
        double ljj = sqrt(d);
        Lw[IDX(j, j, m)] = ljj;
        for (int i = j + 1; i < m; ++i) {
            double s = A[IDX(i, j, m)];
            for (int k = 0; k < j; ++k) s -= Lw[IDX(i, k, m)] * Lw[IDX(j, k, m)];
            Lw[IDX(i, j, m)] = s / ljj;
        }
    }
    return 0;
}

/* solve L z = b (forward substitution), L lower row-major */
static void forward_sub(int m, const double* Lw, const double* b, double* z) {
    for (int i = 0; i < m; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= Lw[IDX(i, k, m)] * z[k];
        z[i] = s / Lw[IDX(i, i, m)];
    }
}
/* solve L^T z = b (back substitution) */
static void back_sub_T(int m, const double* Lw, const double* b, double* z) {
    for (int i = m - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < m; ++k) s -= Lw[IDX(k, i, m)] * z[k];
        z[i] = s / Lw[IDX(i, i, m)];
    }
}

/* Cyclic (row-cyclic) Jacobi for symmetric A; classical rotation formulas
 * (Golub-Van Loan sym.Schur2).  Stops when off(A)/|A|_F <= 1e-15 or a sweep
 * rotates nothing; cap 50 sweeps.  evecs columns are eigenvectors. */
int orc_jacobi(int m, const double* A0, double* evals, double* evecs) {
    double* A = dalloc((size_t)m * m);
    memcpy(A, A0, sizeof(double) * (size_t)m * m);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) evecs[IDX(i, j, m)] = (i == j) ? 1.0 : 0.0;
    double fro = 0.0;
    for (size_t e = 0; e < (size_t)m * m; ++e) fro += A[e] * A[e];
    fro = sqrt(fro);
    int sweep;
    for (sweep = 0; sweep < 50; ++sweep) {
        double off = 0.0;
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j)
                if (i != j) off += A[IDX(i, j, m)] * A[IDX(i, j, m)];
        off = sqrt(off);
        if (off <= 1e-15 * fro || off == 0.0) break;
        int rotated = 0;
        for (int p = 0; p < m - 1; ++p) {
            for (int q = p + 1; q < m; ++q) {
                double apq = A[IDX(p, q, m)];
                if (apq == 0.0) continue;
                double app = A[IDX(p, p, m)], aqq = A[IDX(q, q, m)];
                double tau = (aqq - app) / (2.0 * apq);
                double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                        : -1.0 / (-tau + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = t * c;
                if (s == 0.0) continue;
                rotated = 1;
                /* A <- J^T A J with J = [[c, s], [-s, c]] in the (p,q) plane */
                for (int k = 0; k < m; ++k) { /* columns p, q */
                    double akp = A[IDX(k, p, m)], akq = A[IDX(k, q, m)];
                    A[IDX(k, p, m)] = c * akp - s * akq;
                    A[IDX(k, q, m)] = s * akp + c * akq;
                }
                for (int k = 0; k < m; ++k) { /* rows p, q */
                    double apk = A[IDX(p, k, m)], aqk = A[IDX(q, k, m)];
                    A[IDX(p, k, m)] = c * apk - s * aqk;
                    A[IDX(q, k, m)] = s * apk + c * aqk;
                }
                A[IDX(p, q, m)] = 0.0;
                A[IDX(q, p, m)] = 0.0;
                for (int k = 0; k < m; ++k) { /* V <- V J */
                    double vkp = evecs[IDX(k, p, m)], vkq = evecs[IDX(k, q, m)];
                    evecs[IDX(k, p, m)] = c * vkp - s * vkq;
                    evecs[IDX(k, q, m)] = s * vkp + c * vkq;
                }
            }
        }
        if (!rotated) break;
    }
    for (int i = 0; i < m; ++i) evals[i] = A[IDX(i, i, m)];
    free(A);
    return sweep >= 50 ? 1 : 0;
}

int orc_sym_eig(int m, const double* A, double* evals, double* evecs) {
    return orc_jacobi(m, A, evals, evecs);
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al. 2011) -- SURVEY 8(c).1 O7                     */
/* ------------------------------------------------------------------------ */

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)M0 * c0;
        uint64_t p1 = (uint64_t)M1 * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += W0;
        k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u = ((a>>6) 2^26 + (b>>6) + 0.5) 2^-52  in [2^-53, 1-2^-53]: never 0 or 1
 * (reading R7; a 53-bit variant rounds its top value to 1.0). */
double orc_u01(uint32_t a, uint32_t b) {
    double hi = (double)(a >> 6);
    double lo = (double)(b >> 6);
    return (hi * 67108864.0 + lo + 0.5) * (1.0 / 4503599627370496.0);
}

void orc_step_draws(uint64_t seed, uint32_t tag, uint32_t chain, uint32_t step, int n,
                    double* g, double* eta) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int nb = (n + 1) / 2;
    const double two_pi = 6.283185307179586476925286766559;
    for (int j = 0; j < nb; ++j) {
        uint32_t ctr[4] = {(uint32_t)j, step, chain, tag};
        uint32_t w[4];
        orc_philox4x32_10(ctr, key, w);
        double u0 = orc_u01(w[0], w[1]);
        double u1 = orc_u01(w[2], w[3]);
        double r = sqrt(-2.0 * log(u0));
        double a = two_pi * u1;
        g[2 * j] = r * cos(a);
        if (2 * j + 1 < n) g[2 * j + 1] = r * sin(a);
    }
    if (eta) {
        uint32_t ctr[4] = {(uint32_t)nb, step, chain, tag};
        uint32_t w[4];
        orc_philox4x32_10(ctr, key, w);
        *eta = orc_u01(w[0], w[1]);
    }
}

/* the two doubles of block ceil(n/2): eta (as orc_step_draws) and the second one, which
   picks the coordinate of a W-CHnR step (R29) */
void orc_step_uniforms(uint64_t seed, uint32_t tag, uint32_t chain, uint32_t step, int n, double* eta,
                       double* u2) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)((n + 1) / 2), step, chain, tag};
    uint32_t w[4];
    orc_philox4x32_10(ctr, key, w);
    *eta = orc_u01(w[0], w[1]);
    *u2 = orc_u01(w[2], w[3]);
}

/* ------------------------------------------------------------------------ */
/* INTERSECTION on one block (Alg. 2; Lemma 3)            */
/* ------------------------------------------------------------------------ */

typedef struct {
    double theta_max, theta_min, theta_2;
} thetas_t;

/* Interior start, F = B_0 > 0, F1 = B_1.  L L^T = F; M = -L^{-1} F1 L^{-T};
 * theta = eig(M) by Jacobi; t+ = 1/theta_max, t- = 1/theta_min;
 * y = L^{-T} z_max is the kernel vector of F + t+ F1. */
static int chord_block_interior(int mb, const double* F, const double* F1, thetas_t* th, double* y) {
    double* Lw = dalloc((size_t)mb * mb);
    if (orc_cholesky(mb, F, Lw)) {
        free(Lw);
        return 1;
    }
    double* X = dalloc((size_t)mb * mb);  /* X = L^{-1} F1 (columns) */
    double* col = dalloc(mb);
    double* z = dalloc(mb);
    for (int j = 0; j < mb; ++j) {
        for (int i = 0; i < mb; ++i) col[i] = F1[IDX(i, j, mb)];
        forward_sub(mb, Lw, col, z);
        for (int i = 0; i < mb; ++i) X[IDX(i, j, mb)] = z[i];
    }
    double* M = dalloc((size_t)mb * mb); /* M = -(L^{-1} X^T)^T = -X L^{-T} */
    for (int j = 0; j < mb; ++j) {
        for (int i = 0; i < mb; ++i) col[i] = X[IDX(j, i, mb)]; /* column j of X^T */
        forward_sub(mb, Lw, col, z);
        for (int i = 0; i < mb; ++i) M[IDX(j, i, mb)] = -z[i];
    }
    for (int i = 0; i < mb; ++i)
        for (int j = 0; j < i; ++j) {
            double s = 0.5 * (M[IDX(i, j, mb)] + M[IDX(j, i, mb)]);
            M[IDX(i, j, mb)] = s;
            M[IDX(j, i, mb)] = s;
        }
    double* ev = dalloc(mb);
    double* V = dalloc((size_t)mb * mb);
    orc_jacobi(mb, M, ev, V);
    int imax = 0, imin = 0;
    for (int i = 1; i < mb; ++i) {
        if (ev[i] > ev[imax]) imax = i;
        if (ev[i] < ev[imin]) imin = i;
    }
    double second = -INFINITY;
    for (int i = 0; i < mb; ++i)
        if (i != imax && ev[i] > second) second = ev[i];
    th->theta_max = ev[imax];
    th->theta_min = ev[imin];
    th->theta_2 = second;
    for (int i = 0; i < mb; ++i) col[i] = V[IDX(i, imax, mb)];
    back_sub_T(mb, Lw, col, y);
    free(Lw); free(X); free(col); free(z); free(M); free(ev); free(V);
    return 0;
}

/* Householder H = I - 2 h h^T/(h^T h), h = u + sign(u_0)|u| e_0: H u = -sign(u_0)|u| e_0 */
static void householder_matrix(int mb, const double* u, double* H) {
    double nu = 0.0;
    for (int i = 0; i < mb; ++i) nu += u[i] * u[i];
    nu = sqrt(nu);
    double* h = dalloc(mb);
    for (int i = 0; i < mb; ++i) h[i] = u[i];
    h[0] += (u[0] >= 0.0 ? 1.0 : -1.0) * nu;
    double hh = 0.0;
    for (int i = 0; i < mb; ++i) hh += h[i] * h[i];
    for (int i = 0; i < mb; ++i)
        for (int j = 0; j < mb; ++j) H[IDX(i, j, mb)] = (i == j ? 1.0 : 0.0) - 2.0 * h[i] * h[j] / hh;
    free(h);
}

static void matmul(int m, const double* A, const double* B, double* C) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += A[IDX(i, k, m)] * B[IDX(k, j, m)];
            C[IDX(i, j, m)] = s;
        }
}

/* H X H for symmetric X */
static void congruence_H(int mb, const double* H, const double* X, double* out) {
    double* T = dalloc((size_t)mb * mb);
    matmul(mb, H, X, T);
    matmul(mb, T, H, out);
    free(T);
}

/* Boundary start (SURVEY O1', reading R6): F u = 0 with unit u known.
 * In the Householder basis F' = H F H = [[0,0],[0,Fh]], F1' = H F1 H =
 * [[a, b^T],[b, V]] and det(F + t F1) = t a det(Fh + t (V - b b^T / a)).
 * Returns 0 ok, 1 Cholesky failure of Fh, 3 outward (a <= 0). */
static int chord_block_boundary(int mb, const double* F, const double* F1, const double* u,
                                thetas_t* th, double* y, int* empty) {
    *empty = 0;
    double* H = dalloc((size_t)mb * mb);
    householder_matrix(mb, u, H);
    double* Fp = dalloc((size_t)mb * mb);
    double* F1p = dalloc((size_t)mb * mb);
    congruence_H(mb, H, F, Fp);
    congruence_H(mb, H, F1, F1p);
    double a = F1p[0];
    int rc = 0;
    if (!(a > 0.0)) {
        rc = 3;
        goto done;
    }
    if (mb == 1) { /* deflated pencil is empty: no constraint from this block */
        *empty = 1;
        th->theta_max = -INFINITY;
        th->theta_min = INFINITY;
        th->theta_2 = -INFINITY;
        y[0] = u[0];
        goto done;
    }
    {
        int md = mb - 1;
        double* Fh = dalloc((size_t)md * md);
        double* S = dalloc((size_t)md * md);
        for (int i = 0; i < md; ++i)
            for (int j = 0; j < md; ++j) {
                Fh[IDX(i, j, md)] = Fp[IDX(i + 1, j + 1, mb)];
                S[IDX(i, j, md)] = F1p[IDX(i + 1, j + 1, mb)] - F1p[IDX(i + 1, 0, mb)] * F1p[IDX(0, j + 1, mb)] / a;
            }
        double* yh = dalloc(md);
        if (chord_block_interior(md, Fh, S, th, yh)) {
            rc = 1;
        } else {
            /* y = H [ -b^T yh / a ; yh ] */
            double bty = 0.0;
            for (int i = 0; i < md; ++i) bty += F1p[IDX(i + 1, 0, mb)] * yh[i];
            double* yt = dalloc(mb);
            yt[0] = -bty / a;
            for (int i = 0; i < md; ++i) yt[i + 1] = yh[i];
            for (int i = 0; i < mb; ++i) {
                double s = 0.0;
                for (int k = 0; k < mb; ++k) s += H[IDX(i, k, mb)] * yt[k];
                y[i] = s;
            }
            free(yt);
        }
        free(Fh); free(S); free(yh);
    }
done:
    free(H); free(Fp); free(F1p);
    return rc;
}

int orc_chord(const orc_lmi* L, const double* x, const double* F0, const double* F1_0,
              const double* v, int bound, const double* u, orc_chord_res* r) {
    r->t_plus = INFINITY;
    r->t_minus = -INFINITY;
    r->binding = -1;
    r->degenerate = 0;
    r->outward = 0;
    r->theta_max = 0.0;
    r->theta_2 = -INFINITY;
    r->ylen = 0;
    int maxmb = 0;
    for (int b = 0; b < L->nblocks; ++b)
        if (L->mb[b] > maxmb) maxmb = L->mb[b];
    if (maxmb > 1024) return 1;
    double* F = dalloc((size_t)maxmb * maxmb);
    double* F1 = dalloc((size_t)maxmb * maxmb);
    double* y = dalloc(maxmb);
    int rc = 0;
    for (int b = 0; b < L->nblocks; ++b) {
        int s = L->mb[b];
        if (b == 0 && F0) memcpy(F, F0, sizeof(double) * (size_t)s * s);
        else orc_eval_block(L, b, x, F);
        if (b == 0 && F1_0) memcpy(F1, F1_0, sizeof(double) * (size_t)s * s);
        else orc_dir_block(L, b, v, F1);
        thetas_t th;
        double tp, tm;
        if (b == bound) {
            int empty = 0;
            int brc = chord_block_boundary(s, F, F1, u, &th, y, &empty);
            if (brc == 3) { /* leaving S immediately */
                r->t_plus = 0.0;
                r->t_minus = 0.0;
                r->binding = b;
                r->outward = 1;
                rc = 0;
                goto out;
            }
            if (brc) { rc = 2; goto out; }
            tm = 0.0;
            tp = (th.theta_max > 0.0) ? 1.0 / th.theta_max : INFINITY;
            if (empty) tp = INFINITY;
        } else {
            if (chord_block_interior(s, F, F1, &th, y)) { rc = 2; goto out; }
            tp = (th.theta_max > 0.0) ? 1.0 / th.theta_max : INFINITY;
            tm = (th.theta_min < 0.0) ? 1.0 / th.theta_min : -INFINITY;
        }
        if (tm > r->t_minus) r->t_minus = tm;
        if (tp < r->t_plus) { /* first strict minimum wins (reading R10) */
            r->t_plus = tp;
            r->binding = b;
            r->theta_max = th.theta_max;
            r->theta_2 = th.theta_2;
            r->ylen = s;
            memcpy(r->y, y, sizeof(double) * s);
            double tol = 1e-12 * fabs(th.theta_max);
            r->degenerate = (s > 1 && th.theta_max - th.theta_2 <= tol) ? 1 : 0;
        }
    }
out:
    free(F); free(F1); free(y);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* REFLECTION (Alg. 3, lemma:gradient P:752-764, eq:reflection)    */
/* ------------------------------------------------------------------------ */

int orc_normal(const orc_lmi* L, int b, const double* y, int ylen, double* w) {
    int s = L->mb[b];
    if (ylen != s) return 1;
    size_t ss = (size_t)s * s;
    double ny = 0.0;
    for (int i = 0; i < s; ++i) ny += y[i] * y[i];
    ny = sqrt(ny);
    if (!(ny > 0.0)) return 1;
    double* u = dalloc(s);
    for (int i = 0; i < s; ++i) u[i] = y[i] / ny;
    double gn = 0.0, cmax = 0.0;
    for (int k = 1; k <= L->n; ++k) {
        const double* Ck = L->C[b] + (size_t)k * ss;
        double g = 0.0;
        for (int i = 0; i < s; ++i) {
            double row = 0.0;
            for (int j = 0; j < s; ++j) row += Ck[IDX(i, j, s)] * u[j];
            g += u[i] * row;
        }
        for (size_t e = 0; e < ss; ++e)
            if (fabs(Ck[e]) > cmax) cmax = fabs(Ck[e]);
        w[k - 1] = g;
        gn += g * g;
    }
    gn = sqrt(gn);
    free(u);
    if (!(gn >= 1e-12 * cmax) || gn == 0.0) return 1;
    for (int k = 0; k < L->n; ++k) w[k] = -w[k] / gn; /* outward */
    return 0;
}

void orc_reflect(int n, const double* u, const double* w, double* s) {
    double d = 0.0;
    for (int i = 0; i < n; ++i) d += u[i] * w[i];
    for (int i = 0; i < n; ++i) s[i] = u[i] - 2.0 * d * w[i];
}

/* MEMBERSHIP (Alg. 1): every block PD with pivots > 1e-10 |F_b|_max */
int orc_membership(const orc_lmi* L, const double* x) {
    int maxmb = 0;
    for (int b = 0; b < L->nblocks; ++b)
        if (L->mb[b] > maxmb) maxmb = L->mb[b];
    double* F = dalloc((size_t)maxmb * maxmb);
    double* Lw = dalloc((size_t)maxmb * maxmb);
    int inside = 1;
    for (int b = 0; b < L->nblocks && inside; ++b) {
        int s = L->mb[b];
        orc_eval_block(L, b, x, F);
        double fmax = 0.0;
        for (size_t e = 0; e < (size_t)s * s; ++e)
            if (fabs(F[e]) > fmax) fmax = fabs(F[e]);
        double eps = 1e-10 * fmax;
        /* Cholesky with the pivot threshold */
        for (size_t e = 0; e < (size_t)s * s; ++e) Lw[e] = 0.0;
        for (int j = 0; j < s && inside; ++j) {
            double d = F[IDX(j, j, s)];
            for (int k = 0; k < j; ++k) d -= Lw[IDX(j, k, s)] * Lw[IDX(j, k, s)];
            if (!(d > eps)) { inside = 0; break; }
            double ljj = sqrt(d);
            Lw[IDX(j, j, s)] = ljj;
            for (int i = j + 1; i < s; ++i) {
                double t = F[IDX(i, j, s)];
                for (int k = 0; k < j; ++k) t -= Lw[IDX(i, k, s)] * Lw[IDX(j, k, s)];
                Lw[IDX(i, j, s)] = t / ljj;
            }
        }
    }
    free(F); free(Lw);
    return inside;
}

/* ------------------------------------------------------------------------ */
/* QEP for HMC-r (P:320-354 companion; eq:boltz_ode P:1440-1446)             */
/* ------------------------------------------------------------------------ */

/* Householder reduction of a general N x N matrix to upper Hessenberg form */
static void hessenberg(int N, double* A) {
    double* v = dalloc(N);
    for (int k = 0; k < N - 2; ++k) {
        double alpha = 0.0;
        for (int i = k + 1; i < N; ++i) alpha += A[IDX(i, k, N)] * A[IDX(i, k, N)];
        alpha = sqrt(alpha);
        if (alpha == 0.0) continue;
        double x0 = A[IDX(k + 1, k, N)];
        if (x0 > 0) alpha = -alpha;
        for (int i = 0; i < N; ++i) v[i] = 0.0;
        v[k + 1] = x0 - alpha;
        for (int i = k + 2; i < N; ++i) v[i] = A[IDX(i, k, N)];
        double vv = 0.0;
        for (int i = k + 1; i < N; ++i) vv += v[i] * v[i];
        if (vv == 0.0) continue;
        /* A <- P A, P = I - 2 v v^T / vv */
        for (int j = 0; j < N; ++j) {
            double s = 0.0;
            for (int i = k + 1; i < N; ++i) s += v[i] * A[IDX(i, j, N)];
            s = 2.0 * s / vv;
            for (int i = k + 1; i < N; ++i) A[IDX(i, j, N)] -= s * v[i];
        }
        /* A <- A P */
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
            for (int j = k + 1; j < N; ++j) s += A[IDX(i, j, N)] * v[j];
            s = 2.0 * s / vv;
            for (int j = k + 1; j < N; ++j) A[IDX(i, j, N)] -= s * v[j];
        }
        for (int i = k + 2; i < N; ++i) A[IDX(i, k, N)] = 0.0;
    }
    free(v);
}

/* eigenvalues of [[a,b],[c,d]] (stable real case) */
static void eig2x2(double a, double b, double c, double d, double* re1, double* im1,
                   double* re2, double* im2) {
    double p = 0.5 * (a - d);
    double disc = p * p + b * c;
    if (disc >= 0.0) {
        double q = sqrt(disc);
        double s = p + (p >= 0.0 ? q : -q);
        *re1 = d + s;
        *re2 = (s != 0.0) ? d - b * c / s : d;
        *im1 = *im2 = 0.0;
    } else {
        *re1 = *re2 = d + p;
        *im1 = sqrt(-disc);
        *im2 = -*im1;
    }
}

/* Francis double-shift QR on an upper Hessenberg matrix (Golub-Van Loan
 * Alg. 7.5.1/7.5.2), eigenvalues only.  Returns 0 ok, 1 no convergence. */
static int francis_qr(int N, double* H, double* wr, double* wi) {
    int hi = N - 1;
    int its = 0, total = 0;
    const double eps = 2.220446049250313e-16;
    double* vtmp = dalloc(3);
    while (hi >= 0) {
        /* find l: smallest index such that H[l..hi] unreduced */
        int l = hi;
        while (l > 0) {
            double s = fabs(H[IDX(l - 1, l - 1, N)]) + fabs(H[IDX(l, l, N)]);
            if (s == 0.0) s = 1.0;
            if (fabs(H[IDX(l, l - 1, N)]) <= eps * s) {
                H[IDX(l, l - 1, N)] = 0.0;
                break;
            }
            --l;
        }
        if (l == hi) {
            wr[hi] = H[IDX(hi, hi, N)];
            wi[hi] = 0.0;
            --hi;
            its = 0;
            continue;
        }
        if (l == hi - 1) {
            eig2x2(H[IDX(hi - 1, hi - 1, N)], H[IDX(hi - 1, hi, N)], H[IDX(hi, hi - 1, N)],
                   H[IDX(hi, hi, N)], &wr[hi - 1], &wi[hi - 1], &wr[hi], &wi[hi]);
            hi -= 2;
            its = 0;
            continue;
        }
        if (++total > 60 * N) { free(vtmp); return 1; }
        ++its;
        int p = l, q = hi;
        double s, t;
        if (its == 10 || its == 20) { /* exceptional shift */
            double w = fabs(H[IDX(q, q - 1, N)]) + fabs(H[IDX(q - 1, q - 2, N)]);
            s = 1.5 * w;
            t = w * w;
        } else {
            s = H[IDX(q - 1, q - 1, N)] + H[IDX(q, q, N)];
            t = H[IDX(q - 1, q - 1, N)] * H[IDX(q, q, N)] - H[IDX(q - 1, q, N)] * H[IDX(q, q - 1, N)];
        }
        double x = H[IDX(p, p, N)] * H[IDX(p, p, N)] + H[IDX(p, p + 1, N)] * H[IDX(p + 1, p, N)] -
                   s * H[IDX(p, p, N)] + t;
        double y = H[IDX(p + 1, p, N)] * (H[IDX(p, p, N)] + H[IDX(p + 1, p + 1, N)] - s);
        double z = H[IDX(p + 1, p, N)] * H[IDX(p + 2, p + 1, N)];
        for (int k = p; k <= q - 2; ++k) {
            /* 3-element Householder zeroing y, z */
            double al = sqrt(x * x + y * y + z * z);
            if (al != 0.0) {
                if (x > 0) al = -al;
                double v0 = x - al, v1 = y, v2 = z;
                double vv = v0 * v0 + v1 * v1 + v2 * v2;
                if (vv != 0.0) {
                    int r = (k - 1 > p) ? k - 1 : p;
                    for (int j = r; j <= q; ++j) {
                        double d = v0 * H[IDX(k, j, N)] + v1 * H[IDX(k + 1, j, N)] + v2 * H[IDX(k + 2, j, N)];
                        d = 2.0 * d / vv;
                        H[IDX(k, j, N)] -= d * v0;
                        H[IDX(k + 1, j, N)] -= d * v1;
                        H[IDX(k + 2, j, N)] -= d * v2;
                    }
                    int rmax = (k + 3 < q) ? k + 3 : q;
                    for (int i = p; i <= rmax; ++i) {
                        double d = v0 * H[IDX(i, k, N)] + v1 * H[IDX(i, k + 1, N)] + v2 * H[IDX(i, k + 2, N)];
                        d = 2.0 * d / vv;
                        H[IDX(i, k, N)] -= d * v0;
                        H[IDX(i, k + 1, N)] -= d * v1;
                        H[IDX(i, k + 2, N)] -= d * v2;
                    }
                }
            }
            x = H[IDX(k + 1, k, N)];
            y = H[IDX(k + 2, k, N)];
            if (k < q - 2) z = H[IDX(k + 3, k, N)];
        }
        /* final 2-element Householder on rows q-1, q */
        {
            double al = sqrt(x * x + y * y);
            if (al != 0.0) {
                if (x > 0) al = -al;
                double v0 = x - al, v1 = y;
                double vv = v0 * v0 + v1 * v1;
                if (vv != 0.0) {
                    for (int j = q - 2; j <= q; ++j) {
                        double d = 2.0 * (v0 * H[IDX(q - 1, j, N)] + v1 * H[IDX(q, j, N)]) / vv;
                        H[IDX(q - 1, j, N)] -= d * v0;
                        H[IDX(q, j, N)] -= d * v1;
                    }
                    for (int i = p; i <= q; ++i) {
                        double d = 2.0 * (v0 * H[IDX(i, q - 1, N)] + v1 * H[IDX(i, q, N)]) / vv;
                        H[IDX(i, q - 1, N)] -= d * v0;
                        H[IDX(i, q, N)] -= d * v1;
                    }
                }
            }
        }
        /* clean below the subdiagonal */
        for (int i = p + 2; i <= q; ++i)
            for (int j = p; j < i - 1; ++j) H[IDX(i, j, N)] = 0.0;
    }
    free(vtmp);
    return 0;
}

/* largest real positive eigenvalue of the mu-companion [[-N1, -N2],[I, 0]] */
static int companion_max_pos(int md, const double* N1, const double* N2, double* mu_out) {
    int N = 2 * md;
    double* Cm = dalloc((size_t)N * N);
    for (int i = 0; i < md; ++i) {
        for (int j = 0; j < md; ++j) {
            Cm[IDX(i, j, N)] = -N1[IDX(i, j, md)];
            Cm[IDX(i, md + j, N)] = -N2[IDX(i, j, md)];
        }
        Cm[IDX(md + i, i, N)] = 1.0;
    }
    hessenberg(N, Cm);
    double* wr = dalloc(N);
    double* wi = dalloc(N);
    int rc = francis_qr(N, Cm, wr, wi);
    double best = 0.0;
    int found = 0;
    for (int i = 0; i < N; ++i) {
        if (fabs(wi[i]) <= 1e-8 * (1.0 + fabs(wr[i])) && wr[i] > 0.0) {
            if (!found || wr[i] > best) best = wr[i];
            found = 1;
        }
    }
    *mu_out = found ? best : 0.0;
    free(Cm); free(wr); free(wi);
    return rc;
}

/* kernel vector of symmetric G: eigenvector of the smallest |eigenvalue| (Jacobi) */
static void null_vector(int mb, const double* G, double* y) {
    double* ev = dalloc(mb);
    double* V = dalloc((size_t)mb * mb);
    orc_jacobi(mb, G, ev, V);
    int best = 0;
    for (int i = 1; i < mb; ++i)
        if (fabs(ev[i]) < fabs(ev[best])) best = i;
    for (int i = 0; i < mb; ++i) y[i] = V[IDX(i, best, mb)];
    free(ev); free(V);
}

/* First positive root of det(B0 + t B1 + t^2 B2) for one block.
 * Interior start (bound == 0): L L^T = B0, M_k = L^{-1} B_k L^{-T},
 * companion [[-M1, -M2],[I,0]] in mu = 1/t.
 * Boundary start (bound != 0, B0 u = 0): Householder basis of u; divide the
 * first row of G(t) by t -> G~(t) = G~0 + t G~1 + t^2 G~2 with
 * G~0 = [[a1, b1^T],[0, Bh]] invertible; companion of G~0^{-1} G~k.
 * t_plus = +inf if no positive root.  y = kernel of G(t_plus) (Jacobi). */
int orc_qep_root(int mb, const double* B0, const double* B1, const double* B2, int bound,
                 const double* u, double* t_plus, double* y) {
    int rc = 0;
    double mu = 0.0;
    if (!bound) {
        double* Lw = dalloc((size_t)mb * mb);
        if (orc_cholesky(mb, B0, Lw)) { free(Lw); return 2; }
        double* M1 = dalloc((size_t)mb * mb);
        double* M2 = dalloc((size_t)mb * mb);
        double* col = dalloc(mb);
        double* z = dalloc(mb);
        double* X = dalloc((size_t)mb * mb);
        for (int pass = 0; pass < 2; ++pass) {
            const double* B = pass ? B2 : B1;
            double* Mo = pass ? M2 : M1;
            for (int j = 0; j < mb; ++j) {
                for (int i = 0; i < mb; ++i) col[i] = B[IDX(i, j, mb)];
                forward_sub(mb, Lw, col, z);
                for (int i = 0; i < mb; ++i) X[IDX(i, j, mb)] = z[i];
            }
            for (int j = 0; j < mb; ++j) {
                for (int i = 0; i < mb; ++i) col[i] = X[IDX(j, i, mb)];
                forward_sub(mb, Lw, col, z);
                for (int i = 0; i < mb; ++i) Mo[IDX(j, i, mb)] = z[i];
            }
        }
        rc = companion_max_pos(mb, M1, M2, &mu);
        free(Lw); free(M1); free(M2); free(col); free(z); free(X);
    } else {
        double* H = dalloc((size_t)mb * mb);
        householder_matrix(mb, u, H);
        double* P0 = dalloc((size_t)mb * mb);
        double* P1 = dalloc((size_t)mb * mb);
        double* P2 = dalloc((size_t)mb * mb);
        congruence_H(mb, H, B0, P0);
        congruence_H(mb, H, B1, P1);
        congruence_H(mb, H, B2, P2);
        double a1 = P1[0];
        if (!(a1 > 0.0)) {
            free(H); free(P0); free(P1); free(P2);
            *t_plus = 0.0;
            return 3;
        }
        /* G~0 = [[a1, b1^T],[0, Bh]], G~1 = [[a2, b2^T],[b1, V1]], G~2 = [[0,0],[b2, V2]] */
        int md = mb;
        double* G1 = dalloc((size_t)md * md);
        double* G2 = dalloc((size_t)md * md);
        for (int j = 0; j < md; ++j) {
            G1[IDX(0, j, md)] = P2[IDX(0, j, mb)];
            G2[IDX(0, j, md)] = 0.0;
        }
        for (int i = 1; i < md; ++i)
            for (int j = 0; j < md; ++j) {
                G1[IDX(i, j, md)] = P1[IDX(i, j, mb)];
                G2[IDX(i, j, md)] = P2[IDX(i, j, mb)];
            }
        /* N_k = G~0^{-1} G~k via Cholesky of Bh and block back substitution */
        int mh = mb - 1;
        double* Lw = dalloc((size_t)(mh > 0 ? mh : 1) * (mh > 0 ? mh : 1));
        double* Bh = dalloc((size_t)(mh > 0 ? mh : 1) * (mh > 0 ? mh : 1));
        for (int i = 0; i < mh; ++i)
            for (int j = 0; j < mh; ++j) Bh[IDX(i, j, mh)] = P0[IDX(i + 1, j + 1, mb)];
        if (mh > 0 && orc_cholesky(mh, Bh, Lw)) rc = 2;
        double* N1 = dalloc((size_t)md * md);
        double* N2 = dalloc((size_t)md * md);
        double* col = dalloc(md);
        double* z = dalloc(md);
        double* z2 = dalloc(md);
        for (int pass = 0; pass < 2 && !rc; ++pass) {
            const double* G = pass ? G2 : G1;
            double* No = pass ? N2 : N1;
            for (int j = 0; j < md; ++j) {
                for (int i = 1; i < md; ++i) col[i - 1] = G[IDX(i, j, md)];
                if (mh > 0) {
                    forward_sub(mh, Lw, col, z);
                    back_sub_T(mh, Lw, z, z2);
                }
                double s = G[IDX(0, j, md)];
                for (int i = 0; i < mh; ++i) s -= P1[IDX(0, i + 1, mb)] * z2[i];
                No[IDX(0, j, md)] = s / a1;
                for (int i = 0; i < mh; ++i) No[IDX(i + 1, j, md)] = z2[i];
            }
        }
        if (!rc) rc = companion_max_pos(md, N1, N2, &mu);
        free(H); free(P0); free(P1); free(P2); free(G1); free(G2); free(Lw); free(Bh);
        free(N1); free(N2); free(col); free(z); free(z2);
    }
    if (rc) return rc;
    *t_plus = (mu > 0.0) ? 1.0 / mu : INFINITY;
    if (y) {
        if (isfinite(*t_plus)) {
            double tp = *t_plus;
            double* G = dalloc((size_t)mb * mb);
            for (size_t e = 0; e < (size_t)mb * mb; ++e) G[e] = B0[e] + tp * B1[e] + tp * tp * B2[e];
            null_vector(mb, G, y);
            free(G);
        } else {
            for (int i = 0; i < mb; ++i) y[i] = 0.0;
        }
    }
    return 0;
}

/* HMC-r chord: G_b(t) = F_b(p) + t F1_b(v) - t^2 F1_b(c)/(2T), per block */
int orc_hmc_chord(const orc_lmi* L, const double* x, const double* F0, const double* v,
                  const double* c, double T, int bound, const double* u, orc_chord_res* r) {
    r->t_plus = INFINITY;
    r->t_minus = -INFINITY;
    r->binding = -1;
    r->degenerate = 0;
    r->outward = 0;
    r->ylen = 0;
    int maxmb = 0;
    for (int b = 0; b < L->nblocks; ++b)
        if (L->mb[b] > maxmb) maxmb = L->mb[b];
    if (maxmb > 1024) return 1;
    double* F = dalloc((size_t)maxmb * maxmb);
    double* F1 = dalloc((size_t)maxmb * maxmb);
    double* F2 = dalloc((size_t)maxmb * maxmb);
    double* y = dalloc(maxmb);
    int rc = 0;
    for (int b = 0; b < L->nblocks; ++b) {
        int s = L->mb[b];
        size_t ss = (size_t)s * s;
        if (b == 0 && F0) memcpy(F, F0, sizeof(double) * ss);
        else orc_eval_block(L, b, x, F);
        orc_dir_block(L, b, v, F1);
        orc_dir_block(L, b, c, F2);
        for (size_t e = 0; e < ss; ++e) F2[e] = -F2[e] / (2.0 * T);
        double tp;
        int brc = orc_qep_root(s, F, F1, F2, b == bound, (b == bound) ? u : NULL, &tp, y);
        if (brc == 3) {
            r->t_plus = 0.0;
            r->binding = b;
            r->outward = 1;
            goto out;
        }
        if (brc) { rc = 2; goto out; }
        if (tp < r->t_plus) {
            r->t_plus = tp;
            r->binding = b;
            r->ylen = s;
            memcpy(r->y, y, sizeof(double) * s);
        }
    }
out:
    free(F); free(F1); free(F2); free(y);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Collocation HMC-r (sec:hmcr P:1116-1158; R33)                    */
/* ------------------------------------------------------------------------ */

/* Chebyshev nodes of [0, 1] and the monomial coefficients of the Lagrange basis:
 * column j of V^{-1}, V[i][k] = s_i^k, by Gaussian elimination with partial pivoting. */
int orc_colloc_basis(int q, double* nodes, double* lcoef) {
    if (q < 1 || q > 16) return 1;
    const double pi = 3.14159265358979323846;
    for (int j = 0; j < q; ++j) nodes[j] = 0.5 * (1.0 - cos((2.0 * j + 1.0) * pi / (2.0 * q)));
    double* A = dalloc((size_t)q * q);
    double* b = dalloc(q);
    for (int j = 0; j < q; ++j) {
        for (int i = 0; i < q; ++i) {
            double p = 1.0;
            for (int k = 0; k < q; ++k) {
                A[IDX(i, k, q)] = p;
                p *= nodes[i];
            }
            b[i] = (i == j) ? 1.0 : 0.0;
        }
        for (int c = 0; c < q; ++c) {
            int piv = c;
            for (int r = c + 1; r < q; ++r)
                if (fabs(A[IDX(r, c, q)]) > fabs(A[IDX(piv, c, q)])) piv = r;
            if (piv != c) {
                for (int k = 0; k < q; ++k) {
                    double t = A[IDX(c, k, q)];
                    A[IDX(c, k, q)] = A[IDX(piv, k, q)];
                    A[IDX(piv, k, q)] = t;
                }
                double t = b[c]; b[c] = b[piv]; b[piv] = t;
            }
            for (int r = c + 1; r < q; ++r) {
                double f = A[IDX(r, c, q)] / A[IDX(c, c, q)];
                for (int k = c; k < q; ++k) A[IDX(r, k, q)] -= f * A[IDX(c, k, q)];
                b[r] -= f * b[c];
            }
        }
        for (int k = q - 1; k >= 0; --k) {
            double s = b[k];
            for (int r = k + 1; r < q; ++r) s -= A[IDX(k, r, q)] * lcoef[(size_t)j * q + r];
            lcoef[(size_t)j * q + k] = s / A[IDX(k, k, q)];
        }
    }
    free(A); free(b);
    return 0;
}

/* grad f (ORC_POT_*) */
static void pot_grad(const orc_walk_params* p, int n, const double* x, double* g) {
    for (int i = 0; i < n; ++i) {
        if (p->pot == ORC_POT_LINEAR) g[i] = p->c[i] / p->T;
        else if (p->pot == ORC_POT_GAUSS) g[i] = (x[i] - p->mu[i]) / (p->sigma * p->sigma);
        else g[i] = tanh((x[i] - p->mu[i]) / p->sigma) / p->sigma;
    }
}

/* coefficients of p(t) from the node forces G (q x n):
 * p(t) = x0 + v0 t + sum_k (sum_j l_jk G_j) t^(k+2) / (h^k (k+1)(k+2)) */
static void colloc_coef(int n, int q, const double* lcoef, const double* G, const double* x0, const double* v0,
                        double h, double* coef) {
    for (int i = 0; i < n; ++i) {
        coef[i] = x0[i];
        coef[n + i] = v0[i];
    }
    double hk = 1.0;
    for (int k = 0; k < q; ++k) {
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < q; ++j) s += lcoef[(size_t)j * q + k] * G[(size_t)j * n + i];
            coef[(size_t)(k + 2) * n + i] = s / (hk * (double)(k + 1) * (double)(k + 2));
        }
        hk *= h;
    }
}

/* p(t) by Horner (coef of degree d, n columns) */
static void poly_eval(int n, int d, const double* coef, double t, double* out) {
    for (int i = 0; i < n; ++i) {
        double a = coef[(size_t)d * n + i];
        for (int k = d - 1; k >= 0; --k) a = a * t + coef[(size_t)k * n + i];
        out[i] = a;
    }
}

/* p'(t) by Horner */
static void poly_deriv(int n, int d, const double* coef, double t, double* out) {
    for (int i = 0; i < n; ++i) {
        double a = (double)d * coef[(size_t)d * n + i];
        for (int k = d - 1; k >= 1; --k) a = a * t + (double)k * coef[(size_t)k * n + i];
        out[i] = a;
    }
}

int orc_colloc_poly(int n, const orc_walk_params* p, const double* x0, const double* v0, double h,
                    double* coef) {
    int q = p->q, d = q + 1;
    double nodes[16], lcoef[256];
    if (orc_colloc_basis(q, nodes, lcoef)) return 0;
    double* G = dalloc((size_t)q * n);
    double* xj = dalloc(n);
    double* gj = dalloc(n);
    pot_grad(p, n, x0, gj);
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < n; ++i) G[(size_t)j * n + i] = -gj[i];
    int used = -ORC_COLLOC_MAXIT;
    for (int it = 0; it < ORC_COLLOC_MAXIT; ++it) {
        colloc_coef(n, q, lcoef, G, x0, v0, h, coef);
        double delta = 0.0, gmax = 0.0;
        for (int j = 0; j < q; ++j) {
            poly_eval(n, d, coef, nodes[j] * h, xj);
            pot_grad(p, n, xj, gj);
            for (int i = 0; i < n; ++i) {
                double gn = -gj[i];
                delta = fmax(delta, fabs(gn - G[(size_t)j * n + i]));
                gmax = fmax(gmax, fabs(gn));
                G[(size_t)j * n + i] = gn;
            }
        }
        if (delta <= 1e-14 * (1.0 + gmax)) {
            used = it + 1;
            break;
        }
    }
    colloc_coef(n, q, lcoef, G, x0, v0, h, coef);
    free(G); free(xj); free(gj);
    return used;
}

/* largest real positive eigenvalue of the degree-d mu-companion
 * [[-N_1, -N_2, ..., -N_d], [I, 0, ..., 0], ..., [0, ..., I, 0]] (P:320-354 for the reversed
 * polynomial mu^d I + mu^(d-1) N_1 + ... + N_d) */
static int companion_max_pos_d(int md, int d, double* const* Nk, double* mu_out) {
    int N = d * md;
    double* Cm = dalloc((size_t)N * N);
    for (int i = 0; i < md; ++i) {
        for (int k = 0; k < d; ++k)
            for (int j = 0; j < md; ++j) Cm[IDX(i, (size_t)k * md + j, N)] = -Nk[k][IDX(i, j, md)];
    }
    for (int r = md; r < N; ++r) Cm[IDX(r, r - md, N)] = 1.0;
    hessenberg(N, Cm);
    double* wr = dalloc(N);
    double* wi = dalloc(N);
    int rc = francis_qr(N, Cm, wr, wi);
    double best = 0.0;
    int found = 0;
    for (int i = 0; i < N; ++i) {
        if (fabs(wi[i]) <= 1e-8 * (1.0 + fabs(wr[i])) && wr[i] > 0.0) {
            if (!found || wr[i] > best) best = wr[i];
            found = 1;
        }
    }
    *mu_out = found ? best : 0.0;
    free(Cm); free(wr); free(wi);
    return rc;
}

int orc_pep_root(int mb, int d, const double* B, int bound, const double* u, double tmax, double* t_plus,
                 double* y) {
    size_t ss = (size_t)mb * mb;
    int rc = 0;
    double mu = 0.0;
    if (d < 1) return 1;
    double** Nk = (double**)xmalloc(sizeof(double*) * d);
    for (int k = 0; k < d; ++k) Nk[k] = dalloc(ss);
    double* col = dalloc(mb);
    double* z = dalloc(mb);
    double* z2 = dalloc(mb);
    if (!bound) {
        /* L L^T = B_0, N_k = L^{-1} B_k L^{-T} */
        double* Lw = dalloc(ss);
        double* X = dalloc(ss);
        if (orc_cholesky(mb, B, Lw)) rc = 2;
        for (int k = 1; k <= d && !rc; ++k) {
            const double* Bk = B + (size_t)k * ss;
            for (int j = 0; j < mb; ++j) {
                for (int i = 0; i < mb; ++i) col[i] = Bk[IDX(i, j, mb)];
                forward_sub(mb, Lw, col, z);
                for (int i = 0; i < mb; ++i) X[IDX(i, j, mb)] = z[i];
            }
            for (int j = 0; j < mb; ++j) {
                for (int i = 0; i < mb; ++i) col[i] = X[IDX(j, i, mb)];
                forward_sub(mb, Lw, col, z);
                for (int i = 0; i < mb; ++i) Nk[k - 1][IDX(j, i, mb)] = z[i];
            }
        }
        if (!rc) rc = companion_max_pos_d(mb, d, Nk, &mu);
        free(Lw); free(X);
    } else {
        /* P_k = H B_k H; the first row of P(t) divided by t: G~_k row 0 = P_(k+1) row 0
         * (k < d; 0 for k = d), rows >= 1 = those of P_k; G~_0 = [[a1, b1^T], [0, Bh]] */
        double* H = dalloc(ss);
        householder_matrix(mb, u, H);
        double** P = (double**)xmalloc(sizeof(double*) * (d + 1));
        for (int k = 0; k <= d; ++k) {
            P[k] = dalloc(ss);
            congruence_H(mb, H, B + (size_t)k * ss, P[k]);
        }
        double a1 = P[1][0];
        int mh = mb - 1;
        double* Lw = dalloc((size_t)(mh > 0 ? mh : 1) * (mh > 0 ? mh : 1));
        double* Bh = dalloc((size_t)(mh > 0 ? mh : 1) * (mh > 0 ? mh : 1));
        double* Gk = dalloc(ss);
        if (!(a1 > 0.0)) {
            rc = 3;
        } else {
            for (int i = 0; i < mh; ++i)
                for (int j = 0; j < mh; ++j) Bh[IDX(i, j, mh)] = P[0][IDX(i + 1, j + 1, mb)];
            if (mh > 0 && orc_cholesky(mh, Bh, Lw)) rc = 2;
        }
        for (int k = 1; k <= d && !rc; ++k) {
            for (int j = 0; j < mb; ++j) {
                Gk[IDX(0, j, mb)] = (k < d) ? P[k + 1][IDX(0, j, mb)] : 0.0;
                for (int i = 1; i < mb; ++i) Gk[IDX(i, j, mb)] = P[k][IDX(i, j, mb)];
            }
            /* N_k = G~_0^{-1} G~_k by block back substitution */
            for (int j = 0; j < mb; ++j) {
                for (int i = 1; i < mb; ++i) col[i - 1] = Gk[IDX(i, j, mb)];
                if (mh > 0) {
                    forward_sub(mh, Lw, col, z);
                    back_sub_T(mh, Lw, z, z2);
                }
                double s = Gk[IDX(0, j, mb)];
                for (int i = 0; i < mh; ++i) s -= P[1][IDX(0, i + 1, mb)] * z2[i];
                Nk[k - 1][IDX(0, j, mb)] = s / a1;
                for (int i = 0; i < mh; ++i) Nk[k - 1][IDX(i + 1, j, mb)] = z2[i];
            }
        }
        if (!rc) rc = companion_max_pos_d(mb, d, Nk, &mu);
        for (int k = 0; k <= d; ++k) free(P[k]);
        free(P); free(H); free(Lw); free(Bh); free(Gk);
    }
    for (int k = 0; k < d; ++k) free(Nk[k]);
    free(Nk); free(col); free(z); free(z2);
    if (rc == 3) {
        *t_plus = 0.0;
        return 3;
    }
    if (rc) return rc;
    *t_plus = (mu > 0.0 && 1.0 / mu <= tmax) ? 1.0 / mu : INFINITY;
    if (y) {
        if (isfinite(*t_plus)) {
            double tp = *t_plus;
            double* G = dalloc(ss);
            for (size_t e = 0; e < ss; ++e) {
                double a = B[(size_t)d * ss + e];
                for (int k = d - 1; k >= 0; --k) a = a * tp + B[(size_t)k * ss + e];
                G[e] = a;
            }
            null_vector(mb, G, y);
            free(G);
        } else {
            for (int i = 0; i < mb; ++i) y[i] = 0.0;
        }
    }
    return 0;
}

int orc_colloc_chord(const orc_lmi* L, const double* F0, const double* coef, int d, double tmax, int bound,
                     const double* u, orc_chord_res* r) {
    int n = L->n;
    r->t_plus = INFINITY;
    r->t_minus = -INFINITY;
    r->binding = -1;
    r->degenerate = 0;
    r->outward = 0;
    r->ylen = 0;
    int maxmb = 0;
    for (int b = 0; b < L->nblocks; ++b)
        if (L->mb[b] > maxmb) maxmb = L->mb[b];
    if (maxmb > 1024) return 1;
    size_t mm = (size_t)maxmb * maxmb;
    double* B = dalloc((size_t)(d + 1) * mm);
    double* y = dalloc(maxmb);
    int rc = 0;
    for (int b = 0; b < L->nblocks; ++b) {
        int s = L->mb[b];
        size_t ss = (size_t)s * s;
        if (b == 0 && F0) memcpy(B, F0, sizeof(double) * ss);
        else orc_eval_block(L, b, coef, B);
        for (int k = 1; k <= d; ++k) orc_dir_block(L, b, coef + (size_t)k * n, B + (size_t)k * ss);
        double tp;
        int brc = orc_pep_root(s, d, B, b == bound, (b == bound) ? u : NULL, tmax, &tp, y);
        if (brc == 3) {
            r->t_plus = 0.0;
            r->binding = b;
            r->outward = 1;
            goto out;
        }
        if (brc) { rc = 2; goto out; }
        if (tp < r->t_plus) {
            r->t_plus = tp;
            r->binding = b;
            r->ylen = s;
            memcpy(r->y, y, sizeof(double) * s);
        }
    }
out:
    free(B); free(y);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Walks                                                                      */
/* ------------------------------------------------------------------------ */

typedef struct {
    double* x;    /* n   */
    double* F;    /* m*m dense block, carried */
    double* xs;   /* saved x_i  */
    double* Fs;   /* saved F(x_i) */
    double* v;
    double* g;
    double* F1;
    double* F2c;  /* dense-block F1(c) for HMC */
    double* w;
    double* u;    /* unit kernel vector of the bound block */
    orc_chord_res* res;
    int64_t budget; /* stop after this many chord calls (-1: none) */
    double* coef; /* collocation polynomial, (q+2) x n (q <= 6) */
    double* Fk;   /* dense-block F1(coef_k), k = 1..q+1 */
} walk_ws;

static void ws_init(walk_ws* W, const orc_lmi* L) {
    int n = L->n, m = L->mb[0];
    W->x = dalloc(n); W->xs = dalloc(n); W->v = dalloc(n); W->g = dalloc(n); W->w = dalloc(n);
    W->F = dalloc((size_t)m * m); W->Fs = dalloc((size_t)m * m); W->F1 = dalloc((size_t)m * m);
    W->F2c = dalloc((size_t)m * m);
    int maxmb = 0;
    for (int b = 0; b < L->nblocks; ++b)
        if (L->mb[b] > maxmb) maxmb = L->mb[b];
    W->u = dalloc(maxmb);
    W->res = (orc_chord_res*)xmalloc(sizeof(orc_chord_res));
    W->budget = -1;
    W->coef = dalloc((size_t)8 * n);
    W->Fk = dalloc((size_t)7 * m * m);
}
static void ws_free(walk_ws* W) {
    free(W->x); free(W->xs); free(W->v); free(W->g); free(W->w); free(W->F); free(W->Fs);
    free(W->F1); free(W->F2c); free(W->u); free(W->res); free(W->coef); free(W->Fk);
}

typedef struct {
    int64_t max_refl, nrec;
    double *hit_x, *t, *w, *v_after;
    int32_t* binding;
    int stop; /* end the walk right after the max_refl-th record (no arithmetic change) */
} trace_rec;

/* One step of the Billiard walk (Alg. 5; readings R4, R5) or
 * of HMC-r (Alg. 6; eq:boltz_ode).  Returns 0, or 2 if the start
 * point is not interior. */
/* A point of the chord [t-, t+] drawn from pi_l (Alg. 4 line 4) for the Boltzmann law
 * pi ~ exp(-c^T x / T) (sec:optimization P:1420-1424): along x + t v the density is
 * proportional to exp(-a t), a = c^T v / T, i.e. a truncated exponential; inverse CDF with
 * s = -log(1 - eta (1 - exp(-|a| d))) / |a| measured from the end where the density is largest
 * (d = t+ - t-), written with log1p / expm1.  |a| d < 1e-12: the uniform point s = eta d.
 * s is kept in [2^-26 d, (1 - 2^-26) d] (R30): near a face the chord ends carry
 * relative errors up to ~eps |M| / |theta|, and a closer point would land on the boundary. */
static double boltz_chord_point(double tm, double tp, double a, double eta) {
    double d = tp - tm, b = fabs(a) * d, s;
    if (b < 1e-12)
        s = eta * d;
    else
        s = -log1p(eta * expm1(-b)) / fabs(a);
    s = fmin(fmax(s, 0x1p-26 * d), (1.0 - 0x1p-26) * d);
    return a >= 0.0 ? tm + s : tp - s;
}

/* One step of Hit-and-Run (Alg. 4 alg:hitandrun P:939-965) or of coordinate-directions
 * Hit-and-Run (W-CHnR) for the uniform law: v ~ U(sphere) (HnR) or v = e_j with
 * j uniform in [n] (CHnR); (t-, t+) = INTERSECTION (one chord, Lemma 3); the next point is
 * drawn from pi restricted to [p + t- v, p + t+ v] -- uniform: p += (t- + eta (t+ - t-)) v;
 * Boltzmann (c given, 0 < T < inf): boltz_chord_point -- and F(p) is carried as
 * F += t F1(v) (for e_j, F1 = A_j: the O(m^2) update of P:988-995). */
static int hnr_step(const orc_lmi* L, const orc_walk_params* p, uint32_t chain, uint32_t step, walk_ws* W,
                    orc_stats* st) {
    int n = L->n, m = L->mb[0];
    size_t mm = (size_t)m * m;
    double eta;
    if (p->kind == ORC_HNR) {
        orc_step_draws(p->seed, p->tag, chain, step, n, W->g, &eta);
        double gn = 0.0;
        for (int i = 0; i < n; ++i) gn += W->g[i] * W->g[i];
        gn = sqrt(gn);
        for (int i = 0; i < n; ++i) W->v[i] = W->g[i] / gn;
    } else {
        double u2;
        orc_step_uniforms(p->seed, p->tag, chain, step, n, &eta, &u2);
        int j = (int)(u2 * (double)n);
        if (j > n - 1) j = n - 1;
        for (int i = 0; i < n; ++i) W->v[i] = (i == j) ? 1.0 : 0.0;
    }
    st->steps += 1;
    if (W->budget >= 0 && st->calls >= W->budget) return 5;
    orc_dir_block(L, 0, W->v, W->F1);
    orc_chord_res* r = W->res;
    int rc = orc_chord(L, W->x, W->F, W->F1, W->v, -1, NULL, r);
    st->calls += 1;
    if (rc) return rc;
    double t;
    if (p->c && p->T > 0.0 && isfinite(p->T)) { /* Boltzmann pi_l (sec:optimization) */
        double cv = 0.0;
        for (int i = 0; i < n; ++i) cv += p->c[i] * W->v[i];
        t = boltz_chord_point(r->t_minus, r->t_plus, cv / p->T, eta);
    } else { /* uniform pi_l */
        t = r->t_minus + eta * (r->t_plus - r->t_minus);
    }
    for (int i = 0; i < n; ++i) W->x[i] += t * W->v[i];
    for (size_t e = 0; e < mm; ++e) W->F[e] += t * W->F1[e];
    return 0;
}

/* One step of collocation HMC-r (Alg. 6 P:1079-1115 with the polynomial trajectories of
 * P:1146-1158; R33): l = tau eta, v ~ N(0, I); then, while l > 0, the segment
 * [0, h'] with h' = min(h, l) follows the collocation polynomial p(t) from (x, v); its chord
 * is the first root of det F(p(t)) in (0, h'] over every block (Lemma 3 for degree d = q + 1).
 * No root: x = p(h'), v = p'(h'), l -= h' (not a reflection).  Root t+: x = p(t+), the
 * velocity p'(t+) is reflected at the hit (Alg. 3), l -= t+, and the reflection counts
 * towards rho.  F(x) is carried as F += sum_k t^k F1(coef_k). */
static int chmc_step(const orc_lmi* L, const orc_walk_params* p, uint32_t chain, uint32_t step, walk_ws* W,
                     orc_stats* st, trace_rec* tr) {
    int n = L->n, m = L->mb[0];
    size_t mm = (size_t)m * m;
    const int d = p->q + 1;
    double eta;
    orc_step_draws(p->seed, p->tag, chain, step, n, W->g, &eta);
    double ell = p->L * eta; /* l = tau eta (Alg. 6 line 1) */
    for (int i = 0; i < n; ++i) W->v[i] = W->g[i]; /* v ~ N(0, I) */
    memcpy(W->xs, W->x, sizeof(double) * n);
    memcpy(W->Fs, W->F, sizeof(double) * mm);
    int64_t refl = 0;
    int bound = -1;
    st->steps += 1;
    double* coef = W->coef;
    for (;;) {
        if (W->budget >= 0 && st->calls >= W->budget) return 5;
        const int last = (ell <= p->h);
        const double hs = last ? ell : p->h;
        orc_colloc_poly(n, p, W->x, W->v, hs, coef);
        for (int k = 1; k <= d; ++k) orc_dir_block(L, 0, coef + (size_t)k * n, W->Fk + (size_t)(k - 1) * mm);
        orc_chord_res* r = W->res;
        int rc = orc_colloc_chord(L, W->F, coef, d, hs, bound, W->u, r);
        st->calls += 1;
        if (rc) return rc;
        if (r->outward) {
            st->degenerates += 1;
            goto reject;
        }
        double tp = r->t_plus;
        const double th = (hs <= tp) ? hs : tp; /* reading R4: a tie ends the segment, no reflection */
        poly_eval(n, d, coef, th, W->x);
        poly_deriv(n, d, coef, th, W->g);
        for (size_t e = 0; e < mm; ++e) {
            double a = W->Fk[(size_t)(d - 1) * mm + e];
            for (int k = d - 1; k >= 1; --k) a = a * th + W->Fk[(size_t)(k - 1) * mm + e];
            W->F[e] += th * a;
        }
        if (hs <= tp) {
            if (last) return 0;
            ell -= hs;
            memcpy(W->v, W->g, sizeof(double) * n);
            bound = -1;
            continue;
        }
        ell -= tp;
        refl += 1;
        st->reflections += 1;
        if (refl > p->rho) {
            st->rejects += 1;
            goto reject;
        }
        if (r->degenerate || orc_normal(L, r->binding, r->y, r->ylen, W->w)) {
            st->degenerates += 1;
            goto reject;
        }
        orc_reflect(n, W->g, W->w, W->v);
        {
            double ny = 0.0;
            for (int i = 0; i < r->ylen; ++i) ny += r->y[i] * r->y[i];
            ny = sqrt(ny);
            for (int i = 0; i < r->ylen; ++i) W->u[i] = r->y[i] / ny;
        }
        bound = r->binding;
        if (tr && tr->nrec < tr->max_refl) {
            int64_t k = tr->nrec;
            memcpy(tr->hit_x + k * n, W->x, sizeof(double) * n);
            tr->t[k] = tp;
            memcpy(tr->w + k * n, W->w, sizeof(double) * n);
            memcpy(tr->v_after + k * n, W->v, sizeof(double) * n);
            tr->binding[k] = r->binding;
            tr->nrec += 1;
            if (tr->stop && tr->nrec >= tr->max_refl) return 6;
        }
    }
reject:
    memcpy(W->x, W->xs, sizeof(double) * n);
    memcpy(W->F, W->Fs, sizeof(double) * mm);
    return 0;
}

static int walk_step(const orc_lmi* L, const orc_walk_params* p, uint32_t chain, uint32_t step,
                     walk_ws* W, orc_stats* st, trace_rec* tr) {
    int n = L->n, m = L->mb[0];
    size_t mm = (size_t)m * m;
    double eta;
    if (p->kind == ORC_HNR || p->kind == ORC_CHNR) return hnr_step(L, p, chain, step, W, st);
    if (p->kind == ORC_CHMC) return chmc_step(L, p, chain, step, W, st, tr);
    orc_step_draws(p->seed, p->tag, chain, step, n, W->g, &eta);
    double ell;
    if (p->kind == ORC_BILLIARD) {
        ell = -p->L * log(eta); /* l = -tau ln eta (Alg. 5 line 1) */
        double gn = 0.0;
        for (int i = 0; i < n; ++i) gn += W->g[i] * W->g[i];
        gn = sqrt(gn);
        for (int i = 0; i < n; ++i) W->v[i] = W->g[i] / gn; /* v ~ U(sphere) */
    } else {
        ell = p->L * eta; /* l = tau eta (Alg. 6 line 1) */
        for (int i = 0; i < n; ++i) W->v[i] = W->g[i]; /* v ~ N(0, I) */
        orc_dir_block(L, 0, p->c, W->F2c);
        for (size_t e = 0; e < mm; ++e) W->F2c[e] = -W->F2c[e] / (2.0 * p->T);
    }
    memcpy(W->xs, W->x, sizeof(double) * n);
    memcpy(W->Fs, W->F, sizeof(double) * mm);
    int64_t refl = 0;
    int bound = -1;
    st->steps += 1;
    for (;;) {
        if (W->budget >= 0 && st->calls >= W->budget) return 5; /* replay budget reached mid-step */
        orc_dir_block(L, 0, W->v, W->F1);
        orc_chord_res* r = W->res;
        int rc;
        if (p->kind == ORC_BILLIARD)
            rc = orc_chord(L, W->x, W->F, W->F1, W->v, bound, W->u, r);
        else
            rc = orc_hmc_chord(L, W->x, W->F, W->v, p->c, p->T, bound, W->u, r);
        st->calls += 1;
        if (rc) return rc;
        if (r->outward) { /* grazing / outward after reflection: reject */
            st->degenerates += 1;
            goto reject;
        }
        double tp = r->t_plus;
        if (ell <= tp) { /* segment ends inside (reading R4: tie -> no reflection) */
            if (p->kind == ORC_BILLIARD) {
                for (int i = 0; i < n; ++i) W->x[i] += ell * W->v[i];
                for (size_t e = 0; e < mm; ++e) W->F[e] += ell * W->F1[e];
            } else {
                double a = -ell * ell / (2.0 * p->T);
                for (int i = 0; i < n; ++i) W->x[i] += ell * W->v[i] + a * p->c[i];
                for (size_t e = 0; e < mm; ++e) W->F[e] += ell * W->F1[e] + ell * ell * W->F2c[e];
            }
            return 0;
        }
        /* move to the boundary point Phi(t+) */
        double* uvel = W->g; /* velocity at the hit */
        if (p->kind == ORC_BILLIARD) {
            for (int i = 0; i < n; ++i) W->x[i] += tp * W->v[i];
            for (size_t e = 0; e < mm; ++e) W->F[e] += tp * W->F1[e];
            for (int i = 0; i < n; ++i) uvel[i] = W->v[i];
        } else {
            double a = -tp * tp / (2.0 * p->T);
            for (int i = 0; i < n; ++i) W->x[i] += tp * W->v[i] + a * p->c[i];
            for (size_t e = 0; e < mm; ++e) W->F[e] += tp * W->F1[e] + tp * tp * W->F2c[e];
            for (int i = 0; i < n; ++i) uvel[i] = W->v[i] - (p->c[i] / p->T) * tp; /* dp/dt(t+) */
        }
        ell -= tp;
        refl += 1;
        st->reflections += 1;
        if (refl > p->rho) { /* reading R5: break as soon as #refl > rho */
            st->rejects += 1;
            goto reject;
        }
        if (r->degenerate || orc_normal(L, r->binding, r->y, r->ylen, W->w)) {
            st->degenerates += 1;
            goto reject;
        }
        orc_reflect(n, uvel, W->w, W->v);
        {
            double ny = 0.0;
            for (int i = 0; i < r->ylen; ++i) ny += r->y[i] * r->y[i];
            ny = sqrt(ny);
            for (int i = 0; i < r->ylen; ++i) W->u[i] = r->y[i] / ny;
        }
        bound = r->binding;
        if (tr && tr->nrec < tr->max_refl) {
            int64_t k = tr->nrec;
            memcpy(tr->hit_x + k * n, W->x, sizeof(double) * n);
            tr->t[k] = tp;
            memcpy(tr->w + k * n, W->w, sizeof(double) * n);
            memcpy(tr->v_after + k * n, W->v, sizeof(double) * n);
            tr->binding[k] = r->binding;
            tr->nrec += 1;
            if (tr->stop && tr->nrec >= tr->max_refl) return 6; /* trace complete */
        }
    }
reject:
    memcpy(W->x, W->xs, sizeof(double) * n);
    memcpy(W->F, W->Fs, sizeof(double) * mm);
    return 0;
}

typedef struct {
    const orc_lmi* L;
    const orc_walk_params* p;
    int64_t cb, ce;
    const double* x0;
    int x0_stride;
    double* final_x;
    int64_t next;
    pthread_mutex_t mu;
    orc_stats st;
    int rc;
} walk_job;

static void* walk_worker(void* arg) {
    walk_job* J = (walk_job*)arg;
    const orc_lmi* L = J->L;
    int n = L->n;
    walk_ws W;
    ws_init(&W, L);
    orc_stats st = {0, 0, 0, 0, 0, 0};
    int rc = 0;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t c = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (c >= J->ce) break;
        const double* x0 = J->x0 + (J->x0_stride ? (c - J->cb) * (int64_t)n : 0);
        memcpy(W.x, x0, sizeof(double) * n);
        orc_eval_block(L, 0, W.x, W.F);
        for (int64_t s = 0; s < J->p->steps; ++s) {
            int r = walk_step(L, J->p, (uint32_t)c, (uint32_t)s, &W, &st, NULL);
            if (r) { rc = r; st.failures += 1; break; }
        }
        memcpy(J->final_x + (c - J->cb) * (int64_t)n, W.x, sizeof(double) * n);
    }
    ws_free(&W);
    pthread_mutex_lock(&J->mu);
    J->st.calls += st.calls;
    J->st.reflections += st.reflections;
    J->st.rejects += st.rejects;
    J->st.degenerates += st.degenerates;
    J->st.steps += st.steps;
    J->st.failures += st.failures;
    if (rc) J->rc = rc;
    pthread_mutex_unlock(&J->mu);
    return NULL;
}

int orc_walk(const orc_lmi* L, const orc_walk_params* p, int64_t chain_begin, int64_t chain_end,
             const double* x0, int x0_stride, double* final_x, orc_stats* st, int nthreads) {
    walk_job J;
    J.L = L; J.p = p; J.cb = chain_begin; J.ce = chain_end; J.x0 = x0; J.x0_stride = x0_stride;
    J.final_x = final_x; J.next = chain_begin; J.rc = 0;
    memset(&J.st, 0, sizeof(J.st));
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)xmalloc(sizeof(pthread_t) * nthreads);
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, walk_worker, &J);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&J.mu);
    if (st) *st = J.st;
    return J.rc;
}

/* State of one chain after exactly max_calls chord calls (the GPU scheduler's
 * state after max_calls rounds).  Returns 0, or 2 if a start was not interior. */
int orc_replay(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0, int64_t max_calls,
               double* x_out, int64_t* calls_out) {
    int n = L->n;
    walk_ws W;
    ws_init(&W, L);
    W.budget = max_calls;
    orc_stats st = {0, 0, 0, 0, 0, 0};
    memcpy(W.x, x0, sizeof(double) * n);
    orc_eval_block(L, 0, W.x, W.F);
    int rc = 0;
    for (int64_t s = 0; s < p->steps && st.calls < max_calls; ++s) {
        rc = walk_step(L, p, (uint32_t)chain, (uint32_t)s, &W, &st, NULL);
        if (rc == 5) { rc = 0; break; }
        if (rc) break;
    }
    memcpy(x_out, W.x, sizeof(double) * n);
    *calls_out = st.calls;
    ws_free(&W);
    return rc;
}

/* orc_trace stops right after the max_refl-th reflection is recorded (the records are
   those of orc_trace_stats; only the unrecorded remainder of that step is skipped) */
static int trace_impl(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0,
                      int64_t max_refl, double* hit_x, double* t, double* w, double* v_after,
                      int32_t* binding, int64_t* nrec, orc_stats* st_out, int stop);
int orc_trace(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0,
              int64_t max_refl, double* hit_x, double* t, double* w, double* v_after,
              int32_t* binding, int64_t* nrec) {
    return trace_impl(L, p, chain, x0, max_refl, hit_x, t, w, v_after, binding, nrec, NULL, 1);
}

/* as orc_trace; st_out (may be NULL) receives the walk statistics: the walk always
   completes the step in which the max_refl-th reflection falls, so st_out->calls
   counts every boundary-oracle call made (>= the recorded reflections) */
int orc_trace_stats(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0,
                    int64_t max_refl, double* hit_x, double* t, double* w, double* v_after,
                    int32_t* binding, int64_t* nrec, orc_stats* st_out) {
    return trace_impl(L, p, chain, x0, max_refl, hit_x, t, w, v_after, binding, nrec, st_out, 0);
}

static int trace_impl(const orc_lmi* L, const orc_walk_params* p, int64_t chain, const double* x0,
                      int64_t max_refl, double* hit_x, double* t, double* w, double* v_after,
                      int32_t* binding, int64_t* nrec, orc_stats* st_out, int stop) {
    int n = L->n;
    walk_ws W;
    ws_init(&W, L);
    orc_stats st = {0, 0, 0, 0, 0, 0};
    trace_rec tr = {max_refl, 0, hit_x, t, w, v_after, binding, stop};
    memcpy(W.x, x0, sizeof(double) * n);
    orc_eval_block(L, 0, W.x, W.F);
    int rc = 0;
    for (int64_t s = 0; s < p->steps && tr.nrec < max_refl; ++s) {
        rc = walk_step(L, p, (uint32_t)chain, (uint32_t)s, &W, &st, &tr);
        if (rc == 6) {
            rc = 0;
            break;
        }
        if (rc) break;
    }
    *nrec = tr.nrec;
    if (st_out) *st_out = st;
    ws_free(&W);
    return rc;
}
