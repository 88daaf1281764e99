/*
 * dg_oracle.c -- plain, slow, obviously-correct CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * It shares no code with the CUDA product path.  See dg_oracle.h for the definitions
 * and citations; every function below follows the weak form written there term by
 * term, with explicit quadrature loops and no blocking, fusion or sum factorisation.
 *
 * Pins (tests/test_oracle_*.py, all "-m 'not gpu'"):
 *   GLL/Gauss tables  -> worked values, closed forms, numpy/scipy
 *   sip_apply         -> brute-force dense matrix (sip_dense) on 2x2 meshes, symmetry,
 *                        null space {1} at lam=0, polynomial reproduction, 1-D critical
 *                        penalty, Bloch spectrum, MMS convergence order P+1
 *   sip_diag          -> diagonal of the dense matrix and of sip_apply(e_I)
 *   pcg_solve         -> LAPACK dense solve (numpy) on small meshes, residual checks
 *   convect           -> constant-v zero, conservation, polynomial exactness,
 *                        Taylor-Green closed-form limit.  LLF Lambda (A12) and Q (A13)
 *                        are readings: parity for those choices is "unpinned" by the paper.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (reading A16: no FMA contraction,
 * no fast-math).
 */
#include "dg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXN 18 /* supports P <= 16 (and Q <= 18 Gauss points) */

/* ------------------------------------------------------------------------- */
/* 1-D tables                                                                  */
/* ------------------------------------------------------------------------- */

/* Legendre P_k(x) by the three-term recurrence; returns P_P, *pm1 = P_{P-1}. */
static long double legendre_pair(int P, long double x, long double *pm1)
{
    long double p0 = 1.0L, p1 = x;
    if (P == 0) { *pm1 = 0.0L; return 1.0L; }
    for (int k = 1; k < P; ++k) {
        long double p2 = ((2.0L * k + 1.0L) * x * p1 - (long double)k * p0) / (k + 1.0L);
        p0 = p1;
        p1 = p2;
    }
    *pm1 = p0;
    return p1;
}

int oracle_gll(int P, double *xi, double *w)
{
    if (P < 1 || P + 1 > MAXN || !xi || !w) return -1;
    const int n = P + 1;
    long double x[MAXN];
    /* Chebyshev-Gauss-Lobatto initial guesses, then Newton on
     * x P_P(x) - P_{P-1}(x) = (1-x^2) P_P'(x) / P  (zero at +-1 and at the roots of P_P'). */
    for (int i = 0; i < n; ++i) x[i] = -cosl(3.14159265358979323846264338327950288L * i / P);
    for (int i = 1; i < P; ++i) {
        for (int it = 0; it < 100; ++it) {
            long double pm1, pp = legendre_pair(P, x[i], &pm1);
            long double dx = (x[i] * pp - pm1) / ((long double)(P + 1) * pp);
            x[i] -= dx;
            if (fabsl(dx) < 1e-19L) break;
        }
    }
    x[0] = -1.0L;
    x[P] = 1.0L;
    for (int i = 0; i < n; ++i) {
        long double pm1, pp = legendre_pair(P, x[i], &pm1);
        xi[i] = (double)x[i];
        w[i] = (double)(2.0L / ((long double)P * (P + 1) * pp * pp));
    }
    return 0;
}

int oracle_gauss(int Q, double *zeta, double *omega)
{
    if (Q < 1 || Q > MAXN || !zeta || !omega) return -1;
    long double x[MAXN], wt[MAXN];
    for (int i = 0; i < Q; ++i) {
        long double z = cosl(3.14159265358979323846264338327950288L * (i + 0.75L) / (Q + 0.5L));
        for (int it = 0; it < 100; ++it) {
            long double pm1, p = legendre_pair(Q, z, &pm1);
            long double dp = (long double)Q * (z * p - pm1) / (z * z - 1.0L);
            long double dz = p / dp;
            z -= dz;
            if (fabsl(dz) < 1e-19L) break;
        }
        long double pm1, p = legendre_pair(Q, z, &pm1);
        long double dp = (long double)Q * (z * p - pm1) / (z * z - 1.0L);
        (void)p;
        x[i] = z;
        wt[i] = 2.0L / ((1.0L - z * z) * dp * dp);
    }
    for (int i = 0; i < Q; ++i) { /* ascending order */
        zeta[i] = (double)x[Q - 1 - i];
        omega[i] = (double)wt[Q - 1 - i];
    }
    return 0;
}

void oracle_lagrange(int P, const double *xi, double x, double *l, double *dl)
{
    const int n = P + 1;
    for (int j = 0; j < n; ++j) {
        long double prod = 1.0L;
        for (int m = 0; m < n; ++m)
            if (m != j) prod *= ((long double)x - xi[m]) / ((long double)xi[j] - xi[m]);
        l[j] = (double)prod;
        long double s = 0.0L;
        for (int k = 0; k < n; ++k) {
            if (k == j) continue;
            long double t = 1.0L / ((long double)xi[j] - xi[k]);
            for (int m = 0; m < n; ++m)
                if (m != j && m != k) t *= ((long double)x - xi[m]) / ((long double)xi[j] - xi[m]);
            s += t;
        }
        dl[j] = (double)s;
    }
}

/* ------------------------------------------------------------------------- */
/* mesh helpers                                                                */
/* ------------------------------------------------------------------------- */

typedef struct {
    int dim, P, n, nd[3], npe;
    long N[3], nel;
    double h[3];
    double xi[MAXN], w[MAXN];
    double Lv[MAXN][MAXN]; /* Lv[a][j] = l_j(xi_a)  (product formula) */
    double Dl[MAXN][MAXN]; /* Dl[a][j] = l_j'(xi_a) (product formula) */
} ctx_t;

static int ctx_init(const oracle_mesh *m, ctx_t *c)
{
    if (!m || (m->dim != 2 && m->dim != 3) || m->P < 1 || m->P + 1 > MAXN) return -1;
    c->dim = m->dim;
    c->P = m->P;
    c->n = m->P + 1;
    c->nel = 1;
    for (int d = 0; d < 3; ++d) {
        int active = d < m->dim;
        c->N[d] = active ? m->N[d] : 1;
        if (c->N[d] < 1) return -1;
        c->nd[d] = active ? c->n : 1;
        c->h[d] = active ? m->L[d] / (double)m->N[d] : 1.0;
        c->nel *= c->N[d];
    }
    c->npe = c->nd[0] * c->nd[1] * c->nd[2];
    if (oracle_gll(c->P, c->xi, c->w)) return -1;
    for (int a = 0; a < c->n; ++a) oracle_lagrange(c->P, c->xi, c->xi[a], c->Lv[a], c->Dl[a]);
    return 0;
}

static void el_coords(const ctx_t *c, long e, long ec[3])
{
    ec[0] = e % c->N[0];
    ec[1] = (e / c->N[0]) % c->N[1];
    ec[2] = e / (c->N[0] * c->N[1]);
}

static long el_index(const ctx_t *c, const long ec[3])
{
    return ec[0] + c->N[0] * (ec[1] + c->N[1] * ec[2]);
}

/* periodic neighbour of e across direction d, side s (+1 / -1) */
static long el_neighbour(const ctx_t *c, long e, int d, int s)
{
    long ec[3];
    el_coords(c, e, ec);
    ec[d] = (ec[d] + s + c->N[d]) % c->N[d];
    return el_index(c, ec);
}

static void nd_coords(const ctx_t *c, int q, int qc[3])
{
    qc[0] = q % c->nd[0];
    qc[1] = (q / c->nd[0]) % c->nd[1];
    qc[2] = q / (c->nd[0] * c->nd[1]);
}

static int nd_index(const ctx_t *c, const int qc[3])
{
    return qc[0] + c->nd[0] * (qc[1] + c->nd[1] * qc[2]);
}

/* node index of qc with component d replaced by a */
static int nd_with(const ctx_t *c, const int qc[3], int d, int a)
{
    int t[3] = {qc[0], qc[1], qc[2]};
    t[d] = a;
    return nd_index(c, t);
}

/* GLL volume weight W_q = prod_d w_{q_d} h_d/2 */
static double vol_weight(const ctx_t *c, const int qc[3])
{
    double W = 1.0;
    for (int d = 0; d < c->dim; ++d) W *= c->w[qc[d]] * c->h[d] * 0.5;
    return W;
}

/* GLL face weight W^F_q = prod_{d' != d} w_{q_d'} h_d'/2 */
static double face_weight(const ctx_t *c, const int qc[3], int d)
{
    double W = 1.0;
    for (int dd = 0; dd < c->dim; ++dd)
        if (dd != d) W *= c->w[qc[dd]] * c->h[dd] * 0.5;
    return W;
}

static double nu_at(const double *nu, double nu_const, long e, int npe, int q)
{
    return nu ? nu[e * (long)npe + q] : nu_const;
}

/* ------------------------------------------------------------------------- */
/* SIP apply (explicit GLL quadrature, collocation identity u(x_q) = u_q)      */
/* ------------------------------------------------------------------------- */

static void sip_apply_element(const ctx_t *c, double lam, const double *nu, double nu_const,
                              const double *u, long e, double *y)
{
    const int npe = c->npe, P = c->P, n = c->n;
    const double *ue = u + e * (long)npe;
    for (int I = 0; I < npe; ++I) y[I] = 0.0;

    /* volume: sum_q W_q [lam phi_I u + nu grad phi_I . grad u](x_q) */
    for (int q = 0; q < npe; ++q) {
        int qc[3];
        nd_coords(c, q, qc);
        const double W = vol_weight(c, qc);
        const double nuq = nu_at(nu, nu_const, e, npe, q);
        y[q] += lam * W * ue[q]; /* phi_I(x_q) = delta_Iq */
        for (int d = 0; d < c->dim; ++d) {
            const double s = 2.0 / c->h[d];
            double g = 0.0; /* d_d u (x_q) */
            for (int j = 0; j < n; ++j) g += s * c->Dl[qc[d]][j] * ue[nd_with(c, qc, d, j)];
            for (int i = 0; i < n; ++i) /* d_d phi_I(x_q) != 0 only for I on the d-line through q */
                y[nd_with(c, qc, d, i)] += W * nuq * (s * c->Dl[qc[d]][i]) * g;
        }
    }

    /* faces: sum_F sum_q W^F_q [-{nu d_n u}[phi_I] - {nu d_n phi_I}[u] + sigma [u][phi_I]] */
    for (int d = 0; d < c->dim; ++d) {
        const double s = 2.0 / c->h[d];
        const double tau = (double)(P + 1) * (double)(P + 1) / c->h[d];
        for (int side = -1; side <= 1; side += 2) {
            const long enb = el_neighbour(c, e, d, side);
            const double *un = u + enb * (long)npe;
            const int a_own = side > 0 ? P : 0, a_nb = side > 0 ? 0 : P;
            const double sgn = side > 0 ? 1.0 : -1.0; /* +1: e is the "-" side (n = +e_d) */
            for (int q = 0; q < npe; ++q) {
                int qc[3];
                nd_coords(c, q, qc);
                if (qc[d] != a_own) continue;
                const double WF = face_weight(c, qc, d);
                const int I_own = q, I_nb = nd_with(c, qc, d, a_nb);
                const double u_o = ue[I_own], u_n = un[I_nb];
                const double nu_o = nu_at(nu, nu_const, e, npe, I_own);
                const double nu_n = nu_at(nu, nu_const, enb, npe, I_nb);
                double dn_o = 0.0, dn_n = 0.0;
                for (int j = 0; j < n; ++j) {
                    dn_o += s * c->Dl[a_own][j] * ue[nd_with(c, qc, d, j)];
                    dn_n += s * c->Dl[a_nb][j] * un[nd_with(c, qc, d, j)];
                }
                double um, up, fm, fp, num, nup;
                if (side > 0) { um = u_o; up = u_n; fm = nu_o * dn_o; fp = nu_n * dn_n; num = nu_o; nup = nu_n; }
                else          { um = u_n; up = u_o; fm = nu_n * dn_n; fp = nu_o * dn_o; num = nu_n; nup = nu_o; }
                const double jump = um - up;
                const double avg = 0.5 * (fm + fp);
                const double sigma = tau * 0.5 * (num + nup);
                /* [phi_I] = sgn * delta(I = I_own) */
                y[I_own] += WF * sgn * (-avg + sigma * jump);
                /* {nu d_n phi_I} = 1/2 nu_o d_d phi_I|_e, nonzero on the d-line through the face node */
                for (int i = 0; i < n; ++i)
                    y[nd_with(c, qc, d, i)] += -WF * 0.5 * nu_o * (s * c->Dl[a_own][i]) * jump;
            }
        }
    }
}

int oracle_sip_apply(const oracle_mesh *m, double lam, const double *nu, double nu_const,
                     const double *u, double *y, const long *elems, long nel)
{
    ctx_t c;
    if (ctx_init(m, &c) || !u || !y) return -1;
    const long cnt = elems ? nel : c.nel;
    for (long k = 0; k < cnt; ++k)
        if (elems && (elems[k] < 0 || elems[k] >= c.nel)) return -1;
#pragma omp parallel for schedule(dynamic, 4)
    for (long k = 0; k < cnt; ++k) {
        const long e = elems ? elems[k] : k;
        sip_apply_element(&c, lam, nu, nu_const, u, e, y + k * (long)c.npe);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* diagonal: quadratic form at the unit vector, full tensor-product evaluation */
/* ------------------------------------------------------------------------- */

/* phi_I and d_d phi_I at reference point given by 1-D tables per direction:
 * L1[d][j] = l_j(r_d), G1[d][j] = l_j'(r_d). */
static double tp_val(const ctx_t *c, double L1[3][MAXN], const int Ic[3])
{
    double v = 1.0;
    for (int d = 0; d < c->dim; ++d) v *= L1[d][Ic[d]];
    return v;
}

static double tp_grad(const ctx_t *c, double L1[3][MAXN], double G1[3][MAXN], const int Ic[3], int dd)
{
    double v = 2.0 / c->h[dd];
    for (int d = 0; d < c->dim; ++d) v *= (d == dd) ? G1[d][Ic[d]] : L1[d][Ic[d]];
    return v;
}

/* 1-D tables at GLL node a of each direction (qc) */
static void tables_at_node(const ctx_t *c, const int qc[3], double L1[3][MAXN], double G1[3][MAXN])
{
    for (int d = 0; d < c->dim; ++d)
        for (int j = 0; j < c->n; ++j) {
            L1[d][j] = c->Lv[qc[d]][j];
            G1[d][j] = c->Dl[qc[d]][j];
        }
}

static void sip_diag_element(const ctx_t *c, double lam, const double *nu, double nu_const, long e, double *dg)
{
    const int npe = c->npe, P = c->P;
    for (int I = 0; I < npe; ++I) {
        int Ic[3];
        nd_coords(c, I, Ic);
        double acc = 0.0;
        /* volume */
        for (int q = 0; q < npe; ++q) {
            int qc[3];
            double L1[3][MAXN], G1[3][MAXN];
            nd_coords(c, q, qc);
            tables_at_node(c, qc, L1, G1);
            const double W = vol_weight(c, qc);
            const double phi = tp_val(c, L1, Ic);
            double g2 = 0.0;
            for (int d = 0; d < c->dim; ++d) {
                const double g = tp_grad(c, L1, G1, Ic, d);
                g2 += g * g;
            }
            acc += W * (lam * phi * phi + nu_at(nu, nu_const, e, npe, q) * g2);
        }
        /* faces: each face F once.  For N_d > 1 the two faces of e in direction d are
         * distinct and phi_I vanishes on the neighbour side; for N_d == 1 the element is
         * its own neighbour and both traces of phi_I live on the single face. */
        for (int d = 0; d < c->dim; ++d) {
            const double tau = (double)(P + 1) * (double)(P + 1) / c->h[d];
            const int self = (c->N[d] == 1);
            for (int side = -1; side <= 1; side += 2) {
                if (self && side < 0) continue;
                const long enb = el_neighbour(c, e, d, side);
                const int a_own = side > 0 ? P : 0, a_nb = side > 0 ? 0 : P;
                for (int q = 0; q < npe; ++q) {
                    int qc[3];
                    nd_coords(c, q, qc);
                    if (qc[d] != a_own) continue;
                    const double WF = face_weight(c, qc, d);
                    double L1[3][MAXN], G1[3][MAXN];
                    /* own-side trace of phi_I */
                    tables_at_node(c, qc, L1, G1);
                    const double t_o = tp_val(c, L1, Ic), dn_o = tp_grad(c, L1, G1, Ic, d);
                    /* neighbour-side trace (nonzero only if the neighbour is e itself) */
                    double t_n = 0.0, dn_n = 0.0;
                    int qn[3] = {qc[0], qc[1], qc[2]};
                    qn[d] = a_nb;
                    if (enb == e) {
                        tables_at_node(c, qn, L1, G1);
                        t_n = tp_val(c, L1, Ic);
                        dn_n = tp_grad(c, L1, G1, Ic, d);
                    }
                    const double nu_o = nu_at(nu, nu_const, e, npe, q);
                    const double nu_n = nu_at(nu, nu_const, enb, npe, nd_index(c, qn));
                    double pm, pp, fm, fp, num, nup;
                    if (side > 0) { pm = t_o; pp = t_n; fm = nu_o * dn_o; fp = nu_n * dn_n; num = nu_o; nup = nu_n; }
                    else          { pm = t_n; pp = t_o; fm = nu_n * dn_n; fp = nu_o * dn_o; num = nu_n; nup = nu_o; }
                    const double jump = pm - pp, avg = 0.5 * (fm + fp);
                    const double sigma = tau * 0.5 * (num + nup);
                    acc += WF * (-2.0 * avg * jump + sigma * jump * jump);
                }
            }
        }
        dg[I] = acc;
    }
}

int oracle_sip_diag(const oracle_mesh *m, double lam, const double *nu, double nu_const,
                    double *diag, const long *elems, long nel)
{
    ctx_t c;
    if (ctx_init(m, &c) || !diag) return -1;
    const long cnt = elems ? nel : c.nel;
    for (long k = 0; k < cnt; ++k)
        if (elems && (elems[k] < 0 || elems[k] >= c.nel)) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (long k = 0; k < cnt; ++k) {
        const long e = elems ? elems[k] : k;
        sip_diag_element(&c, lam, nu, nu_const, e, diag + k * (long)c.npe);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* brute-force dense matrix                                                    */
/* ------------------------------------------------------------------------- */

int oracle_sip_dense(const oracle_mesh *m, double lam, const double *nu, double nu_const, double *A)
{
    ctx_t c;
    if (ctx_init(m, &c) || !A) return -1;
    const int npe = c.npe, P = c.P;
    const long ndof = c.nel * npe;
    if (ndof > 20000) return -2;
    memset(A, 0, sizeof(double) * ndof * ndof);
    double *phi = malloc(sizeof(double) * ndof);
    double *gr = malloc(sizeof(double) * ndof * 3);
    double *phm = malloc(sizeof(double) * ndof), *php = malloc(sizeof(double) * ndof);
    double *dnm = malloc(sizeof(double) * ndof), *dnp = malloc(sizeof(double) * ndof);
    if (!phi || !gr || !phm || !php || !dnm || !dnp) return -3;

    /* volume: all (I, J, q); phi_I(x_q) = 0 unless I lives on element K (broken space) */
    for (long K = 0; K < c.nel; ++K) {
        for (int q = 0; q < npe; ++q) {
            int qc[3];
            double L1[3][MAXN], G1[3][MAXN];
            nd_coords(&c, q, qc);
            tables_at_node(&c, qc, L1, G1);
            const double W = vol_weight(&c, qc);
            const double nuq = nu_at(nu, nu_const, K, npe, q);
            for (long I = 0; I < ndof; ++I) {
                int Ic[3];
                const long eI = I / npe;
                nd_coords(&c, (int)(I % npe), Ic);
                phi[I] = (eI == K) ? tp_val(&c, L1, Ic) : 0.0;
                for (int d = 0; d < 3; ++d)
                    gr[3 * I + d] = (eI == K && d < c.dim) ? tp_grad(&c, L1, G1, Ic, d) : 0.0;
            }
            for (long I = 0; I < ndof; ++I)
                for (long J = 0; J < ndof; ++J) {
                    double gg = 0.0;
                    for (int d = 0; d < c.dim; ++d) gg += gr[3 * I + d] * gr[3 * J + d];
                    A[I * ndof + J] += W * (lam * phi[I] * phi[J] + nuq * gg);
                }
        }
    }
    /* faces: every face once, as the face on the +d side of its "-" element */
    for (int d = 0; d < c.dim; ++d) {
        const double tau = (double)(P + 1) * (double)(P + 1) / c.h[d];
        for (long em = 0; em < c.nel; ++em) {
            const long ep = el_neighbour(&c, em, d, +1);
            for (int q = 0; q < npe; ++q) {
                int qc[3];
                nd_coords(&c, q, qc);
                if (qc[d] != P) continue;
                int qp[3] = {qc[0], qc[1], qc[2]};
                qp[d] = 0;
                const double WF = face_weight(&c, qc, d);
                double Lm[3][MAXN], Gm[3][MAXN], Lp[3][MAXN], Gp[3][MAXN];
                tables_at_node(&c, qc, Lm, Gm); /* reference point xi_d = +1 in em */
                tables_at_node(&c, qp, Lp, Gp); /* reference point xi_d = -1 in ep */
                const double num = nu_at(nu, nu_const, em, npe, q);
                const double nup = nu_at(nu, nu_const, ep, npe, nd_index(&c, qp));
                const double sigma = tau * 0.5 * (num + nup);
                for (long I = 0; I < ndof; ++I) {
                    int Ic[3];
                    const long eI = I / npe;
                    nd_coords(&c, (int)(I % npe), Ic);
                    phm[I] = (eI == em) ? tp_val(&c, Lm, Ic) : 0.0;
                    dnm[I] = (eI == em) ? tp_grad(&c, Lm, Gm, Ic, d) : 0.0;
                    php[I] = (eI == ep) ? tp_val(&c, Lp, Ic) : 0.0;
                    dnp[I] = (eI == ep) ? tp_grad(&c, Lp, Gp, Ic, d) : 0.0;
                }
                for (long I = 0; I < ndof; ++I) {
                    const double jI = phm[I] - php[I];
                    const double aI = 0.5 * (num * dnm[I] + nup * dnp[I]);
                    for (long J = 0; J < ndof; ++J) {
                        const double jJ = phm[J] - php[J];
                        const double aJ = 0.5 * (num * dnm[J] + nup * dnp[J]);
                        A[I * ndof + J] += WF * (-aJ * jI - aI * jJ + sigma * jJ * jI);
                    }
                }
            }
        }
    }
    free(phi); free(gr); free(phm); free(php); free(dnm); free(dnp);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* (P)CG solve                                                                 */
/* ------------------------------------------------------------------------- */

static double dot(const double *a, const double *b, long n)
{
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

int oracle_pcg_solve(const oracle_mesh *m, double lam, const double *nu, double nu_const,
                     const double *f, double tol, int maxit, int precond, double *u,
                     int *iters, double *relres, double *removed_mean)
{
    ctx_t c;
    if (ctx_init(m, &c) || !f || !u || lam < 0.0) return -1;
    const int npe = c.npe;
    const long ndof = c.nel * npe;
    double *mass = malloc(sizeof(double) * ndof), *fp = malloc(sizeof(double) * ndof);
    double *r = malloc(sizeof(double) * ndof), *z = malloc(sizeof(double) * ndof);
    double *p = malloc(sizeof(double) * ndof), *q = malloc(sizeof(double) * ndof);
    double *dinv = malloc(sizeof(double) * ndof);
    if (!mass || !fp || !r || !z || !p || !q || !dinv) return -3;

    for (long e = 0; e < c.nel; ++e)
        for (int I = 0; I < npe; ++I) {
            int Ic[3];
            nd_coords(&c, I, Ic);
            mass[e * npe + I] = vol_weight(&c, Ic); /* m_I = prod w h/2 */
        }
    double fmean = 0.0;
    if (lam == 0.0) { /* project f to zero mass-weighted mean (reading A8) */
        double sm = 0.0, smf = 0.0;
        for (long i = 0; i < ndof; ++i) { sm += mass[i]; smf += mass[i] * f[i]; }
        fmean = smf / sm;
    }
    for (long i = 0; i < ndof; ++i) fp[i] = f[i] - fmean;
    if (removed_mean) *removed_mean = fmean;
    const double fnorm = sqrt(dot(fp, fp, ndof));

    if (precond) {
        if (oracle_sip_diag(m, lam, nu, nu_const, dinv, NULL, 0)) return -1;
        for (long i = 0; i < ndof; ++i) dinv[i] = 1.0 / dinv[i];
    } else {
        for (long i = 0; i < ndof; ++i) dinv[i] = 1.0;
    }

    /* r = M f - A u */
    oracle_sip_apply(m, lam, nu, nu_const, u, q, NULL, 0);
    for (long i = 0; i < ndof; ++i) r[i] = mass[i] * fp[i] - q[i];
    if (lam == 0.0) {
        double mr = 0.0;
        for (long i = 0; i < ndof; ++i) mr += r[i];
        mr /= (double)ndof;
        for (long i = 0; i < ndof; ++i) r[i] -= mr;
    }
    for (long i = 0; i < ndof; ++i) { z[i] = dinv[i] * r[i]; p[i] = z[i]; }
    double rz = dot(r, z, ndof);

    int k = 0, status = 1;
    double best = INFINITY;
    int since_best = 0;
    double res = 0.0;
    for (;;) {
        double s = 0.0;
        for (long i = 0; i < ndof; ++i) s += (r[i] / mass[i]) * (r[i] / mass[i]);
        res = (fnorm > 0.0) ? sqrt(s) / fnorm : sqrt(s);
        if (res <= tol) { status = 0; break; }
        if (res < 0.999 * best) { best = res; since_best = 0; }
        else if (++since_best > 400) break; /* stagnation */
        if (k >= maxit) break;
        oracle_sip_apply(m, lam, nu, nu_const, p, q, NULL, 0);
        const double pq = dot(p, q, ndof);
        if (!(pq > 0.0)) { status = -4; break; }
        const double alpha = rz / pq;
        for (long i = 0; i < ndof; ++i) { u[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
        if (lam == 0.0) {
            double mr = 0.0;
            for (long i = 0; i < ndof; ++i) mr += r[i];
            mr /= (double)ndof;
            for (long i = 0; i < ndof; ++i) r[i] -= mr;
        }
        for (long i = 0; i < ndof; ++i) z[i] = dinv[i] * r[i];
        const double rz_new = dot(r, z, ndof);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (long i = 0; i < ndof; ++i) p[i] = z[i] + beta * p[i];
        ++k;
    }
    if (lam == 0.0) { /* zero mass-weighted mean */
        double sm = 0.0, smu = 0.0;
        for (long i = 0; i < ndof; ++i) { sm += mass[i]; smu += mass[i] * u[i]; }
        for (long i = 0; i < ndof; ++i) u[i] -= smu / sm;
    }
    if (iters) *iters = k;
    if (relres) *relres = res;
    free(mass); free(fp); free(r); free(z); free(p); free(q); free(dinv);
    return status;
}

/* ------------------------------------------------------------------------- */
/* LLF convection (explicit Gauss quadrature, dense basis evaluation)          */
/* ------------------------------------------------------------------------- */

static void convect_element(const ctx_t *c, int Q, const double *zeta, const double *omega,
                            double Bq[MAXN][MAXN], double Gq[MAXN][MAXN],
                            double Bend[2][MAXN], double Gend[2][MAXN],
                            const double *const *v, long e, double *const *outk, long k)
{
    const int npe = c->npe, dim = c->dim;
    const int nq[3] = {Q, Q, dim == 3 ? Q : 1};
    const int nqe = nq[0] * nq[1] * nq[2];
    double y[3][MAXN * MAXN * MAXN];
    for (int cc = 0; cc < dim; ++cc)
        for (int I = 0; I < npe; ++I) y[cc][I] = 0.0;
    (void)zeta;

    /* volume: sum_q W_q sum_e v_c v_e d_e phi_I */
    for (int g = 0; g < nqe; ++g) {
        int gc[3] = {g % nq[0], (g / nq[0]) % nq[1], g / (nq[0] * nq[1])};
        double L1[3][MAXN], G1[3][MAXN];
        double W = 1.0;
        for (int d = 0; d < dim; ++d) {
            W *= omega[gc[d]] * c->h[d] * 0.5;
            for (int j = 0; j < c->n; ++j) { L1[d][j] = Bq[gc[d]][j]; G1[d][j] = Gq[gc[d]][j]; }
        }
        double vq[3] = {0.0, 0.0, 0.0};
        for (int J = 0; J < npe; ++J) {
            int Jc[3];
            nd_coords(c, J, Jc);
            const double phi = tp_val(c, L1, Jc);
            for (int cc = 0; cc < dim; ++cc) vq[cc] += v[cc][e * (long)npe + J] * phi;
        }
        for (int I = 0; I < npe; ++I) {
            int Ic[3];
            nd_coords(c, I, Ic);
            for (int ed = 0; ed < dim; ++ed) {
                const double dphi = tp_grad(c, L1, G1, Ic, ed);
                for (int cc = 0; cc < dim; ++cc) y[cc][I] += W * vq[cc] * vq[ed] * dphi;
            }
        }
    }
    /* faces: - sum_q W^F_q h_c [phi_I], own-side test traces */
    for (int d = 0; d < dim; ++d) {
        for (int side = -1; side <= 1; side += 2) {
            const long enb = el_neighbour(c, e, d, side);
            const int own_end = side > 0 ? 1 : 0, nb_end = side > 0 ? 0 : 1; /* 0: xi=-1, 1: xi=+1 */
            const double sgn = side > 0 ? 1.0 : -1.0;
            int nf[3] = {nq[0], nq[1], nq[2]};
            nf[d] = 1;
            const int nfe = nf[0] * nf[1] * nf[2];
            for (int g = 0; g < nfe; ++g) {
                int gc[3] = {g % nf[0], (g / nf[0]) % nf[1], g / (nf[0] * nf[1])};
                double Lo[3][MAXN], Go[3][MAXN], Ln[3][MAXN], Gn[3][MAXN];
                double WF = 1.0;
                for (int dd = 0; dd < dim; ++dd) {
                    for (int j = 0; j < c->n; ++j) {
                        if (dd == d) {
                            Lo[dd][j] = Bend[own_end][j]; Go[dd][j] = Gend[own_end][j];
                            Ln[dd][j] = Bend[nb_end][j];  Gn[dd][j] = Gend[nb_end][j];
                        } else {
                            Lo[dd][j] = Ln[dd][j] = Bq[gc[dd]][j];
                            Go[dd][j] = Gn[dd][j] = Gq[gc[dd]][j];
                        }
                    }
                    if (dd != d) WF *= omega[gc[dd]] * c->h[dd] * 0.5;
                }
                double vo[3] = {0, 0, 0}, vn[3] = {0, 0, 0};
                for (int J = 0; J < npe; ++J) {
                    int Jc[3];
                    nd_coords(c, J, Jc);
                    const double po = tp_val(c, Lo, Jc), pn = tp_val(c, Ln, Jc);
                    for (int cc = 0; cc < dim; ++cc) {
                        vo[cc] += v[cc][e * (long)npe + J] * po;
                        vn[cc] += v[cc][enb * (long)npe + J] * pn;
                    }
                }
                const double *vm = side > 0 ? vo : vn, *vp = side > 0 ? vn : vo;
                const double vnm = vm[d], vnp = vp[d]; /* v.n with n = +e_d */
                const double Lam = 2.0 * fmax(fabs(vnm), fabs(vnp));
                double hflux[3];
                for (int cc = 0; cc < dim; ++cc)
                    hflux[cc] = 0.5 * (vnm * vm[cc] + vnp * vp[cc]) + 0.5 * Lam * (vm[cc] - vp[cc]);
                for (int I = 0; I < npe; ++I) {
                    int Ic[3];
                    nd_coords(c, I, Ic);
                    const double jphi = sgn * tp_val(c, Lo, Ic); /* [phi_I], own-side trace */
                    for (int cc = 0; cc < dim; ++cc) y[cc][I] -= WF * hflux[cc] * jphi;
                }
            }
        }
    }
    /* M^{-1}, GLL-lumped */
    for (int I = 0; I < npe; ++I) {
        int Ic[3];
        nd_coords(c, I, Ic);
        const double mI = vol_weight(c, Ic);
        for (int cc = 0; cc < dim; ++cc) outk[cc][k * (long)npe + I] = y[cc][I] / mI;
    }
}

int oracle_convect(const oracle_mesh *m, const double *const *v, double *const *out,
                   const long *elems, long nel)
{
    /* reading A13: Q = floor(3P/2) + 1 Gauss points per direction (2Q - 1 >= 3P) */
    return oracle_convect_q(m, (3 * m->P) / 2 + 1, v, out, elems, nel);
}

int oracle_convect_q(const oracle_mesh *m, int Q, const double *const *v, double *const *out,
                     const long *elems, long nel)
{
    ctx_t c;
    if (ctx_init(m, &c) || !v || !out) return -1;
    for (int cc = 0; cc < c.dim; ++cc)
        if (!v[cc] || !out[cc]) return -1;
    if (Q < 1 || Q > MAXN) return -1;
    double zeta[MAXN], omega[MAXN];
    double Bq[MAXN][MAXN], Gq[MAXN][MAXN], Bend[2][MAXN], Gend[2][MAXN];
    if (oracle_gauss(Q, zeta, omega)) return -1;
    for (int g = 0; g < Q; ++g) oracle_lagrange(c.P, c.xi, zeta[g], Bq[g], Gq[g]);
    oracle_lagrange(c.P, c.xi, -1.0, Bend[0], Gend[0]);
    oracle_lagrange(c.P, c.xi, +1.0, Bend[1], Gend[1]);
    const long cnt = elems ? nel : c.nel;
    for (long k = 0; k < cnt; ++k)
        if (elems && (elems[k] < 0 || elems[k] >= c.nel)) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (long k = 0; k < cnt; ++k) {
        const long e = elems ? elems[k] : k;
        convect_element(&c, Q, zeta, omega, Bq, Gq, Bend, Gend, v, e, out, k);
    }
    return 0;
}
