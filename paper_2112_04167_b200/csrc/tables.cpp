// tables.cpp -- 1-D GLL / Gauss tables of the product path.
//
// GLL nodes: xi_0 = -1, xi_P = 1, interior roots of P_P'(x) ("Lagrange polynomials
// based on GLL points"), found by Newton on P_P' with P_P'' from the Legendre ODE
// (1-x^2) P'' = 2x P' - P(P+1) P.  Weights w_i = 2 / (P(P+1) P_P(xi_i)^2).
// Differentiation matrix (collocation differentiation on GLL points) in the
// closed form  D_ij = P_P(xi_i) / (P_P(xi_j) (xi_i - xi_j)) (i != j),
// D_00 = -P(P+1)/4, D_PP = P(P+1)/4, else 0.
// Gauss points for the convective term (reading A13: Q = floor(3P/2)+1); interpolation
// matrix by the barycentric formula; derivative interpolation Gq = Bq D.
// All in long double, rounded once.
#include <cmath>
#include <mutex>

#include "dg_internal.h"

namespace dg {
namespace {

// P_k(x) and P_k'(x) by recurrences
void legendre(int k, long double x, long double *p, long double *dp)
{
    long double a = 1.0L, b = x, da = 0.0L, db = 1.0L;
    if (k == 0) { *p = 1.0L; *dp = 0.0L; return; }
    for (int m = 1; m < k; ++m) {
        long double c = ((2.0L * m + 1.0L) * x * b - (long double)m * a) / (m + 1.0L);
        long double dc = da + (2.0L * m + 1.0L) * b;  // P'_{m+1} = P'_{m-1} + (2m+1) P_m
        a = b; b = c; da = db; db = dc;
    }
    *p = b;
    *dp = db;
}

const long double PI_L = 3.14159265358979323846264338327950288L;

}  // namespace

static void build_eo(int P, const long double X[NMAX][NMAX], EOTab *e);

void build_tab(int P, Tab *t)
{
    const int n = P + 1;
    long double x[NMAX], lp[NMAX];
    for (int i = 0; i < n; ++i) {
        long double xi = -cosl(PI_L * i / P);
        if (i > 0 && i < P) {
            for (int it = 0; it < 200; ++it) {
                long double p, dp;
                legendre(P, xi, &p, &dp);
                long double d2p = (2.0L * xi * dp - (long double)P * (P + 1) * p) / (1.0L - xi * xi);
                long double dx = dp / d2p;
                xi -= dx;
                if (fabsl(dx) < 1e-19L) break;
            }
        }
        x[i] = xi;
        long double dp;
        legendre(P, xi, &lp[i], &dp);
    }
    for (int i = 0; i < n; ++i) {
        t->xi[i] = (double)x[i];
        t->w[i] = (double)(2.0L / ((long double)P * (P + 1) * lp[i] * lp[i]));
    }
    long double D[NMAX][NMAX];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (i != j) D[i][j] = lp[i] / (lp[j] * (x[i] - x[j]));
            else if (i == 0) D[i][j] = -(long double)P * (P + 1) / 4.0L;
            else if (i == P) D[i][j] = (long double)P * (P + 1) / 4.0L;
            else D[i][j] = 0.0L;
            t->D[i][j] = (double)D[i][j];
        }

    // constant-nu reference line matrix and even-odd tables
    {
        long double Kr[NMAX][NMAX], Dt[NMAX][NMAX];
        long double wl[NMAX];
        for (int i = 0; i < n; ++i) wl[i] = 2.0L / ((long double)P * (P + 1) * lp[i] * lp[i]);
        const long double kap = (long double)(P + 1) * (P + 1) / 2.0L;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                long double s = 0.0L;
                for (int k = 0; k < n; ++k) s += wl[k] * D[k][i] * D[k][j];
                if (i == P) s += -0.5L * D[P][j];
                if (j == P) s += -0.5L * D[P][i];
                if (i == 0) s += 0.5L * D[0][j];
                if (j == 0) s += 0.5L * D[0][i];
                if (i == j && (i == 0 || i == P)) s += kap;
                Kr[i][j] = s;
                Dt[i][j] = D[j][i];
            }
        for (int i = 0; i < NMAX; ++i)
            for (int j = 0; j < NMAX; ++j) t->Kref[i][j] = (i < n && j < n) ? (double)Kr[i][j] : 0.0;
        build_eo(P, D, &t->eD);
        build_eo(P, Dt, &t->eE);
        build_eo(P, Kr, &t->eK);
    }

    // Gauss-Legendre points for convection
    const int Q = (3 * P) / 2 + 1;
    t->Q = Q;
    for (int q = 0; q < Q; ++q) {
        // Tricomi-type initial guess, descending; stored ascending below
        long double z = (1.0L - (Q - 1.0L) / (8.0L * Q * Q * Q)) * cosl(PI_L * (4.0L * (q + 1) - 1.0L) / (4.0L * Q + 2.0L));
        for (int it = 0; it < 200; ++it) {
            long double p, dp;
            legendre(Q, z, &p, &dp);
            long double dz = p / dp;
            z -= dz;
            if (fabsl(dz) < 1e-19L) break;
        }
        long double p, dp;
        legendre(Q, z, &p, &dp);
        const int qa = Q - 1 - q;
        t->zq[qa] = (double)z;
        t->wq[qa] = (double)(2.0L / ((1.0L - z * z) * dp * dp));
        // barycentric interpolation to z:  l_j(z) = (lam_j/(z - x_j)) / sum_m lam_m/(z - x_m)
        long double lamb[NMAX], s = 0.0L;
        for (int j = 0; j < n; ++j) {
            long double pr = 1.0L;
            for (int m = 0; m < n; ++m)
                if (m != j) pr *= (x[j] - x[m]);
            lamb[j] = 1.0L / pr;
            s += lamb[j] / (z - x[j]);
        }
        long double B[NMAX];
        for (int j = 0; j < n; ++j) B[j] = (lamb[j] / (z - x[j])) / s;
        for (int j = 0; j < n; ++j) {
            t->Bq[qa][j] = (double)B[j];
            long double g = 0.0L;
            for (int k = 0; k < n; ++k) g += B[k] * D[k][j];
            t->Gq[qa][j] = (double)g;
        }
    }
}

static void build_eo(int P, const long double X[NMAX][NMAX], EOTab *e)
{
    const int n = P + 1, h = n / 2, mid = P / 2;
    for (int i = 0; i < HMAX; ++i) {
        for (int j = 0; j < HMAX; ++j) e->Te[i][j] = e->To[i][j] = 0.0;
        e->Tc[i] = e->Mr[i] = 0.0;
    }
    e->Mmid = 0.0;
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < h; ++j) {
            e->Te[i][j] = (double)((X[i][j] + X[i][P - j]) / 2.0L);
            e->To[i][j] = (double)((X[i][j] - X[i][P - j]) / 2.0L);
        }
    if (n % 2 == 1) {
        for (int i = 0; i < h; ++i) {
            e->Tc[i] = (double)X[i][mid];
            e->Mr[i] = (double)X[mid][i];
        }
        e->Mmid = (double)X[mid][mid];
    }
}

const Tab &host_tab(int P)
{
    static Tab tabs[PMAX + 1];
    static std::once_flag once;
    std::call_once(once, [] {
        for (int p = 1; p <= PMAX; ++p) build_tab(p, &tabs[p]);
    });
    return tabs[P];
}

}  // namespace dg
