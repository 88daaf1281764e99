/*
 * dg_oracle.h -- plain, slow CPU oracle for the SIP-DG implicit-stage hot path of
 * arXiv 2112.04167 (Guesmi, Grotteschi, Stiller).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library.  It shares no code, header, table or constant with the CUDA product path
 * (paper_2112_04167_b200/csrc, include/dg.h), and neither side includes the other.
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L (the paper's text), with the
 * section / equation / algorithm line.  Readings where the paper is silent are
 * SURVEY.md §8(c) A1..A21 and are listed in DESIGN.md "Readings".
 *
 * Mesh / layout (input recipe): periodic box [0,L0]x[0,L1](x[0,L2]),
 * N[d] uniform elements per direction, element e = ex + N0*(ey + N1*ez),
 * node index i + n*(j + n*k), n = P+1; every nodal array is [N_el][n^dim] double.
 *
 * Parity status of every function is stated in its comment and in DESIGN.md.
 */
#ifndef DG_ORACLE_H
#define DG_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int dim;          /* 2 or 3                                   */
    int N[3];         /* elements per direction (N[2]=1 in 2D)    */
    double L[3];      /* box lengths                              */
    int P;            /* polynomial degree, n = P+1 GLL points    */
} oracle_mesh;

/* GLL nodes/weights on [-1,1] ("tensor-product Lagrange polynomials based on GLL
 * points"): xi_0=-1, xi_P=1, interior = roots of P_P'(x); w_i = 2/(P(P+1) P_P(xi_i)^2).
 * Newton in long double.  Returns 0 on success. */
int oracle_gll(int P, double *xi, double *w);

/* Gauss-Legendre points/weights, Q points (used for "consistent integration" of the
 * convective term; reading A13: Q = floor(3P/2)+1). */
int oracle_gauss(int Q, double *zeta, double *omega);

/* Lagrange basis on the nodes xi[0..P] and its derivative at x by the PRODUCT formula:
 * l_j(x) = prod_{m!=j} (x-xi_m)/(xi_j-xi_m). */
void oracle_lagrange(int P, const double *xi, double x, double *l, double *dl);

/* SIP-DG Helmholtz operator action, weak form (reading A5):
 *   (A u)_I = sum_K sum_{q in GLL^d(K)} W_q [lam phi_I u + nu grad phi_I . grad u](x_q)
 *           + sum_F sum_{q in GLL^{d-1}(F)} W^F_q [ -{nu d_n u}[phi_I] - {nu d_n phi_I}[u]
 *                                                  + sigma [u][phi_I] ]
 * sigma = tau (nu^- + nu^+)/2, tau = (P+1)^2/h  (BASELINE configs[0]; reading A1).
 * P:1039 (interior penalty), P:852-861 (Alg. 3 line 9), P:829-838 (Alg. 3 line 5, lam=0).
 * Explicit GLL quadrature (reading A2), uses the collocation identity l_j(xi_q)=delta_jq
 * of the product-formula basis.  nu==NULL -> constant nu_const.
 * Rows of the elements elems[0..nel-1] (elems==NULL -> all elements, nel ignored) are
 * written compactly to y[k*n^d + node]. */
int oracle_sip_apply(const oracle_mesh *m, double lam, const double *nu, double nu_const,
                     const double *u, double *y, const long *elems, long nel);

/* diag(A)_I = e_I^T A e_I evaluated by explicit quadrature of the quadratic form with the
 * full tensor-product basis evaluation (no collocation shortcut).  Same element
 * selection / compact output convention as oracle_sip_apply. */
int oracle_sip_diag(const oracle_mesh *m, double lam, const double *nu, double nu_const,
                    double *diag, const long *elems, long nel);

/* Brute-force dense matrix A (ndof x ndof, row-major) by explicit quadrature over all
 * (I, J, q) triples with the full tensor-product basis evaluated at every quadrature
 * point; no sparsity logic.  For tiny meshes (ndof <= ~4096). */
int oracle_sip_dense(const oracle_mesh *m, double lam, const double *nu, double nu_const,
                     double *A);

/* Solve A u = M f, M = GLL-lumped mass (reading A6), by Jacobi-preconditioned CG on
 * oracle_sip_apply / oracle_sip_diag (precond=0: plain CG).  lam==0 (periodic
 * pressure Poisson): f is projected to zero mass-weighted mean, the residual is kept in
 * 1-perp, u is returned with zero mass-weighted mean (reading A8).  Stops when
 * ||M^{-1} r||_2 <= tol ||f||_2 (RMS residual at collocation points; reading A7),
 * on stagnation, or at maxit.  u holds the initial guess on entry.  Returns 0 converged,
 * 1 not converged (iters/relres still filled), <0 error. */
int oracle_pcg_solve(const oracle_mesh *m, double lam, const double *nu, double nu_const,
                     const double *f, double tol, int maxit, int precond, double *u,
                     int *iters, double *relres, double *removed_mean);

/* Explicit DG convective tendency with local Lax-Friedrichs flux (P:693 F_c = -div(vv);
 * P:1038 "consistent integration and local Lax-Friedrichs fluxes"), GLL-lumped M^{-1}:
 *   F_c,c = M^{-1} [ sum_K sum_{q in Gauss^d} W_q sum_e v_c v_e d_e phi_I
 *                  - sum_F sum_{q in Gauss^{d-1}} W_q h_c [phi_I] ]
 *   h = 1/2((v^-.n) v^- + (v^+.n) v^+) + 1/2 Lambda (v^- - v^+),
 *   Lambda = 2 max(|v^-.n|, |v^+.n|)               (readings A12, A13, A14)
 * v[c] are dim nodal velocity components; out[c] compact per elems (see apply).
 * Values at Gauss points by dense basis evaluation sum_J v_J phi_J(x_q). */
int oracle_convect(const oracle_mesh *m, const double *const *v, double *const *out,
                   const long *elems, long nel);
/* The same with an explicit Gauss point count Q per direction (1 <= Q <= 18): used by the
 * pins that show Q = floor(3P/2)+1 is the smallest exact rule (tests/test_oracle_convect.py). */
int oracle_convect_q(const oracle_mesh *m, int Q, const double *const *v, double *const *out,
                     const long *elems, long nel);

#ifdef __cplusplus
}
#endif
#endif
