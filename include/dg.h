/*
 * dg.h -- C-ABI of libdgsip.so, the B200-native (sm_100a) implicit-stage hot path of
 * arXiv 2112.04167 (Guesmi, Grotteschi, Stiller, "Assessment of high-order IMEX methods
 * for incompressible flow").  Citations "P:L" are lines of the paper text
 * (/root/reference/PAPER.md); readings A1..A21 are SURVEY.md §8(c), A22..A25 DESIGN.md's, all listed in DESIGN.md.
 *
 * What is computed.  Each IMEX-RK stage (Alg. 3) solves
 *   line 5:  a periodic pressure Poisson problem  -lap psi = rhs  (lam = 0)
 *   line 9:  per velocity component  v - dt a_ii div(nu grad v) = g,
 *                        i.e.  lam v - div(nu grad v) = f  with lam = 1/(dt a_ii), f = lam g
 * discretised by the symmetric interior-penalty DG method on tensor-product
 * GLL elements of degree P, plus the explicit DG convective term
 * F_c = -div(v v) with local Lax-Friedrichs fluxes.  Built on these:
 * the DG divergence/gradient pair of the projection (lines 5-6), whole IMEX-RK steps for
 * constant viscosity and for the solution-dependent viscosity of P:1222 (with F_d2/F_d3,
 * forcing and the final projection), and a two-level Schwarz preconditioner for the solves
 * (readings A22-A25 in DESIGN.md).
 *
 * Mesh and data layout (all calls).  Periodic box [0,L0]x[0,L1](x[0,L2]) with N[d]
 * uniform elements per direction.  Global element index e = ex + N0*(ey + N1*ez);
 * node index i + n*(j + n*k), n = P+1.  Every field is a caller-owned DEVICE array of
 * double, [local_elements][n^dim], holding the contiguous slab of elements owned by this
 * rank: ranks split the slowest direction (z in 3-D, y in 2-D) into equal slabs, rank r
 * owning global elements [r*E, (r+1)*E), E = N_el / nranks.
 *
 * Operator (dg_helmholtz_apply, weak form, reading A5):
 *   (A u)_I = sum_K sum_{q in GLL^d} W_q [lam phi_I u + nu grad phi_I . grad u](x_q)
 *           + sum_F sum_{q in GLL^{d-1}} W^F_q [-{nu d_n u}[phi_I] - {nu d_n phi_I}[u]
 *                                              + sigma [u][phi_I]],
 *   W_q = prod_d w_{q_d} h_d/2 (GLL collocation, reading A2), sigma = tau (nu^- + nu^+)/2,
 *   tau = (P+1)^2 / h_d  (readings A1, A3).  A is symmetric; PSD with null space {1} at
 *   lam = 0, SPD for lam > 0.
 *
 * Streams.  Every call is enqueued on the mesh's stream (set at create or by
 * dg_mesh_set_stream; NULL = legacy default stream).  apply/diag/convect are
 * asynchronous; dg_pcg_solve returns after convergence (it synchronises with the host
 * every few iterations to test convergence).
 *
 * Errors.  No exception crosses the ABI.  Every call returns a dg_status; the message of
 * the last failing call on this thread is dg_last_error().  Invalid arguments
 * (null pointers, P outside [1,10], N[d] < 1, slab split not exact, lam < 0, nu_const <= 0
 * when nu == NULL, tol <= 0, maxit < 1) return DG_EINVAL before anything is enqueued.
 * A nu field is not scanned for positivity on the hot path (it is the caller's
 * precondition, "nu_field > 0"); dg_check_field() does that on request.
 */
#ifndef DG_H
#define DG_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct dg_mesh dg_mesh; /* opaque; owns all workspace, NCCL comm and halo buffers */

typedef enum {
    DG_OK = 0,
    DG_EINVAL = 1,       /* invalid argument                                   */
    DG_ECUDA = 2,        /* CUDA runtime error (message has cudaGetErrorString) */
    DG_ENCCL = 3,        /* NCCL error                                          */
    DG_ENOMEM = 4,       /* device allocation failed                            */
    DG_ENOTCONV = 5,     /* maxit reached; info holds the final residual        */
    DG_EBREAKDOWN = 6,   /* CG breakdown: p^T A p <= 0 or a non-finite scalar  */
    DG_EUNSUPPORTED = 7  /* configuration not compiled (e.g. P > 10)            */
} dg_status;

typedef struct {
    int iters;           /* CG iterations performed                             */
    double rel_res;      /* ||M^-1 r||_2 / ||f||_2 at exit (RMS residual at the
                            collocation points; reading A7)             */
    double removed_mean; /* lam == 0: mass-weighted mean removed from f (A8)    */
    double f_norm;       /* ||f||_2 after the lam == 0 projection               */
    double kappa_est;    /* Lanczos estimate of cond(B A) from CG alpha/beta (B = the
                            mesh's preconditioner, dg_mesh_set_precond)        */
} dg_solve_info;

/* NCCL unique id for multi-rank meshes (call on rank 0, broadcast the 128 bytes with
 * torch.distributed, pass to dg_mesh_create on every rank). */
dg_status dg_nccl_unique_id(unsigned char out[128]);

/* Create a mesh: GLL tables for degree P, periodic
 * structured connectivity, the slab of rank `rank` out of `nranks`, and all workspace
 * (PCG vectors, reduction scratch, halo buffers, NCCL communicator and exchange stream:
 * the hot calls never allocate).
 * dim in {2,3}; N[d] >= 1; L[d] > 0; 1 <= P <= 10; N[dim-1] % nranks == 0.
 * nccl_uid: required when nranks > 1.  With nranks == 1, NULL gives the plain single-GPU
 * mesh (the slab wraps onto itself); a non-NULL id selects the HALO MODE: a 1-rank NCCL
 * communicator, and every slab-boundary face of the slowest direction goes through the same
 * face-trace exchange (self send/recv) and halo-consuming kernels as a multi-rank slab -- the
 * multi-GPU data plane, testable on one GPU (SURVEY.md:311; results equal the plain mesh's).
 * Face-trace halo (operator apply, diagonal, PCG): per face node of the neighbour's boundary
 * layer, u, nu d_n u and nu (nu once per solve), exchanged on a separate stream while the
 * interior element layers are applied; the once-per-stage kernels (convection,
 * DG pair, DG derivative) exchange the boundary element layers.
 * cuda_stream: a cudaStream_t (may be NULL).
 * The caller must have selected the device (cudaSetDevice) before the call.  */
dg_status dg_mesh_create(int dim, const int N[3], const double L[3], int P, int rank, int nranks,
                         const unsigned char *nccl_uid, void *cuda_stream, dg_mesh **out);
void dg_mesh_destroy(dg_mesh *m);
dg_status dg_mesh_set_stream(dg_mesh *m, void *cuda_stream);

long long dg_mesh_local_ndof(const dg_mesh *m);      /* local_elements * (P+1)^dim    */
long long dg_mesh_local_elements(const dg_mesh *m);
long long dg_mesh_element_offset(const dg_mesh *m);  /* first global element owned   */

/* Node coordinates of the local slab: xyz is a DEVICE array [dim][local_ndof]. */
dg_status dg_mesh_node_coords(const dg_mesh *m, double *xyz);

/* GLL lumped mass m_I = prod_d w h_d/2 of the local slab, DEVICE [local_ndof]. */
dg_status dg_mesh_mass(const dg_mesh *m, double *mass);

/* out = A u (weak form, see above).  nu: DEVICE nodal viscosity [local_ndof] or NULL for
 * the constant nu_const.  u and out must not alias.  lam >= 0.  Multi-rank: collective
 * (face halos are exchanged with NCCL over NVLink). */
dg_status dg_helmholtz_apply(dg_mesh *m, double lam, const double *nu, double nu_const,
                             const double *u, double *out);

/* diag = diag(A) (the Jacobi preconditioner of the north star). */
dg_status dg_helmholtz_diag(dg_mesh *m, double lam, const double *nu, double nu_const, double *diag);

/* Solve A u = M f (M = GLL-lumped mass, reading A6) by preconditioned CG (Jacobi unless
 * dg_mesh_set_precond chose the two-level Schwarz preconditioner).
 * f: DEVICE nodal rhs.  u: DEVICE, initial guess on entry, solution on exit.
 * Stops when ||M^-1 r||_2 <= tol ||f||_2 (reading A7) -> DG_OK, or after maxit
 * iterations -> DG_ENOTCONV (u and info hold the last iterate).  lam == 0 (pressure
 * Poisson, Alg. 3 line 5): f is projected to zero mass-weighted mean (info.removed_mean),
 * the residual is kept orthogonal to constants, u is returned with zero mass-weighted
 * mean (reading A8).  info may be NULL.  Collective for multi-rank meshes. */
dg_status dg_pcg_solve(dg_mesh *m, double lam, const double *nu, double nu_const, const double *f,
                       double tol, int maxit, double *u, dg_solve_info *info);

/* Preconditioner of every later dg_pcg_solve on this mesh (including the solves inside
 * dg_imex_stage / dg_imex_rk_step).  DG_PC_JACOBI (default): diag(A)^-1 (the north star).
 * DG_PC_SCHWARZ2: two-level additive Schwarz (the paper solves with
 * "Krylov-accelerated Schwarz/multigrid methods", formula not given; reading in
 * DESIGN.md §9):
 *     B r = sum_K R_K^T A_KK^-1 R_K r + P_1 A_c^+ P_1^T r,   A_c = P_1^T A P_1,
 * non-overlapping element blocks (exact, by fast diagonalisation of the Kronecker-sum block)
 * plus the continuous vertex-based Q1 space on the same mesh as coarse space (exact solve by
 * a real Fourier diagonalisation; pseudo-inverse on the constants for lam = 0).  Exact
 * blocks / coarse operator for a constant viscosity; for a nu field both are built with the
 * mass-weighted mean viscosity (computed on the device per solve): a spectrally equivalent
 * preconditioner (constant max nu / min nu).  In dg_pcg_solve the coarse term is used while
 * diffusion dominates at the element scale, lam min_d h_d^2 <= 50 nu (above, the element
 * blocks alone converge faster: measured); dg_schwarz_apply always applies the full B.
 * Needs 2 <= N_d <= 64 and P >= 2 (else DG_EUNSUPPORTED here).  Multi-rank: the coarse residual is all-reduced
 * (NV = prod N_d doubles per iteration) and every rank solves the coarse problem. */
#define DG_PC_JACOBI 0
#define DG_PC_SCHWARZ2 1
dg_status dg_mesh_set_precond(dg_mesh *m, int precond);
int dg_mesh_get_precond(const dg_mesh *m);

/* z = B r with the DG_PC_SCHWARZ2 preconditioner above for (lam, nu_const) (independent of
 * the mesh's setting; for tests and for use as a smoother).  r, z: DEVICE [local_ndof], no
 * aliasing.  Collective for multi-rank meshes. */
dg_status dg_schwarz_apply(dg_mesh *m, double lam, double nu_const, const double *r, double *z);

/* Explicit convective tendency F_c = -div(v v) with LLF fluxes, nodal (M^-1 applied,
 * GLL-lumped), Gauss quadrature with Q = floor(3P/2)+1 points per direction
 * (readings A12-A14).  v[c], out[c]: DEVICE [local_ndof], c < dim.
 * out must not alias v. */
dg_status dg_convect_rhs(dg_mesh *m, const double *const v[3], double *const out[3]);

/* DG divergence / gradient pair of the projection step (Alg. 3 lines 5-6; SURVEY
 * NEXT-1).  mv: velocity mesh (degree P >= 2), mp: pressure mesh with the same dim, N, L,
 * rank/nranks and degree P-1.  Integrals on the velocity GLL grid (exact for these
 * integrands), central fluxes {.} = (minus + plus)/2, [.] = minus - plus, n from the minus to
 * the plus element:
 *   dg_divergence: div_weak_a = -sum_K sum_q W_q v(x_q).grad phi^p_a(x_q)
 *                               + sum_F sum_q W^F_q ({v}.n)[phi^p_a]        (pressure layout)
 *   dg_gradient:   grad_weak_{c,i} = -sum_K sum_q W_q psi_h(x_q) d_c phi^v_i(x_q)
 *                               + sum_F sum_q W^F_q {psi_h} n_c [phi^v_i]   (velocity layout)
 * with psi_h the pressure interpolant at the velocity nodes.  -grad is the transpose of div;
 * both are exact (= the weak forms of div v and grad psi) for continuous polynomial fields of
 * degree <= P-1.  Weak vectors: nodal values are M^-1 times them.  DEVICE arrays; the call
 * runs on mv's stream; collective for multi-rank meshes (face halos over NCCL).  The
 * div/mass-flux stabilisation of P:1040 is not part of the pair (its formula is not in the
 * paper). */
dg_status dg_divergence(dg_mesh *mv, dg_mesh *mp, const double *const v[3], double *div_weak);
dg_status dg_gradient(dg_mesh *mp, dg_mesh *mv, const double *psi, double *const grad_weak[3]);

/* One IMEX-RK stage i = 2 of Alg. 3 for constant viscosity nu, F_s = 0 and
 * periodic boundaries (the config-4 composition):
 *   line 4: v' = v + dt a_ex21 (F_c + F_d + F_d3)(v),  F_c by dg_convect_rhs (LLF),
 *           F_d1 = -M^-1 A_0 v (the SIP operator at lam = 0, P:693 F_d1 = div nu grad v) and,
 *           for constant nu, F_d2 = -F_d3 = nu grad div v = nu M^-1 G M_p^-1 D v with the DG
 *           pair below (F_d + F_d3 = F_d1 - nu grad div v: the rotational form);
 *   line 5: -lap psi = -div v' on the pressure mesh mp (degree P-1; reading A9):
 *           SIP Poisson with the weak DG divergence of v' as rhs (b = -D v'), solved
 *           by dg_pcg_solve (lam = 0: mean projection, reading A8) from psi = 0;
 *   line 6: v'' = v' - M^-1 G psi with the weak DG gradient G (dg_gradient);
 *   line 8: g = v'' + dt [(a_im21 - a_ex21) F_d1(v) - a_ex21 F_d3(v)];
 *   line 9: per component, solve v - dt a_im22 nu lap v = g, i.e. lam = 1/(dt a_im22),
 *           f = lam g (reading A4), by dg_pcg_solve from the initial guess v''.
 * The projection is approximate (the SIP pressure operator is not -D M^-1 G), as in the
 * paper's splitting; the final projection (lines 12-15) is skipped for constant nu.
 * mv: velocity mesh (degree P >= 2); mp: pressure mesh with the same dim, N, L, rank/nranks
 * and degree P-1.  v[c], vout[c] (c < dim): DEVICE [local_ndof of mv], vout must not alias
 * v; psi: DEVICE [local_ndof of mp].  Runs on mv's stream; synchronous (it contains solves).
 * The stage workspace (2 dim velocity fields, one pressure field) is allocated on first use
 * and owned by the meshes.  Errors: DG_EINVAL for mismatched meshes or non-positive dt,
 * a_im22, nu, tol or maxit; solver errors as dg_pcg_solve (info holds every solve). */
typedef struct {
    dg_solve_info pressure;
    dg_solve_info velocity[3];
    dg_solve_info stab;  /* the divergence / mass-flux stabilisation solve (0 iterations when off) */
} dg_stage_info;

dg_status dg_imex_stage(dg_mesh *mv, dg_mesh *mp, double dt, double a_ex21, double a_im21, double a_im22,
                        double nu, const double *const v[3], double *const vout[3], double *psi, double tol,
                        int maxit, dg_stage_info *info);

/* One step of an IMEX Runge-Kutta method (Alg. 3) for constant nu,
 * F_s = 0, periodic boundaries, with the CK-type tableaux of the paper's appendix
 * (implicit DIRK with a_im[0][0] = 0 and a strictly lower explicit tableau, equal
 * nodes c).  With constant nu, F_d2 = -F_d3 = nu grad(div u), formed with the DG
 * pair as nu M^-1 G M_p^-1 D u, so that the explicit viscous part of line 4 is the rotational,
 * divergence-free form F_d + F_d3 = F_d1 - nu grad div u.  Stage 1: v_1 = v.
 * Stages i = 2..s: line 4 v'_i = v + dt sum_j a_ex[i][j] (F_c + F_d1 - nu grad div u)_j,
 * lines 5-6 (projection with the DG divergence/gradient pair and the SIP Poisson solve on
 * mp), line 8 g_i = v''_i + dt sum_j [(a_im - a_ex)[i][j] F_d1,j + a_ex[i][j] nu grad div u_j],
 * line 9 (Helmholtz solves, lam = 1/(dt a_im[i][i]), from the guess v''_i; a stage with
 * a_im[i][i] = 0 takes v_i = g_i); line 11: v = v_s + dt sum_i [(b_ex - a_ex[s])_i F_c,i +
 * (b_im - a_im[s])_i F_d1,i] (F_d2 + F_d3 = 0).  The final projection (lines 12-15) is
 * skipped for constant nu.
 * v[c] (c < dim): DEVICE velocity, in: v^n, out: v^{n+1}; psi: DEVICE pressure workspace (the
 * last stage's psi'' on exit; the first implicit stage's Poisson solve starts from 0, later
 * stages from the previous stage's psi'').  Workspace (3 s + 2) dim velocity fields, owned by mv.
 * Synchronous.  DG_EINVAL for a malformed tableau (s outside [2, 8], a non-explicit first
 * stage, upper-triangular entries) or bad scalars; solver errors as dg_pcg_solve. */
#define DG_RK_MAX_STAGES 8
typedef struct {
    int s;
    double c[DG_RK_MAX_STAGES];
    double a_im[DG_RK_MAX_STAGES][DG_RK_MAX_STAGES];
    double a_ex[DG_RK_MAX_STAGES][DG_RK_MAX_STAGES];
    double b_im[DG_RK_MAX_STAGES];
    double b_ex[DG_RK_MAX_STAGES];
} dg_tableau;

typedef struct {
    int stages;          /* implicit stages performed (s - 1)                 */
    int pressure_iters;  /* CG iterations summed over the Poisson solves     */
    int velocity_iters;  /* CG iterations summed over the Helmholtz solves   */
    int stab_iters;      /* CG iterations of the divergence stabilisation    */
} dg_step_info;

dg_status dg_imex_rk_step(dg_mesh *mv, dg_mesh *mp, const dg_tableau *tab, double dt, double nu,
                          double *const v[3], double *psi, double tol, int maxit, dg_step_info *info);

/* One step of Alg. 3 with the solution-dependent viscosity of P:1218-1224,
 * nu(v) = nu0 + nu1 (|v| / vmax)^2, forcing F_s and the final projection:
 *   stage 1: v_1 = v, nu_1 = nu(v);  stages i = 2..s:
 *   line 4:  v'_i = v + dt [sum_{j<i} a_ex[i][j] (F_c + F_d1 + F_d2 + 2 F_d3)_j
 *                          + sum_{j<=i} a_im[i][j] F_s,j]   (F_d + F_d3)
 *   lines 5-6: projection with the DG pair and the SIP Poisson solve on mp (as dg_imex_rk_step);
 *   line 7:  nu_i = nu(v''_i) at the nodes;
 *   line 8:  g_i = v''_i + dt sum_{j<i} [(a_im - a_ex)[i][j] F_d1,j - a_ex[i][j] F_d3,j];
 *   line 9:  v_i - dt a_im[i][i] div(nu_i grad v_i) = g_i  (variable-nu SIP Helmholtz, Jacobi-PCG);
 *   line 11: v = v_s + dt sum_i [(b_ex - a_ex[s])_i (F_c + F_d2 + F_d3)_i
 *                               + (b_im - a_im[s])_i (F_d1 + F_s)_i];
 *   lines 12-15 (final_projection != 0): lap psi = div v, v <- v - grad psi.
 * Stage forces of stage i use nu_i (the viscosity of its implicit solve; stage 1: nu(v)):
 * F_c by dg_convect_rhs, F_d1 = -M^-1 A_0(nu_i) u (SIP, lam = 0, nodal nu field), and, with the
 * velocity-level central-flux DG derivative (D_c u)_i = m_i^-1 [-sum_K (u, d_c phi_i)_GLL +
 * sum_F ({u} n_c, [phi_i])_GLL]:  F_d2,c = sum_e D_e(nu D_c u_e),  F_d3,c = -D_c(nu sum_e D_e u_e)
 * (readings in DESIGN.md §9; for constant nu F_d2 + F_d3 = 0 exactly, the D_c commute).
 * fs: NULL (F_s = 0) or s*dim DEVICE pointers, fs[j*dim + c] = F_s,c at t + c_j dt (nodal).
 * The Helmholtz solves (variable nu) and the Poisson solves use the preconditioner set on mv
 * and mp respectively (DG_PC_SCHWARZ2 uses the mean viscosity for the variable-nu solves).  Workspace (4 s + 2) dim + dim^2 + 2 velocity fields, owned by mv.
 * Synchronous.  Errors as dg_imex_rk_step; DG_EINVAL for nu0 <= 0, nu1 < 0 or vmax <= 0. */
typedef struct {
    double nu0, nu1, vmax;
} dg_visc_model;

dg_status dg_imex_rk_step_vv(dg_mesh *mv, dg_mesh *mp, const dg_tableau *tab, double dt, const dg_visc_model *visc,
                             const double *const *fs, int final_projection, double *const v[3], double *psi,
                             double tol, int maxit, dg_step_info *info);

/* Velocity-level central-flux DG derivatives out[c] = D_c u (c < dim; out[c] may be NULL to
 * skip a direction), the operator of dg_imex_rk_step_vv's F_d2 / F_d3.  DEVICE arrays of m;
 * no aliasing of u with out.  Collective for multi-rank meshes. */
dg_status dg_derivative(dg_mesh *m, const double *u, double *const out[3]);

/* Divergence / mass-flux stabilisation of the projection step (§3.3: "For
 * pressure robustness a divergence/mass-flux stabilization is added as proposed in [Joshi
 * 2016, Akbas 2018]"; the formula is not in the paper -- reading A26; SURVEY
 * NEXT-1).  After the projection v'' = v' - M^-1 G psi, solve for v^ in the velocity DG space
 *   (M + a_D K_D + a_C K_C) v^ = M v'',
 *   (K_D v)_{c,I} = sum_K sum_q W_q (div v)(x_q) d_c phi_I(x_q)       broken (element) divergence
 *   (K_C v)_{c,I} = sum_{F normal to c} sum_q W^F_q [v_c] [phi_I]       normal-velocity jumps
 * (GLL collocation quadrature, [g] = g^- - g^+), a_D = dt zeta_D U h / (P+1), a_C = dt zeta_C U,
 * U = sqrt(sum m |v''|^2 / sum m) the RMS velocity, h = (prod_d h_d)^(1/dim).  SPD; Jacobi-
 * preconditioned CG over the dim components, stopped at ||M^-1 r|| <= tol ||v''||, from v''.
 *
 * dg_mesh_set_div_stab(mv, zeta_D, zeta_C): zeta > 0 switches the step on for every projection
 *   of dg_imex_stage, dg_imex_rk_step and dg_imex_rk_step_vv on this velocity mesh (after line 6
 *   and after the final projection) and allocates its workspace (4 dim ndof doubles); 0, 0
 *   switches it off.  Not a hot call.
 * dg_div_stab_apply: out[c] = ((M + a_D K_D + a_C K_C) v)_c (weak), explicit coefficients.
 * dg_div_stab_solve: v (in: v'', out: v^) for (dt, zeta_D, zeta_C); coef (may be NULL) returns
 *   (a_D, a_C, U).  Needs the workspace of dg_mesh_set_div_stab (DG_EINVAL otherwise).
 * DEVICE arrays [local_ndof]; collective for multi-rank meshes (element-layer halos). */
dg_status dg_mesh_set_div_stab(dg_mesh *mv, double zeta_D, double zeta_C);
dg_status dg_div_stab_apply(dg_mesh *m, double a_D, double a_C, const double *const v[3], double *const out[3]);
dg_status dg_div_stab_solve(dg_mesh *m, double dt, double zeta_D, double zeta_C, double *const v[3], double tol,
                            int maxit, double coef[3], dg_solve_info *info);

/* Host-buffer variants: same operations on HOST arrays; H2D and D2H copies through
 * mesh-owned device staging buffers are part of the call (allocated on first use). */
dg_status dg_helmholtz_apply_host(dg_mesh *m, double lam, const double *nu_host, double nu_const,
                                  const double *u_host, double *out_host);
dg_status dg_pcg_solve_host(dg_mesh *m, double lam, const double *nu_host, double nu_const,
                            const double *f_host, double tol, int maxit, double *u_host,
                            dg_solve_info *info);

/* Validate a nodal field (finite and, if positive != 0, > 0).  Synchronous. */
dg_status dg_check_field(dg_mesh *m, const double *x, int positive);

/* The product path's 1-D tables for degree P (host arrays): GLL nodes xi[P+1], weights
 * w[P+1] and the differentiation matrix D[(P+1)*(P+1)] (row-major, D[i][j] = l_j'(xi_i)).
 * Introspection only (tests pin them against closed forms); no CUDA call. */
dg_status dg_gll_tables(int P, double *xi, double *w, double *D);

/* Number of kernel launches this mesh enqueued since creation (evidence for bench.py). */
long long dg_mesh_launch_count(const dg_mesh *m);

/* The last operator-apply kernel this thread dispatched (generation, template parameters, grid,
 * brick shape), e.g. "v6::k_apply6<dim=3,P=5,varnu=1,mode=0> grid=148 brick=4x4x1" (evidence for
 * bench.py's roofline line). */
const char *dg_last_apply_kernel(void);

/* Message for the last failing call on this thread ("" if none). */
const char *dg_last_error(void);

/* Library version string. */
const char *dg_version(void);

#ifdef __cplusplus
}
#endif
#endif
