// dg_internal.h -- internal declarations of libdgsip.so (product path; no oracle code).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "dg.h"

// Development switches (A/B measurements quoted in DESIGN.md) exist only in builds with
// -DDG_DEVELOPMENT (DG_EXTRA_DEFS=-DDG_DEVELOPMENT python paper_2112_04167_b200/build.py);
// the default build reads no environment variable on the product path.
#ifdef DG_DEVELOPMENT
#define DG_DEV_ENV(name) getenv(name)
#else
#define DG_DEV_ENV(name) ((const char *)nullptr)
#endif

namespace dg {

constexpr int PMAX = 10;         // highest compiled degree
constexpr int NMAX = PMAX + 1;   // GLL points per direction
constexpr int QMAX = (3 * PMAX) / 2 + 1;  // Gauss points for convection (reading A13)

constexpr int HMAX = NMAX / 2 + 1;  // even-odd half size

// Even-odd (Kopriva) factorisation of an n x n matrix X that is centro-symmetric (sym:
// X[P-i][P-j] = X[i][j]) or anti-centro-symmetric (anti: X[P-i][P-j] = -X[i][j]).
// h = n/2, mid = P/2 (odd n only):
//   Te[i][j] = (X[i][j] + X[i][P-j])/2,  To[i][j] = (X[i][j] - X[i][P-j])/2   (i, j < h)
//   Tc[i] = X[i][mid],  Mr[j] = X[mid][j],  Mmid = X[mid][mid]
struct EOTab {
    double Te[HMAX][HMAX];
    double To[HMAX][HMAX];
    double Tc[HMAX];
    double Mr[HMAX];
    double Mmid;
};

// Per-degree 1-D tables (host copy; uploaded to __constant__ memory by the kernels TU).
struct Tab {
    double xi[NMAX];          // GLL nodes on [-1,1]
    double w[NMAX];           // GLL weights
    double D[NMAX][NMAX];     // D[i][j] = l_j'(xi_i), closed form
    int Q;                    // Gauss points, floor(3P/2)+1        (reading A13)
    double zq[QMAX];          // Gauss nodes
    double wq[QMAX];          // Gauss weights
    double Bq[QMAX][NMAX];    // Bq[q][j] = l_j(zq_q)  (barycentric form)
    double Gq[QMAX][NMAX];    // Gq[q][j] = l_j'(zq_q) = (Bq D)[q][j]
    // Reference SIP line matrix for constant nu (reading A1: tau = (P+1)^2/h = (P+1)^2/2 * (2/h)):
    //   Kref = Kvol + F1 + (P+1)^2/2 F2,  Kvol[i][j] = sum_k w_k D[k][i] D[k][j],
    //   F1 = -1/2 (e_P D[P]^T + D[P] e_P^T) + 1/2 (e_0 D[0]^T + D[0] e_0^T),  F2 = e_0 e_0^T + e_P e_P^T
    // so that one element line contributes  (nu 2/h) Kref v  plus the neighbour terms.
    double Kref[NMAX][NMAX];
    EOTab eD, eE, eK;         // even-odd forms of D (anti), D^T (anti), Kref (sym)
};

// tables.cpp
void build_tab(int P, Tab *t);
const Tab &host_tab(int P);

// error plumbing (capi.cpp)
dg_status set_error(dg_status s, const std::string &msg);
char *last_apply_kernel();  // thread-local buffer (160 bytes): the last dispatched apply kernel

// ---------------------------------------------------------------------------
// kernel launch interface (kernels.cu)
// ---------------------------------------------------------------------------
struct Geom {
    int dim, P, n, npe;
    int N[3];        // global elements per direction (N[2] = 1 in 2-D)
    int Nl[3];       // local elements per direction (slowest one split by ranks)
    int B[3];        // brick (elements per CTA) per direction
    int nbk[3];      // bricks per direction (local)
    double h[3];     // element size per direction
    double tau[3];   // penalty (P+1)^2 / h_d (reading A1)
    double sd[3];    // 2 / h_d (reference-to-physical derivative factor)
    double wfac[3];  // transverse Jacobian of a line along d: prod_{d' != d} h_d'/2
    double mfac;     // element Jacobian prod_d h_d/2 (GLL mass m_I = w_i w_j (w_k) mfac)
    double wsd[3][NMAX];  // w_k * 2/h_d (GLL weight times derivative factor)
    long long nel;   // local elements
};

// Face-trace halos of the slab boundary faces of the slowest direction S (multi-rank slabs and
// the 1-rank halo mode): per face node of the neighbouring rank's boundary layer,
//   tr[0 F + f] = u,   tr[1 F + f] = s = nu d u / d x_S (physical, +S direction),   tr[2 F + f] = nu,
// F = face nodes of one layer = Nl_0 (Nl_1) n^(dim-1); f = face element (c_0 + Nl_0 c_1) * n^(dim-1)
// + the node's in-face index (a + n b).  tr_lo: the top face of the layer below the slab
// (rank - 1), tr_hi: the bottom face of the layer above (rank + 1).  Null: the slab wraps
// periodically onto itself (one rank, no halo mode).
struct Halo {
    const double *tr_lo = nullptr, *tr_hi = nullptr;
};

// Fused epilogue for the PCG apply: partial[blk*2 + 0] += dotv . out,  partial[blk*2+1] += sum(out)
struct DotEpi {
    const double *dotv = nullptr;
    double *partial = nullptr;
};

// Prologue for the PCG apply: the operand is p = z + beta * p_old (computed on the fly, also
// for neighbour lines), and p is written to p_out for the owned elements.
struct PProl {
    bool on = false;
    const double *z = nullptr, *p_old = nullptr;   // z = D^-1 r (written by the update kernel)
    double *p_out = nullptr;
    const double *beta = nullptr;  // device scalar
    const int *done = nullptr;     // device flag: skip all work when set
};                                 // (single-rank only; multi-rank runs the unfused path)

// Weight-folded constants of the v6 variable-nu apply (apply6.cuh): the staged
// viscosity is nu~ = nu w_i w_j w_k, so every transverse weight W = w_a w_b wfac_d and the
// derivative factor 2/h_d fold into per-direction constants and one scaled D^T table.
struct V6Fold {
    EOTab eE[3];      // C_d D^T (even-odd form), C_d = wfac_d (2/h_d)
    double kF[3];     // tau_d wfac_d / (2 w_0):      W sigma (nu- + nu+)  = kF (nu~- + nu~+)
    double kS[3];     // wfac_d (2/h_d) / (2 w_0):    W (s- + s+) / 2     = kS (s~- + s~+)
    double kL;        // 1 / (2 w_0):                  lifting coefficient of nu~ (before C_d D^T)
    double kCL[3];    // C_d kL
};

struct ApplyParams {
    Geom g;
    double lam, nu_const;
    const double *u, *nu;
    double *out;
    Halo halo;
    DotEpi epi;
    PProl pro;
    long long b0, b1;   // brick range [b0, b1)
    int seglen = 1, nseg = 1;  // column segments along the slowest direction (apply kernel)
    V6Fold f6;                 // filled by the v6 dispatch (variable nu)
    int zlo = 0, zhi = -1;     // element layers [zlo, zhi) of the slowest direction to apply
                               // (3-D v5 kernel only; -1 = all), for the pipelined host call
};

struct ConvParams {
    Geom g;
    const double *v[3];
    double *out[3];
    const double *lo[3];
    const double *hi[3];
};

// apply2.cu / apply3.cu / convect.cu
// grid: out, the number of CTAs launched (persistent; <= 148 x 8)
cudaError_t launch_apply2(const ApplyParams &a, bool varnu, int mode, int *grid, int smem, cudaStream_t st);
cudaError_t launch_apply3(const ApplyParams &a, bool varnu, int mode, int *grid, int smem, cudaStream_t st);
bool apply3_ranges_ok(const Geom &g);  // layer-range applies available (pipelined host call)
bool apply3_split_pcg_ok(const Geom &g, const double *nu);  // apply MODE 2 (dot epilogue) available
// invert != 0: write 1/diag (closed-form meshes only; cudaErrorInvalidValue otherwise)
cudaError_t launch_diag2(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                         cudaStream_t st, int invert = 0);
cudaError_t launch_diag3(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                         cudaStream_t st, int invert = 0);
cudaError_t launch_convect_k(const ConvParams &a, cudaStream_t st);
cudaError_t launch_coords(const Geom &g, long long el_offset, double *xyz, cudaStream_t st);
// face traces (u, s, nu) of the slab's bottom face (layer 0, -> send_lo) and top face (layer
// Nl_S - 1, -> send_hi) in the Halo layout; with_nu = 0 writes only u and s
cudaError_t launch_slab_traces(const Geom &g, const double *u, const double *nu, double nu_const, double *send_lo,
                               double *send_hi, int with_nu, cudaStream_t st);
cudaError_t launch_mass(const Geom &g, double *mass, cudaStream_t st);
cudaError_t upload_tables();   // all kernel TUs (capi.cpp)
cudaError_t upload_tables_vec();
cudaError_t upload_tables_apply2();
cudaError_t upload_tables_apply3();
cudaError_t upload_tables_convect();
cudaError_t upload_tables_halo();
cudaError_t upload_tables_stage();
cudaError_t upload_tables_stage_interp();

// stage.cu (config-4 IMEX-RK stage pieces)
cudaError_t launch_stage_combine(const Geom &g, const double *mass_e, double a_ex, double c_g, double lamH,
                                 const double *v, const double *Fc, const double *Av, double *vp, double *fH,
                                 cudaStream_t st);
struct DivGradParams {  // geometry: the velocity mesh's (degree P); pressure degree P-1
    const double *v[3] = {nullptr, nullptr, nullptr};     // div: velocity components
    const double *vlo[3] = {nullptr, nullptr, nullptr}, *vhi[3] = {nullptr, nullptr, nullptr};
    double *out = nullptr;                               // div: weak divergence (pressure layout)
    const double *psi = nullptr, *plo = nullptr, *phi = nullptr;  // grad: pressure (+ halos)
    double *gout[3] = {nullptr, nullptr, nullptr};      // grad: weak gradient (velocity layout)
};
cudaError_t launch_dg_div(const Geom &gv, const DivGradParams &a, cudaStream_t st);
struct LinComb {  // out = c0 x0 + sum_k c[k] y[k] (+ cm w / m)
    static constexpr int MAXT = 40;
    const double *x0 = nullptr;
    double c0 = 0.0;
    int n = 0;
    double c[MAXT];
    const double *y[MAXT];
    const double *w = nullptr;
    double cm = 0.0;
};
cudaError_t launch_lincomb(const Geom &g, const LinComb &lc, const double *mass_e, double *out, cudaStream_t st);
cudaError_t launch_scale_minv(const Geom &g, const double *mass_e, double c, const double *in, double *out,
                              cudaStream_t st);
cudaError_t launch_stage_project(const Geom &g, const double *mass_e, double lamH, const double *gw, double *vp,
                                 double *fH, cudaStream_t st);
cudaError_t launch_dg_grad(const Geom &gv, const DivGradParams &a, cudaStream_t st);

// PCG vector kernels -------------------------------------------------------
struct PcgScal {                 // device-resident scalars of one solve
    double rz, pq, alpha, beta, qmean, res2, fnorm2, fmean, sum_m, tol2;
    double nu_eff;                 // Schwarz preconditioner viscosity (mass-weighted mean of nu)
    double lam;
    long long ndof_global;
    int iter, done, status, maxit;
    int hist_cap;                  // alpha/beta history capacity (iterations), fixed at mesh creation
};
constexpr int PCG_HIST_CAP = 8192;
enum { PCG_ST_RUN = 0, PCG_ST_CONV = 1, PCG_ST_MAXIT = 2, PCG_ST_BREAKDOWN = 3 };

cudaError_t launch_abssum(const Geom &g, const double *u, double *partial, cudaStream_t st);
int vec_grid();       // grid (and partial count) of the reduction vector kernels
int vec_grid_wide();  // grid of the streaming vector kernels (and of k_pcg_update_t's partials)
// partial sums of m*f and m over the local slab -> partial[blk*2 + {0,1}]
cudaError_t launch_mass_moments(const Geom &g, const double *f, const double *mass_e, double *partial,
                                cudaStream_t st);
// r = m (f - fmean) - Ar ; partial: sum r, sum (f-fmean)^2
cudaError_t launch_pcg_init(const Geom &g, const double *f, const double *Ar, double *r, const double *mass_e,
                            const PcgScal *s, double *partial, cudaStream_t st);
// lam > 0: r = M f - Ar (Ar may be null), z = D^-1 r (dinv_table: dinv is the [npe] table, z may be
// null), partials [r.z, sum (r/m)^2] -> partial, [0, sum f^2] -> partial2
cudaError_t launch_pcg_init_fused(const Geom &g, const double *f, const double *Ar, double *r, const double *dinv,
                                  int dinv_table, double *z, const double *mass_e, double *partial, double *partial2,
                                  cudaStream_t st);
// r -= rmean (lam==0) ; z = dinv r ; partial: r.z, sum (r/m)^2
cudaError_t launch_pcg_init2(const Geom &g, double *r, const double *dinv, double *z, const double *mass_e,
                             const PcgScal *s, double *partial, cudaStream_t st);
// x += a p ; r -= a (q - qmean) ; z = dinv r ; partial: r.z, sum (r/m)^2
cudaError_t launch_pcg_update(const Geom &g, double *x, double *r, const double *p, const double *q,
                              const double *dinv, double *z, const double *mass_e, const PcgScal *s, double *partial,
                              cudaStream_t st);
// u -= (sum m u)/(sum m)  (lam == 0), partial for the moment is computed separately
cudaError_t launch_shift(const Geom &g, double *x, const double *shift, cudaStream_t st);
// deterministic reduction of partial[G][K] into sums[K] (single CTA, fixed order)
cudaError_t launch_reduce(const double *partial, int G, int K, double *sums, cudaStream_t st);
// scalar finalisation steps (single thread), mode-dependent
enum FinMode { FIN_FMEAN = 0, FIN_INIT = 1, FIN_INIT2 = 2, FIN_ALPHA = 3, FIN_BETA = 4, FIN_UMEAN = 5, FIN_NUMEAN = 6, FIN_ABSSUM = 7 };
cudaError_t launch_finalize(int mode, const double *sums, PcgScal *s, double *hist, double *aux, cudaStream_t st);
cudaError_t launch_reduce_s(const double *partial, int G, int K, double *sums, const PcgScal *s, cudaStream_t st);
cudaError_t launch_reduce_fin(const double *partial, int G, int K, double *sums, int mode, PcgScal *s, double *hist,
                              double *aux, cudaStream_t st);
cudaError_t launch_pcg_pupd(const Geom &g, double *p, const double *z, const PcgScal *s, cudaStream_t st);
// split step with the x update deferred by one iteration (single rank)
cudaError_t launch_pcg_pupd_x(const Geom &g, double *x, double *p, const double *z, const PcgScal *s, cudaStream_t st);
cudaError_t launch_pcg_update_nox(const Geom &g, double *r, const double *q, const double *dinv, double *z,
                                  const double *mass_e, const PcgScal *s, double *partial, cudaStream_t st);
// constant-nu uniform-mesh split step (dinv_t: the [npe] diagonal-inverse table)
cudaError_t launch_pcg_update_t(const Geom &g, double *r, const double *q, const double *dinv_t,
                                const double *mass_e, const PcgScal *s, double *partial, cudaStream_t st);
cudaError_t launch_pcg_pupd_xt(const Geom &g, double *x, double *p, const double *r, const double *dinv_t,
                               const PcgScal *s, cudaStream_t st);
cudaError_t launch_pcg_xfinal(const Geom &g, double *x, const double *p, const PcgScal *s, cudaStream_t st);
cudaError_t launch_dot_pq(const Geom &g, const double *p, const double *q, const PcgScal *s, double *partial,
                          cudaStream_t st);
cudaError_t launch_recip(const Geom &g, const double *d, double *dinv, cudaStream_t st);
cudaError_t launch_check_field(long long n, const double *x, int positive, int *bad, cudaStream_t st);

// schwarz.cu -- two-level additive Schwarz preconditioner
constexpr int SW_NCMAX = 64;     // coarse (vertex) grid: N_d <= 64 per direction
struct SwTab {                   // device-resident tables of one (mesh, nu)
    int Nc[3];                   // vertices per direction (= N_d; 1 for an absent direction)
    double nu;
    double S[3][NMAX * NMAX];    // S_d[i*n + k]: M-orthonormal eigenvectors of the 1-D block
    double Lam[3][NMAX];         // its eigenvalues (K_d S = M_d S Lam)
    double hat[2][NMAX];         // Q1 hats (1 - xi)/2, (1 + xi)/2 at the GLL nodes
    double eK[3][SW_NCMAX], eM[3][SW_NCMAX];  // 1-D coarse circulant symbols per Fourier column
};
enum { SW_APPLY = 0, SW_INIT = 1, SW_UPDATE = 2 };
struct SwBlockParams {
    const SwTab *T = nullptr;
    double lam = 0.0;
    double nu = 1.0;                // viscosity of the blocks (tables are for nu = 1) ...
    const double *nu_eff = nullptr; // ... or read from the device (PCG: PcgScal::nu_eff)
    int mode = SW_APPLY;
    long long nel = 0;
    double *r = nullptr;            // INIT/UPDATE: residual, updated in place
    const double *rin = nullptr;    // APPLY: input
    const double *q = nullptr;      // UPDATE: A p
    double *z = nullptr;            // out: block part z_b
    double *rc_el = nullptr;        // out: [2^dim][nel] hat moments of r
    const double *mass_e = nullptr; // element mass table [npe]
    const PcgScal *s = nullptr;
    double *partial = nullptr;      // [grid][2]: r.z_b, sum (r/m)^2
};
struct SwCoarseParams {
    const SwTab *T = nullptr;
    const double *F = nullptr;      // [3][SW_NCMAX^2] Fourier bases F_d[j*N + col]
    int dim = 3;
    double lam = 0.0;
    double nu = 1.0;
    const double *nu_eff = nullptr;
    const double *rc_el = nullptr;  // element moments [2^dim][nel] (single rank: gathered directly)
    long long nel = 0;              // local elements
    double *rc = nullptr;           // multi-rank: the all-reduced vertex vector (cfwd input)
    double *chat = nullptr;         // spectral workspace [NV]
    double *xc = nullptr;           // out: coarse solution [NV]
    double *partial = nullptr;
    int pslot = 0;                  // first partial slot of the column kernel
    int count_dot = 1;              // multi-rank: only rank 0 contributes r_c.x_c
    const int *done = nullptr;      // PCG converged: skip (the host checks convergence per chunk)
};
struct SwPupdParams {
    const SwTab *T = nullptr;
    long long nel = 0, el_off = 0;
    const double *zb = nullptr, *xc = nullptr;
    const double *p_old = nullptr;  // null: p = z_b + P_1 x_c (preconditioner apply); else == p (in place)
    double *p = nullptr, *x = nullptr;
    const PcgScal *s = nullptr;     // alpha, beta, done (null: beta = 0)
};
bool schwarz_supported(const Geom &g, const char **why);
void build_sw_tab(const Geom &g, double nu, SwTab *t, std::vector<double> &F);
cudaError_t launch_sw_block(const Geom &g, const SwTab &h, const SwBlockParams &a, cudaStream_t st, int *grid);
cudaError_t launch_sw_pupd(const Geom &g, const SwTab &h, const SwPupdParams &a, cudaStream_t st);
cudaError_t launch_sw_coarse(const SwCoarseParams &a, const SwTab &h, int stage, cudaStream_t st);
cudaError_t launch_sw_gather_local(const SwCoarseParams &a, int S, int off, int nl, cudaStream_t st);
int sw_cz_grid(const SwTab &h);

// stab.cu -- divergence / mass-flux stabilisation of the projection (reading A26)
struct StabParams {
    const double *in[3] = {nullptr, nullptr, nullptr};   // velocity components (apply operand)
    const double *lo[3] = {nullptr, nullptr, nullptr}, *hi[3] = {nullptr, nullptr, nullptr};  // rank halo layers
    double *out[3] = {nullptr, nullptr, nullptr};        // (M + a_D K_D + a_C K_C) in (weak)
    double aD = 0.0, aC = 0.0;
    double *partial = nullptr;                           // [grid][2]: in . out, 0
    const PcgScal *s = nullptr;                          // done flag (CG) or null
};
struct StabVec {                                          // CG vectors: r, p, q are [dim][ndof] blocks
    int dim = 3, npe = 0;
    long long ndof = 0;
    double *x[3] = {nullptr, nullptr, nullptr};           // the solution (in place: v'' on entry)
    double *r = nullptr, *p = nullptr, *q = nullptr;
    const double *dinv = nullptr;                         // [dim][npe] Jacobi table
    const double *mass_e = nullptr;                       // [npe] m, [npe] 1/m
    const PcgScal *s = nullptr;
    double *partial = nullptr, *partial2 = nullptr;
};
enum { STAB_INIT = 0, STAB_PUPD = 1, STAB_UPDATE = 2, STAB_U2 = 3 };
int stab_grid();
cudaError_t launch_stab_apply(const Geom &g, const StabParams &a, cudaStream_t st, int *grid = nullptr);
cudaError_t launch_stab_vec(int op, const StabVec &a, cudaStream_t st);
cudaError_t upload_tables_stab();

// visc.cu -- variable-viscosity step pieces
struct DerivParams {
    const double *u = nullptr;
    const double *lo = nullptr, *hi = nullptr;  // neighbour slab layers (multi-rank)
    double *out[3] = {nullptr, nullptr, nullptr};
    int dirs = 7;           // bit c: compute D_c u into out[c]
    int accumulate = 0;     // out += scale D_c u  (else out = scale D_c u)
    double scale = 1.0;
};
cudaError_t launch_dg_deriv(const Geom &g, const DerivParams &a, cudaStream_t st);
cudaError_t launch_visc_model(const Geom &g, const double *const v[3], double nu0, double nu1, double vmax, double *nu,
                              cudaStream_t st);
cudaError_t launch_nu_mul(const Geom &g, const double *nu, const double *x, const double *y, double *out,
                          cudaStream_t st);
cudaError_t upload_tables_visc();

}  // namespace dg
