// apply.cuh -- SIP-DG Helmholtz operator apply and Jacobi diagonal (sm_100a, FP64).
//
// Operator (include/dg.h; P:1039 interior penalty; Alg. 3 lines 5/9):
//   (A u)_I = lam m_I u_I + sum_d W_perp,d(I) (K_d u)_I
// where, because the GLL collocation quadrature (reading A2) makes grad phi_I(x_q)
// non-zero only on the d lines through q, the form splits into independent 1-D SIP line
// operators along each direction d, weighted by the transverse GLL weights
// W_perp,d = prod_{d' != d} w h_d'/2.  For one element line v[0..P] with
// neighbour traces (u, nu d_n u, nu) at both ends, the 1-D operator is
//   r_i  = sum_k D_ki w_k nu_k g_k,              g = (2/h) D v        (volume)
//   r_P += -1/2 (s_P + s_R) + sigma_R (v_P - u_R)                       (right face, own = "-")
//   r_i += -1/2 nu_P (2/h) D_Pi (v_P - u_R)                             (symmetry term)
//   r_0 += +1/2 (s_L + s_0) - sigma_L (u_L - v_0)                       (left face, own = "+")
//   r_i += -1/2 nu_0 (2/h) D_0i (u_L - v_0)
// with s = nu (2/h) (D v) the flux at a line end and sigma = tau (nu^- + nu^+)/2.
//
// Kernel design: one CTA per brick of B0 x B1 (x B2) elements.
// The brick's u (and nu) is staged once into shared memory (odd row pitch: conflict-free
// 8-byte line reads in all three directions).  Each direction is one pass in which a
// thread owns a whole brick-row line (B_d elements x n nodes): it streams the line
// element by element in registers, so faces inside the brick use the neighbouring line
// already in shared memory, and only the two line ends outside the brick read the
// neighbour element's line from global memory (L2-resident in z-slowest brick order).
// Results accumulate in a shared-memory tile; the last phase adds lam m u and writes
// out (coalesced).  The PCG variant computes its operand p = D^-1 r + beta p_old on the
// fly (prologue, also for the neighbour lines), stores p, and reduces p.q and sum(q) in
// the epilogue.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "dev_common.cuh"

namespace dg {

// ---------------------------------------------------------------------------
// 1-D line operator
// ---------------------------------------------------------------------------
template <int P, bool VARNU>
__device__ __forceinline__ void line_op(const DevTab &T, const double (&v)[P + 1], const double (&nv)[P + 1],
                                        double nuc, double uL, double sL, double nuL, double uR, double sR,
                                        double nuR, double sd, double tau, double (&r)[P + 1], double &sP)
{
    constexpr int n = P + 1;
    double t[n];
    double s0 = 0.0;
#pragma unroll
    for (int k = 0; k < n; ++k) {
        double g = 0.0;
#pragma unroll
        for (int j = 0; j < n; ++j) g = fma(T.D[k][j], v[j], g);
        g *= sd;
        const double nuk = VARNU ? nv[k] : nuc;
        t[k] = T.w[k] * nuk * g;
        if (k == 0) s0 = nuk * g;        // own flux at node 0
        if (k == P) sP = nuk * g;        // own flux at node P
    }
#pragma unroll
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k) acc = fma(T.D[k][i], t[k], acc);
        r[i] = acc;
    }
    const double nu0 = VARNU ? nv[0] : nuc, nuP = VARNU ? nv[P] : nuc;
    const double JR = v[P] - uR, JL = uL - v[0];
    r[P] += -0.5 * (sP + sR) + tau * 0.5 * (nuP + nuR) * JR;
    r[0] += 0.5 * (sL + s0) - tau * 0.5 * (nuL + nu0) * JL;
    const double cR = -0.5 * nuP * sd * JR, cL = -0.5 * nu0 * sd * JL;
#pragma unroll
    for (int i = 0; i < n; ++i) r[i] = fma(cR, T.D[P][i], fma(cL, T.D[0][i], r[i]));
}

template <int P>
__device__ __forceinline__ double end_flux(const DevTab &T, const double (&v)[P + 1], int end, double nu, double sd)
{
    double g = 0.0;
#pragma unroll
    for (int j = 0; j <= P; ++j) g = fma(T.D[end ? P : 0][j], v[j], g);
    return nu * sd * g;
}

}  // namespace dg

#include "apply_kernel.cuh"
#include "apply5.cuh"
#include "apply6.cuh"

namespace dg {

// ---------------------------------------------------------------------------
// Jacobi diagonal: diag_I = lam m_I + sum_d W_perp,d (K_d e_I)_I, evaluated by the same
// line operator on the unit vector (the neighbour line is e_I itself when the element is
// its own periodic neighbour, N_d = 1, else zero).  One thread per node.
// ---------------------------------------------------------------------------
// Closed-form Jacobi diagonal for meshes with N_d > 1 in every direction:
// per direction d of node I (index i along d):
//   W_perp [ (2/h) sum_k w_k nu_k D_ki^2  + [i == P] (-nu_P (2/h) D_PP + tau (nu_P + nu_R)/2)
//                                         + [i == 0] ( nu_0 (2/h) D_00 + tau (nu_0 + nu_L)/2) ]
// plus lam m_I.  One CTA per element (grid-stride), the element's nu and the 1-D tables in
// shared memory (per-lane table indices would serialise constant-cache reads).
// invert: write 1/diag (the Jacobi preconditioner of the PCG) instead of diag.
template <int DIM, int P, bool VARNU>
__global__ void __launch_bounds__(256) k_diag_cf(const Geom g, double lam, const double *nu, double nu_const,
                                                 Halo halo, double *diag, int invert)
{
    using C = Cfg<DIM, P>;
    constexpr int n = C::n, NPE = C::NPE;
    const DevTab &T = c_tab[P];
    __shared__ double swd2[n * n], sw[n], sdd[n], snu[VARNU ? NPE : 1];
    for (int q = threadIdx.x; q < n * n; q += blockDim.x) {
        const int k = q / n, i = q % n;
        swd2[q] = T.w[k] * T.D[k][i] * T.D[k][i];
        if (q < n) {
            sw[q] = T.w[q];
            sdd[q] = T.D[q][q];
        }
    }
    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        __syncthreads();
        if (VARNU)
            for (int q = threadIdx.x; q < NPE; q += blockDim.x) snu[q] = nu[e * NPE + q];
        __syncthreads();
        const int ec[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                           DIM == 3 ? (int)(e / ((long long)g.Nl[0] * g.Nl[1])) : 0};
        for (int q = threadIdx.x; q < NPE; q += blockDim.x) {
            const int qc[3] = {q % n, (q / n) % n, DIM == 3 ? q / (n * n) : 0};
            double m = g.mfac;
#pragma unroll
            for (int d = 0; d < DIM; ++d) m *= sw[qc[d]];
            double dg = lam * m;
#pragma unroll
            for (int D = 0; D < DIM; ++D) {
                const int GS = D == 0 ? 1 : (D == 1 ? n : n * n);
                const int i = qc[D];
                const int goff = q - i * GS;
                const double sd = g.sd[D];
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < n; ++k) acc = fma(swd2[k * n + i], VARNU ? snu[goff + k * GS] : nu_const, acc);
                acc *= sd;
                if (i == P || i == 0) {
                    int cn[3] = {ec[0], ec[1], ec[2]};
                    cn[D] += (i == P) ? 1 : -1;
                    const double nown = VARNU ? snu[q] : nu_const;
                    const double nnb = VARNU ? nbr_face_nu(g, nu, halo, n, cn, D, goff, i == P ? 0 : P * GS)
                                             : nu_const;
                    acc += (i == P ? -1.0 : 1.0) * nown * sd * sdd[i] + 0.5 * g.tau[D] * (nown + nnb);
                }
                double W = g.wfac[D];  // W_perp = prod_{d != D} w_{q_d} h_d / 2 (no division)
#pragma unroll
                for (int d = 0; d < DIM; ++d)
                    if (d != D) W *= sw[qc[d]];
                dg += W * acc;
            }
            diag[e * NPE + q] = invert ? 1.0 / dg : dg;
        }
    }
}

// Same closed form, one thread per node (grid-stride over the slab's nodes, no barriers): the
// element's nu lines come through L1 (every element is read by its npe consecutive threads),
// the w_k D_ki^2 table from shared memory.  The once-per-solve setup of the variable-nu PCG.
template <int DIM, int P, bool VARNU>
__global__ void __launch_bounds__(256) k_diag_cf2(const Geom g, double lam, const double *__restrict__ nu,
                                                  double nu_const, Halo halo, double *__restrict__ diag, int invert)
{
    using C = Cfg<DIM, P>;
    constexpr int n = C::n, NPE = C::NPE;
    const DevTab &T = c_tab[P];
    __shared__ double swd2[n * n], sw[n], sdd[n];
    for (int q = threadIdx.x; q < n * n; q += blockDim.x) {
        const int k = q / n, i = q % n;
        swd2[q] = T.w[k] * T.D[k][i] * T.D[k][i];
        if (q < n) {
            sw[q] = T.w[q];
            sdd[q] = T.D[q][q];
        }
    }
    __syncthreads();
    const long long tot = g.nel * NPE;
    // element coordinates in 32-bit arithmetic (local meshes below 2^31 elements: every config)
    const unsigned nx = (unsigned)g.Nl[0], ny = (unsigned)g.Nl[1];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const long long e = t / NPE;  // constant divisor: a multiply-shift
        const int q = (int)(t - e * NPE);
        const unsigned e32 = (unsigned)e, exy = e32 / nx;
        const int ec[3] = {(int)(e32 - exy * nx), (int)(DIM == 3 ? exy % ny : exy), DIM == 3 ? (int)(exy / ny) : 0};
        const int qc[3] = {q % n, (q / n) % n, DIM == 3 ? q / (n * n) : 0};
        const double *ne = VARNU ? nu + e * NPE : nullptr;
        double m = g.mfac;
#pragma unroll
        for (int d = 0; d < DIM; ++d) m *= sw[qc[d]];
        double dg = lam * m;
#pragma unroll
        for (int D = 0; D < DIM; ++D) {
            const int GS = D == 0 ? 1 : (D == 1 ? n : n * n);
            const int i = qc[D];
            const int goff = q - i * GS;
            const double sd = g.sd[D];
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < n; ++k) acc = fma(swd2[k * n + i], VARNU ? __ldg(ne + goff + k * GS) : nu_const, acc);
            acc *= sd;
            if (i == P || i == 0) {
                int cn[3] = {ec[0], ec[1], ec[2]};
                cn[D] += (i == P) ? 1 : -1;
                const double nown = VARNU ? __ldg(ne + q) : nu_const;
                const double nnb = VARNU ? nbr_face_nu(g, nu, halo, n, cn, D, goff, i == P ? 0 : P * GS)
                                         : nu_const;
                acc += (i == P ? -1.0 : 1.0) * nown * sd * sdd[i] + 0.5 * g.tau[D] * (nown + nnb);
            }
            double W = g.wfac[D];
#pragma unroll
            for (int d = 0; d < DIM; ++d)
                if (d != D) W *= sw[qc[d]];
            dg += W * acc;
        }
        diag[t] = invert ? 1.0 / dg : dg;
    }
}

// Same closed form for variable nu in 3-D, by line passes over tiles of E elements in shared
// memory (the apply's sum-factorised structure with the line matrix w_k D_ki^2 acting on the
// nu line): the tile's nu is read from HBM once (coalesced), each pass reads one nu line per
// thread and accumulates its direction's term into a shared tile; the z pass inverts and the
// tile leaves with coalesced stores.  ~72 B of shared traffic per node instead of 18 scattered
// L1 loads.  Tables in the kernel parameters (uniform constant-bank operands).
struct DiagTab {
    double wd2[NMAX][NMAX];  // w_k D_ki^2  [k][i]
    double dd0, ddP;          // D_00, D_PP
};

template <int P>
struct DiagCfg3 {
    static constexpr int n = P + 1, NN = n * n, NPE = NN * n;
    static constexpr int PX = (n % 2 == 0) ? n + 1 : n;  // odd x pitch: conflict-free strided lines
    static constexpr int SPE = PX * NN;
    static constexpr int E = 256 / NN > 0 ? 256 / NN : 1;  // elements per tile
    static constexpr int SMEM = (2 * E * SPE + 6 * E * NN + 6 * E) * 8;
};

// line L of direction D in a tile: element le, shared base of node 0, global in-element offset of node 0
template <int P, int D>
__device__ __forceinline__ int diag3_line(int L, int &base, int &goff, int &a, int &b)
{
    using C = DiagCfg3<P>;
    constexpr int n = C::n, NN = C::NN, PX = C::PX;
    const int le = L / NN, ab = L - le * NN;
    a = ab % n;
    b = ab / n;
    if (D == 0) {
        base = PX * ab;
        goff = n * a + NN * b;
    } else if (D == 1) {
        base = a + PX * n * b;
        goff = a + NN * b;
    } else {
        base = a + PX * b;
        goff = a + n * b;
    }
    base += le * C::SPE;
    return le;
}

// the face-neighbour nu of every line of direction D in the tile -> snb[2D + side][L]
template <int P, int D>
__device__ __forceinline__ void diag3_nbr(const Geom &g, const double *__restrict__ nu, const Halo &halo, bool hmesh,
                                          long long e0, int cnt, const long long *sne, double *snb)
{
    using C = DiagCfg3<P>;
    constexpr int n = C::n, NN = C::NN, NPE = C::NPE, E = C::E;
    constexpr int GS = D == 0 ? 1 : (D == 1 ? n : NN);
    for (int L = threadIdx.x; L < cnt * NN; L += blockDim.x) {
        int base, goff, a, b;
        const int le = diag3_line<P, D>(L, base, goff, a, b);
        double vl, vr;
        if (!hmesh) {
            vl = __ldg(nu + sne[le * 6 + 2 * D] * NPE + goff + P * GS);
            vr = __ldg(nu + sne[le * 6 + 2 * D + 1] * NPE + goff);
        } else {
            const unsigned e32 = (unsigned)(e0 + le), exy = e32 / (unsigned)g.Nl[0];
            const int c0 = (int)(e32 - exy * (unsigned)g.Nl[0]), c1 = (int)(exy % (unsigned)g.Nl[1]),
                      c2 = (int)(exy / (unsigned)g.Nl[1]);
            const int cl[3] = {c0 - (D == 0), c1 - (D == 1), c2 - (D == 2)};
            const int cr[3] = {c0 + (D == 0), c1 + (D == 1), c2 + (D == 2)};
            vl = nbr_face_nu(g, nu, halo, n, cl, D, goff, P * GS);
            vr = nbr_face_nu(g, nu, halo, n, cr, D, goff, 0);
        }
        snb[(2 * D) * E * NN + L] = vl;
        snb[(2 * D + 1) * E * NN + L] = vr;
    }
}

// one pass: every line of direction D accumulates its term into sacc (D = 2 also inverts)
template <int P, int D>
__device__ __forceinline__ void diag3_pass(const Geom &g, double lam, int invert, const DiagTab &dt, int cnt,
                                           const double *snu, const double *snb, double *sacc)
{
    using C = DiagCfg3<P>;
    constexpr int n = C::n, NN = C::NN, PX = C::PX, E = C::E;
    constexpr int SS = D == 0 ? 1 : (D == 1 ? PX : PX * n);
    const DevTab &T = c_tab[P];
    const double sd = g.sd[D], tau = g.tau[D];
    for (int L = threadIdx.x; L < cnt * NN; L += blockDim.x) {
        int base, goff, a, b;
        diag3_line<P, D>(L, base, goff, a, b);
        double v[n];
#pragma unroll
        for (int m = 0; m < n; ++m) v[m] = snu[base + m * SS];
        const double nuL = snb[(2 * D) * E * NN + L], nuR = snb[(2 * D + 1) * E * NN + L];
        const double W = g.wfac[D] * T.w[a] * T.w[b];
        double r[n];
#pragma unroll
        for (int i = 0; i < n; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < n; ++k) acc = fma(dt.wd2[k][i], v[k], acc);
            r[i] = acc * sd;
        }
        r[0] += v[0] * sd * dt.dd0 + 0.5 * tau * (v[0] + nuL);
        r[P] += -v[P] * sd * dt.ddP + 0.5 * tau * (v[P] + nuR);
        if (D == 0) {
            const double lm = lam * g.mfac * T.w[a] * T.w[b];
#pragma unroll
            for (int i = 0; i < n; ++i) sacc[base + i] = fma(W, r[i], lm * T.w[i]);
        } else if (D == 1) {
#pragma unroll
            for (int i = 0; i < n; ++i) sacc[base + i * SS] = fma(W, r[i], sacc[base + i * SS]);
        } else {
#pragma unroll
            for (int i = 0; i < n; ++i) {
                const double dgv = fma(W, r[i], sacc[base + i * SS]);
                double rv = dgv;
                if (invert) {  // reciprocal: approximate + two Newton steps (no DDIV slow path)
                    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rv) : "d"(dgv));
                    rv = fma(rv, fma(-dgv, rv, 1.0), rv);
                    rv = fma(rv, fma(-dgv, rv, 1.0), rv);
                }
                sacc[base + i * SS] = rv;
            }
        }
    }
}

template <int P>
__global__ void __launch_bounds__(256, 3) k_diag_cf3(const Geom g, double lam, const double *__restrict__ nu,
                                                     Halo halo, double *__restrict__ diag, int invert,
                                                     const __grid_constant__ DiagTab dt)
{
    using C = DiagCfg3<P>;
    constexpr int n = C::n, NN = C::NN, NPE = C::NPE, PX = C::PX, SPE = C::SPE, E = C::E;
    extern __shared__ __align__(16) double dsm[];
    double *snu = dsm, *sacc = dsm + E * SPE;
    double *snb = dsm + 2 * E * SPE;  // [D][side][line]: the neighbours' nu at the tile's face nodes
    long long *sne = reinterpret_cast<long long *>(snb + 6 * E * NN);  // [le][D][side] neighbour elements
    const int tid = threadIdx.x, bd = blockDim.x;
    const long long ntile = (g.nel + E - 1) / E;
    const unsigned nx = (unsigned)g.Nl[0], ny = (unsigned)g.Nl[1];
    // slab meshes without halos: neighbour element indices once per (element, direction, side);
    // halo meshes take the generic per-line lookup
    const bool hmesh = halo.tr_lo != nullptr || halo.tr_hi != nullptr;
    for (long long tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const long long e0 = tile * E;
        const int cnt = (int)(g.nel - e0 < E ? g.nel - e0 : E);
        __syncthreads();  // the previous tile's store has read sacc
        for (int q = tid; q < cnt * NPE; q += bd) {
            const int le = q / NPE, r = q - le * NPE;
            snu[le * SPE + r % n + PX * (r / n)] = __ldg(nu + e0 * NPE + q);
        }
        if (!hmesh) {
            for (int x = tid; x < cnt * 6; x += bd) {
                const int le = x / 6, D = (x >> 1) % 3, side = x & 1;
                const unsigned e32 = (unsigned)(e0 + le), exy = e32 / nx;
                int c0 = (int)(e32 - exy * nx), c1 = (int)(exy % ny), c2 = (int)(exy / ny);
                const int dd = side ? 1 : -1;
                if (D == 0) c0 = (c0 + dd + g.Nl[0]) % g.Nl[0];
                else if (D == 1) c1 = (c1 + dd + g.Nl[1]) % g.Nl[1];
                else c2 = (c2 + dd + g.Nl[2]) % g.Nl[2];
                sne[x] = (long long)c0 + (long long)g.Nl[0] * (c1 + (long long)g.Nl[1] * c2);
            }
            __syncthreads();
        }
        diag3_nbr<P, 0>(g, nu, halo, hmesh, e0, cnt, sne, snb);
        diag3_nbr<P, 1>(g, nu, halo, hmesh, e0, cnt, sne, snb);
        diag3_nbr<P, 2>(g, nu, halo, hmesh, e0, cnt, sne, snb);
        __syncthreads();
        diag3_pass<P, 0>(g, lam, invert, dt, cnt, snu, snb, sacc);
        __syncthreads();
        diag3_pass<P, 1>(g, lam, invert, dt, cnt, snu, snb, sacc);
        __syncthreads();
        diag3_pass<P, 2>(g, lam, invert, dt, cnt, snu, snb, sacc);
        __syncthreads();
        for (int q = tid; q < cnt * NPE; q += bd) {  // coalesced store
            const int le = q / NPE, r = q - le * NPE;
            diag[e0 * NPE + q] = sacc[le * SPE + r % n + PX * (r / n)];
        }
    }
}

template <int DIM, int P, bool VARNU>
__global__ void __launch_bounds__(256) k_diag(const Geom g, double lam, const double *nu, double nu_const,
                                              Halo halo, double *diag)
{
    using C = Cfg<DIM, P>;
    constexpr int n = C::n;
    const DevTab &T = c_tab[P];
    const long long tot = g.nel * C::NPE;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const long long e = t / C::NPE;
        const int q = (int)(t - e * C::NPE);
        int ec[3];
        ec[0] = (int)(e % g.Nl[0]);
        ec[1] = (int)((e / g.Nl[0]) % g.Nl[1]);
        ec[2] = (int)(e / ((long long)g.Nl[0] * g.Nl[1]));
        const int qc[3] = {q % n, (q / n) % n, DIM == 3 ? q / (n * n) : 0};
        double m = 1.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) m *= T.w[qc[d]] * 0.5 * g.h[d];
        double dg = lam * m;
#pragma unroll
        for (int D = 0; D < DIM; ++D) {
            const int GS = D == 0 ? 1 : (D == 1 ? n : n * n);
            const int i = qc[D];
            const double W = m / (T.w[i] * 0.5 * g.h[D]);
            const double sd = 2.0 / g.h[D];
            const int goff = q - i * GS;
            double v[n], vn[n];
#pragma unroll
            for (int k = 0; k < n; ++k) {
                v[k] = (k == i) ? 1.0 : 0.0;
                vn[k] = VARNU ? __ldg(nu + e * C::NPE + goff + k * GS) : nu_const;
            }
            const bool self = (g.N[D] == 1);
            if (!self) {
                // closed form: (2/h) sum_k w_k nu_k D_ki^2, plus at node P
                // -nu_P (2/h) D_PP + tau (nu_P + nu_R)/2 and at node 0 +nu_0 (2/h) D_00 + tau (nu_0 + nu_L)/2
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    const double nk = VARNU ? __ldg(nu + e * C::NPE + goff + k * GS) : nu_const;
                    acc = fma(T.w[k] * T.D[k][i] * T.D[k][i], nk, acc);
                }
                acc *= sd;
                if (i == P || i == 0) {
                    int cn[3] = {ec[0], ec[1], ec[2]};
                    cn[D] += (i == P) ? 1 : -1;
                    const double nown = VARNU ? __ldg(nu + e * C::NPE + goff + i * GS) : nu_const;
                    const double nnb = VARNU ? nbr_face_nu(g, nu, halo, n, cn, D, goff, i == P ? 0 : P * GS)
                                             : nu_const;
                    acc += (i == P ? -1.0 : 1.0) * nown * sd * T.D[i][i] + 0.5 * g.tau[D] * (nown + nnb);
                }
                dg += W * acc;
                continue;
            }
            double uL, sL, nuL, uR, sR, nuR;
            if (self) {
                uL = v[P]; nuL = vn[P]; sL = end_flux<P>(T, v, 1, nuL, sd);
                uR = v[0]; nuR = vn[0]; sR = end_flux<P>(T, v, 0, nuR, sd);
            } else {
                int cl[3] = {ec[0], ec[1], ec[2]}, cr[3] = {ec[0], ec[1], ec[2]};
                cl[D] -= 1;
                cr[D] += 1;
                uL = sL = uR = sR = 0.0;
                if (VARNU) {
                    nuL = nbr_face_nu(g, nu, halo, n, cl, D, goff, P * GS);
                    nuR = nbr_face_nu(g, nu, halo, n, cr, D, goff, 0);
                } else {
                    nuL = nuR = nu_const;
                }
            }
            double r[n], sP;
            line_op<P, VARNU>(T, v, vn, nu_const, uL, sL, nuL, uR, sR, nuR, sd, g.tau[D], r, sP);
            dg += W * r[i];
        }
        diag[t] = dg;
    }
}

// ---------------------------------------------------------------------------
// host-side dispatch for one dimension
// ---------------------------------------------------------------------------
// name of the last dispatched apply kernel of this thread (bench / profiling evidence)
inline void note_kernel(const char *gen, int dim, int P, bool varnu, int mode, int grid, int bx, int by, int bz)
{
    snprintf(last_apply_kernel(), 160, "%s<dim=%d,P=%d,varnu=%d,mode=%d> grid=%d brick=%dx%dx%d", gen, dim, P, varnu ? 1 : 0,
             mode, grid, bx, by, bz);
}

template <int DIM>
struct ApplyDispatch {
    // launch one compile-time brick shape (persistent grid: #SM x occupancy, <= 148 x 8)
    template <int P, bool VARNU, int MODE, int BX, int BY, int BZ>
    static cudaError_t go(ApplyParams a, int *grid, cudaStream_t st)
    {
        using K = KC<DIM, P, VARNU, MODE, BX, BY, BZ>;
        if constexpr (K::SMEM_BYTES > 227 * 1024) {
            return cudaErrorNotSupported;
        } else {
            auto kern = k_apply<DIM, P, VARNU, MODE, BX, BY, BZ>;
            static int occ = -1, nsm = 0;  // per instantiation (one device per process is assumed)
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM_BYTES);
            if (e != cudaSuccess) return e;
            if (occ < 0) {
                int dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, K::NT, K::SMEM_BYTES);
                if (e != cudaSuccess) return e;
                if (occ < 1) return cudaErrorInvalidConfiguration;
            }
            a.g.B[0] = BX;
            a.g.B[1] = BY;
            a.g.B[2] = BZ;
            for (int d = 0; d < 3; ++d) a.g.nbk[d] = a.g.Nl[d] / a.g.B[d];
            a.b0 = 0;
            a.b1 = (long long)a.g.nbk[0] * a.g.nbk[1] * a.g.nbk[2];
            long long gsz = (long long)nsm * std::min(occ, 8);
            // column segments along the slowest direction: enough units (>= 3 per CTA) for
            // balance, as long as possible for the on-chip slowest-direction traces
            const int S = DIM - 1;
            const long long ncols = DIM == 3 ? (long long)a.g.nbk[0] * a.g.nbk[1] : a.g.nbk[0];
            const int nbS = a.g.nbk[S];
            int nseg = 1;
            while (ncols * nseg < 3 * gsz && nbS % (2 * nseg) == 0) nseg *= 2;
            a.nseg = nseg;
            a.seglen = nbS / nseg;
            const long long nunits = ncols * nseg;
            if (gsz > nunits) gsz = nunits;
            if (gsz < 1) gsz = 1;
            *grid = (int)gsz;
            note_kernel("k_apply(v4)", DIM, P, VARNU, MODE, (int)gsz, BX, BY, BZ);
            kern<<<(int)gsz, K::NT, K::SMEM_BYTES, st>>>(a);
            return cudaGetLastError();
        }
    }
    // v5 (3-D): warp-specialised TMA/mbarrier kernel on 2x2x2 bricks (apply5.cuh)
    template <int P, bool VARNU, int MODE>
    static cudaError_t go5(ApplyParams a, int *grid, cudaStream_t st)
    {
        using K = v5::KC5<P, VARNU, MODE>;
        if constexpr (K::SMEM_BYTES > 227 * 1024) {
            return cudaErrorNotSupported;
        } else {
            auto kern = v5::k_apply5<P, VARNU, MODE>;
            static int occ = -1, nsm = 0;
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM_BYTES);
            if (e != cudaSuccess) return e;
            if (occ < 0) {
                int dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, K::NT, K::SMEM_BYTES);
                if (e != cudaSuccess) return e;
                if (occ < 1) return cudaErrorInvalidConfiguration;
            }
            long long gsz = (long long)nsm * std::min(occ, 4);
            const long long ncols = (long long)(a.g.Nl[0] / 2) * (a.g.Nl[1] / 2);
            if (a.zhi < 0) {
                a.zlo = 0;
                a.zhi = a.g.Nl[2];
            }
            const int nbS = (a.zhi - a.zlo) / 2;
            // segments per column by the same load-balance model as v6, with a per-segment cost
            // of ~1.5 bricks (fitted on the c4 P = 6 / P = 7 applies: nseg = 1, 2, 4, 8, 16 ->
            // Poisson 276, 284, 292, 298, 325 us per Jacobi-PCG iteration); near-ties: fewer
            // segments (the z carry pays more than balance here)
            int nseg = 1;
            {
                double best = 1e300;
                for (int ns = 1; ns <= nbS; ++ns) {
                    if (nbS % ns) continue;
                    const double cost = (double)((ncols * ns + gsz - 1) / gsz) * (nbS / ns + 1.5);
                    if (cost < best * 0.99) {
                        best = cost;
                        nseg = ns;
                    }
                }
            }
            if (const char *ev = DG_DEV_ENV("DG_V5_NSEG")) {  // development override
                const int want = atoi(ev);
                if (want >= 1 && nbS % want == 0) nseg = want;
            }
            a.nseg = nseg;
            a.seglen = nbS / nseg;
            const long long nunits = ncols * nseg;
            if (gsz > nunits) gsz = nunits;
            if (gsz < 1) gsz = 1;
            *grid = (int)gsz;
            note_kernel("v5::k_apply5", 3, P, VARNU, MODE, (int)gsz, 2, 2, 2);
            kern<<<(int)gsz, K::NT, K::SMEM_BYTES, st>>>(a);
            return cudaGetLastError();
        }
    }
    // degrees / viscosity kinds the v6 kernel has: P odd <= 5, and P = 6 with constant nu
    template <int P, bool VARNU>
    static constexpr bool v6_shape() { return (P <= 5 && P % 2 == 1) || ((P == 6 || P == 7) && !VARNU); }
    // v6 (3-D, n <= 6): one CTA per SM, 4x4x1 bricks, warpgroup-specialised (apply6.cuh)
    template <int P, bool VARNU, int MODE>
    static cudaError_t go6(ApplyParams a, int *grid, cudaStream_t st)
    {
        if constexpr (!v6_shape<P, VARNU>() || MODE == 1) {
            return cudaErrorNotSupported;
        } else if constexpr (v6::KC6<P, VARNU, MODE>::SMEM_BYTES > 227 * 1024) {
            return cudaErrorNotSupported;
        } else {
            using K = v6::KC6<P, VARNU, MODE>;
            auto kern = v6::k_apply6<P, VARNU, MODE>;
            if (VARNU) {  // weight-folded constants (V6Fold, dg_internal.h)
                const Tab &t = host_tab(P);
                const double w0 = t.w[0];
                a.f6.kL = 0.5 / w0;
                for (int d = 0; d < 3; ++d) {
                    const double C = a.g.wfac[d] * a.g.sd[d];
                    a.f6.kF[d] = a.g.tau[d] * a.g.wfac[d] / (2.0 * w0);
                    a.f6.kS[d] = 0.5 * C / w0;
                    a.f6.kCL[d] = C * a.f6.kL;
                    EOTab e = t.eE;
                    for (int i = 0; i < HMAX; ++i) {
                        for (int j = 0; j < HMAX; ++j) {
                            e.Te[i][j] *= C;
                            e.To[i][j] *= C;
                        }
                        e.Tc[i] *= C;
                        e.Mr[i] *= C;
                    }
                    e.Mmid *= C;
                    a.f6.eE[d] = e;
                }
            }
            static int nsm = 0;
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM_BYTES);
            if (e != cudaSuccess) return e;
            if (nsm == 0) {
                int dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            }
            long long gsz = nsm;
            const long long ncols = (long long)(a.g.Nl[0] / K::BX) * (a.g.Nl[1] / K::BY);
            if (a.zhi < 0) {
                a.zlo = 0;
                a.zhi = a.g.Nl[2];
            }
            const int nbS = a.zhi - a.zlo;  // one element layer per brick
            // column segments per column: the persistent CTAs take ceil(units / grid) units of
            // seglen bricks each plus a per-segment cost (the two halo bricks of the segment's z
            // ends) of ~1.1 bricks (fitted on c5: nseg = 2, 4, 8, 16 -> 0.544, 0.494, 0.526,
            // 0.579 ms; 3.3 bricks with the earlier segment-end trace loads); pick the divisor of
            // nbS (seglen >= 2) with the least modelled time
            int nseg = 1;
            double best = 1e300;
            for (int ns = 1; ns <= nbS / 2; ++ns) {
                if (nbS % ns) continue;
                const long long units = ncols * ns;
                const double cost = (double)((units + gsz - 1) / gsz) * (nbS / ns + 1.1);
                if (cost <= best * 1.01) {  // near-ties: more units (finer balance; measured)
                    best = cost < best ? cost : best;
                    nseg = ns;
                }
            }
            if (nbS < 2) nseg = 1;
            if (const char *ev = DG_DEV_ENV("DG_V6_NSEG")) {  // development override
                const int want = atoi(ev);
                if (want >= 1 && nbS % want == 0 && nbS / want >= 2) nseg = want;
            }
            a.nseg = nseg;
            a.seglen = nbS / nseg;
            const long long nunits = ncols * nseg;
            if (gsz > nunits) gsz = nunits;
            if (gsz < 1) gsz = 1;
            *grid = (int)gsz;
            note_kernel("v6::k_apply6", 3, P, VARNU, MODE, (int)gsz, K::BX, K::BY, 1);
            kern<<<(int)gsz, K::NT, K::SMEM_BYTES, st>>>(a);
            return cudaGetLastError();
        }
    }
    static bool v6_ok(const ApplyParams &a, bool pcg)
    {
        static const bool off = [] {
            const char *e = DG_DEV_ENV("DG_APPLY_IMPL");
            return e && e[0] == 'v' && (e[1] == '4' || e[1] == '5');
        }();
        // TMA copies single elements (n even) or brick rows (P = 6, constant nu); P = 7 (constant
        // nu) takes 4 x 2 x 1 bricks
        if (off || DIM != 3) return false;
        if (!((a.g.P <= 5 && a.g.P % 2 == 1) || ((a.g.P == 6 || a.g.P == 7) && !a.nu))) return false;
        const int by = v6::v6_by(a.g.P);
        if (a.g.Nl[0] % 4 || a.g.Nl[1] % by || a.g.Nl[2] < 2) return false;
        const int nz = a.zhi >= 0 ? a.zhi - a.zlo : a.g.Nl[2];
        if (nz < 2) return false;
        auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        if (pcg) return al(a.pro.z) && al(a.pro.p_old) && al(a.pro.p_out) && (!a.nu || al(a.nu));
        return al(a.u) && (!a.nu || al(a.nu));
    }
    // can this mesh be applied per range of slowest-direction layers (v5/v6 only)?
    template <int P, bool VARNU>
    static constexpr bool mode2_fits6()
    {
        if constexpr (v6_shape<P, VARNU>()) return v6::KC6<P, VARNU, 2>::SMEM_BYTES <= 227 * 1024;
        else return false;
    }
    template <int P, bool VARNU>
    static constexpr bool mode2_fits5() { return v5::KC5<P, VARNU, 2>::SMEM_BYTES <= 227 * 1024; }
    static bool mode2_compiled(int P, bool varnu, bool six)
    {
        switch (P) {
#define DG_M2(p)                                                                                           \
    case p:                                                                                                \
        if constexpr (DG_HAS_P(p) && DIM == 3)                                                             \
            return six ? (varnu ? mode2_fits6<p, true>() : mode2_fits6<p, false>())                        \
                       : (varnu ? mode2_fits5<p, true>() : mode2_fits5<p, false>());                       \
        else                                                                                               \
            return false;
            DG_M2(1) DG_M2(2) DG_M2(3) DG_M2(4) DG_M2(5) DG_M2(6) DG_M2(7) DG_M2(8) DG_M2(9) DG_M2(10)
#undef DG_M2
        default:
            return false;
        }
    }
    static bool split_pcg_ok(const Geom &g, const double *nu)
    {
        ApplyParams a{};
        a.g = g;
        a.u = nu ? nu : reinterpret_cast<const double *>(256);  // alignment probe only
        a.nu = nu;
        a.zhi = -1;
        // the MODE-2 (dot epilogue) kernel the apply dispatch would pick must exist for this P
        if (v6_ok(a, false)) return mode2_compiled(g.P, nu != nullptr, true);
        return v5_ok(a, false) && mode2_compiled(g.P, nu != nullptr, false);
    }
    static bool ranges_ok(const Geom &g)
    {
        const char *e = DG_DEV_ENV("DG_APPLY_IMPL");
        if (e && e[0] == 'v' && e[1] == '4') return false;
        return DIM == 3 && g.Nl[0] % 2 == 0 && g.Nl[1] % 2 == 0 && g.Nl[2] % 2 == 0;
    }
    static bool v5_ok(const ApplyParams &a, bool pcg)
    {
        static const bool off = [] {
            const char *e = DG_DEV_ENV("DG_APPLY_IMPL");
            return e && e[0] == 'v' && e[1] == '4';
        }();
        if (off || DIM != 3) return false;
        for (int d = 0; d < 3; ++d)
            if (a.g.Nl[d] % 2) return false;
        if (a.zhi >= 0 && (a.zlo % 2 || a.zhi % 2 || a.zhi <= a.zlo || a.zhi > a.g.Nl[2])) return false;
        auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        if (pcg) return al(a.pro.z) && al(a.pro.p_old) && al(a.pro.p_out) && (!a.nu || al(a.nu));
        return al(a.u) && (!a.nu || al(a.nu));
    }
    // brick shape: the largest of the candidates that divides the local mesh and fits the
    // shared-memory budget (default 110 KB = two CTAs per SM; DG_SMEM_BUDGET_KB overrides)
    template <int P, bool VARNU, int MODE>
    static cudaError_t pick(const ApplyParams &a, int *grid, cudaStream_t st)
    {
        static const int budget = [] {
            const char *e = DG_DEV_ENV("DG_SMEM_BUDGET_KB");
            return (e ? atoi(e) : 110) * 1024;
        }();
        const int *N = a.g.Nl;
        if constexpr (DIM == 3) {
            if (MODE == 0 && v6_ok(a, false)) {  // the fused PCG operand stays on v5 (measured faster)
                const cudaError_t e = go6<P, VARNU, MODE>(a, grid, st);
                if (e != cudaErrorNotSupported) return e;
            }
            if (v5_ok(a, MODE == 1)) {
                const cudaError_t e = go5<P, VARNU, MODE>(a, grid, st);
                if (e != cudaErrorNotSupported) return e;
            }
            if (a.zhi >= 0) return cudaErrorNotSupported;  // layer ranges need the v5 kernel
            if (N[0] % 2 == 0 && N[1] % 2 == 0 && N[2] % 2 == 0 && KC<3, P, VARNU, MODE, 2, 2, 2>::SMEM_BYTES <= budget)
                return go<P, VARNU, MODE, 2, 2, 2>(a, grid, st);
            if (N[0] % 2 == 0 && N[1] % 2 == 0 && KC<3, P, VARNU, MODE, 2, 2, 1>::SMEM_BYTES <= budget)
                return go<P, VARNU, MODE, 2, 2, 1>(a, grid, st);
            return go<P, VARNU, MODE, 1, 1, 1>(a, grid, st);
        } else {
            if (N[0] % 4 == 0 && N[1] % 4 == 0 && KC<2, P, VARNU, MODE, 4, 4, 1>::SMEM_BYTES <= budget)
                return go<P, VARNU, MODE, 4, 4, 1>(a, grid, st);
            if (N[0] % 2 == 0 && N[1] % 2 == 0 && KC<2, P, VARNU, MODE, 2, 2, 1>::SMEM_BYTES <= budget)
                return go<P, VARNU, MODE, 2, 2, 1>(a, grid, st);
            return go<P, VARNU, MODE, 1, 1, 1>(a, grid, st);
        }
    }
    template <int P>
    static cudaError_t go_p(const ApplyParams &a, bool varnu, int mode, int *grid, cudaStream_t st)
    {
        if (mode == 2) {  // dot epilogue only (split PCG path): 3-D meshes the v6 or v5 kernel runs
            if constexpr (DIM == 3) {
                if (v6_ok(a, false)) {
                    if (a.lam > 0.0)  // sum(q) unused: the epilogue variant without it
                        return varnu ? go6<P, true, 3>(a, grid, st) : go6<P, false, 3>(a, grid, st);
                    return varnu ? go6<P, true, 2>(a, grid, st) : go6<P, false, 2>(a, grid, st);
                }
                if (v5_ok(a, false)) return varnu ? go5<P, true, 2>(a, grid, st) : go5<P, false, 2>(a, grid, st);
                return cudaErrorNotSupported;
            } else {
                return cudaErrorNotSupported;
            }
        }
        const bool pcg = mode == 1;
        if (varnu) return pcg ? pick<P, true, 1>(a, grid, st) : pick<P, true, 0>(a, grid, st);
        return pcg ? pick<P, false, 1>(a, grid, st) : pick<P, false, 0>(a, grid, st);
    }
    static cudaError_t apply(const ApplyParams &a, bool varnu, int pcg, int *grid, int smem, cudaStream_t st)
    {
        (void)smem;
        switch (a.g.P) {
        case 1: if constexpr (DG_HAS_P(1)) return go_p<1>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 2: if constexpr (DG_HAS_P(2)) return go_p<2>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 3: if constexpr (DG_HAS_P(3)) return go_p<3>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 4: if constexpr (DG_HAS_P(4)) return go_p<4>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 5: if constexpr (DG_HAS_P(5)) return go_p<5>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 6: if constexpr (DG_HAS_P(6)) return go_p<6>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 7: if constexpr (DG_HAS_P(7)) return go_p<7>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 8: if constexpr (DG_HAS_P(8)) return go_p<8>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 9: if constexpr (DG_HAS_P(9)) return go_p<9>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        case 10: if constexpr (DG_HAS_P(10)) return go_p<10>(a, varnu, pcg, grid, st); else return cudaErrorNotSupported;
        default: return cudaErrorInvalidValue;
        }
    }
    template <int P>
    static cudaError_t diag_p(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                              int invert, cudaStream_t st)
    {
        const long long tot = g.nel * Cfg<DIM, P>::NPE;
        bool self = false;
        for (int dd = 0; dd < DIM; ++dd) self = self || g.N[dd] == 1;
        if (!self) {  // closed form, one CTA per element (grid-stride)
#ifdef DG_DEVELOPMENT  // DG_DIAG_V1: the first one-CTA-per-element closed-form kernel (A/B only)
            if (DG_DEV_ENV("DG_DIAG_V1")) {
                const long long blocks = g.nel < 148LL * 16 ? g.nel : 148LL * 16;
                if (nu) k_diag_cf<DIM, P, true><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d, invert);
                else k_diag_cf<DIM, P, false><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d, invert);
                return cudaGetLastError();
            }
#endif
            if constexpr (DIM == 3) {
                if (nu && !DG_DEV_ENV("DG_DIAG_CF2")) {  // variable nu: tiled line passes (k_diag_cf3)
                    using C3 = DiagCfg3<P>;
                    static DiagTab dt;
                    static int resident = 0;
                    if (!resident) {
                        const Tab &t = host_tab(P);
                        for (int k = 0; k <= P; ++k)
                            for (int i = 0; i <= P; ++i) dt.wd2[k][i] = t.w[k] * t.D[k][i] * t.D[k][i];
                        dt.dd0 = t.D[0][0];
                        dt.ddP = t.D[P][P];
                        cudaError_t e = cudaFuncSetAttribute(k_diag_cf3<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, C3::SMEM);
                        if (e != cudaSuccess) return e;
                        int dev = 0, nsm = 148, occ = 1;
                        cudaGetDevice(&dev);
                        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_diag_cf3<P>, 256, C3::SMEM);
                        if (e != cudaSuccess || occ < 1) occ = 1;
                        resident = nsm * occ;
                    }
                    const long long ntile = (g.nel + C3::E - 1) / C3::E;
                    const int blocks = (int)(ntile < resident ? ntile : resident);
                    k_diag_cf3<P><<<blocks, 256, C3::SMEM, st>>>(g, lam, nu, h, d, invert, dt);
                    return cudaGetLastError();
                }
            }
            {  // one thread per node (measured faster than one CTA per element: 1.39 vs 1.73 ms on c5), one resident wave
                static int resident[2] = {0, 0};
                const int vi = nu ? 1 : 0;
                if (!resident[vi]) {
                    int dev = 0, nsm = 148, occ = 1;
                    cudaGetDevice(&dev);
                    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                    cudaError_t e = nu ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_diag_cf2<DIM, P, true>, 256, 0)
                                       : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_diag_cf2<DIM, P, false>, 256, 0);
                    if (e != cudaSuccess || occ < 1) occ = 1;
                    resident[vi] = nsm * occ;
                }
                long long blocks = (tot + 255) / 256;
                if (blocks > resident[vi]) blocks = resident[vi];
                if (nu) k_diag_cf2<DIM, P, true><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d, invert);
                else k_diag_cf2<DIM, P, false><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d, invert);
                return cudaGetLastError();
            }
        }
        if (invert) return cudaErrorInvalidValue;  // N_d = 1 meshes: caller inverts separately
        long long blocks = (tot + 255) / 256;
        if (blocks > 148 * 64) blocks = 148 * 64;
        if (nu) k_diag<DIM, P, true><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d);
        else k_diag<DIM, P, false><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d);
        return cudaGetLastError();
    }
    static cudaError_t diag(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                            int invert, cudaStream_t st)
    {
        switch (g.P) {
        case 1: if constexpr (DG_HAS_P(1)) return diag_p<1>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 2: if constexpr (DG_HAS_P(2)) return diag_p<2>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 3: if constexpr (DG_HAS_P(3)) return diag_p<3>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 4: if constexpr (DG_HAS_P(4)) return diag_p<4>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 5: if constexpr (DG_HAS_P(5)) return diag_p<5>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 6: if constexpr (DG_HAS_P(6)) return diag_p<6>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 7: if constexpr (DG_HAS_P(7)) return diag_p<7>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 8: if constexpr (DG_HAS_P(8)) return diag_p<8>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 9: if constexpr (DG_HAS_P(9)) return diag_p<9>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        case 10: if constexpr (DG_HAS_P(10)) return diag_p<10>(g, lam, nu, nuc, h, d, invert, st); else return cudaErrorNotSupported;
        default: return cudaErrorInvalidValue;
        }
    }
};

}  // namespace dg
