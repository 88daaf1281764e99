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

// ---------------------------------------------------------------------------
// one direction pass over the brick
// ---------------------------------------------------------------------------
template <int DIM, int P, bool VARNU, bool PCG, int D>
__device__ __forceinline__ void apply_pass(const ApplyParams &a, const DevTab &T, const double *su,
                                           const double *snu, double *sacc, const int (&e0)[3], double beta)
{
    using C = Cfg<DIM, P>;
    constexpr int n = C::n;
    constexpr int O1 = (D == 0) ? 1 : 0;
    constexpr int O2 = (DIM == 3) ? ((D == 2) ? 1 : 2) : 2;
    const Geom &g = a.g;
    const int Bd = g.B[D];
    const int BE = g.B[0] * g.B[1] * g.B[2];
    const int ncross = BE / Bd;
    const int nlines = ncross * C::NT;
    // shared-memory strides per node coordinate (x pitch PX), global strides (pitch n)
    constexpr int SS[3] = {1, C::PX, C::PX * n};
    constexpr int GS[3] = {1, n, n * n};
    const double sd = 2.0 / g.h[D];
    const double tau = g.tau[D];

    for (int L = threadIdx.x; L < nlines; L += blockDim.x) {
        const int tn = L % C::NT, ce = L / C::NT;
        const int ta = tn % n, tb = (DIM == 3) ? tn / n : 0;
        int lc[3] = {0, 0, 0};
        lc[O1] = ce % g.B[O1];
        if (DIM == 3) lc[O2] = ce / g.B[O1];
        int nd[3] = {0, 0, 0};
        nd[O1] = ta;
        if (DIM == 3) nd[O2] = tb;
        const int soff = nd[0] * SS[0] + nd[1] * SS[1] + nd[2] * SS[2];  // node offset, i_D = 0
        const int goff = nd[0] * GS[0] + nd[1] * GS[1] + nd[2] * GS[2];
        double W = T.w[ta] * 0.5 * g.h[O1];
        if (DIM == 3) W *= T.w[tb] * 0.5 * g.h[O2];

        auto slot = [&](int l) {
            int c[3] = {lc[0], lc[1], lc[2]};
            c[D] = l;
            return c[0] + g.B[0] * (c[1] + g.B[1] * c[2]);
        };
        // global neighbour line (outside the brick) along D at brick-row position l (-1 or Bd)
        auto load_global = [&](int l, double (&v)[n], double &nu_face, int face_node) {
            int c[3] = {e0[0] + lc[0], e0[1] + lc[1], e0[2] + lc[2]};
            c[D] = e0[D] + l;
            const double *pu;
            if (PCG) {
                const double *pr = elem_ptr(g, a.pro.r, nullptr, nullptr, c[0], c[1], c[2]) + goff;
                const double *pd = elem_ptr(g, a.pro.dinv, nullptr, nullptr, c[0], c[1], c[2]) + goff;
                const double *pp = elem_ptr(g, a.pro.p_old, nullptr, nullptr, c[0], c[1], c[2]) + goff;
#pragma unroll
                for (int i = 0; i < n; ++i)
                    v[i] = fma(beta, __ldg(pp + i * GS[D]), __ldg(pd + i * GS[D]) * __ldg(pr + i * GS[D]));
            } else {
                pu = elem_ptr(g, a.u, a.halo.u_lo, a.halo.u_hi, c[0], c[1], c[2]) + goff;
#pragma unroll
                for (int i = 0; i < n; ++i) v[i] = __ldg(pu + i * GS[D]);
            }
            if (VARNU) {
                const double *pn = elem_ptr(g, a.nu, a.halo.nu_lo, a.halo.nu_hi, c[0], c[1], c[2]) + goff;
                nu_face = __ldg(pn + face_node * GS[D]);
            } else {
                nu_face = a.nu_const;
            }
        };
        auto load_smem = [&](int l, double (&v)[n], double (&vn)[n]) {
            const int base = slot(l) * C::SPE + soff;
#pragma unroll
            for (int i = 0; i < n; ++i) v[i] = su[base + i * SS[D]];
            if (VARNU) {
#pragma unroll
                for (int i = 0; i < n; ++i) vn[i] = snu[base + i * SS[D]];
            }
        };

        double cur[n], cnu[n], nxt[n], nnu[n];
        double uL, sL, nuL;
        {
            double nb[n];
            load_global(-1, nb, nuL, P);
            uL = nb[P];
            sL = end_flux<P>(T, nb, 1, nuL, sd);
        }
        load_smem(0, cur, cnu);
        for (int l = 0; l < Bd; ++l) {
            double uR, sR, nuR;
            if (l + 1 < Bd) {
                load_smem(l + 1, nxt, nnu);
                nuR = VARNU ? nnu[0] : a.nu_const;
            } else {
                load_global(Bd, nxt, nuR, 0);
            }
            uR = nxt[0];
            sR = end_flux<P>(T, nxt, 0, nuR, sd);
            double r[n], sP;
            line_op<P, VARNU>(T, cur, cnu, a.nu_const, uL, sL, nuL, uR, sR, nuR, sd, tau, r, sP);
            const int base = slot(l) * C::SPE + soff;
#pragma unroll
            for (int i = 0; i < n; ++i) sacc[base + i * SS[D]] += W * r[i];
            uL = cur[P];
            sL = sP;
            nuL = VARNU ? cnu[P] : a.nu_const;
#pragma unroll
            for (int i = 0; i < n; ++i) {
                cur[i] = nxt[i];
                if (VARNU) cnu[i] = nnu[i];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// apply kernel
// ---------------------------------------------------------------------------
template <int DIM, int P, bool VARNU, bool PCG>
__global__ void __launch_bounds__(256, 1) k_apply(const ApplyParams a)
{
    using C = Cfg<DIM, P>;
    constexpr int n = C::n;
    const Geom &g = a.g;
    const DevTab &T = c_tab[P];
    extern __shared__ double sm[];
    const int BE = g.B[0] * g.B[1] * g.B[2];
    double *su = sm;
    double *snu = su + BE * C::SPE;
    double *sacc = snu + (VARNU ? BE * C::SPE : 0);
    double *sred = sacc + BE * C::SPE;  // 64 doubles
    double *smass = sred + 64;          // NPE doubles: element mass m_q
    if (PCG && *a.pro.done) return;
    const double beta = PCG ? *a.pro.beta : 0.0;

    for (int q = threadIdx.x; q < C::NPE; q += blockDim.x) {
        const int i = q % n, j = (q / n) % n, k = q / (n * n);
        double m = T.w[i] * 0.5 * g.h[0] * T.w[j] * 0.5 * g.h[1];
        if (DIM == 3) m *= T.w[k] * 0.5 * g.h[2];
        smass[q] = m;
    }
    double acc2[2] = {0.0, 0.0};

    for (long long bk = a.b0 + blockIdx.x; bk < a.b1; bk += gridDim.x) {
        const int bx = (int)(bk % g.nbk[0]);
        const int by = (int)((bk / g.nbk[0]) % g.nbk[1]);
        const int bz = (int)(bk / ((long long)g.nbk[0] * g.nbk[1]));
        const int e0[3] = {bx * g.B[0], by * g.B[1], bz * g.B[2]};
        __syncthreads();
        // ---- stage the brick (coalesced per element chunk)
        for (int t = threadIdx.x; t < BE * C::NPE; t += blockDim.x) {
            const int el = t / C::NPE, q = t - el * C::NPE;
            const int lx = el % g.B[0], ly = (el / g.B[0]) % g.B[1], lz = el / (g.B[0] * g.B[1]);
            const long long gi = elem_index(g, e0[0] + lx, e0[1] + ly, e0[2] + lz) * C::NPE + q;
            const int si = el * C::SPE + (q % n) + C::PX * (q / n);
            double val;
            if (PCG) {
                val = fma(beta, a.pro.p_old[gi], a.pro.dinv[gi] * a.pro.r[gi]);
                a.pro.p_out[gi] = val;
            } else {
                val = a.u[gi];
            }
            su[si] = val;
            if (VARNU) snu[si] = a.nu[gi];
            sacc[si] = 0.0;
        }
        __syncthreads();
        apply_pass<DIM, P, VARNU, PCG, 0>(a, T, su, snu, sacc, e0, beta);
        __syncthreads();
        apply_pass<DIM, P, VARNU, PCG, 1>(a, T, su, snu, sacc, e0, beta);
        __syncthreads();
        if (DIM == 3) {
            apply_pass<DIM, P, VARNU, PCG, (DIM == 3 ? 2 : 1)>(a, T, su, snu, sacc, e0, beta);
            __syncthreads();
        }
        // ---- write out = acc + lam m u
        for (int t = threadIdx.x; t < BE * C::NPE; t += blockDim.x) {
            const int el = t / C::NPE, q = t - el * C::NPE;
            const int lx = el % g.B[0], ly = (el / g.B[0]) % g.B[1], lz = el / (g.B[0] * g.B[1]);
            const long long gi = elem_index(g, e0[0] + lx, e0[1] + ly, e0[2] + lz) * C::NPE + q;
            const int si = el * C::SPE + (q % n) + C::PX * (q / n);
            const double uu = su[si];
            const double o = fma(a.lam * smass[q], uu, sacc[si]);
            a.out[gi] = o;
            if (PCG) {
                acc2[0] = fma(uu, o, acc2[0]);
                acc2[1] += o;
            }
        }
    }
    if (PCG) {
        block_sum<2>(acc2, sred);
        if (threadIdx.x == 0) {
            a.epi.partial[2 * blockIdx.x + 0] = acc2[0];
            a.epi.partial[2 * blockIdx.x + 1] = acc2[1];
        }
    }
}

// ---------------------------------------------------------------------------
// Jacobi diagonal: diag_I = lam m_I + sum_d W_perp,d (K_d e_I)_I, evaluated by the same
// line operator on the unit vector (the neighbour line is e_I itself when the element is
// its own periodic neighbour, N_d = 1, else zero).  One thread per node.
// ---------------------------------------------------------------------------
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
                    nuL = __ldg(elem_ptr(g, nu, halo.nu_lo, halo.nu_hi, cl[0], cl[1], cl[2]) + goff + P * GS);
                    nuR = __ldg(elem_ptr(g, nu, halo.nu_lo, halo.nu_hi, cr[0], cr[1], cr[2]) + goff);
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
template <int DIM>
struct ApplyDispatch {
    template <int P, bool VARNU, bool PCG>
    static cudaError_t go(const ApplyParams &a, int grid, int smem, cudaStream_t st)
    {
        auto kern = k_apply<DIM, P, VARNU, PCG>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, 256, smem, st>>>(a);
        return cudaGetLastError();
    }
    template <int P>
    static cudaError_t go_p(const ApplyParams &a, bool varnu, bool pcg, int grid, int smem, cudaStream_t st)
    {
        if (varnu) return pcg ? go<P, true, true>(a, grid, smem, st) : go<P, true, false>(a, grid, smem, st);
        return pcg ? go<P, false, true>(a, grid, smem, st) : go<P, false, false>(a, grid, smem, st);
    }
    static cudaError_t apply(const ApplyParams &a, bool varnu, bool pcg, int grid, int smem, cudaStream_t st)
    {
        switch (a.g.P) {
        case 1: if constexpr (DG_HAS_P(1)) return go_p<1>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 2: if constexpr (DG_HAS_P(2)) return go_p<2>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 3: if constexpr (DG_HAS_P(3)) return go_p<3>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 4: if constexpr (DG_HAS_P(4)) return go_p<4>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 5: if constexpr (DG_HAS_P(5)) return go_p<5>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 6: if constexpr (DG_HAS_P(6)) return go_p<6>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 7: if constexpr (DG_HAS_P(7)) return go_p<7>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 8: if constexpr (DG_HAS_P(8)) return go_p<8>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 9: if constexpr (DG_HAS_P(9)) return go_p<9>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        case 10: if constexpr (DG_HAS_P(10)) return go_p<10>(a, varnu, pcg, grid, smem, st); else return cudaErrorNotSupported;
        default: return cudaErrorInvalidValue;
        }
    }
    template <int P>
    static cudaError_t diag_p(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                              cudaStream_t st)
    {
        const long long tot = g.nel * Cfg<DIM, P>::NPE;
        long long blocks = (tot + 255) / 256;
        if (blocks > 148 * 64) blocks = 148 * 64;
        if (nu) k_diag<DIM, P, true><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d);
        else k_diag<DIM, P, false><<<(int)blocks, 256, 0, st>>>(g, lam, nu, nuc, h, d);
        return cudaGetLastError();
    }
    static cudaError_t diag(const Geom &g, double lam, const double *nu, double nuc, const Halo &h, double *d,
                            cudaStream_t st)
    {
        switch (g.P) {
        case 1: if constexpr (DG_HAS_P(1)) return diag_p<1>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 2: if constexpr (DG_HAS_P(2)) return diag_p<2>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 3: if constexpr (DG_HAS_P(3)) return diag_p<3>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 4: if constexpr (DG_HAS_P(4)) return diag_p<4>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 5: if constexpr (DG_HAS_P(5)) return diag_p<5>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 6: if constexpr (DG_HAS_P(6)) return diag_p<6>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 7: if constexpr (DG_HAS_P(7)) return diag_p<7>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 8: if constexpr (DG_HAS_P(8)) return diag_p<8>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 9: if constexpr (DG_HAS_P(9)) return diag_p<9>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        case 10: if constexpr (DG_HAS_P(10)) return diag_p<10>(g, lam, nu, nuc, h, d, st); else return cudaErrorNotSupported;
        default: return cudaErrorInvalidValue;
        }
    }
};

}  // namespace dg
