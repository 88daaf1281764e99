// apply5.cuh -- 3-D SIP-DG apply, v5: warp-specialised producer/consumer bricks.
//
// Same operator as apply.cuh (P:1039 interior penalty, Alg. 3 lines 5/9, readings A1-A5);
// this file only changes HOW it is scheduled on sm_100a (DESIGN.md §6 "k_apply5"):
//
//   * a persistent CTA walks z-column segments of 2x2x2-element bricks (z slowest, so the
//     x/y neighbour columns are processed concurrently by neighbouring CTAs and their data
//     is L2-resident);
//   * PRODUCER warps (4) run one brick ahead: they stage the brick's u and nu into shared
//     memory with TMA bulk copies (cp.async.bulk, completion on an mbarrier with
//     expect_tx), and compute every brick-surface neighbour trace (u, nu (2/h) d_n u, nu) of
//     the six faces from the neighbour element lines in L2 into a trace table.  PCG mode
//     (MODE 1) instead forms p = z + beta p_old in registers, stores it to shared memory and
//     to p_out (the fused CG prologue), and takes the neighbour traces of p;
//   * CONSUMER warps wait on the brick's "full" mbarrier and run three line passes (x, y, z):
//     a thread owns one brick-row line (2 elements) and keeps it in registers: even-odd
//     D / D^T (variable nu) or K_ref (constant nu) products, the in-brick face in registers,
//     the two brick faces from the trace table; x writes W r into the accumulator tile, y
//     adds, z adds lam m u and stores `out` to global memory (coalesced), with the PCG dot
//     epilogue; then the consumers arrive on the brick's "empty" mbarrier.
//   * no division, no 64-bit div/mod and no per-element address arithmetic on the hot
//     path: all strides are compile-time, scalars (2/h, tau, Jacobians) come precomputed.
//
// Shared memory (doubles): U[2][8 n^3], NU[2][8 n^3] (variable nu), ACC[8 n^3],
// TR[2][sum_d 2 * 4 n^2 * NV] (NV = 3 values per trace, 2 for constant nu), 4 mbarriers.
#pragma once

#include <cstdint>

#include "dev_common.cuh"

namespace dg {
namespace v5 {

#ifdef DG_V5_DEBUG
// development instrumentation: per-role cycle counters (see dg_debug_counters in apply3.cu)
__device__ unsigned long long g_dbg[16];
#define V5_T0(var) const long long var = clock64()
#define V5_ACC(idx, var) atomicAdd(&g_dbg[idx], (unsigned long long)(clock64() - (var)))
#else
#define V5_T0(var)
#define V5_ACC(idx, var)
#endif

__device__ __forceinline__ unsigned su32(const void *p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(su32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared (this CTA), completion counted on mbarrier b
__device__ __forceinline__ void tma_load(void *sdst, const void *gsrc, unsigned bytes, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(su32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(su32(b))
        : "memory");
}
// bulk L2 prefetch of [p, p + bytes) (rounded out to 16-byte granules)
__device__ __forceinline__ void l2_prefetch(const void *p, unsigned bytes)
{
    const unsigned long long a0 = reinterpret_cast<unsigned long long>(p) & ~15ull;
    const unsigned long long a1 = (reinterpret_cast<unsigned long long>(p) + bytes + 15ull) & ~15ull;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int count)
{
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// out = X v for a (anti-)centro-symmetric X in even-odd form (see EOTab) -- as apply_kernel.cuh
template <int P, bool ANTI>
__device__ __forceinline__ void eo(const EOTab &E, const double (&v)[P + 1], double (&out)[P + 1])
{
    constexpr int n = P + 1, h = n / 2, mid = P / 2;
    constexpr bool odd = (n % 2) == 1;
    double ve[h], vo[h];
#pragma unroll
    for (int j = 0; j < h; ++j) {
        ve[j] = v[j] + v[P - j];
        vo[j] = v[j] - v[P - j];
    }
    const double vm = odd ? v[mid] : 0.0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
        double se = odd ? E.Tc[i] * vm : E.Te[i][0] * ve[0];
        double so = E.To[i][0] * vo[0];
#pragma unroll
        for (int j = odd ? 0 : 1; j < h; ++j) se = fma(E.Te[i][j], ve[j], se);
#pragma unroll
        for (int j = 1; j < h; ++j) so = fma(E.To[i][j], vo[j], so);
        out[i] = se + so;
        out[P - i] = ANTI ? so - se : se - so;
    }
    if (odd) {
        double m = ANTI ? 0.0 : E.Mmid * vm;
#pragma unroll
        for (int j = 0; j < h; ++j) m = fma(E.Mr[j], ANTI ? vo[j] : ve[j], m);
        out[mid] = m;
    }
}

template <int P>
__device__ __forceinline__ double rdot(const DevTab &T, int row, const double (&v)[P + 1])
{
    double g = T.D[row][0] * v[0];
#pragma unroll
    for (int j = 1; j <= P; ++j) g = fma(T.D[row][j], v[j], g);
    return g;
}

template <int P_, bool VARNU_, int MODE_>
struct KC5 {
    static constexpr int P = P_;
    static constexpr bool VARNU = VARNU_;
    static constexpr int MODE = MODE_;
    static constexpr int n = P + 1;
    static constexpr int NN = n * n;
    static constexpr int NPE = n * n * n;
    static constexpr int B = 2;                 // brick edge (elements) in every direction
    static constexpr int BE = B * B * B;
    static constexpr int LN = (BE / B) * NN;     // brick-row lines per pass (4 n^2)
    static constexpr int NC = (LN + 31) / 32 * 32;  // consumer threads
    static constexpr int NP = 96;                // producer threads (3 warps)
    static constexpr int NT = NC + NP;
    static constexpr int NV = VARNU ? 3 : 2;     // values per trace entry: u, s (, nu)
    static constexpr int TRD = 2 * NV * LN;      // trace entries per direction
    static constexpr int TRB = 3 * TRD;          // per buffer
    static constexpr int BRK = BE * NPE;         // doubles per staged field
    static constexpr int OFF_U = 0;
    static constexpr int OFF_NU = OFF_U + 2 * BRK;
    static constexpr int OFF_ACC = OFF_NU + (VARNU ? 2 * BRK : 0);
    static constexpr int OFF_TR = OFF_ACC + BRK;
    static constexpr int OFF_RED = OFF_TR + 2 * TRB;
    static constexpr int OFF_BAR = OFF_RED + 64;  // 4 mbarriers (uint64)
    static constexpr int SMEM_DOUBLES = OFF_BAR + 4;
    static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
    static constexpr int KTD = (2 * LN + NP - 1) / NP;  // producer trace tasks per thread per direction
    static constexpr int MINB = (SMEM_BYTES + 1024) * 2 <= 228 * 1024 ? 2 : 1;
    // registers per thread for MINB resident CTAs: each of the 4 SM sub-partitions has a
    // 16K-register file and receives ceil(warps / 4) of the resident warps
    static constexpr int NW = (NT + 31) / 32;
    static constexpr int MAXREG0 = 16384 / (((MINB * NW + 3) / 4) * 32) / 8 * 8;
    static constexpr int MAXREG = MAXREG0 > 255 ? 255 : MAXREG0;
};

// transverse directions of D
template <int D>
struct Tr {
    static constexpr int O1 = D == 0 ? 1 : 0;
    static constexpr int O2 = D == 2 ? 1 : 2;
};

// ---------------------------------------------------------------------------
// consumer: one direction pass over the brick
// ---------------------------------------------------------------------------
// z-pass carry of one consumer thread (its z line L is the same in every brick): the output
// of the brick's TOP element line is held back until the next brick of the column supplies
// the other side of the shared face, so no brick ever waits for its upper neighbour.
template <int n>
struct ZCarry {
    bool held = false;
    double o[n];          // top-element output without its top-face terms
    double *po = nullptr; // its destination
    double u, gP, nu;     // top-face own trace: u_P, (D v)_P, nu_P
};

template <class K, int D, bool FIRST, bool LAST>
__device__ __forceinline__ void cpass(const ApplyParams &a, const DevTab &T, const double *su, const double *snu,
                                      double *sacc, const double *tr, long long ebase, int L, double &epi0,
                                      double &epi1, ZCarry<K::n> &zc, bool zfirst, bool zlast)
{
    constexpr int P = K::P, n = K::n, NN = K::NN, NPE = K::NPE, B = K::B, LN = K::LN, NV = K::NV;
    constexpr int O1 = Tr<D>::O1, O2 = Tr<D>::O2;
    constexpr int SS[3] = {1, n, NN};                         // node strides (smem == global)
    constexpr int ES[3] = {NPE, B * NPE, B * B * NPE};        // element strides in the brick
    constexpr bool ZC = (D == 2) && LAST;                     // column carry active in this pass
    if (L >= LN) return;
    const Geom &g = a.g;
    const int ce = L / NN, tn = L - ce * NN;
    const int ta = tn % n, tb = tn / n;
    const int c1 = ce % B, c2 = ce / B;
    const int soff = c1 * ES[O1] + c2 * ES[O2] + ta * SS[O1] + tb * SS[O2];
    const double W = T.w[ta] * T.w[tb] * g.wfac[D];
    const double sd = g.sd[D], htau = 0.5 * g.tau[D];
    const double *trd = tr + D * K::TRD;
    // brick-face traces: side 0 (left/bottom neighbour, its node P), side 1 (its node 0)
    const bool use_lo = !ZC || zfirst, use_hi = !ZC || zlast;
    const double nu_c = a.nu_const;
    double uLb, sLb, nuLb, uRb = 0.0, sRb = 0.0, nuRb = nu_c;
    if (use_lo) {
        uLb = trd[0 * LN + L];
        sLb = trd[1 * LN + L];
        nuLb = K::VARNU ? trd[2 * LN + L] : nu_c;
    } else {
        uLb = zc.u;
        nuLb = K::VARNU ? zc.nu : nu_c;
        sLb = nuLb * sd * zc.gP;
    }
    if (use_hi) {
        uRb = trd[NV * LN + L];
        sRb = trd[(NV + 1) * LN + L];
        nuRb = K::VARNU ? trd[(NV + 2) * LN + L] : nu_c;
    }

    double v[B][n], nv[B][n];
#pragma unroll
    for (int l = 0; l < B; ++l) {
        const double *pu = su + soff + l * ES[D];
        if (D == 0 && (n % 2) == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 2) {
                const double2 x = *reinterpret_cast<const double2 *>(pu + i);
                v[l][i] = x.x;
                v[l][i + 1] = x.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < n; ++i) v[l][i] = pu[i * SS[D]];
        }
        if (K::VARNU) {
            const double *pn = snu + soff + l * ES[D];
            if (D == 0 && (n % 2) == 0) {
#pragma unroll
                for (int i = 0; i < n; i += 2) {
                    const double2 x = *reinterpret_cast<const double2 *>(pn + i);
                    nv[l][i] = x.x;
                    nv[l][i + 1] = x.y;
                }
            } else {
#pragma unroll
                for (int i = 0; i < n; ++i) nv[l][i] = pn[i * SS[D]];
            }
        }
    }

    // release the held top element of the previous brick: add its top-face terms
    // dr_i = c D_{P,i} + [i == P] f0 (c: lifting / neighbour-value coefficient, f0: flux part)
    auto release = [&](double c, double f0) {
        double s1 = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
            const double d = W * fma(c, T.D[P][i], i == P ? f0 : 0.0);
            zc.po[i * SS[D]] = zc.o[i] + d;
            s1 += d;
        }
        if (K::MODE >= 1) {
            epi0 = fma(W, fma(c, zc.gP, f0 * zc.u), epi0);  // sum_i v_i dr_i W
            epi1 += s1;
        }
        zc.held = false;
    };

    // accumulate / store (or hold) the line result r of element l of the brick row
    auto emit = [&](int l, const double (&r)[n], bool hold) {
        double *pa = sacc + soff + l * ES[D];
        if (FIRST) {
#pragma unroll
            for (int i = 0; i < n; ++i) pa[i * SS[D]] = W * r[i];
        } else if (!LAST) {
#pragma unroll
            for (int i = 0; i < n; ++i) pa[i * SS[D]] = fma(W, r[i], pa[i * SS[D]]);
        } else {
            int lc[3];
            lc[O1] = c1;
            lc[O2] = c2;
            lc[D] = l;
            const long long ge = ebase + lc[0] + (long long)g.Nl[0] * (lc[1] + (long long)g.Nl[1] * lc[2]);
            double *po = a.out + ge * NPE + ta * SS[O1] + tb * SS[O2];
            const double lw = a.lam * W * (0.5 * g.h[D]);  // lam m_I = lam W w_i h_D/2
#pragma unroll
            for (int i = 0; i < n; ++i) {
                const double ui = v[l][i];
                const double o = fma(lw * T.w[i], ui, fma(W, r[i], pa[i * SS[D]]));
                if (ZC && hold) zc.o[i] = o;
                else po[i * SS[D]] = o;
                if (K::MODE >= 1) {
                    epi0 = fma(ui, o, epi0);
                    epi1 += o;
                }
            }
            if (ZC && hold) zc.po = po;
        }
    };

    if (K::VARNU) {
        double gg[B][n];
#pragma unroll
        for (int l = 0; l < B; ++l) eo<P, true>(T.eD, v[l], gg[l]);
        // faces f = 0..B: F_f = -1/2 (s- + s+) + tau/2 (nu- + nu+) J,  J = u- - u+,
        // own end fluxes s = nu (2/h) (D v) at nodes 0 and P
        double F[B + 1], J[B + 1];
#pragma unroll
        for (int f = 0; f <= B; ++f) {
            const double um = f == 0 ? uLb : v[f - 1][P];
            const double sm = f == 0 ? sLb : nv[f - 1][P] * sd * gg[f - 1][P];
            const double nm = f == 0 ? nuLb : nv[f - 1][P];
            const double up = f == B ? uRb : v[f][0];
            const double sp = f == B ? sRb : nv[f][0] * sd * gg[f][0];
            const double np = f == B ? nuRb : nv[f][0];
            J[f] = um - up;
            F[f] = fma(htau * (nm + np), J[f], -0.5 * (sm + sp));
        }
        if (ZC && !use_hi) {  // top face deferred to the next brick
            F[B] = 0.0;
            J[B] = 0.0;
        }
        if (ZC && !use_lo && zc.held) release(-0.5 * sd * zc.nu * J[0], F[0]);
#pragma unroll
        for (int l = 0; l < B; ++l) {
            double t[n], r[n];
#pragma unroll
            for (int k = 0; k < n; ++k) t[k] = g.wsd[D][k] * (nv[l][k] * gg[l][k]);
            // symmetry (lifting) terms -1/2 nu (2/h) D_{end,i} J folded into the D^T operand
            t[P] = fma(-0.5 * sd * nv[l][P], J[l + 1], t[P]);
            t[0] = fma(-0.5 * sd * nv[l][0], J[l], t[0]);
            eo<P, true>(T.eE, t, r);
            r[P] += F[l + 1];
            r[0] -= F[l];
            emit(l, r, l == B - 1 && !use_hi);
        }
        if (ZC && !use_hi) {
            zc.held = true;
            zc.u = v[B - 1][P];
            zc.gP = gg[B - 1][P];
            zc.nu = nv[B - 1][P];
        }
    } else {
        const double c = nu_c * sd;
        const double ck = c * (0.5 * (P + 1) * (P + 1));
        double d0[B], dP[B];
#pragma unroll
        for (int l = 0; l < B; ++l) {
            d0[l] = rdot<P>(T, 0, v[l]);
            dP[l] = rdot<P>(T, P, v[l]);
        }
        // previous top element: neighbour terms (1/2 c u+) D_P + [P] (-1/2 s+ - c kappa u+)
        if (ZC && !use_lo && zc.held) release(0.5 * c * v[0][0], fma(-ck, v[0][0], -0.5 * c * d0[0]));
#pragma unroll
        for (int l = 0; l < B; ++l) {
            const double uL = l == 0 ? uLb : v[l - 1][P];
            const double sL = l == 0 ? sLb : c * dP[l - 1];
            const double uR = l == B - 1 ? uRb : v[l + 1][0];
            const double sR = l == B - 1 ? sRb : c * d0[l + 1];
            double kv[n], r[n];
            eo<P, false>(T.eK, v[l], kv);
            const double aR = 0.5 * c * uR, aL = -0.5 * c * uL;
#pragma unroll
            for (int i = 0; i < n; ++i) r[i] = fma(c, kv[i], fma(aR, T.D[P][i], aL * T.D[0][i]));
            r[P] += fma(-ck, uR, -0.5 * sR);
            r[0] += fma(-ck, uL, 0.5 * sL);
            emit(l, r, l == B - 1 && !use_hi);
        }
        if (ZC && !use_hi) {
            zc.held = true;
            zc.u = v[B - 1][P];
            zc.gP = dP[B - 1];
        }
    }
}

// pointer to the element with local coordinates c (only c[D] may be one step outside the
// slab; x/y wrap periodically, z wraps or reads the rank-neighbour halo layer)
template <int D>
__device__ __forceinline__ const double *nbr(const Geom &g, const double *base, const double *lo, const double *hi,
                                             int c0, int c1, int c2, int npe)
{
    if (D == 0) c0 = c0 < 0 ? c0 + g.Nl[0] : (c0 >= g.Nl[0] ? c0 - g.Nl[0] : c0);
    if (D == 1) c1 = c1 < 0 ? c1 + g.Nl[1] : (c1 >= g.Nl[1] ? c1 - g.Nl[1] : c1);
    if (D == 2) {
        if (c2 < 0) {
            if (lo) return lo + ((long long)c0 + (long long)g.Nl[0] * c1) * npe;
            c2 += g.Nl[2];
        } else if (c2 >= g.Nl[2]) {
            if (hi) return hi + ((long long)c0 + (long long)g.Nl[0] * c1) * npe;
            c2 -= g.Nl[2];
        }
    }
    return base + ((long long)c0 + (long long)g.Nl[0] * ((long long)c1 + (long long)g.Nl[1] * c2)) * npe;
}

// ---------------------------------------------------------------------------
// producer: neighbour traces of one direction for the brick at e0
// ---------------------------------------------------------------------------
template <class K, int D>
__device__ __noinline__ void ptraces(const ApplyParams &a, const DevTab &T, double *tr, const int (&e0)[3],
                                     int ptid, double beta, int smask)
{
    constexpr int P = K::P, n = K::n, NN = K::NN, NPE = K::NPE, B = K::B, LN = K::LN, NV = K::NV, KT = K::KTD;
    constexpr int O1 = Tr<D>::O1, O2 = Tr<D>::O2;
    constexpr int GS[3] = {1, n, NN};
    const Geom &g = a.g;
    const double sd = g.sd[D];
    const double *fu = K::MODE == 1 ? a.pro.z : a.u;
    double v[KT][n], nuf[KT];
    int slot[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int t = ptid + k * K::NP;
        slot[k] = -1;
        if (t >= 2 * LN) continue;
        const int side = t >= LN ? 1 : 0;
        if (!((smask >> side) & 1)) continue;
        const int L = t - side * LN;
        const int ce = L / NN, tn = L - ce * NN;
        const int ta = tn % n, tb = tn / n;
        int c[3];
        c[O1] = e0[O1] + ce % B;
        c[O2] = e0[O2] + ce / B;
        c[D] = side ? e0[D] + B : e0[D] - 1;
        const int goff = ta * GS[O1] + tb * GS[O2] + (side ? 0 : P * GS[D]);  // face node of the line
        const int step = side ? GS[D] : -GS[D];  // walk away from the shared face
        if (D == 2 && K::MODE != 1) {  // slab boundary of a multi-rank / halo-mode mesh: received trace
            const double *trh = halo_trace(g, a.halo, c[2]);
            if (trh) {  // (u, s = nu d_z u, nu): the table's canonical form, stored directly
                const long long F = halo_F(g, n), f = halo_f(g, n, c[0], c[1], ta + n * tb);
                double *o = tr + D * K::TRD + side * NV * LN + L;
                o[0] = __ldg(trh + f);
                o[LN] = __ldg(trh + F + f);
                if (K::VARNU) o[2 * LN] = __ldg(trh + 2 * F + f);
                continue;
            }
        }
        const double *pu = nbr<D>(g, fu, nullptr, nullptr, c[0], c[1], c[2], NPE) + goff;
        if (K::MODE == 1) {
            const long long off = pu - fu;
            const double *pp = a.pro.p_old + off;
#pragma unroll
            for (int i = 0; i < n; ++i) v[k][i] = fma(beta, __ldg(pp + i * step), __ldg(pu + i * step));
        } else {
#pragma unroll
            for (int i = 0; i < n; ++i) v[k][i] = __ldg(pu + i * step);
        }
        nuf[k] = K::VARNU ? __ldg(nbr<D>(g, a.nu, nullptr, nullptr, c[0], c[1], c[2], NPE) + goff) : a.nu_const;
        slot[k] = side * NV * LN + L;
    }
    double *trd = tr + D * K::TRD;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        if (slot[k] < 0) continue;
        // v[k][0] is the face node; D[0] . v is the derivative there for the right
        // neighbour; for the left neighbour the line was read reversed, so its node-P
        // derivative D[P] . line = -D[0] . (reversed line)
        const double dd = rdot<P>(T, 0, v[k]);
        const bool side = slot[k] >= NV * LN;
        trd[slot[k]] = v[k][0];
        trd[slot[k] + LN] = nuf[k] * sd * (side ? dd : -dd);
        if (K::VARNU) trd[slot[k] + 2 * LN] = nuf[k];
    }
}

template <int P, bool VARNU, int MODE>
__global__ void __launch_bounds__((KC5<P, VARNU, MODE>::NT)) __maxnreg__((KC5<P, VARNU, MODE>::MAXREG)) k_apply5(const __grid_constant__ ApplyParams a)
{
    using K = KC5<P, VARNU, MODE>;
    constexpr int NPE = K::NPE, B = K::B, BRK = K::BRK, NC = K::NC, NP = K::NP;
    const Geom &g = a.g;
    const DevTab &T = c_tab[P];
    extern __shared__ __align__(16) double sm[];
    // full[0..1] (producers + TMA bytes), empty[0..1] (consumers)
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + K::OFF_BAR);
    const int tid = threadIdx.x;
    if (MODE >= 1 && *a.pro.done) return;  // PCG converged: nothing to do
    const double beta = MODE == 1 ? *a.pro.beta : 0.0;
    if (tid == 0) {
        mbar_init(&bar[0], NP);
        mbar_init(&bar[1], NP);
        mbar_init(&bar[2], NC);
        mbar_init(&bar[3], NC);
        fence_proxy_async();
    }
    __syncthreads();

    const int nb0 = g.Nl[0] / B, nb1 = g.Nl[1] / B;
    const int ncols = nb0 * nb1;
    const int nunits = ncols * a.nseg;
    const int seglen = a.seglen;
    const long long s1 = g.Nl[0], s2 = (long long)g.Nl[0] * g.Nl[1];

    if (tid >= NC) {
        // ------------------------------- producer -------------------------------
        const int ptid = tid - NC;
        int it = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int col = u % ncols, zs = u / ncols;
            int e0[3] = {(col % nb0) * B, (col / nb0) * B, a.zlo + zs * seglen * B};
            for (int j = 0; j < seglen; ++j, ++it, e0[2] += B) {
                const int buf = it & 1;
                V5_T0(tw);
                if (it >= 2) mbar_wait(&bar[2 + buf], ((it >> 1) - 1) & 1);
                if (ptid == 0) V5_ACC(2, tw);
                V5_T0(tt);
                double *su = sm + K::OFF_U + buf * BRK;
                double *snu = sm + K::OFF_NU + buf * BRK;
                const long long eb = e0[0] + s1 * e0[1] + s2 * e0[2];
                constexpr unsigned CH = 2u * NPE * 8u;  // bytes of one x-pair of elements
                if (ptid == 0) {
                    const unsigned bytes = (MODE != 1 ? 4u * CH : 0u) + (VARNU ? 4u * CH : 0u);
                    if (bytes) mbar_expect_tx(&bar[buf], bytes);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {  // (y, z) rows of the brick; x pairs contiguous
                        const long long ge = eb + (q & 1) * s1 + (q >> 1) * s2;
                        if (MODE != 1) tma_load(su + q * 2 * NPE, a.u + ge * NPE, CH, &bar[buf]);
                        if (VARNU) tma_load(snu + q * 2 * NPE, a.nu + ge * NPE, CH, &bar[buf]);
                    }
                }
                if (MODE == 1) {  // p = z + beta p_old -> shared (operand) and p_out (fused CG prologue)
                    constexpr int NQ = 4 * NPE;  // double2 per brick (4 chunks of 2 n^3 doubles)
                    for (int q = ptid; q < NQ; q += NP) {
                        const int ch = q / NPE, w = q - ch * NPE;
                        const long long go = (eb + (ch & 1) * s1 + (ch >> 1) * s2) * NPE + 2 * w;
                        const double2 z = __ldg(reinterpret_cast<const double2 *>(a.pro.z + go));
                        const double2 po = __ldg(reinterpret_cast<const double2 *>(a.pro.p_old + go));
                        double2 p;
                        p.x = fma(beta, po.x, z.x);
                        p.y = fma(beta, po.y, z.y);
                        *reinterpret_cast<double2 *>(su + ch * 2 * NPE + 2 * w) = p;
                        *reinterpret_cast<double2 *>(a.pro.p_out + go) = p;
                    }
                }
                double *tr = sm + K::OFF_TR + buf * K::TRB;
                if (ptid == 0) V5_ACC(4, tt);
                V5_T0(tx);
                ptraces<K, 0>(a, T, tr, e0, ptid, beta, 3);
                if (ptid == 0) V5_ACC(9, tx);
                V5_T0(ty);
                ptraces<K, 1>(a, T, tr, e0, ptid, beta, 3);
                if (ptid == 0) V5_ACC(10, ty);
                // z faces: from global memory only at segment ends; inside a segment the
                // consumers carry the shared face from one brick to the next (ZCarry)
                const int zm = (j == 0 ? 1 : 0) | (j == seglen - 1 ? 2 : 0);
                if (zm) ptraces<K, 2>(a, T, tr, e0, ptid, beta, zm);
                if (ptid == 0) V5_ACC(3, tx);
                mbar_arrive(&bar[buf]);
            }
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    double epi0 = 0.0, epi1 = 0.0;
    int it = 0;
    ZCarry<K::n> zc;
    double *sacc = sm + K::OFF_ACC;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int col = u % ncols, zs = u / ncols;
        int e0[3] = {(col % nb0) * B, (col / nb0) * B, a.zlo + zs * seglen * B};
        for (int j = 0; j < seglen; ++j, ++it, e0[2] += B) {
            const int buf = it & 1;
            const double *su = sm + K::OFF_U + buf * BRK;
            const double *snu = sm + K::OFF_NU + buf * BRK;
            const double *tr = sm + K::OFF_TR + buf * K::TRB;
            const long long eb = e0[0] + s1 * e0[1] + s2 * e0[2];
            V5_T0(tw);
            mbar_wait(&bar[buf], (it >> 1) & 1);
            if (tid == 0) V5_ACC(0, tw);
            V5_T0(tp);
            const bool zf = j == 0, zl = j == seglen - 1;
            cpass<K, 0, true, false>(a, T, su, snu, sacc, tr, eb, tid, epi0, epi1, zc, zf, zl);
            if (tid == 0) V5_ACC(6, tp);
            named_sync(1, NC);
            V5_T0(t1);
            cpass<K, 1, false, false>(a, T, su, snu, sacc, tr, eb, tid, epi0, epi1, zc, zf, zl);
            if (tid == 0) V5_ACC(7, t1);
            named_sync(1, NC);
            V5_T0(t2);
            cpass<K, 2, false, true>(a, T, su, snu, sacc, tr, eb, tid, epi0, epi1, zc, zf, zl);
            if (tid == 0) V5_ACC(8, t2);
            mbar_arrive(&bar[2 + buf]);
            named_sync(1, NC);  // ACC is rewritten by the next brick's x pass
            if (tid == 0) {
                V5_ACC(1, tp);
#ifdef DG_V5_DEBUG
                atomicAdd(&g_dbg[5], 1ull);
#endif
            }
        }
    }
    if (MODE >= 1) {  // dot epilogue: block partials of u.out and sum(out)
        double *red = sm + K::OFF_RED;
        const int lane = tid & 31, wid = tid >> 5;
        epi0 = warp_sum(epi0);
        epi1 = warp_sum(epi1);
        if (lane == 0) {
            red[wid] = epi0;
            red[32 + wid] = epi1;
        }
        named_sync(1, NC);
        if (tid == 0) {
            double s0 = 0.0, s1v = 0.0;
            for (int w = 0; w < NC / 32; ++w) {
                s0 += red[w];
                s1v += red[32 + w];
            }
            a.epi.partial[2 * blockIdx.x + 0] = s0;
            a.epi.partial[2 * blockIdx.x + 1] = s1v;
        }
    }
}

}  // namespace v5
}  // namespace dg
