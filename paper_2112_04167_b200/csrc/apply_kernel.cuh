// apply_kernel.cuh -- the SIP-DG apply kernel: persistent CTAs over element bricks.
//
// Per brick (BX x BY x BZ elements, compile-time shape):
//   0. staging: the NEXT brick's u (and nu; PCG mode: z and p_old) is copied global ->
//      shared with cp.async (LDGSTS, one contiguous x-row of n values per task, into an
//      odd-pitch padded layout) while the current brick computes (double buffer), so DRAM
//      latency hides behind the FP64 work;
//   1. traces: every line end on the brick surface needs the neighbour element's trace
//      (u, s = nu (2/h) d_n u, nu) at the shared face; all of them are computed in one
//      parallel phase (one neighbour line per task, L2-resident reads) into a shared-memory
//      trace table;
//   2. three line passes (x, y, z): a thread owns one brick row of B_d element lines and
//      streams it in registers: even-odd (Kopriva) matrix-vector products, in-brick faces
//      from the next line in shared memory, brick faces from the trace table;
//      x stores W r into the accumulator tile, y adds, and the last pass adds lam m u and
//      writes `out` straight to global memory (coalesced along the transverse index).
// PCG mode (MODE 1) stages z = D^-1 r and p_old, forms p = z + beta p_old, writes p, and
// reduces p.q and sum(q) in the epilogue (fused Jacobi-PCG: one HBM pass for q = A p).
// All index arithmetic inside a brick is compile-time (shape and degree are template
// parameters); only brick coordinates and global element offsets are runtime.
#pragma once

#include "dev_common.cuh"

namespace dg {

__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// out = X v for a (anti-)centro-symmetric X in even-odd form (see EOTab)
template <int P, bool ANTI>
__device__ __forceinline__ void eo_mv(const EOTab &E, const double (&v)[P + 1], double (&out)[P + 1])
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
        double se = odd ? E.Tc[i] * vm : 0.0, so = 0.0;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            se = fma(E.Te[i][j], ve[j], se);
            so = fma(E.To[i][j], vo[j], so);
        }
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
__device__ __forceinline__ double row_dot(const DevTab &T, int row, const double (&v)[P + 1])
{
    double g = 0.0;
#pragma unroll
    for (int j = 0; j <= P; ++j) g = fma(T.D[row][j], v[j], g);
    return g;
}

// compile-time configuration of one kernel instance
template <int DIM, int P, bool VARNU, int MODE, int BX, int BY, int BZ>
struct KC {
    static constexpr int n = P + 1;
    static constexpr int PX = (n % 2 == 0) ? n + 1 : n;
    static constexpr int NPE = DIM == 3 ? n * n * n : n * n;
    static constexpr int SPE = DIM == 3 ? PX * n * n : PX * n;
    static constexpr int NTL = DIM == 3 ? n * n : n;  // lines (= x rows) per element and direction
    static constexpr int B[3] = {BX, BY, BZ};
    static constexpr int BE = BX * BY * BZ;
    static constexpr int NST = 1 + (VARNU ? 1 : 0) + (MODE == 1 ? 1 : 0);
    static constexpr int LN[3] = {BE / BX * NTL, BE / BY * NTL, BE / BZ * NTL};  // brick-row lines per pass
    static constexpr int LN0 = BE / BX * NTL, LN1 = BE / BY * NTL;  // scalar copies for runtime use
    static constexpr int LM01 = LN[0] > LN[1] ? LN[0] : LN[1];
    static constexpr int LMAX = (DIM == 3 && LN[2] > LM01) ? LN[2] : LM01;  // widest pass
    static constexpr int NT0 = (LMAX + 31) / 32 * 32;
    static constexpr int NT = NT0 < 64 ? 64 : (NT0 > 512 ? 512 : NT0);     // threads per CTA
    static constexpr int TRO[3] = {0, 6 * LN[0], 6 * LN[0] + 6 * LN[1]};  // trace table offsets
    static constexpr int TRTOT = 6 * LN[0] + 6 * LN[1] + (DIM == 3 ? 6 * LN[2] : 0);
    static constexpr int STSZ = NST * BE * SPE;
    static constexpr int SMEM_DOUBLES = 2 * STSZ + BE * SPE + TRTOT + NPE + 16 + 64;
    static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
};

// neighbour element of brick-local position lc (only coordinate D may be outside the brick)
template <int DIM, int D>
__device__ __forceinline__ const double *nb_elem(const Geom &g, const double *base, const double *lo,
                                                 const double *hi, int c0, int c1, int c2)
{
    constexpr int S = DIM - 1;
    int c[3] = {c0, c1, c2};
    if (c[D] < 0) {
        if (D == S && lo) {
            const long long li = (S == 2) ? (long long)c[0] + (long long)g.Nl[0] * c[1] : (long long)c[0];
            return lo + li * g.npe;
        }
        c[D] += g.Nl[D];
    } else if (c[D] >= g.Nl[D]) {
        if (D == S && hi) {
            const long long li = (S == 2) ? (long long)c[0] + (long long)g.Nl[0] * c[1] : (long long)c[0];
            return hi + li * g.npe;
        }
        c[D] -= g.Nl[D];
    }
    return base + elem_index(g, c[0], c[1], c[2]) * g.npe;
}

// phase 1 for direction D: neighbour traces of both brick faces normal to D
template <typename K, int DIM, int P, bool VARNU, int MODE, int D>
__device__ __forceinline__ void traces(const ApplyParams &a, const DevTab &T, double *str, const int (&e0)[3],
                                       double beta, bool do0 = true, bool do1 = true)
{
    constexpr int n = K::n, NTL = K::NTL, LN = K::LN[D];
    constexpr int O1 = (D == 0) ? 1 : 0;
    constexpr int O2 = (DIM == 3) ? ((D == 2) ? 1 : 2) : 2;
    constexpr int GS[3] = {1, n, n * n};
    constexpr int BO1 = K::B[O1];
    const Geom &g = a.g;
    const double sd = 2.0 / g.h[D];
    for (int L = threadIdx.x; L < 2 * LN; L += blockDim.x) {
        const int side = L / LN, rem = L % LN;
        if (side ? !do1 : !do0) continue;
        const int ce = rem / NTL, tn = rem % NTL;
        const int ta = tn % n, tb = (DIM == 3) ? tn / n : 0;
        int c[3] = {e0[0], e0[1], e0[2]};
        c[O1] += ce % BO1;
        if (DIM == 3) c[O2] += ce / BO1;
        c[D] += side ? K::B[D] : -1;
        const int goff = ta * GS[O1] + (DIM == 3 ? tb * GS[O2] : 0);
        if (D == DIM - 1) {  // slab boundary of a multi-rank / halo-mode mesh: received face trace
            const double *tr = halo_trace(g, a.halo, c[D]);
            if (tr) {
                const long long F = halo_F(g, n), f = halo_f(g, n, c[0], c[1], goff);
                double *o = str + K::TRO[D] + L * 3;
                o[0] = __ldg(tr + f);
                o[1] = __ldg(tr + F + f);
                o[2] = VARNU ? __ldg(tr + 2 * F + f) : a.nu_const;
                continue;
            }
        }
        double v[n];
        if (MODE == 1) {
            const double *pz = nb_elem<DIM, D>(g, a.pro.z, nullptr, nullptr, c[0], c[1], c[2]) + goff;
            const double *pp = nb_elem<DIM, D>(g, a.pro.p_old, nullptr, nullptr, c[0], c[1], c[2]) + goff;
#pragma unroll
            for (int i = 0; i < n; ++i) v[i] = fma(beta, __ldg(pp + i * GS[D]), __ldg(pz + i * GS[D]));
        } else {
            const double *pu = nb_elem<DIM, D>(g, a.u, nullptr, nullptr, c[0], c[1], c[2]) + goff;
#pragma unroll
            for (int i = 0; i < n; ++i) v[i] = __ldg(pu + i * GS[D]);
        }
        double nuf = a.nu_const;
        // side 1: right neighbour, its node 0 faces us; side 0: left neighbour, its node P
        if (VARNU)
            nuf = __ldg(nb_elem<DIM, D>(g, a.nu, nullptr, nullptr, c[0], c[1], c[2]) + goff +
                        (side ? 0 : P * GS[D]));
        const double s = nuf * sd * (side ? row_dot<P>(T, 0, v) : row_dot<P>(T, P, v));
        double *o = str + K::TRO[D] + L * 3;
        o[0] = side ? v[0] : v[P];
        o[1] = s;
        o[2] = nuf;
    }
}


// Fast phase 1 for the directions D < S (never split across ranks): per-thread task
// descriptors (relative neighbour-line offset from the brick origin, direction, side) are
// computed once per kernel; per brick only the periodic wrap correction is added.  All
// loads of a thread's tasks are issued before any is consumed (memory-level parallelism).
template <typename K, int DIM>
struct SideTasks {
    static constexpr int S = DIM - 1;
    static constexpr int TOT = 2 * K::LN[0] + (DIM == 3 ? 2 * K::LN[1] : 0);  // tasks of dirs < S
    static constexpr int KT = (TOT + K::NT - 1) / K::NT;                        // per thread
};

template <typename K, int DIM, int P, bool VARNU, int MODE>
__device__ __forceinline__ void side_traces(const ApplyParams &a, const DevTab &T, double *str, long long ebase,
                                            const int (&e0)[3], const int (&toff)[SideTasks<K, DIM>::KT],
                                            const int (&tmeta)[SideTasks<K, DIM>::KT], double beta)
{
    using ST = SideTasks<K, DIM>;
    constexpr int n = K::n, NPE = K::NPE, KT = ST::KT;
    const Geom &g = a.g;
    // periodic wrap corrections (in doubles) per (direction, side) for this brick
    const long long strd1 = (long long)g.Nl[0] * NPE;  // y element stride (3-D)
    const long long cx0 = (e0[0] == 0) ? (long long)g.Nl[0] * NPE : 0;
    const long long cx1 = (e0[0] + K::B[0] == g.Nl[0]) ? -(long long)g.Nl[0] * NPE : 0;
    const long long cy0 = (DIM == 3 && e0[1] == 0) ? (long long)g.Nl[1] * strd1 : 0;
    const long long cy1 = (DIM == 3 && e0[1] + K::B[1] == g.Nl[1]) ? -(long long)g.Nl[1] * strd1 : 0;
    const long long eo = ebase * NPE;  // brick origin element, in doubles
    const double sd0 = 2.0 / g.h[0], sd1 = 2.0 / g.h[1];
    const double *ub = (MODE == 1 ? a.pro.z : a.u) + eo;
    const double *pb = MODE == 1 ? a.pro.p_old + eo : nullptr;
    const double *nb = VARNU ? a.nu + eo : nullptr;
    double v[KT][n];
    double nuf[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int meta = tmeta[k];
        if (meta < 0) continue;
        const int D = meta & 3, side = (meta >> 2) & 1;
        const long long corr = D == 0 ? (side ? cx1 : cx0) : (side ? cy1 : cy0);
        const int gs = D == 0 ? 1 : n;
        // read the line towards the shared face: side 1 (right neighbour) from node 0 up,
        // side 0 (left neighbour) from node P down, so v[0] is the face node in both cases
        const long long o0 = toff[k] + corr + (side ? 0 : P * gs);
        const int step = side ? gs : -gs;
#pragma unroll
        for (int i = 0; i < n; ++i) {
            const long long oi = o0 + i * step;
            v[k][i] = MODE == 1 ? fma(beta, __ldg(pb + oi), __ldg(ub + oi)) : __ldg(ub + oi);
        }
        nuf[k] = VARNU ? __ldg(nb + o0) : a.nu_const;
    }
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int meta = tmeta[k];
        if (meta < 0) continue;
        const int D = meta & 3, side = (meta >> 2) & 1, slot = meta >> 3;
        // flux n.(nu grad u) with n = +e_D: the right neighbour's node-0 derivative is D[0].v;
        // the left neighbour's node-P derivative is D[P].line = -D[0].(reversed line)
        double dd = 0.0;
#pragma unroll
        for (int j = 0; j < n; ++j) dd = fma(T.D[0][j], v[k][j], dd);
        const double s = nuf[k] * (D == 0 ? sd0 : sd1) * (side ? dd : -dd);
        double *o = str + slot * 3;
        o[0] = v[k][0];
        o[1] = s;
        o[2] = nuf[k];
    }
}

// z+ (slowest direction, side 1) traces from the next brick of the same column, already
// staged in shared memory
template <typename K, int DIM, int P, bool VARNU, int MODE>
__device__ __forceinline__ void next_traces(const ApplyParams &a, const DevTab &T, double *str, const double *stn,
                                            double beta)
{
    constexpr int S = DIM - 1, n = K::n, NTL = K::NTL, SPE = K::SPE, BE = K::BE, LN = K::LN[S];
    constexpr int O1 = (S == 0) ? 1 : 0;
    constexpr int O2 = (DIM == 3) ? ((S == 2) ? 1 : 2) : 2;
    constexpr int SS[3] = {1, K::PX, K::PX * n};
    constexpr int BO1 = K::B[O1];
    const double sd = 2.0 / a.g.h[S];
    for (int L = threadIdx.x; L < LN; L += blockDim.x) {
        const int ce = L / NTL, tn = L % NTL;
        const int ta = tn % n, tb = (DIM == 3) ? tn / n : 0;
        int lc[3] = {0, 0, 0};
        lc[O1] = ce % BO1;
        if (DIM == 3) lc[O2] = ce / BO1;
        const int slot = lc[0] + K::B[0] * (lc[1] + K::B[1] * lc[2]);  // lc[S] = 0: bottom layer
        const int base = slot * SPE + ta * SS[O1] + (DIM == 3 ? tb * SS[O2] : 0);
        double v[n];
#pragma unroll
        for (int i = 0; i < n; ++i) {
            const double z = stn[base + i * SS[S]];
            v[i] = MODE == 1 ? fma(beta, stn[(K::NST - 1) * BE * SPE + base + i * SS[S]], z) : z;
        }
        const double nuf = VARNU ? stn[BE * SPE + base] : a.nu_const;
        double *o = str + K::TRO[S] + (LN + L) * 3;
        o[0] = v[0];
        o[1] = nuf * sd * row_dot<P>(T, 0, v);
        o[2] = nuf;
    }
}

// phase 2 for direction D
template <typename K, int DIM, int P, bool VARNU, int MODE, int D, bool FIRST, bool LAST>
__device__ __forceinline__ void pass3(const ApplyParams &a, const DevTab &T, const double *su, const double *snu,
                                      double *sacc, double *str, long long ebase, const double *smass,
                                      const double *sw, double &epi0, double &epi1)
{
    constexpr int n = K::n, NTL = K::NTL, SPE = K::SPE, LN = K::LN[D], BD = K::B[D];
    constexpr int O1 = (D == 0) ? 1 : 0;
    constexpr int O2 = (DIM == 3) ? ((D == 2) ? 1 : 2) : 2;
    constexpr int BO1 = K::B[O1];
    constexpr int SS[3] = {1, K::PX, K::PX * n};
    constexpr int GS[3] = {1, n, n * n};
    constexpr double kap = 0.5 * (P + 1) * (P + 1);
    const Geom &g = a.g;
    const double sd = 2.0 / g.h[D];
    const double c = a.nu_const * sd;
    const double nuc = a.nu_const;
    const double lam = a.lam;
    const double tau = g.tau[D];
    double wsd[n];
#pragma unroll
    for (int k = 0; k < n; ++k) wsd[k] = sw[k] * sd;
    // global element strides of the brick-local coordinates
    const long long es[3] = {1, (long long)g.Nl[0], (long long)g.Nl[0] * g.Nl[1]};

    for (int L = threadIdx.x; L < LN; L += blockDim.x) {
        const int ce = L / NTL, tn = L % NTL;
        const int ta = tn % n, tb = (DIM == 3) ? tn / n : 0;
        int lc[3] = {0, 0, 0};
        lc[O1] = ce % BO1;
        if (DIM == 3) lc[O2] = ce / BO1;
        const int soff = ta * SS[O1] + (DIM == 3 ? tb * SS[O2] : 0);
        const int goff = ta * GS[O1] + (DIM == 3 ? tb * GS[O2] : 0);
        double W = sw[ta] * 0.5 * g.h[O1];
        if (DIM == 3) W *= sw[tb] * 0.5 * g.h[O2];
        double *trL = str + K::TRO[D] + L * 3;
        const double *trR = str + K::TRO[D] + (LN + L) * 3;
        double uL = trL[0], sL = trL[1], nuL = trL[2];
        const int slot0 = lc[0] + K::B[0] * (lc[1] + K::B[1] * lc[2]);
        constexpr int SLS = (D == 0) ? 1 : (D == 1 ? K::B[0] : K::B[0] * K::B[1]);  // slot stride along D
        double cur[n], cnu[n];
#pragma unroll
        for (int i = 0; i < n; ++i) {
            cur[i] = su[slot0 * SPE + soff + i * SS[D]];
            cnu[i] = VARNU ? snu[slot0 * SPE + soff + i * SS[D]] : nuc;
        }
#pragma unroll
        for (int l = 0; l < BD; ++l) {
            const int sl = slot0 + l * SLS;
            double nxt[n], nnu[n];
            double uR, sR, nuR;
            if (l + 1 < BD) {
                const int base = (sl + SLS) * SPE + soff;
#pragma unroll
                for (int i = 0; i < n; ++i) {
                    nxt[i] = su[base + i * SS[D]];
                    nnu[i] = VARNU ? snu[base + i * SS[D]] : nuc;
                }
                uR = nxt[0];
                nuR = nnu[0];
                sR = nuR * sd * row_dot<P>(T, 0, nxt);
            } else {
                uR = trR[0];
                sR = trR[1];
                nuR = trR[2];
            }
            double r[n];
            double sPown;
            if (VARNU) {
                double gg[n], t[n];
                eo_mv<P, true>(T.eD, cur, gg);  // D v (reference derivative)
                const double s0 = cnu[0] * sd * gg[0];
                sPown = cnu[P] * sd * gg[P];
#pragma unroll
                for (int k = 0; k < n; ++k) t[k] = wsd[k] * cnu[k] * gg[k];
                const double JR = cur[P] - uR, JL = uL - cur[0];
                // symmetry (lifting) terms c D[P][i] + c' D[0][i] = D^T (c e_P + c' e_0): fold into t
                t[P] = fma(-0.5 * cnu[P] * sd, JR, t[P]);
                t[0] = fma(-0.5 * cnu[0] * sd, JL, t[0]);
                eo_mv<P, true>(T.eE, t, r);
                r[P] += -0.5 * (sPown + sR) + tau * 0.5 * (cnu[P] + nuR) * JR;
                r[0] += 0.5 * (sL + s0) - tau * 0.5 * (nuL + cnu[0]) * JL;
            } else {
                double kv[n];
                eo_mv<P, false>(T.eK, cur, kv);
                const double aR = 0.5 * c * uR, aL = -0.5 * c * uL;
#pragma unroll
                for (int i = 0; i < n; ++i) r[i] = fma(c, kv[i], fma(aR, T.D[P][i], aL * T.D[0][i]));
                r[P] += -0.5 * sR - c * kap * uR;
                r[0] += 0.5 * sL - c * kap * uL;
                sPown = c * row_dot<P>(T, P, cur);
            }
            const int sb = sl * SPE + soff;
            if (FIRST) {
#pragma unroll
                for (int i = 0; i < n; ++i) sacc[sb + i * SS[D]] = W * r[i];
            } else if (!LAST) {
#pragma unroll
                for (int i = 0; i < n; ++i) sacc[sb + i * SS[D]] = fma(W, r[i], sacc[sb + i * SS[D]]);
            } else {
                int cc[3] = {lc[0], lc[1], lc[2]};
                cc[D] = l;
                const long long gb = (ebase + cc[0] * es[0] + cc[1] * es[1] + cc[2] * es[2]) * K::NPE + goff;
#pragma unroll
                for (int i = 0; i < n; ++i) {
                    const double o = fma(lam * smass[goff + i * GS[D]], cur[i], fma(W, r[i], sacc[sb + i * SS[D]]));
                    a.out[gb + i * GS[D]] = o;
                    if (MODE == 1) {
                        epi0 = fma(cur[i], o, epi0);
                        epi1 += o;
                    }
                }
            }
            uL = cur[P];
            sL = sPown;
            nuL = cnu[P];
            if (l + 1 < BD) {
#pragma unroll
                for (int i = 0; i < n; ++i) {
                    cur[i] = nxt[i];
                    cnu[i] = nnu[i];
                }
            }
        }
        if (LAST) {  // carry: this row's top-face trace is the next brick's bottom-face trace
            trL[0] = uL;
            trL[1] = sL;
            trL[2] = nuL;
        }
    }
}

// Work decomposition: the bricks of one column along the slowest direction S are split
// into nseg segments of seglen bricks; a unit is (column, segment) and CTA b processes units
// b, b + G, b + 2G, ... walking each segment bottom-up, so the bottom-face traces of a brick
// are the top-face traces its predecessor computed (carry) and the top-face traces come from
// the next brick's staged data.  Only segment ends read slowest-direction neighbours.
template <int DIM, int P, bool VARNU, int MODE, int BX, int BY, int BZ>
__global__ void __launch_bounds__(KC<DIM, P, VARNU, MODE, BX, BY, BZ>::NT,
                                  (KC<DIM, P, VARNU, MODE, BX, BY, BZ>::NT <= 192 ? 2 : 1)) k_apply(const ApplyParams a)
{
    using K = KC<DIM, P, VARNU, MODE, BX, BY, BZ>;
    using ST = SideTasks<K, DIM>;
    constexpr int S = DIM - 1;
    constexpr int n = K::n, NPE = K::NPE, SPE = K::SPE, PX = K::PX, NTL = K::NTL, BE = K::BE, NST = K::NST;
    constexpr int NT = K::NT, STSZ = K::STSZ, KT = ST::KT;
    const Geom &g = a.g;
    const DevTab &T = c_tab[P];
    extern __shared__ double sm[];
    double *sacc = sm + 2 * STSZ;
    double *str = sacc + BE * SPE;
    double *smass = str + K::TRTOT;
    double *sw = smass + NPE;  // n GLL weights
    double *sred = sw + 16;    // 64
    const int tid = threadIdx.x;

    if (MODE == 1 && *a.pro.done) return;
    const double beta = MODE == 1 ? *a.pro.beta : 0.0;
    for (int q = tid; q < NPE; q += NT) {
        const int i = q % n, j = (q / n) % n, k = q / (n * n);
        double m = T.w[i] * 0.5 * g.h[0] * T.w[j] * 0.5 * g.h[1];
        if (DIM == 3) m *= T.w[k] * 0.5 * g.h[2];
        smass[q] = m;
    }
    if (tid < n) sw[tid] = T.w[tid];

    // per-thread side-trace task descriptors (relative offsets, in doubles)
    int toff[KT], tmeta[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int L = tid + k * NT;
        tmeta[k] = -1;
        toff[k] = 0;
        if (L < ST::TOT) {
            const int D = (DIM == 3 && L >= 2 * K::LN0) ? 1 : 0;
            const int rem0 = L - (D ? 2 * K::LN0 : 0);
            const int LN = D ? K::LN1 : K::LN0;
            const int side = rem0 / LN, rem = rem0 % LN;
            const int ce = rem / NTL, tn = rem % NTL;
            const int ta = tn % n, tb = (DIM == 3) ? tn / n : 0;
            const int o1 = (D == 0) ? 1 : 0, o2 = 2;  // D < S: for 3-D D in {0,1}, o2 = 2 (z)
            int lc[3] = {0, 0, 0};
            const int bo1 = o1 == 0 ? BX : BY;
            if (DIM == 3) {
                lc[o1] = ce % bo1;
                lc[o2] = ce / bo1;
            } else {
                lc[1] = ce;  // 2-D, D = 0: cross-section along y
            }
            lc[D] = side ? (D == 0 ? BX : BY) : -1;
            const int gs1 = (o1 == 0) ? 1 : n, gs2 = n * n;
            const int goff = ta * gs1 + (DIM == 3 ? tb * gs2 : 0);
            const int de = lc[0] + g.Nl[0] * (lc[1] + (DIM == 3 ? g.Nl[1] * lc[2] : 0));
            toff[k] = de * NPE + goff;
            const int slot = (D == 0 ? 0 : 2 * K::LN0) + side * LN + rem;  // trace-table entry
            tmeta[k] = D | (side << 2) | (slot << 3);
        }
    }

    const int nb0 = g.nbk[0];
    const int ncols = DIM == 3 ? g.nbk[0] * g.nbk[1] : g.nbk[0];
    const long long nunits = (long long)ncols * a.nseg;
    const int seglen = a.seglen;
    // brick coordinates of the bi-th brick of this CTA; false when past the end
    auto brick_of = [&](int bi, int (&e0)[3], int &j) -> bool {
        const long long u = blockIdx.x + (long long)(bi / seglen) * gridDim.x;
        if (u >= nunits) return false;
        j = bi % seglen;
        const int col = (int)(u % ncols), zs = (int)(u / ncols);
        const int bs = zs * seglen + j;
        if (DIM == 3) {
            e0[0] = (col % nb0) * BX;
            e0[1] = (col / nb0) * BY;
            e0[2] = bs * BZ;
        } else {
            e0[0] = col * BX;
            e0[1] = bs * BY;
            e0[2] = 0;
        }
        return true;
    };
    auto ebase_of = [&](const int (&e0)[3]) {
        return (long long)e0[0] + (long long)g.Nl[0] * ((long long)e0[1] + (long long)g.Nl[1] * e0[2]);
    };
    // stage one brick: BE * NTL contiguous rows of n values per field
    auto issue = [&](const int (&e0)[3], double *st) {
        const long long eb = ebase_of(e0);
        for (int t = tid; t < BE * NTL; t += NT) {
            const int el = t / NTL, row = t % NTL;
            const int lx = el % BX, ly = (el / BX) % BY, lz = el / (BX * BY);
            const long long go =
                (eb + lx + (long long)g.Nl[0] * (ly + (long long)g.Nl[1] * lz)) * NPE + row * n;
            double *dst = st + el * SPE + row * PX;
            const double *s0 = (MODE == 1 ? a.pro.z : a.u) + go;
#pragma unroll
            for (int i = 0; i < n; ++i) cp_async8(dst + i, s0 + i);
            if (VARNU) {
#pragma unroll
                for (int i = 0; i < n; ++i) cp_async8(dst + BE * SPE + i, a.nu + go + i);
            }
            if (MODE == 1) {
#pragma unroll
                for (int i = 0; i < n; ++i) cp_async8(dst + (NST - 1) * BE * SPE + i, a.pro.p_old + go + i);
            }
        }
    };

    double epi0 = 0.0, epi1 = 0.0;
    int e0[3], jcur;
    bool have = brick_of(0, e0, jcur);
    if (have) issue(e0, sm);
    cp_async_commit();
    for (int bi = 0; have; ++bi) {
        double *st = sm + (bi & 1) * STSZ;
        double *stn = sm + ((bi + 1) & 1) * STSZ;
        int e1[3], jn;
        const bool haven = brick_of(bi + 1, e1, jn);
        if (haven) issue(e1, stn);
        cp_async_commit();
        const long long eb = ebase_of(e0);
        const bool seg_first = (jcur == 0), seg_last = (jcur == seglen - 1);
        // phase 1: side traces (global, L2-resident); slowest-direction traces only at
        // segment ends (elsewhere: carry from the previous brick / next brick's stage)
        side_traces<K, DIM, P, VARNU, MODE>(a, T, str, eb, e0, toff, tmeta, beta);
        if (seg_first || seg_last) traces<K, DIM, P, VARNU, MODE, S>(a, T, str, e0, beta, seg_first, seg_last);
        cp_async_wait1();
        __syncthreads();
        double *su = st;
        const double *snu = st + BE * SPE;
        if (MODE == 1) {
            const double *spo = st + (NST - 1) * BE * SPE;
            for (int t = tid; t < BE * NTL; t += NT) {
                const int el = t / NTL, row = t % NTL;
                const int lx = el % BX, ly = (el / BX) % BY, lz = el / (BX * BY);
                const long long go =
                    (eb + lx + (long long)g.Nl[0] * (ly + (long long)g.Nl[1] * lz)) * NPE + row * n;
                const int so = el * SPE + row * PX;
#pragma unroll
                for (int i = 0; i < n; ++i) {
                    const double p = fma(beta, spo[so + i], su[so + i]);
                    su[so + i] = p;
                    a.pro.p_out[go + i] = p;
                }
            }
            __syncthreads();
        }
        if (DIM == 3) {
            pass3<K, DIM, P, VARNU, MODE, 0, true, false>(a, T, su, snu, sacc, str, eb, smass, sw, epi0, epi1);
            __syncthreads();
            pass3<K, DIM, P, VARNU, MODE, 1, false, false>(a, T, su, snu, sacc, str, eb, smass, sw, epi0, epi1);
        } else {
            pass3<K, DIM, P, VARNU, MODE, 0, true, false>(a, T, su, snu, sacc, str, eb, smass, sw, epi0, epi1);
        }
        if (!seg_last) {  // the next brick (same column) must have landed for its bottom traces
            cp_async_wait0();
            __syncthreads();
            next_traces<K, DIM, P, VARNU, MODE>(a, T, str, stn, beta);
        }
        __syncthreads();
        pass3<K, DIM, P, VARNU, MODE, S, false, true>(a, T, su, snu, sacc, str, eb, smass, sw, epi0, epi1);
        __syncthreads();
        have = haven;
        e0[0] = e1[0];
        e0[1] = e1[1];
        e0[2] = e1[2];
        jcur = jn;
    }
    if (MODE == 1) {
        double v2[2] = {epi0, epi1};
        block_sum<2>(v2, sred);
        if (tid == 0) {
            a.epi.partial[2 * blockIdx.x + 0] = v2[0];
            a.epi.partial[2 * blockIdx.x + 1] = v2[1];
        }
    }
}

}  // namespace dg
