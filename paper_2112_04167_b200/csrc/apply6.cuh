// MODE: 0 plain apply; 1 fused PCG operand (prologue p = z + beta p_old, dot epilogue);
// 2 apply with the dot epilogue only (the split PCG path: p formed by k_pcg_pupd); 3 as 2
// without sum(out) (lam > 0: the mean of q is not used; one accumulator fewer at 80 registers).
//
// apply6.cuh -- 3-D SIP-DG apply, v6: one persistent CTA per SM, 4x4x1-element bricks,
// warp-specialised producer / consumers, one element line per consumer thread with warp
// shuffles across the in-brick faces.
//
// Same operator as apply.cuh / apply5.cuh (P:1039 interior penalty; Alg. 3 lines 5/9;
// readings A1-A5).  What changes against v5 (DESIGN.md §6 "k_apply6"):
//
//   * bricks of 4x4x1 elements (a z-column segment is walked one element layer at a time):
//     x/y brick faces per element halve against 2x2x2 (the producer's L2 trace work), and
//     every z face is carried by the consumer that owns the z line in consecutive bricks;
//   * 5 consumer warpgroups (one thread per element line: 16 n^2 lines per pass) and one
//     producer warpgroup; the producer loads a brick's x/y neighbour lines in two memory
//     rounds (at most 3 lines per thread in flight at 80 registers);
//   * in the x and y passes the 4 elements of a brick row sit on 4 adjacent lanes: the
//     in-brick faces exchange (u, nu (2/h) d_n u, nu) with __shfl_up/down, only the two
//     brick-end lanes read the producer's trace table;
//   * z pass: the bottom face comes from the thread's own carry (the previous brick's top
//     line), the top face is deferred -- the element output is parked in shared memory and
//     completed by the next brick (the v5 ZCarry, per element line);
//   * segment ends: each column segment is walked with one halo brick below and above it,
//     staged by TMA like the others (periodic layers; received face traces at the slab ends of
//     a halo mesh): the bottom halo seeds the z carry, the top halo releases the last parked
//     outputs -- no per-line global loads for the segment-end z traces (round 3: c5
//     0.517 -> 0.493 ms, per-segment cost 3.3 -> 1.1 bricks);
//   * staging: TMA bulk copies, one element per lane, into odd-chunk padded slots
//     (conflict-free 16-byte x-line loads); odd n (P = 6, constant nu only): one copy per
//     brick row of 4 x-consecutive elements (an element is not a multiple of 16 bytes).
#pragma once

#ifndef DG_V6_EXP
#define DG_V6_EXP 0  // development bound experiments: 1 = no x/y traces, 2 = consumers skip the passes
#endif

#include "apply5.cuh"

namespace dg {
namespace v6 {
#ifdef DG_V5_DEBUG
using v5::g_dbg;
#endif

using v5::eo;
using v5::fence_proxy_async;
using v5::mbar_arrive;
using v5::mbar_arrive_expect_tx;
using v5::mbar_expect_tx;
using v5::mbar_init;
using v5::mbar_wait;
using v5::named_sync;
using v5::rdot;
using v5::tma_load;

#ifndef DG_V6_BY6
#define DG_V6_BY6 4  // brick rows along y at P = 6
#endif
#ifndef DG_V6_REGCAP
#define DG_V6_REGCAP 80  // register cap per thread
#endif
// brick rows along y (the host's divisibility check uses the same function)
__host__ __device__ constexpr int v6_by(int P) { return P == 7 ? 2 : (P == 6 ? DG_V6_BY6 : 4); }

// y-pass line order at n = 7 (dense row-TMA slots): a y-pass lane (l_y, line (ta, tb)) hits bank pair
// 4 l_y + ta + tb + const (mod 16), so a warp is conflict-free when its 8 lines hold two of every
// class of (ta + tb) mod 4 -- the lines taken round-robin over the four classes (any 8 consecutive
// entries qualify).  Consecutive lines gave 490 wavefronts per field pass of a brick, this order 364
// (ideal 343).
static __constant__ unsigned char c_yperm7[49] = {0,  1,  2,  3,  4,  5,  6,  9,  10, 7,  8,  13, 16, 11, 12, 15, 20,
                                           17, 14, 19, 22, 23, 18, 21, 26, 27, 24, 25, 28, 29, 30, 31, 32, 33,
                                           34, 37, 38, 35, 36, 41, 44, 39, 40, 43, 48, 45, 42, 47, 46};

template <int P_, bool VARNU_, int MODE_>
struct KC6 {
    static constexpr int P = P_;
    static constexpr bool VARNU = VARNU_;
    static constexpr int MODE = MODE_;
    static constexpr int n = P + 1;
    static constexpr int NN = n * n;
    static constexpr int NPE = n * n * n;
    // brick: 4 x 4 x 1 elements (n = 8: 4 x 2 x 1, the shared-memory budget; n = 7: DG_V6_BY6)
    static constexpr int BX = 4, BY = v6_by(P), BE = BX * BY;
    // odd n (P = 6, constant nu): an element is not a multiple of 16 bytes, so the TMA copies
    // whole brick rows (4 x-consecutive elements, contiguous in HBM and in shared memory)
    static constexpr bool ROWTMA = (NPE % 2) != 0;
    static_assert(!(ROWTMA && VARNU_), "odd n: constant nu only");
#ifndef DG_V6_SE228
#define DG_V6_SE228 1
#endif
#ifndef DG_V6_SE514
#define DG_V6_SE514 1
#endif
    // element slot (doubles); n = 6: SE = 228 == NN (mod 16) keeps the z-pass lines (stride NN,
    // consecutive lanes crossing slot boundaries) and the x-line LDS.128 loads conflict-free
    // n = 8: SE = 514 (== 2 mod 4) with rows 4 SE apart keeps all three passes conflict-free (bank
    // model validated against ncu on c5); SE = 516 with rows 4 mod 16 apart cost 2 wavefronts per
    // quarter-warp LDS.128 in the x pass and 4 instead of 2 per request in the y pass
    static constexpr int SE = ROWTMA ? NPE : (n == 6 && DG_V6_SE228) ? 228 : (n == 8 && DG_V6_SE514) ? 514 : ((NPE + 1) / 2) * 2 + 4;
#ifndef DG_V6_PITCH
#define DG_V6_PITCH 0  // development: measured 0.913 vs 0.444 ms on c5 (192 bulk copies of 288 bytes per brick)
#endif
    // n = 6: the slot's 12 padding doubles are spread over its z planes (plane pitch 38, SE = 6 * 38)
    // and the brick rows sit 8 (mod 16) doubles apart: a y-pass request (4 rows x 8 consecutive
    // lines, line offsets == L mod 16) then touches every bank pair exactly twice -- with the
    // dense planes (pitch 36 == 4 mod 16, rows 4 mod 16 apart) it needed 3 wavefronts instead of
    // 2 (ncu: 4.7 M of 60 M shared-memory wavefronts on c5).  The x-pass LDS.128 quarter-warps and
    // the z-pass 16-lane runs stay conflict-free; the TMA warp copies plane by plane (288 bytes).
    static constexpr bool PITCH = n == 6 && !ROWTMA && DG_V6_SE228 && DG_V6_PITCH;
    static constexpr int NNS = PITCH ? 38 : NN;                  // z-plane pitch inside a slot
    static constexpr int SY0 = ROWTMA ? 4 * SE : (PITCH ? 4 * SE + 8 : (n == 8 && DG_V6_SE514) ? 4 * SE : 4 * SE + 4);
    static constexpr int SY = ROWTMA ? SY0 + ((4 - SY0 % 16) + 16) % 16 : SY0;  // row stride (== 4 mod 16)
    static constexpr int NCL = BE * NN;                          // consumer lines per pass
    // consumer warps, warpgroup-aligned (18 of 20 busy at P = 5; measured: 18 consumer + 6 producer
    // warps 0.573 ms, 18 + 5 0.605 ms, 20 + 4 0.520 ms on c5)
    static constexpr int NCW = ROWTMA ? (NCL + 31) / 32 : ((NCL + 31) / 32 + 3) / 4 * 4;
    static constexpr int NC = NCW * 32;
    // producer: one TMA warp and NTW trace warps (n = 7: 25 consumer + 1 + 6 = 32 warps at 64 registers)
    static constexpr int NTW = (ROWTMA || n == 8) ? 6 : 3;
    static constexpr int NP = 32 * (1 + NTW);
    static constexpr int NT = NC + NP;
    static constexpr int NV = VARNU ? 3 : 2;                     // trace values: u, s (, nu)
    // brick-face lines per side: x faces BY rows of n^2 lines, y faces BX columns
    static constexpr int LRX = BY * NN, LRY = BX * NN;
    static constexpr int NTASK = 2 * (LRX + LRY);                 // x/y trace lines per brick
    static constexpr int TRXY = NV * NTASK;                      // x/y trace table per slot: [d][side][c][LR_d]
    template <int D>
    __host__ __device__ static constexpr int lr() { return D == 0 ? LRX : LRY; }
    template <int D>
    __host__ __device__ static constexpr int troff() { return D == 0 ? 0 : 2 * NV * LRX; }
    // trace threads: producer warps 1..NTW (the TMA warp joining them delayed its next copies:
    // measured 0.677 vs 0.516 ms in round 2)
    static constexpr int NPT = NP - 32;
    static constexpr int KT = (NTASK + NPT - 1) / NPT;          // producer x/y tasks per thread
    static constexpr int BRK = BY * SY;
    static constexpr int OFF_U = 0;
    static constexpr int OFF_NU = OFF_U + 2 * BRK;
    static constexpr int OFF_ACC = OFF_NU + (VARNU ? 2 * BRK : 0);
#ifndef DG_V6_ACC2
#define DG_V6_ACC2 0
#endif
    // development: two accumulator tiles (even n) let brick k+1's x pass start while brick k's
    // z pass finishes (one named barrier less per brick; then only two trace-table slots fit):
    // measured unchanged on c5 (0.449 ms), so one tile and three trace slots
    static constexpr int NACC = (DG_V6_ACC2 && !ROWTMA) ? 2 : 1;
    static constexpr int OFF_TR = OFF_ACC + NACC * BRK;          // [NTR][d][side][c][LR]
    static constexpr int NTR = NACC == 2 ? 2 : 3;                // trace-table slots (traces run ahead)
    static constexpr int OFF_ZO = OFF_TR + NTR * TRXY;           // parked z-pass outputs [n][NCL]
    static constexpr int OFF_RED = OFF_ZO + n * NCL;
    static constexpr int OFF_BAR = OFF_RED + 64;
    static constexpr int OFF_W = OFF_BAR + 10;         // full_uv[2] empty_uv[2] full_tr[3] empty_tr[3]
    static constexpr int OFF_PERM = OFF_W + n;         // n = 7: the y-pass line order (49 bytes)
    static constexpr int SMEM_DOUBLES = OFF_PERM + (ROWTMA ? 8 : 0);  // GLL weights (per-lane indexed reads)
    static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
    static constexpr int REG_C = 65536 / NT / 8 * 8 > DG_V6_REGCAP ? DG_V6_REGCAP : 65536 / NT / 8 * 8;  // launch registers
};

// consumer z-line carry (the same thread owns the same z line in every brick of a column)
struct ZC6 {
    bool held = false;
    double *po = nullptr;
    double u, gP, nu, s;  // top node: u, reference derivative, nu (VARNU: nu~), flux s (VARNU: s~)
};

// ---------------------------------------------------------------------------
// consumer x / y pass: one element line per thread, 4 lanes per brick row
// ---------------------------------------------------------------------------
template <class K, int D, bool FIRST>
__device__ __forceinline__ void cpass_xy(const ApplyParams &a, const DevTab &T, const double *su, double *snu,
                                         double *sacc, const double *tr, int t, const double *sw)
{
    constexpr int P = K::P, n = K::n, NN = K::NN, NNS = K::NNS, LR = K::template lr<D>(), NV = K::NV, SE = K::SE;
    constexpr int SSD = D == 0 ? 1 : n;
    constexpr int BD = D == 0 ? K::BX : K::BY;  // elements along D in a brick row (adjacent lanes)
    if ((t & ~31) >= K::NCL) return;  // fully idle warp (warp-uniform: no shuffle partners lost)
    const bool act = t < K::NCL;
    const int tt = act ? t : 0;
    const int l = tt % BD;               // position along D in the brick row
    int L = tt / BD;                     // row index
    const int ce = L / NN;
    int tn = L - ce * NN;
#ifndef DG_V6_XPERM
#define DG_V6_XPERM 1
#endif
    if (DG_V6_XPERM && D == 0 && K::ROWTMA && n == 7) {
        // dense row-TMA slots (slot stride n^3 == 7, line stride 7): lane (l_x, line t) of the x pass
        // hits bank pair 7 (l_x + t) mod 16, so 4 elements x 8 consecutive lines need 4 wavefronts
        // where 2 suffice.  Lines taken in class-major order of t mod 4 (0, 4, .., 48, 1, 5, ..) put
        // lines 4 apart on a warp: l_x + 4 j covers every residue mod 16 twice (ncu: 13.1 M
        // shared-memory wavefronts against 7.6 M ideal on the config-4 pressure apply before)
        const int c = tn < 13 ? 0 : (tn - 13) / 12 + 1;
        tn = 4 * (tn - (c ? 13 + 12 * (c - 1) : 0)) + c;
        L = ce * NN + tn;
    }
    if (DG_V6_XPERM && D == 1 && K::ROWTMA && n == 7) {  // y pass: round-robin class order (c_yperm7)
        tn = reinterpret_cast<const unsigned char *>(sw + n)[tn];
        L = ce * NN + tn;
    }
    const int ta = tn % n, tb = tn / n;
    const int lx = D == 0 ? l : ce, ly = D == 0 ? ce : l;
    const int base = lx * SE + ly * K::SY + (D == 0 ? ta * n + tb * NNS : ta + tb * NNS);
    const Geom &g = a.g;
    const double sd = g.sd[D];

    double v[n], nv[n];
    if (D == 0 && (n % 2) == 0) {
        // VARNU: the x pass folds the GLL weights into the staged viscosity, nu~ = nu w_i w_j w_k
        // (V6Fold), in registers and in place for the y and z passes (each x line has one owner)
        const double wjk = K::VARNU ? sw[ta] * sw[tb] : 0.0;
#pragma unroll
        for (int i = 0; i < n; i += 2) {
            const double2 x = *reinterpret_cast<const double2 *>(su + base + i);
            v[i] = x.x;
            v[i + 1] = x.y;
            if (K::VARNU) {
                double2 y = *reinterpret_cast<const double2 *>(snu + base + i);
                y.x *= T.w[i] * wjk;
                y.y *= T.w[i + 1] * wjk;
                nv[i] = y.x;
                nv[i + 1] = y.y;
                if (act) *reinterpret_cast<double2 *>(snu + base + i) = y;
            }
        }
        // generic-proxy writes into a TMA-refilled slot: order them before later async-proxy writes
        if (K::VARNU) fence_proxy_async();
    } else {
#pragma unroll
        for (int i = 0; i < n; ++i) {
            v[i] = su[base + i * SSD];
            nv[i] = K::VARNU ? snu[base + i * SSD] : a.nu_const;
        }
    }
    // brick-face traces (only the end lanes use them)
    const double *trd = tr + K::template troff<D>();
    double uL = 0.0, sL = 0.0, nuL = a.nu_const, uR = 0.0, sR = 0.0, nuR = a.nu_const;
    if (act && l == 0) {
        uL = trd[L];
        sL = trd[LR + L];
        if (K::VARNU) nuL = trd[2 * LR + L];
    }
    if (act && l == BD - 1) {
        uR = trd[NV * LR + L];
        sR = trd[(NV + 1) * LR + L];
        if (K::VARNU) nuR = trd[(NV + 2) * LR + L];
    }
    double r[n];
    if (K::VARNU) {
        // weight-folded form (V6Fold): nv = nu~ = nu w_i w_j w_k (staged by the producers), so
        // W (w_k (2/h) nu_k g_k) = C nu~_k g_k with g = D v on the reference line, the own flux
        // s~ = nu~ g at the line ends, and the whole line result is already W-weighted
        const V6Fold &F = a.f6;
        double gg[n], tv[n];
        eo<P, true>(T.eD, v, gg);
#pragma unroll
        for (int k = 0; k < n; ++k) tv[k] = nv[k] * gg[k];
        const double s0 = tv[0], sP = tv[P];
        // in-brick faces: the left neighbour's right end arrives from lane - 1, the right
        // neighbour's left end from lane + 1
        const double xu = __shfl_up_sync(0xffffffffu, v[P], 1), xs = __shfl_up_sync(0xffffffffu, sP, 1),
                     xn = __shfl_up_sync(0xffffffffu, nv[P], 1);
        const double yu = __shfl_down_sync(0xffffffffu, v[0], 1), ys = __shfl_down_sync(0xffffffffu, s0, 1),
                     yn = __shfl_down_sync(0xffffffffu, nv[0], 1);
        if (l != 0) {
            uL = xu;
            sL = xs;
            nuL = xn;
        }
        if (l != BD - 1) {
            uR = yu;
            sR = ys;
            nuR = yn;
        }
        const double JL = uL - v[0], JR = v[P] - uR;
        const double FL = fma(F.kF[D] * (nuL + nv[0]), JL, -F.kS[D] * (sL + s0));
        const double FR = fma(F.kF[D] * (nv[P] + nuR), JR, -F.kS[D] * (sP + sR));
        tv[P] = fma(-F.kL * nv[P], JR, tv[P]);
        tv[0] = fma(-F.kL * nv[0], JL, tv[0]);
        eo<P, true>(F.eE[D], tv, r);
        r[P] += FR;
        r[0] -= FL;
        if (!act) return;
        double *pa = sacc + base;
        if (D == 0 && FIRST && (n % 2) == 0 && DG_V6_SE228) {  // contiguous x line: 16-byte stores
#pragma unroll
            for (int i = 0; i < n; i += 2) *reinterpret_cast<double2 *>(pa + i) = make_double2(r[i], r[i + 1]);
            return;
        }
#pragma unroll
        for (int i = 0; i < n; ++i) pa[i * SSD] = FIRST ? r[i] : pa[i * SSD] + r[i];
        return;
    } else {
        const double c = a.nu_const * sd, ck = c * (0.5 * (P + 1) * (P + 1));
        const double d0 = rdot<P>(T, 0, v), dP = rdot<P>(T, P, v);
        const double xu = __shfl_up_sync(0xffffffffu, v[P], 1), xs = __shfl_up_sync(0xffffffffu, c * dP, 1);
        const double yu = __shfl_down_sync(0xffffffffu, v[0], 1), ys = __shfl_down_sync(0xffffffffu, c * d0, 1);
        if (l != 0) {
            uL = xu;
            sL = xs;
        }
        if (l != BD - 1) {
            uR = yu;
            sR = ys;
        }
        double kv[n];
        eo<P, false>(T.eK, v, kv);
        const double aR = 0.5 * c * uR, aL = -0.5 * c * uL;
#pragma unroll
        for (int i = 0; i < n; ++i) r[i] = fma(c, kv[i], fma(aR, T.D[P][i], aL * T.D[0][i]));
        r[P] += fma(-ck, uR, -0.5 * sR);
        r[0] += fma(-ck, uL, 0.5 * sL);
    }
    if (!act) return;
    const double W = sw[ta] * sw[tb] * g.wfac[D];
    double *pa = sacc + base;
    if (D == 0 && FIRST && (n % 2) == 0) {  // contiguous x line: 16-byte stores (a quarter-warp per wavefront)
#pragma unroll
        for (int i = 0; i < n; i += 2) *reinterpret_cast<double2 *>(pa + i) = make_double2(W * r[i], W * r[i + 1]);
        return;
    }
#pragma unroll
    for (int i = 0; i < n; ++i) pa[i * SSD] = FIRST ? W * r[i] : fma(W, r[i], pa[i * SSD]);
}

// ---------------------------------------------------------------------------
// consumer z pass (last): carry, deferred top face, output
// ---------------------------------------------------------------------------
// release the previous brick's parked output: its top-face terms dr_i = c D_{P,i} + [i == P] f0
// with the face shared with the current bottom (VARNU: c and f0 arrive W-weighted)
template <class K>
__device__ __forceinline__ void zrelease(const DevTab &T, double c, double f0, double W, const double *zo, int t,
                                         ZC6 &zc, double &epi0, double &epi1)
{
    constexpr int P = K::P, n = K::n, NN = K::NN, NCL = K::NCL;
    const double Wr = K::VARNU ? 1.0 : W;
    double s1 = 0.0;
#pragma unroll
    for (int i = 0; i < n; ++i) {
        const double d = K::VARNU ? fma(c, T.D[P][i], i == P ? f0 : 0.0) : W * fma(c, T.D[P][i], i == P ? f0 : 0.0);
        zc.po[i * NN] = zo[i * NCL + t] + d;
        s1 += d;
    }
    if (K::MODE >= 1) {
        epi0 = fma(Wr, fma(c, zc.gP, f0 * zc.u), epi0);
        if (K::MODE != 3) epi1 += s1;
    }
    zc.held = false;
}

template <class K>
__device__ __forceinline__ void cpass_z(const ApplyParams &a, const DevTab &T, const double *su, const double *snu,
                                        const double *sacc, double *zo, long long eb, int t, ZC6 &zc, double &epi0,
                                        double &epi1, const double *sw)
{
    constexpr int P = K::P, n = K::n, NN = K::NN, NNS = K::NNS, NPE = K::NPE, NCL = K::NCL, SE = K::SE;
    if (t >= NCL) return;
    const Geom &g = a.g;
    const int slot = t / NN, tn = t - slot * NN;
    const int ta = tn % n, tb = tn / n;
    const int base = (slot & 3) * SE + (slot >> 2) * K::SY + ta + tb * n;
    const double W = sw[ta] * sw[tb] * g.wfac[2];
    const double sd = g.sd[2];
    double v[n], nv[n];
#pragma unroll
    for (int i = 0; i < n; ++i) {
        v[i] = su[base + i * NNS];
        nv[i] = K::VARNU ? snu[base + i * NNS] : a.nu_const;
    }
    // bottom face: the carry of the brick below (or of the segment's bottom halo brick)
    const double uL = zc.u, nuL = K::VARNU ? zc.nu : a.nu_const, sL = zc.s;
    double r[n], gP, sP;
    if (K::VARNU) {
        // weight-folded form (see cpass_xy): results are W-weighted, the parked output and
        // its release too
        const V6Fold &F = a.f6;
        double gg[n], tv[n];
        eo<P, true>(T.eD, v, gg);
#pragma unroll
        for (int k = 0; k < n; ++k) tv[k] = nv[k] * gg[k];
        const double s0 = tv[0];
        sP = tv[P];
        const double JL = uL - v[0];
        const double FL = fma(F.kF[2] * (nuL + nv[0]), JL, -F.kS[2] * (sL + s0));
        if (zc.held) zrelease<K>(T, -F.kCL[2] * zc.nu * JL, FL, W, zo, t, zc, epi0, epi1);
        tv[0] = fma(-F.kL * nv[0], JL, tv[0]);
        eo<P, true>(F.eE[2], tv, r);
        r[0] -= FL;
        gP = gg[P];
    } else {
        const double c = a.nu_const * sd, ck = c * (0.5 * (P + 1) * (P + 1));
        const double d0 = rdot<P>(T, 0, v), dP = rdot<P>(T, P, v);
        if (zc.held) zrelease<K>(T, 0.5 * c * v[0], fma(-ck, v[0], -0.5 * c * d0), W, zo, t, zc, epi0, epi1);
        double kv[n];
        eo<P, false>(T.eK, v, kv);
        const double aL = -0.5 * c * uL;
#pragma unroll
        for (int i = 0; i < n; ++i) r[i] = fma(c, kv[i], aL * T.D[0][i]);
        r[0] += fma(-ck, uL, 0.5 * sL);
        gP = dP;
        sP = c * dP;
    }
    // output of element (slot % 4, slot / 4) of the brick layer: parked without its top-face
    // terms until the brick above (or the top halo brick) supplies the other side
    const long long ge = eb + (slot & 3) + (long long)g.Nl[0] * (slot >> 2);
    const double lw = a.lam * W * (0.5 * g.h[2]);
    const double *pa = sacc + base;
#pragma unroll
    for (int i = 0; i < n; ++i) {
        const double o = fma(lw * T.w[i], v[i], K::VARNU ? r[i] + pa[i * NNS] : fma(W, r[i], pa[i * NNS]));
        zo[i * NCL + t] = o;
        if (K::MODE >= 1) {
            epi0 = fma(v[i], o, epi0);
            if (K::MODE != 3) epi1 += o;
        }
    }
    zc.held = true;
    zc.po = a.out + ge * NPE + ta + tb * n;
    zc.u = v[P];
    zc.gP = gP;
    zc.nu = nv[P];
    zc.s = sP;
}

// the halo bricks of a column segment (the layer below its first brick, TOP: above its last):
// only their face lines adjacent to the segment are used -- the bottom halo sets the z carry,
// the top halo releases the parked outputs of the last brick.  The brick was staged like any
// other (TMA, local or periodic layer); at a slab boundary of a halo mesh the face traces
// received from the neighbouring rank are read instead (su == nullptr).
template <class K, bool TOP>
__device__ __forceinline__ void czhalo(const ApplyParams &a, const DevTab &T, const double *su, const double *snu,
                                       const double *zo, const int (&e0)[3], int cz, int t, ZC6 &zc, double &epi0,
                                       double &epi1, const double *sw)
{
    constexpr int P = K::P, n = K::n, NN = K::NN, NNS = K::NNS, NCL = K::NCL, SE = K::SE;
    if (t >= NCL) return;
    const Geom &g = a.g;
    const int slot = t / NN, tn = t - slot * NN;
    const int ta = tn % n, tb = tn / n;
    const double W = sw[ta] * sw[tb] * g.wfac[2];
    const double sd = g.sd[2];
    constexpr int fi = TOP ? 0 : P;  // the face node of the halo element
    double uf, nuf, sf, gf = 0.0;    // face u, nu (VARNU: nu~), flux (VARNU: s~), reference derivative
    if (su) {
        const int base = (slot & 3) * SE + (slot >> 2) * K::SY + ta + tb * n;
        double v[n];
#pragma unroll
        for (int i = 0; i < n; ++i) v[i] = su[base + i * NNS];
        gf = rdot<P>(T, fi, v);
        uf = v[fi];
        nuf = K::VARNU ? snu[base + fi * NNS] * (sw[ta] * sw[tb] * T.w[fi]) : a.nu_const;
        sf = K::VARNU ? nuf * gf : a.nu_const * sd * gf;
    } else {
        const double *trh = halo_trace(g, a.halo, cz);
        const long long F = halo_F(g, n), f = halo_f(g, n, e0[0] + (slot & 3), e0[1] + (slot >> 2), ta + tb * n);
        uf = __ldg(trh + f);
        const double hs = __ldg(trh + F + f);  // physical s = nu d u / d x_S
        if (K::VARNU) {  // weight-folded: nu~ = nu w_a w_b w_0, s~ = s w_a w_b w_0 h_z / 2
            const double wab = sw[ta] * sw[tb] * sw[0];
            nuf = __ldg(trh + 2 * F + f) * wab;
            sf = hs * wab * (0.5 * g.h[2]);
        } else {
            nuf = a.nu_const;
            sf = hs;
        }
    }
    if (!TOP) {
        zc.held = false;
        zc.u = uf;
        zc.gP = gf;
        zc.nu = nuf;
        zc.s = sf;
        return;
    }
    if (!zc.held) return;
    if (K::VARNU) {
        const V6Fold &F = a.f6;
        const double JL = zc.u - uf;
        const double FL = fma(F.kF[2] * (zc.nu + nuf), JL, -F.kS[2] * (zc.s + sf));
        zrelease<K>(T, -F.kCL[2] * zc.nu * JL, FL, W, zo, t, zc, epi0, epi1);
    } else {
        const double c = a.nu_const * sd, ck = c * (0.5 * (P + 1) * (P + 1));
        zrelease<K>(T, 0.5 * c * uf, fma(-ck, uf, -0.5 * sf), W, zo, t, zc, epi0, epi1);
    }
}

// ---------------------------------------------------------------------------
// producer: x and y brick-face traces, one memory round (KT lines per thread in flight)
// ---------------------------------------------------------------------------
template <class K, int K0, int K1>
__device__ __forceinline__ void ptraces_xy(const ApplyParams &a, const DevTab &T, double *tr, const int (&e0)[3],
                                           long long eb, int ptid, double beta, const double *sw)
{
    constexpr int P = K::P, n = K::n, NN = K::NN, NPE = K::NPE, LRX = K::LRX, LRY = K::LRY, NV = K::NV, KT = K1 - K0;
    const Geom &g = a.g;
    const long long lay = (long long)g.Nl[0] * g.Nl[1];
    // task tk: x faces [0, 2 LRX) (side-major), then y faces [2 LRX, 2 LRX + 2 LRY)
    auto decode = [&](int tk, int &D, int &side, int &L) {
        D = tk >= 2 * LRX;
        const int r = D ? tk - 2 * LRX : tk, lr = D ? LRY : LRX;
        side = r / lr;
        L = r - side * lr;
    };
    const double *fu = K::MODE == 1 ? a.pro.z : a.u;
    // every neighbour line is read forward from its node 0 (x lines: contiguous, n even ->
    // 16-byte vector loads); the face node is node P of the left / node 0 of the right neighbour
    double v[KT][n], nuf[KT];
    int meta[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int tk = ptid + (K0 + k) * K::NPT;
        meta[k] = -1;
        if (tk >= K::NTASK) continue;
        int D, side, L;
        decode(tk, D, side, L);
        const int ce = L / NN, tn = L - ce * NN;
        const int ta = tn % n, tb = tn / n;
        int cx, cy, off, step;
        if (D == 0) {
            cx = side ? e0[0] + K::BX : e0[0] - 1;
            cx = cx < 0 ? cx + g.Nl[0] : (cx >= g.Nl[0] ? cx - g.Nl[0] : cx);
            cy = e0[1] + ce;
            off = ta * n + tb * NN;
            step = 1;
        } else {
            cy = side ? e0[1] + K::BY : e0[1] - 1;
            cy = cy < 0 ? cy + g.Nl[1] : (cy >= g.Nl[1] ? cy - g.Nl[1] : cy);
            cx = e0[0] + ce;
            off = ta + tb * NN;
            step = n;
        }
        const long long o = (cx + (long long)g.Nl[0] * cy + lay * e0[2]) * NPE + off;
        if (K::MODE == 1) {
#pragma unroll
            for (int i = 0; i < n; ++i) v[k][i] = fma(beta, __ldg(a.pro.p_old + o + i * step), __ldg(fu + o + i * step));
        } else if ((n % 2) == 0 && D == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 2) {
                const double2 x = __ldg(reinterpret_cast<const double2 *>(fu + o + i));
                v[k][i] = x.x;
                v[k][i + 1] = x.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < n; ++i) v[k][i] = __ldg(fu + o + i * step);
        }
        nuf[k] = K::VARNU ? __ldg(a.nu + o + (side ? 0 : P * step)) : a.nu_const;
        meta[k] = tk;
    }
    (void)eb;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
        const int tk = meta[k];
        if (tk < 0) continue;
        int D, side, L;
        decode(tk, D, side, L);
        const int LR = D ? LRY : LRX;
        // the neighbour's face node and its derivative along +d there (reference coordinates)
        const double uf = side ? v[k][0] : v[k][P];
        const double dd = side ? rdot<P>(T, 0, v[k]) : rdot<P>(T, P, v[k]);
        double *trd = tr + (D ? 2 * NV * LRX : 0) + side * NV * LR;
        trd[L] = uf;
        if (K::VARNU) {  // weight-folded: nu~ = nu w_a w_b w_0, s~ = nu~ (D v)_face (reference derivative)
            const int tn = L % NN;
            const double nw = nuf[k] * (sw[tn % n] * sw[tn / n] * sw[0]);
            trd[LR + L] = nw * dd;
            trd[2 * LR + L] = nw;
        } else {
            trd[LR + L] = nuf[k] * g.sd[D] * dd;
        }
    }
}

template <int P, bool VARNU, int MODE>
__global__ void __launch_bounds__((KC6<P, VARNU, MODE>::NT)) __maxnreg__((KC6<P, VARNU, MODE>::REG_C))
    k_apply6(const __grid_constant__ ApplyParams a)
{
    using K = KC6<P, VARNU, MODE>;
    static_assert(MODE != 1, "v6 has no fused-PCG (MODE 1) variant");
    constexpr int NPE = K::NPE, SE = K::SE, BRK = K::BRK, NC = K::NC, NCL = K::NCL, NTR = K::NTR;
    const Geom &g = a.g;
    const DevTab &T = c_tab[P];
    extern __shared__ __align__(16) double sm[];
    // the TMA warp runs on two u / nu slots, the trace warps on NTR trace-table slots: the
    // brick-face traces are formed up to NTR - 1 bricks ahead of the consumers
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + K::OFF_BAR);
    uint64_t *full_uv = bar, *empty_uv = bar + 2, *full_tr = bar + 4, *empty_tr = bar + 4 + NTR;
    double *sw = sm + K::OFF_W;
    const int tid = threadIdx.x;
    if (tid < K::n) sw[tid] = T.w[tid];
    if (K::ROWTMA && K::n == 7 && tid < K::NN) reinterpret_cast<unsigned char *>(sw + K::n)[tid] = c_yperm7[tid];
    if (MODE >= 1 && *a.pro.done) return;  // PCG converged: nothing to do
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full_uv[b], 1);
            mbar_init(&empty_uv[b], NC);
        }
        for (int b = 0; b < NTR; ++b) {
            mbar_init(&full_tr[b], K::NPT);
            mbar_init(&empty_tr[b], NC);
        }
        fence_proxy_async();
    }
    __syncthreads();

    const int nb0 = g.Nl[0] / K::BX, nb1 = g.Nl[1] / K::BY;
    const int ncols = nb0 * nb1;
    const int nunits = ncols * a.nseg;
    const int seglen = a.seglen;
    const long long s1 = g.Nl[0], s2 = (long long)g.Nl[0] * g.Nl[1];
    const bool hmesh = a.halo.tr_lo != nullptr || a.halo.tr_hi != nullptr;

    if (tid >= NC + 32) {
        // ------------------------------ trace warps ------------------------------
        const int pt = tid - NC - 32;
        int it = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int col = u % ncols, zs = u / ncols;
            // bricks j = -1 and j = seglen are the segment's halo bricks (z faces of its ends)
            int e0[3] = {(col % nb0) * K::BX, (col / nb0) * K::BY, a.zlo + zs * seglen - 1};
            for (int j = -1; j <= seglen; ++j, ++it, ++e0[2]) {
                const int slot = it % NTR;
                V5_T0(tw);
                if (it >= NTR) mbar_wait(&empty_tr[slot], ((it / NTR) - 1) & 1);
                if (pt == 0) V5_ACC(2, tw);
                V5_T0(tx);
                if (j >= 0 && j < seglen && (DG_V6_EXP & 1) == 0) {
                    double *tr = sm + K::OFF_TR + slot * K::TRXY;
                    constexpr int R = 3;  // lines in flight per thread (register budget)
                    ptraces_xy<K, 0, (K::KT < R ? K::KT : R)>(a, T, tr, e0, 0, pt, 0.0, sw);
                    if constexpr (K::KT > R) ptraces_xy<K, R, (K::KT < 2 * R ? K::KT : 2 * R)>(a, T, tr, e0, 0, pt, 0.0, sw);
                    if constexpr (K::KT > 2 * R) ptraces_xy<K, 2 * R, K::KT>(a, T, tr, e0, 0, pt, 0.0, sw);
                }
                if (pt == 0) V5_ACC(3, tx);
                mbar_arrive(&full_tr[slot]);
            }
        }
        return;
    }
    if (tid >= NC) {
        // ------------------------------- TMA warp -------------------------------
        const int lane = tid - NC;
        int it = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int col = u % ncols, zs = u / ncols;
            int e0[3] = {(col % nb0) * K::BX, (col / nb0) * K::BY, a.zlo + zs * seglen - 1};
            for (int j = -1; j <= seglen; ++j, ++it, ++e0[2]) {
                const int buf = it & 1;
                V5_T0(tw);
                if (it >= 2) mbar_wait(&empty_uv[buf], ((it >> 1) - 1) & 1);
                if (lane == 0) V5_ACC(4, tw);
                double *su = sm + K::OFF_U + buf * BRK;
                double *snu = sm + K::OFF_NU + buf * BRK;
                // halo layer outside the slab: periodic wrap on a plain mesh; on a halo mesh the
                // consumers read the received face traces instead (nothing staged)
                int zl = e0[2];
                bool staged = true;
                if (zl < 0 || zl >= g.Nl[2]) {
                    if (hmesh) staged = false;
                    else zl = zl < 0 ? zl + g.Nl[2] : zl - g.Nl[2];
                }
                const long long eb = e0[0] + s1 * e0[1] + s2 * zl;
                constexpr unsigned EB = NPE * 8u;
                constexpr unsigned BE = K::BE;
                if (lane == 0) {
                    if (staged) mbar_arrive_expect_tx(&full_uv[buf], BE * EB + (VARNU ? BE * EB : 0u));
                    else mbar_arrive(&full_uv[buf]);
                }
                __syncwarp();
                if (staged) {
                    if (K::ROWTMA) {  // brick row r = lane: elements (e0x .. e0x + 3, e0y + r)
                        if (lane < K::BY) tma_load(su + lane * K::SY, a.u + (eb + s1 * lane) * NPE, 4 * EB, &full_uv[buf]);
                    } else {  // one element per lane into its padded slot (u lanes 0-15, nu 16-31)
                        const int el = lane & 15;
                        const long long ge = eb + (el & 3) + s1 * (el >> 2);
                        const int so = (el & 3) * SE + (el >> 2) * K::SY;
                        if (K::PITCH) {  // plane by plane into the pitched slot
                            const bool isu = lane < (int)BE, isnu = lane >= 16 && el < (int)BE && VARNU;
                            if (isu || isnu) {
                                double *dst = (isu ? su : snu) + so;
                                const double *src = (isu ? a.u : a.nu) + ge * NPE;
#pragma unroll
                                for (int k = 0; k < K::n; ++k)
                                    tma_load(dst + k * K::NNS, src + k * K::NN, K::NN * 8u, &full_uv[buf]);
                            }
                        } else {
                            if (lane < (int)BE) tma_load(su + so, a.u + ge * NPE, EB, &full_uv[buf]);
                            if (lane >= 16 && el < (int)BE && VARNU) tma_load(snu + so, a.nu + ge * NPE, EB, &full_uv[buf]);
                        }
                    }
                }
                if (j >= 0 && j + 1 < seglen) {
                    // L2 prefetch of the x/y brick-face neighbour elements of the next brick
                    // (their trace loads then hit L2; measured on c5: 0.517 vs 0.525 ms;
                    // two layers ahead 0.519, four 0.54, eight 0.60)
                    // lanes 0-15 u, 16-31 nu: neighbour nb < 2 BY on the x sides, then 2 BX on the y sides
                    const int nb = lane & 15;
                    int cx, cy;
                    if (nb < 2 * K::BY) {
                        const int side = nb / K::BY, r = nb % K::BY;
                        cx = side ? e0[0] + K::BX : e0[0] - 1;
                        cx = cx < 0 ? cx + g.Nl[0] : (cx >= g.Nl[0] ? cx - g.Nl[0] : cx);
                        cy = e0[1] + r;
                    } else {
                        const int q = nb - 2 * K::BY, side = q / K::BX, r = q % K::BX;
                        cy = side ? e0[1] + K::BY : e0[1] - 1;
                        cy = cy < 0 ? cy + g.Nl[1] : (cy >= g.Nl[1] ? cy - g.Nl[1] : cy);
                        cx = e0[0] + r;
                    }
                    const long long pe = cx + s1 * cy + s2 * (e0[2] + 1);
                    if (nb < 2 * (K::BX + K::BY)) {
                        if (lane < 16) v5::l2_prefetch(a.u + pe * NPE, EB);
                        else if (VARNU) v5::l2_prefetch(a.nu + pe * NPE, EB);
                    }
                }
            }
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    double epi0 = 0.0, epi1 = 0.0;
    int it = 0;
    ZC6 zc;
    double *zo = sm + K::OFF_ZO;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int col = u % ncols, zs = u / ncols;
        int e0[3] = {(col % nb0) * K::BX, (col / nb0) * K::BY, a.zlo + zs * seglen - 1};
        for (int j = -1; j <= seglen; ++j, ++it, ++e0[2]) {
            const int buf = it & 1, slot = it % NTR;
            const double *su = sm + K::OFF_U + buf * BRK;
            double *snu = sm + K::OFF_NU + buf * BRK;
            const double *tr = sm + K::OFF_TR + slot * K::TRXY;
            double *sacc = sm + K::OFF_ACC + (K::NACC == 2 ? buf * BRK : 0);
            const long long eb = e0[0] + s1 * e0[1] + s2 * e0[2];
            V5_T0(tw);
            mbar_wait(&full_uv[buf], (it >> 1) & 1);
            mbar_wait(&full_tr[slot], (it / NTR) & 1);
            if (tid == 0) V5_ACC(0, tw);
            if (j < 0 || j == seglen) {  // halo brick: the segment's bottom carry / top release
                const bool staged = !((e0[2] < 0 || e0[2] >= g.Nl[2]) && hmesh);
                if (j < 0) czhalo<K, false>(a, T, staged ? su : nullptr, snu, zo, e0, e0[2], tid, zc, epi0, epi1, sw);
                else czhalo<K, true>(a, T, staged ? su : nullptr, snu, zo, e0, e0[2], tid, zc, epi0, epi1, sw);
                mbar_arrive(&empty_tr[slot]);
                mbar_arrive(&empty_uv[buf]);
                if (K::NACC == 1) named_sync(1, NC);  // ACC is rewritten by the next brick
                continue;
            }
            V5_T0(tp);
            if (DG_V6_EXP & 2) {
                mbar_arrive(&empty_tr[slot]);
                mbar_arrive(&empty_uv[buf]);
                continue;
            }
            cpass_xy<K, 0, true>(a, T, su, snu, sacc, tr, tid, sw);
            if (tid == 0) V5_ACC(6, tp);
            named_sync(1, NC);
            V5_T0(t1);
            cpass_xy<K, 1, false>(a, T, su, snu, sacc, tr, tid, sw);
            if (tid == 0) V5_ACC(7, t1);
            mbar_arrive(&empty_tr[slot]);  // the trace table is read by the x and y passes only
            named_sync(1, NC);
            V5_T0(t2);
            cpass_z<K>(a, T, su, snu, sacc, zo, eb, tid, zc, epi0, epi1, sw);
            if (tid == 0) V5_ACC(8, t2);
            mbar_arrive(&empty_uv[buf]);
            // single ACC: rewritten by the next brick's x pass (the parked outputs are
            // thread-private); two ACC tiles: the next x pass writes the other one
            if (K::NACC == 1) named_sync(1, NC);
            if (tid == 0) {
                V5_ACC(1, tp);
#ifdef DG_V5_DEBUG
                atomicAdd(&v5::g_dbg[5], 1ull);
#endif
            }
        }
    }
    if (MODE >= 1) {  // dot epilogue: block partials of u.out and sum(out)
        double *red = sm + K::OFF_RED;
        const int lane = tid & 31, wid = tid >> 5;
        epi0 = warp_sum(epi0);
        if (MODE != 3) epi1 = warp_sum(epi1);
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
    (void)NCL;
}

}  // namespace v6
}  // namespace dg
