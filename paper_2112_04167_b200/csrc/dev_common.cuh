// dev_common.cuh -- device-side helpers shared by the kernel translation units of
// libdgsip.so.  Each TU gets its own (internal-linkage) copy of the __constant__ tables
// and its own upload function.
#pragma once

#include <cuda_runtime.h>

#include "dg_internal.h"

// DG_PSET: bit mask of compiled polynomial degrees (default: all of 1..PMAX).  Development
// builds may restrict it to shorten compile time; dispatch of other degrees then fails
// with cudaErrorNotSupported (DG_EUNSUPPORTED at the C-ABI).
#ifndef DG_PSET
#define DG_PSET 0x7FE
#endif
#define DG_HAS_P(p) (((DG_PSET) >> (p)) & 1)

namespace dg {

// operator tables (apply / diag / vec TUs)
struct DevTab {
    double xi[NMAX];
    double w[NMAX];
    double D[NMAX][NMAX];
    double Kref[NMAX][NMAX];
    EOTab eD, eE, eK;
};

// convection tables (convect TU)
constexpr int HQMAX = QMAX / 2 + 1;  // even-odd half size of the Gauss rows
struct CvTab {
    double w[NMAX];
    double zq[QMAX];
    double wq[QMAX];
    double Bq[QMAX][NMAX];
    double Gq[QMAX][NMAX];
    // even-odd forms of the rectangular Gauss tables: Gauss points and GLL nodes are both
    // symmetric about 0, so B[Q-1-q][P-j] = B[q][j] and G[Q-1-q][P-j] = -G[q][j]; for q < Q/2 + 1,
    // j < n/2:  Xe[q][j] = (X[q][j] + X[q][P-j]) / 2,  Xo[q][j] = (X[q][j] - X[q][P-j]) / 2,
    // Xc[q] = X[q][P/2] (odd n).  Half the multiply-adds of X v and X^T f (convect.cuh eo_fwd / eo_acc).
    double Be[HQMAX][HMAX], Bo[HQMAX][HMAX], Bc[HQMAX];
    double Ge[HQMAX][HMAX], Go[HQMAX][HMAX], Gc[HQMAX];
};

inline void to_devtab(const Tab &t, DevTab *d)
{
    for (int i = 0; i < NMAX; ++i) {
        d->xi[i] = t.xi[i];
        d->w[i] = t.w[i];
        for (int j = 0; j < NMAX; ++j) {
            d->D[i][j] = t.D[i][j];
            d->Kref[i][j] = t.Kref[i][j];
        }
    }
    d->eD = t.eD;
    d->eE = t.eE;
    d->eK = t.eK;
}

inline void to_cvtab(const Tab &t, int P, CvTab *d)
{
    *d = CvTab{};
    for (int i = 0; i < NMAX; ++i) d->w[i] = t.w[i];
    for (int q = 0; q < QMAX; ++q) {
        d->zq[q] = t.zq[q];
        d->wq[q] = t.wq[q];
        for (int j = 0; j < NMAX; ++j) {
            d->Bq[q][j] = t.Bq[q][j];
            d->Gq[q][j] = t.Gq[q][j];
        }
    }
    const int n = P + 1, Q = t.Q;
    for (int q = 0; q <= Q / 2; ++q) {
        for (int j = 0; j < n / 2; ++j) {
            d->Be[q][j] = 0.5 * (t.Bq[q][j] + t.Bq[q][P - j]);
            d->Bo[q][j] = 0.5 * (t.Bq[q][j] - t.Bq[q][P - j]);
            d->Ge[q][j] = 0.5 * (t.Gq[q][j] + t.Gq[q][P - j]);
            d->Go[q][j] = 0.5 * (t.Gq[q][j] - t.Gq[q][P - j]);
        }
        d->Bc[q] = (n % 2) ? t.Bq[q][P / 2] : 0.0;
        d->Gc[q] = (n % 2) ? t.Gq[q][P / 2] : 0.0;
    }
}

#define DG_DEFINE_CONST_TABLES(fn_name)                                                     \
    static __constant__ DevTab c_tab[PMAX + 1];                                             \
    cudaError_t fn_name()                                                                   \
    {                                                                                       \
        static DevTab h[PMAX + 1];                                                          \
        for (int p = 1; p <= PMAX; ++p) to_devtab(host_tab(p), &h[p]);                      \
        return cudaMemcpyToSymbol(c_tab, h, sizeof(h));                                     \
    }

#define DG_DEFINE_CONV_TABLES(fn_name)                                                      \
    static __constant__ CvTab c_ctab[PMAX + 1];                                             \
    cudaError_t fn_name()                                                                   \
    {                                                                                       \
        static CvTab h[PMAX + 1];                                                           \
        for (int p = 1; p <= PMAX; ++p) to_cvtab(host_tab(p), p, &h[p]);                       \
        return cudaMemcpyToSymbol(c_ctab, h, sizeof(h));                                    \
    }

template <int DIM, int P>
struct Cfg {
    static constexpr int n = P + 1;
    static constexpr int PX = (n % 2 == 0) ? n + 1 : n;  // odd x-pitch in shared memory
    static constexpr int NPE = DIM == 3 ? n * n * n : n * n;
    static constexpr int SPE = DIM == 3 ? PX * n * n : PX * n;
    static constexpr int NT = DIM == 3 ? n * n : n;      // lines per element per direction
};

// local-slab element index; c[] already wrapped / in range
__device__ __forceinline__ long long elem_index(const Geom &g, int c0, int c1, int c2)
{
    return (long long)c0 + (long long)g.Nl[0] * ((long long)c1 + (long long)g.Nl[1] * c2);
}

// Face-trace halo (dg_internal.h Halo) of the slowest direction: is the neighbour at local
// slowest-direction coordinate cS outside the slab with a received trace, and where is it.
// Returns the trace array of that side (or nullptr: wrap / local element), f = face node index.
__device__ __forceinline__ const double *halo_trace(const Geom &g, const Halo &h, int cS)
{
    const int S = g.dim - 1;
    if (cS < 0) return h.tr_lo;
    if (cS >= g.Nl[S]) return h.tr_hi;
    return nullptr;
}
__device__ __forceinline__ long long halo_F(const Geom &g, int n)
{
    return g.dim == 3 ? (long long)g.Nl[0] * g.Nl[1] * n * n : (long long)g.Nl[0] * n;
}
__device__ __forceinline__ long long halo_f(const Geom &g, int n, int c0, int c1, int inface)
{
    return g.dim == 3 ? ((long long)c0 + (long long)g.Nl[0] * c1) * (n * n) + inface : (long long)c0 * n + inface;
}

// Pointer to the nodal data of the element with local coordinates c (any direction may be
// one step outside the slab).  Non-slowest directions wrap periodically (they are never
// split).  The slowest direction wraps locally when the halo pointers are null (one rank),
// otherwise reads the neighbour layer received from the adjacent rank.
__device__ __forceinline__ const double *elem_ptr(const Geom &g, const double *base, const double *lo,
                                                  const double *hi, int c0, int c1, int c2)
{
    const int S = g.dim - 1;
    int c[3] = {c0, c1, c2};
    for (int d = 0; d < S; ++d) {
        if (c[d] < 0) c[d] += g.Nl[d];
        else if (c[d] >= g.Nl[d]) c[d] -= g.Nl[d];
    }
    if (c[S] < 0) {
        if (lo) {
            long long li = (S == 2) ? (long long)c[0] + (long long)g.Nl[0] * c[1] : (long long)c[0];
            return lo + li * g.npe;
        }
        c[S] += g.Nl[S];
    } else if (c[S] >= g.Nl[S]) {
        if (hi) {
            long long li = (S == 2) ? (long long)c[0] + (long long)g.Nl[0] * c[1] : (long long)c[0];
            return hi + li * g.npe;
        }
        c[S] -= g.Nl[S];
    }
    return base + elem_index(g, c[0], c[1], c[2]) * g.npe;
}

// viscosity at the neighbour element's face node across a face normal to D: the neighbour cn is
// one step from the own element along D; goff = the node's offset with its D-coordinate removed
// (= the in-face index for D = S), nboff = the neighbour face node's D-offset (0 or P * stride)
__device__ __forceinline__ double nbr_face_nu(const Geom &g, const double *nu, const Halo &h, int n, const int (&cn)[3],
                                              int D, int goff, int nboff)
{
    if (D == g.dim - 1) {
        const double *tr = halo_trace(g, h, cn[D]);
        if (tr) return __ldg(tr + 2 * halo_F(g, n) + halo_f(g, n, cn[0], cn[1], goff));
    }
    return __ldg(elem_ptr(g, nu, nullptr, nullptr, cn[0], cn[1], cn[2]) + goff + nboff);
}

__device__ __forceinline__ double warp_sum(double v)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide sum of K values (K <= 4), result valid in thread 0; red must hold 32*K doubles
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double *red)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) red[k * 32 + wid] = v[k];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double t = lane < nw ? red[k * 32 + lane] : 0.0;
            v[k] = warp_sum(t);
        }
    }
    __syncthreads();
}

}  // namespace dg
