// convect.cuh -- explicit DG convective tendency with local Lax-Friedrichs fluxes.
//
// F_c = -div(v v), DG-SEM "with consistent integration and local Lax-Friedrichs
// fluxes for convection":
//   M F_c,c = sum_K sum_{q in Gauss^d} W_q sum_e v_c v_e d_e phi_I
//           - sum_F sum_{q in Gauss^{d-1}} W_q h_c [phi_I],
//   h = 1/2 ((v^-.n) v^- + (v^+.n) v^+) + 1/2 Lambda (v^- - v^+), Lambda = 2 max|v^+-.n|
// (readings A12-A14: Q = floor(3P/2)+1 Gauss points per direction, GLL-lumped M).
//
// One CTA per element.  Sum-factorised: v is interpolated GLL -> Gauss by three 1-D
// contractions with Bq; the volume term is tested back with three passes that apply
// Bq^T or Gq^T per direction, the three directional terms sharing the x pass; each face
// interpolates its own and the neighbour's trace (GLL end nodes are exact traces) to the
// face Gauss points, forms the LLF flux and projects back with Bq^T.  FP64-ALU bound
// (~400 flop per component-DOF at P=7), shared-memory resident.
#pragma once

#include <cstdlib>

#include "dev_common.cuh"

namespace dg {

template <int DIM, int P>
struct CCfg {
    static constexpr int n = P + 1;
    static constexpr int Q = (3 * P) / 2 + 1;
    static constexpr int NZ = DIM == 3 ? n : 1;
    static constexpr int QZ = DIM == 3 ? Q : 1;
    static constexpr int NPE = n * n * NZ;
    static constexpr int NQ = Q * Q * QZ;
    static constexpr int T12 = 3 * NZ * n * Q + 3 * NZ * Q * Q;
    static constexpr int STG = (DIM == 3) ? (3 * n * Q * Q + 2 * n * n * Q) : (2 * n * Q);
    static constexpr int FACE = 2 * 3 * n * n + 2 * 3 * n * Q + 2 * 3 * Q * Q + 3 * Q * Q + 3 * Q * n;
    static constexpr int SCR = T12 > STG ? (T12 > FACE ? T12 : FACE) : (STG > FACE ? STG : FACE);
    static constexpr int SMEM = (3 * NPE + 3 * NQ + 3 * NPE + SCR + 2 * Q * n + Q) * 8;
};

template <int DIM, int P>
__global__ void __launch_bounds__(256) k_convect(const ConvParams a)
{
    using C = CCfg<DIM, P>;
    constexpr int n = C::n, Q = C::Q, NZ = C::NZ, QZ = C::QZ, NPE = C::NPE, NQ = C::NQ;
    const Geom &g = a.g;
    const CvTab &T = c_ctab[P];
    extern __shared__ double sm[];
    double *sv = sm;                 // [3][NPE]
    double *vg = sv + 3 * NPE;       // [3][NQ]
    double *sy = vg + 3 * NQ;        // [3][NPE]
    double *scr = sy + 3 * NPE;      // scratch
    double *sB = scr + C::SCR;       // [Q][n] interpolation, staged from __constant__
    double *sG = sB + Q * n;         // [Q][n] derivative interpolation
    double *swq = sG + Q * n;        // [Q] Gauss weights
    const int tid = threadIdx.x, nth = blockDim.x;
    for (int t = tid; t < Q * n; t += nth) {
        sB[t] = T.Bq[t / n][t % n];
        sG[t] = T.Gq[t / n][t % n];
    }
    for (int t = tid; t < Q; t += nth) swq[t] = T.wq[t];

    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        const int ec[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                           (int)(e / ((long long)g.Nl[0] * g.Nl[1]))};
        __syncthreads();
        for (int t = tid; t < DIM * NPE; t += nth) {
            const int c = t / NPE, q = t - c * NPE;
            sv[t] = a.v[c][e * NPE + q];
            sy[t] = 0.0;
        }
        __syncthreads();
        // ---- interpolate to Gauss points: T1[c][k][j][qx], T2[c][k][qy][qx], vg[c][qz][qy][qx]
        double *T1 = scr, *T2 = scr + 3 * NZ * n * Q;
        for (int t = tid; t < DIM * NZ * n * Q; t += nth) {
            const int qx = t % Q, j = (t / Q) % n, k = (t / (Q * n)) % NZ, c = t / (Q * n * NZ);
            const double *src = sv + c * NPE + n * (j + n * k);
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < n; ++i) s = fma(sB[(qx) * n + (i)], src[i], s);
            T1[t] = s;
        }
        __syncthreads();
        for (int t = tid; t < DIM * NZ * Q * Q; t += nth) {
            const int qx = t % Q, qy = (t / Q) % Q, k = (t / (Q * Q)) % NZ, c = t / (Q * Q * NZ);
            const double *src = T1 + ((c * NZ + k) * n) * Q + qx;
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < n; ++j) s = fma(sB[(qy) * n + (j)], src[j * Q], s);
            if (DIM == 3) T2[t] = s;
            else vg[c * NQ + qx + Q * qy] = s;
        }
        __syncthreads();
        if (DIM == 3) {
            for (int t = tid; t < DIM * NQ; t += nth) {
                const int qx = t % Q, qy = (t / Q) % Q, qz = (t / (Q * Q)) % QZ, c = t / NQ;
                const double *src = T2 + (c * NZ) * Q * Q + qx + Q * qy;
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < NZ; ++k) s = fma(sB[(qz) * n + (k)], src[k * Q * Q], s);
                vg[t] = s;
            }
            __syncthreads();
        }
        // ---- volume term, one component at a time
        const double hx2 = 0.5 * g.h[0], hy2 = 0.5 * g.h[1], hz2 = DIM == 3 ? 0.5 * g.h[2] : 1.0;
        const double Wc = hx2 * hy2 * hz2;
        for (int c = 0; c < DIM; ++c) {
            if (DIM == 3) {
                double *Ax = scr, *Ay = Ax + n * Q * Q, *Az = Ay + n * Q * Q;
                double *D1 = Az + n * Q * Q, *D2 = D1 + n * n * Q;
                for (int t = tid; t < n * Q * Q; t += nth) {
                    const int qx = t % Q, qy = (t / Q) % Q, k = t / (Q * Q);
                    double sx = 0.0, sy_ = 0.0, sz = 0.0;
                    const double wxy = swq[qx] * swq[qy] * Wc;
#pragma unroll
                    for (int qz = 0; qz < QZ; ++qz) {
                        const int qi = qx + Q * (qy + Q * qz);
                        const double vc = vg[c * NQ + qi];
                        const double w = wxy * swq[qz] * vc;
                        const double fx = w * vg[0 * NQ + qi], fy = w * vg[1 * NQ + qi], fz = w * vg[2 * NQ + qi];
                        sx = fma(sB[(qz) * n + (k)], fx, sx);
                        sy_ = fma(sB[(qz) * n + (k)], fy, sy_);
                        sz = fma(sG[(qz) * n + (k)], fz, sz);
                    }
                    Ax[t] = sx;
                    Ay[t] = sy_;
                    Az[t] = sz * (2.0 / g.h[2]);
                }
                __syncthreads();
                for (int t = tid; t < n * n * Q; t += nth) {
                    const int qx = t % Q, j = (t / Q) % n, k = t / (Q * n);
                    double d1 = 0.0, d2a = 0.0, d2b = 0.0;
#pragma unroll
                    for (int qy = 0; qy < Q; ++qy) {
                        const int si = qx + Q * (qy + Q * k);
                        d1 = fma(sB[(qy) * n + (j)], Ax[si], d1);
                        d2a = fma(sG[(qy) * n + (j)], Ay[si], d2a);
                        d2b = fma(sB[(qy) * n + (j)], Az[si], d2b);
                    }
                    D1[t] = d1;
                    D2[t] = fma(d2a, 2.0 / g.h[1], d2b);
                }
                __syncthreads();
                for (int t = tid; t < NPE; t += nth) {
                    const int i = t % n, j = (t / n) % n, k = t / (n * n);
                    double s1 = 0.0, s2 = 0.0;
#pragma unroll
                    for (int qx = 0; qx < Q; ++qx) {
                        const int si = qx + Q * (j + n * k);
                        s1 = fma(sG[(qx) * n + (i)], D1[si], s1);
                        s2 = fma(sB[(qx) * n + (i)], D2[si], s2);
                    }
                    sy[c * NPE + t] += fma(s1, 2.0 / g.h[0], s2);
                }
                __syncthreads();
            } else {
                double *D1 = scr, *D2 = scr + n * Q;
                for (int t = tid; t < n * Q; t += nth) {
                    const int qx = t % Q, j = t / Q;
                    double d1 = 0.0, d2 = 0.0;
#pragma unroll
                    for (int qy = 0; qy < Q; ++qy) {
                        const int qi = qx + Q * qy;
                        const double w = swq[qx] * swq[qy] * Wc * vg[c * NQ + qi];
                        d1 = fma(sB[(qy) * n + (j)], w * vg[0 * NQ + qi], d1);
                        d2 = fma(sG[(qy) * n + (j)], w * vg[1 * NQ + qi], d2);
                    }
                    D1[t] = d1;
                    D2[t] = d2 * (2.0 / g.h[1]);
                }
                __syncthreads();
                for (int t = tid; t < NPE; t += nth) {
                    const int i = t % n, j = t / n;
                    double s1 = 0.0, s2 = 0.0;
#pragma unroll
                    for (int qx = 0; qx < Q; ++qx) {
                        s1 = fma(sG[(qx) * n + (i)], D1[qx + Q * j], s1);
                        s2 = fma(sB[(qx) * n + (i)], D2[qx + Q * j], s2);
                    }
                    sy[c * NPE + t] += fma(s1, 2.0 / g.h[0], s2);
                }
                __syncthreads();
            }
        }
        // ---- faces
        constexpr int NF = DIM == 3 ? n * n : n;  // face nodes
        constexpr int QF = DIM == 3 ? Q * Q : Q;  // face Gauss points
        double *fo = scr, *fn = fo + 3 * NF;               // [3][NF] own / neighbour traces
        double *F1o = fn + 3 * NF, *F1n = F1o + 3 * n * Q; // 3-D intermediates [3][b][qa]
        double *Go = F1n + 3 * n * Q, *Gn = Go + 3 * QF;   // [3][QF]
        double *H = Gn + 3 * QF;                           // [3][QF]
        double *P1 = H + 3 * QF;                           // [3][qb][a]
        for (int d = 0; d < DIM; ++d) {
            const int o1 = (d == 0) ? 1 : 0;
            const int o2 = (d == 2) ? 1 : 2;
            const double ho1 = 0.5 * g.h[o1], ho2 = DIM == 3 ? 0.5 * g.h[o2] : 1.0;
            for (int side = -1; side <= 1; side += 2) {
                const int a_own = side > 0 ? P : 0, a_nb = side > 0 ? 0 : P;
                int cn[3] = {ec[0], ec[1], ec[2]};
                cn[d] += side;
                for (int t = tid; t < DIM * NF; t += nth) {
                    const int c = t / NF, f = t - c * NF;
                    const int fa = f % n, fb = f / n;
                    int nd[3] = {0, 0, 0};
                    nd[o1] = fa;
                    if (DIM == 3) nd[o2] = fb;
                    nd[d] = a_own;
                    const int qo = nd[0] + n * (nd[1] + n * nd[2]);
                    nd[d] = a_nb;
                    const int qn = nd[0] + n * (nd[1] + n * nd[2]);
                    fo[t] = sv[c * NPE + qo];
                    fn[t] = __ldg(elem_ptr(g, a.v[c], a.lo[c], a.hi[c], cn[0], cn[1], cn[2]) + qn);
                }
                __syncthreads();
                if (DIM == 3) {
                    for (int t = tid; t < 2 * DIM * n * Q; t += nth) {
                        const int side2 = t / (DIM * n * Q), r = t - side2 * DIM * n * Q;
                        const int qa = r % Q, b = (r / Q) % n, c = r / (Q * n);
                        const double *src = (side2 ? fn : fo) + c * NF + b * n;
                        double s = 0.0;
#pragma unroll
                        for (int aa = 0; aa < n; ++aa) s = fma(sB[(qa) * n + (aa)], src[aa], s);
                        (side2 ? F1n : F1o)[r] = s;
                    }
                    __syncthreads();
                    for (int t = tid; t < 2 * DIM * QF; t += nth) {
                        const int side2 = t / (DIM * QF), r = t - side2 * DIM * QF;
                        const int qa = r % Q, qb = (r / Q) % Q, c = r / QF;
                        const double *src = (side2 ? F1n : F1o) + c * n * Q + qa;
                        double s = 0.0;
#pragma unroll
                        for (int b = 0; b < n; ++b) s = fma(sB[(qb) * n + (b)], src[b * Q], s);
                        (side2 ? Gn : Go)[r] = s;
                    }
                } else {
                    for (int t = tid; t < 2 * DIM * QF; t += nth) {
                        const int side2 = t / (DIM * QF), r = t - side2 * DIM * QF;
                        const int qa = r % Q, c = r / Q;
                        const double *src = (side2 ? fn : fo) + c * NF;
                        double s = 0.0;
#pragma unroll
                        for (int aa = 0; aa < n; ++aa) s = fma(sB[(qa) * n + (aa)], src[aa], s);
                        (side2 ? Gn : Go)[r] = s;
                    }
                }
                __syncthreads();
                for (int t = tid; t < QF; t += nth) {
                    const int qa = t % Q, qb = t / Q;
                    const double WF = swq[qa] * ho1 * (DIM == 3 ? swq[qb] * ho2 : 1.0);
                    const double sgn = side > 0 ? 1.0 : -1.0;
                    const double *vm = side > 0 ? Go : Gn, *vp = side > 0 ? Gn : Go;
                    const double vnm = vm[d * QF + t], vnp = vp[d * QF + t];
                    const double Lam = 2.0 * fmax(fabs(vnm), fabs(vnp));
                    for (int c = 0; c < DIM; ++c) {
                        const double hc = 0.5 * (vnm * vm[c * QF + t] + vnp * vp[c * QF + t]) +
                                          0.5 * Lam * (vm[c * QF + t] - vp[c * QF + t]);
                        H[c * QF + t] = sgn * WF * hc;
                    }
                }
                __syncthreads();
                if (DIM == 3) {
                    for (int t = tid; t < DIM * Q * n; t += nth) {
                        const int aa = t % n, qb = (t / n) % Q, c = t / (n * Q);
                        const double *src = H + c * QF + Q * qb;
                        double s = 0.0;
#pragma unroll
                        for (int qa = 0; qa < Q; ++qa) s = fma(sB[(qa) * n + (aa)], src[qa], s);
                        P1[t] = s;
                    }
                    __syncthreads();
                }
                for (int t = tid; t < DIM * NF; t += nth) {
                    const int c = t / NF, f = t - c * NF;
                    const int fa = f % n, fb = f / n;
                    double s = 0.0;
                    if (DIM == 3) {
                        const double *src = P1 + c * Q * n + fa;
#pragma unroll
                        for (int qb = 0; qb < Q; ++qb) s = fma(sB[(qb) * n + (fb)], src[qb * n], s);
                    } else {
                        const double *src = H + c * QF;
#pragma unroll
                        for (int qa = 0; qa < Q; ++qa) s = fma(sB[(qa) * n + (fa)], src[qa], s);
                    }
                    int nd[3] = {0, 0, 0};
                    nd[o1] = fa;
                    if (DIM == 3) nd[o2] = fb;
                    nd[d] = a_own;
                    sy[c * NPE + nd[0] + n * (nd[1] + n * nd[2])] -= s;
                }
                __syncthreads();
            }
        }
        // ---- M^-1 (GLL-lumped) and store
        for (int t = tid; t < DIM * NPE; t += nth) {
            const int c = t / NPE, q = t - c * NPE;
            const int i = q % n, j = (q / n) % n, k = q / (n * n);
            double m = T.w[i] * hx2 * T.w[j] * hy2;
            if (DIM == 3) m *= T.w[k] * hz2;
            a.out[c][e * NPE + q] = sy[t] / m;
        }
    }
}

// ---------------------------------------------------------------------------
// even-odd products with the rectangular Gauss tables (CvTab Xe / Xo / Xc): X is B
// (centro-symmetric, ANTI = false) or G (centro-antisymmetric, ANTI = true)
// ---------------------------------------------------------------------------
// out[q] = sum_j X[q][j] v[j], q < Q
template <int n, int Q, bool ANTI>
__device__ __forceinline__ void eo_fwd(const double (&Xe)[HQMAX][HMAX], const double (&Xo)[HQMAX][HMAX],
                                       const double (&Xc)[HQMAX], const double (&v)[n], double (&out)[Q])
{
    constexpr int hn = n / 2, hq = Q / 2;
    constexpr bool nodd = (n % 2) == 1, qodd = (Q % 2) == 1;
    double ve[hn], vo[hn];
#pragma unroll
    for (int j = 0; j < hn; ++j) {
        ve[j] = v[j] + v[n - 1 - j];
        vo[j] = v[j] - v[n - 1 - j];
    }
    const double vm = nodd ? v[n / 2] : 0.0;
#pragma unroll
    for (int q = 0; q < hq; ++q) {
        double e = nodd ? Xc[q] * vm : Xe[q][0] * ve[0];
        double o = Xo[q][0] * vo[0];
#pragma unroll
        for (int j = nodd ? 0 : 1; j < hn; ++j) e = fma(Xe[q][j], ve[j], e);
#pragma unroll
        for (int j = 1; j < hn; ++j) o = fma(Xo[q][j], vo[j], o);
        out[q] = e + o;
        out[Q - 1 - q] = ANTI ? o - e : e - o;
    }
    if (qodd) {
        double m;
        if (!ANTI) {
            m = nodd ? Xc[hq] * vm : 0.0;
#pragma unroll
            for (int j = 0; j < hn; ++j) m = fma(Xe[hq][j], ve[j], m);
        } else {
            m = 0.0;
#pragma unroll
            for (int j = 0; j < hn; ++j) m = fma(Xo[hq][j], vo[j], m);
        }
        out[hq] = m;
    }
}

// transposed products out[j] = sum_q X[q][j] f[q], accumulated one Gauss pair (q, Q-1-q) at a
// time into the even / odd halves E[j] = (out[j] + out[P-j]) / 2, O[j] = (out[j] - out[P-j]) / 2
// and the middle output (odd n); eo_fin forms out
template <int n, bool ANTI>
__device__ __forceinline__ void eo_acc(const double (&Xe)[HQMAX][HMAX], const double (&Xo)[HQMAX][HMAX],
                                       const double (&Xc)[HQMAX], int q, double f1, double f2, double (&E)[n / 2],
                                       double (&O)[n / 2], double &M)
{
    const double fe = f1 + f2, fo = f1 - f2;
#pragma unroll
    for (int j = 0; j < n / 2; ++j) {
        E[j] = fma(Xe[q][j], ANTI ? fo : fe, E[j]);
        O[j] = fma(Xo[q][j], ANTI ? fe : fo, O[j]);
    }
    if (n % 2) M = fma(Xc[q], ANTI ? fo : fe, M);
}
// the middle Gauss point (odd Q)
template <int n, bool ANTI>
__device__ __forceinline__ void eo_acc_mid(const double (&Xe)[HQMAX][HMAX], const double (&Xo)[HQMAX][HMAX],
                                           const double (&Xc)[HQMAX], int q, double f, double (&E)[n / 2],
                                           double (&O)[n / 2], double &M)
{
#pragma unroll
    for (int j = 0; j < n / 2; ++j) {
        if (ANTI) O[j] = fma(Xo[q][j], f, O[j]);
        else E[j] = fma(Xe[q][j], f, E[j]);
    }
    if ((n % 2) && !ANTI) M = fma(Xc[q], f, M);
}
template <int n>
__device__ __forceinline__ void eo_zero(double (&E)[n / 2], double (&O)[n / 2], double &M)
{
#pragma unroll
    for (int j = 0; j < n / 2; ++j) E[j] = O[j] = 0.0;
    M = 0.0;
}
template <int n>
__device__ __forceinline__ void eo_fin(const double (&E)[n / 2], const double (&O)[n / 2], double M, double (&out)[n])
{
#pragma unroll
    for (int j = 0; j < n / 2; ++j) {
        out[j] = E[j] + O[j];
        out[n - 1 - j] = E[j] - O[j];
    }
    if (n % 2) out[n / 2] = M;
}
// out[j] = sum_q X[q][j] f[q] with f in registers
template <int n, int Q, bool ANTI>
__device__ __forceinline__ void eo_bwd(const double (&Xe)[HQMAX][HMAX], const double (&Xo)[HQMAX][HMAX],
                                       const double (&Xc)[HQMAX], const double (&f)[Q], double (&out)[n])
{
    double E[n / 2], O[n / 2], M;
    eo_zero<n>(E, O, M);
#pragma unroll
    for (int q = 0; q < Q / 2; ++q) eo_acc<n, ANTI>(Xe, Xo, Xc, q, f[q], f[Q - 1 - q], E, O, M);
    if (Q % 2) eo_acc_mid<n, ANTI>(Xe, Xo, Xc, Q / 2, f[Q / 2], E, O, M);
    eo_fin<n>(E, O, M, out);
}

// ---------------------------------------------------------------------------
// k_convect3 (3-D, the dispatched kernel): one thread per element line, the 1-D tables of
// __constant__ c_ctab as uniform operands of fully unrolled contractions.
//   interpolation GLL -> Gauss: x lines (n^2), y lines (Q n), z lines (Q^2; the Gauss column
//   of all three components stays in the thread's registers);
//   volume, per component c: fluxes W v_c v_e at the column's Gauss points, tested along z
//   (B, B, G'), then y (lines (qx, k): B and G'), then x (lines (j, k): G' and B);
//   faces: per direction d both sides at once: own (shared) and neighbour (global) traces
//   interpolated to the face Gauss points along o1 then o2, the LLF flux, projected back.
// Shared memory: nodal v, the accumulator, two work regions (the interpolation arrays, then
// the test arrays, then the face arrays).
// ---------------------------------------------------------------------------
template <int P>
struct C3Cfg {
    static constexpr int n = P + 1, Q = (3 * P) / 2 + 1;
    static constexpr int NPE = n * n * n;
    static constexpr int NX = n % 2 == 0 ? n + 1 : n;   // padded x-line pitch of sv / sy (odd:
    static constexpr int NPEP = NX * n * n;             //  conflict-free strided line access)
#ifndef DG_CONV_NT
#define DG_CONV_NT 0  // development: threads per CTA (0: the Gauss column count rounded to warps, >= 128)
#endif
    static constexpr int NT0 = ((Q * Q + 31) / 32) * 32 < 128 ? 128 : ((Q * Q + 31) / 32) * 32;
    static constexpr int NT = DG_CONV_NT > NT0 ? DG_CONV_NT : NT0;
    static constexpr int MINB = NT > 128 ? 2 : (P >= 7 ? 3 : 1);
    static constexpr int W1 = 3 * n * n * Q;            // T1 / D region
    static constexpr int W2a = 3 * n * Q * Q, W2b = 2 * 3 * Q * (n + 1);
    static constexpr int W2 = W2a > W2b ? W2a : W2b;    // T2 / A / face G2, P1 region
    static constexpr int FACE1 = 2 * 3 * n * Q;         // per direction: F1 (both sides)
    static constexpr int FACE2 = 2 * 3 * Q * Q;         // G (both sides)
    static_assert(FACE1 <= W1 && FACE2 <= W2 && 2 * 3 * Q * (n + 1) <= W2, "face arrays fit the work regions");
    static constexpr int SMEM = (2 * 3 * NPEP + W1 + W2) * 8;
};

template <int P>
__global__ void __launch_bounds__(C3Cfg<P>::NT, C3Cfg<P>::MINB) k_convect3(const ConvParams a)
{
    using C = C3Cfg<P>;
    constexpr int n = C::n, Q = C::Q, NPE = C::NPE, NT = C::NT, NX = C::NX, NPEP = C::NPEP;
    const Geom &g = a.g;
    const CvTab &T = c_ctab[P];
    extern __shared__ double sm[];
    double *sv = sm;                // [3][NPEP] nodal v (x-line pitch NX)
    double *sy = sv + 3 * NPEP;     // [3][NPEP] accumulator (weak form)
    double *R1 = sy + 3 * NPEP;     // W1 doubles
    double *R2 = R1 + C::W1;        // W2 doubles
    const int tid = threadIdx.x;
    const double hx2 = 0.5 * g.h[0], hy2 = 0.5 * g.h[1], hz2 = 0.5 * g.h[2];
    const double Wc = hx2 * hy2 * hz2;
    const double sdx = 2.0 / g.h[0], sdy = 2.0 / g.h[1], sdz = 2.0 / g.h[2];
    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        const int ec[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                           (int)(e / ((long long)g.Nl[0] * g.Nl[1]))};
        __syncthreads();
        for (int t = tid; t < 3 * NPE; t += NT) {
            const int c = t / NPE, q = t - c * NPE;
            sv[c * NPEP + (q / n) * NX + q % n] = a.v[c][e * NPE + q];
        }
        __syncthreads();
        // ---- interpolation x: lines (c, j, k) -> T1[c][(k n + j) Q + qx]
        for (int l = tid; l < 3 * n * n; l += NT) {
            const double *src = sv + (l / (n * n)) * NPEP + (l % (n * n)) * NX;
            double v[n], o[Q];
#pragma unroll
            for (int i = 0; i < n; ++i) v[i] = src[i];
            eo_fwd<n, Q, false>(T.Be, T.Bo, T.Bc, v, o);
#pragma unroll
            for (int q = 0; q < Q; ++q) R1[l * Q + q] = o[q];
        }
        __syncthreads();
        // ---- y: lines (c, k, qx) over j -> T2[c][(k Q + qy) Q + qx]
        for (int l = tid; l < 3 * n * Q; l += NT) {
            const int qx = l % Q, ck = l / Q;  // ck = c n + k
            double v[n], o[Q];
#pragma unroll
            for (int j = 0; j < n; ++j) v[j] = R1[(ck * n + j) * Q + qx];
            eo_fwd<n, Q, false>(T.Be, T.Bo, T.Bc, v, o);
#pragma unroll
            for (int q = 0; q < Q; ++q) R2[(ck * Q + q) * Q + qx] = o[q];
        }
        __syncthreads();
        // ---- z: column (qx, qy) of all three components, kept in registers
        const bool col = tid < Q * Q;
        const int qx = tid % Q, qy = tid / Q;
        double vz[3][Q];
        if (col) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double v[n];
#pragma unroll
                for (int k = 0; k < n; ++k) v[k] = R2[((c * n + k) * Q + qy) * Q + qx];
                eo_fwd<n, Q, false>(T.Be, T.Bo, T.Bc, v, vz[c]);
            }
        }
        // ---- volume, per component
        for (int c = 0; c < 3; ++c) {
            // c = 0: T2 (R2) has been read by the z interpolation.  c > 0: no barrier -- the z
            // test writes R2 (read by the previous y test, behind its barrier) while slower
            // threads finish the previous x test (R1 -> sy); the barrier after the z test orders
            // that x test before the next y test rewrites R1
            if (c == 0) __syncthreads();
            if (col) {
                const double wxy = T.wq[qx] * T.wq[qy] * Wc;
                double ax[n], ay[n], az[n];
                {
                    constexpr int hn = n / 2;
                    double Ex[hn], Ox[hn], Mx, Ey[hn], Oy[hn], My, Ez[hn], Oz[hn], Mz;
                    eo_zero<n>(Ex, Ox, Mx);
                    eo_zero<n>(Ey, Oy, My);
                    eo_zero<n>(Ez, Oz, Mz);
#pragma unroll
                    for (int q = 0; q < Q / 2; ++q) {
                        const int q2 = Q - 1 - q;
                        const double w1 = wxy * T.wq[q] * vz[c][q], w2 = wxy * T.wq[q2] * vz[c][q2];
                        eo_acc<n, false>(T.Be, T.Bo, T.Bc, q, w1 * vz[0][q], w2 * vz[0][q2], Ex, Ox, Mx);
                        eo_acc<n, false>(T.Be, T.Bo, T.Bc, q, w1 * vz[1][q], w2 * vz[1][q2], Ey, Oy, My);
                        eo_acc<n, true>(T.Ge, T.Go, T.Gc, q, w1 * vz[2][q], w2 * vz[2][q2], Ez, Oz, Mz);
                    }
                    if (Q % 2) {
                        constexpr int qm = Q / 2;
                        const double w = wxy * T.wq[qm] * vz[c][qm];
                        eo_acc_mid<n, false>(T.Be, T.Bo, T.Bc, qm, w * vz[0][qm], Ex, Ox, Mx);
                        eo_acc_mid<n, false>(T.Be, T.Bo, T.Bc, qm, w * vz[1][qm], Ey, Oy, My);
                        eo_acc_mid<n, true>(T.Ge, T.Go, T.Gc, qm, w * vz[2][qm], Ez, Oz, Mz);
                    }
                    eo_fin<n>(Ex, Ox, Mx, ax);
                    eo_fin<n>(Ey, Oy, My, ay);
                    eo_fin<n>(Ez, Oz, Mz, az);
                }
                // A[t][(k Q + qy) Q + qx], t = x, y, z term
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    const int o = (k * Q + qy) * Q + qx;
                    R2[o] = ax[k];
                    R2[n * Q * Q + o] = ay[k];
                    R2[2 * n * Q * Q + o] = az[k] * sdz;
                }
            }
            __syncthreads();
            // y: lines (k, qx): D1 = B_y A_x, D2 = (2/hy) G_y A_y + B_y A_z -> R1[t][(k n + j) Q + qx]
            // (q-outer: the inputs stream through, 3 n accumulators stay in registers next to
            // the Gauss column)
            for (int l = tid; l < n * Q; l += NT) {
                const int lqx = l % Q, k = l / Q;
                double d1[n], d2[n], d3[n];
                {
                    constexpr int hn = n / 2;
                    double E1[hn], O1[hn], M1, E2[hn], O2[hn], M2, E3[hn], O3[hn], M3;
                    eo_zero<n>(E1, O1, M1);
                    eo_zero<n>(E2, O2, M2);
                    eo_zero<n>(E3, O3, M3);
#pragma unroll
                    for (int q = 0; q < Q / 2; ++q) {
                        const int o = (k * Q + q) * Q + lqx, o2 = (k * Q + (Q - 1 - q)) * Q + lqx;
                        eo_acc<n, false>(T.Be, T.Bo, T.Bc, q, R2[o], R2[o2], E1, O1, M1);
                        eo_acc<n, true>(T.Ge, T.Go, T.Gc, q, R2[n * Q * Q + o], R2[n * Q * Q + o2], E2, O2, M2);
                        eo_acc<n, false>(T.Be, T.Bo, T.Bc, q, R2[2 * n * Q * Q + o], R2[2 * n * Q * Q + o2], E3, O3, M3);
                    }
                    if (Q % 2) {
                        constexpr int qm = Q / 2;
                        const int o = (k * Q + qm) * Q + lqx;
                        eo_acc_mid<n, false>(T.Be, T.Bo, T.Bc, qm, R2[o], E1, O1, M1);
                        eo_acc_mid<n, true>(T.Ge, T.Go, T.Gc, qm, R2[n * Q * Q + o], E2, O2, M2);
                        eo_acc_mid<n, false>(T.Be, T.Bo, T.Bc, qm, R2[2 * n * Q * Q + o], E3, O3, M3);
                    }
                    eo_fin<n>(E1, O1, M1, d1);
                    eo_fin<n>(E2, O2, M2, d2);
                    eo_fin<n>(E3, O3, M3, d3);
                }
#pragma unroll
                for (int j = 0; j < n; ++j) {
                    R1[(k * n + j) * Q + lqx] = d1[j];
                    R1[n * n * Q + (k * n + j) * Q + lqx] = fma(d2[j], sdy, d3[j]);
                }
            }
            __syncthreads();
            // x: lines (j, k): out_i = (2/hx) sum G D1 + sum B D2 (q-outer)
            for (int l = tid; l < n * n; l += NT) {
                double s1[n], s2[n];
                {
                    constexpr int hn = n / 2;
                    double E1[hn], O1[hn], M1, E2[hn], O2[hn], M2;
                    eo_zero<n>(E1, O1, M1);
                    eo_zero<n>(E2, O2, M2);
                    const double *r1 = R1 + l * Q, *r2 = R1 + n * n * Q + l * Q;
#pragma unroll
                    for (int q = 0; q < Q / 2; ++q) {
                        eo_acc<n, true>(T.Ge, T.Go, T.Gc, q, r1[q], r1[Q - 1 - q], E1, O1, M1);
                        eo_acc<n, false>(T.Be, T.Bo, T.Bc, q, r2[q], r2[Q - 1 - q], E2, O2, M2);
                    }
                    if (Q % 2) {
                        eo_acc_mid<n, true>(T.Ge, T.Go, T.Gc, Q / 2, r1[Q / 2], E1, O1, M1);
                        eo_acc_mid<n, false>(T.Be, T.Bo, T.Bc, Q / 2, r2[Q / 2], E2, O2, M2);
                    }
                    eo_fin<n>(E1, O1, M1, s1);
                    eo_fin<n>(E2, O2, M2, s2);
                }
#pragma unroll
                for (int i = 0; i < n; ++i) sy[c * NPEP + l * NX + i] = fma(s1[i], sdx, s2[i]);
            }
        }
        // ---- faces, per direction d (both sides): node of face index (fa along o1, fb along o2)
        for (int d = 0; d < 3; ++d) {
            const int o1 = d == 0 ? 1 : 0, o2 = d == 2 ? 1 : 2;
            const int S[3] = {1, NX, NX * n};
            const double ho1 = 0.5 * g.h[o1], ho2 = 0.5 * g.h[o2];
            // d = 0: the volume's x test has read R1.  d > 0: no barrier -- F1 (R1) was last read
            // by the previous direction's P1 phase (behind its barrier); the previous back phase
            // (reads R2, updates sy) is ordered before G2 rewrites R2 by the barrier after F1
            if (d == 0) __syncthreads();
            // F1[s][side2][c][fb][qa]: along o1, n -> Q; s = 0: face at node 0 (side -1), s = 1: node P
            // side2 = 0: own trace, 1: neighbour trace
            double *F1 = R1, *G2 = R2;
            for (int l = tid; l < 2 * 2 * 3 * n; l += NT) {
                const int fb = l % n, c = (l / n) % 3, side2 = (l / (3 * n)) % 2, s = l / (6 * n);
                double v[n];
                if (side2 == 0) {
                    const int base = c * NPEP + fb * S[o2] + (s ? P : 0) * S[d];
#pragma unroll
                    for (int fa = 0; fa < n; ++fa) v[fa] = sv[base + fa * S[o1]];
                } else {
                    int cn[3] = {ec[0], ec[1], ec[2]};
                    cn[d] += s ? 1 : -1;
                    const int G[3] = {1, n, n * n};  // global (unpadded) strides
                    const double *nb = elem_ptr(g, a.v[c], a.lo[c], a.hi[c], cn[0], cn[1], cn[2]) + fb * G[o2] +
                                       (s ? 0 : P) * G[d];
#pragma unroll
                    for (int fa = 0; fa < n; ++fa) v[fa] = __ldg(nb + fa * G[o1]);
                }
                double o[Q];
                eo_fwd<n, Q, false>(T.Be, T.Bo, T.Bc, v, o);
#pragma unroll
                for (int q = 0; q < Q; ++q) F1[l * Q + q] = o[q];
            }
            __syncthreads();
            // G2[s][side2][c][qb][qa]: along o2, n -> Q
            for (int l = tid; l < 2 * 2 * 3 * Q; l += NT) {
                const int qa = l % Q, r = l / Q;  // r = (s 2 + side2) 3 + c
                double v[n];
#pragma unroll
                for (int fb = 0; fb < n; ++fb) v[fb] = F1[(r * n + fb) * Q + qa];
                double o[Q];
                eo_fwd<n, Q, false>(T.Be, T.Bo, T.Bc, v, o);
#pragma unroll
                for (int q = 0; q < Q; ++q) G2[(r * Q + q) * Q + qa] = o[q];
            }
            __syncthreads();
            // LLF flux at the face Gauss points -> H[s][c][qb][qa] (in F1's region)
            double *H = F1;
            for (int l = tid; l < 2 * Q * Q; l += NT) {
                const int t = l % (Q * Q), s = l / (Q * Q);
                const int qa = t % Q, qb = t / Q;
                const double WF = T.wq[qa] * ho1 * T.wq[qb] * ho2;
                // side s = 1 (node P): own is '-', neighbour '+'; s = 0: neighbour '-', own '+'
                const double *own = G2 + (s * 2 + 0) * 3 * Q * Q, *nbr = G2 + (s * 2 + 1) * 3 * Q * Q;
                const double *vm = s ? own : nbr, *vp = s ? nbr : own;
                const double vnm = vm[d * Q * Q + t], vnp = vp[d * Q * Q + t];
                const double Lam = 2.0 * fmax(fabs(vnm), fabs(vnp));
                const double sgn = s ? 1.0 : -1.0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double hc = 0.5 * (vnm * vm[c * Q * Q + t] + vnp * vp[c * Q * Q + t]) +
                                      0.5 * Lam * (vm[c * Q * Q + t] - vp[c * Q * Q + t]);
                    H[(s * 3 + c) * Q * Q + t] = sgn * WF * hc;
                }
            }
            __syncthreads();
            // back along o1: lines (s, c, qb): Q -> n  -> P1[s][c][qb][fa] (in G2's region)
            double *P1 = G2;
            for (int l = tid; l < 2 * 3 * Q; l += NT) {
                double v[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) v[q] = H[l * Q + q];
                double o[n];
                eo_bwd<n, Q, false>(T.Be, T.Bo, T.Bc, v, o);
#pragma unroll
                for (int fa = 0; fa < n; ++fa) P1[l * NX + fa] = o[fa];
            }
            __syncthreads();
            // back along o2: lines (s, c, fa): Q -> n, subtract at the face nodes
            for (int l = tid; l < 2 * 3 * n; l += NT) {
                const int fa = l % n, c = (l / n) % 3, s = l / (3 * n);
                double v[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) v[q] = P1[((s * 3 + c) * Q + q) * NX + fa];
                double o[n];
                eo_bwd<n, Q, false>(T.Be, T.Bo, T.Bc, v, o);
#pragma unroll
                for (int fb = 0; fb < n; ++fb) sy[c * NPEP + fa * S[o1] + fb * S[o2] + (s ? P : 0) * S[d]] -= o[fb];
            }
        }
        __syncthreads();
        // ---- M^-1 (GLL-lumped) and store
        for (int t = tid; t < 3 * NPE; t += NT) {
            const int c = t / NPE, q = t - c * NPE;
            const int i = q % n, j = (q / n) % n, k = q / (n * n);
            const double m = T.w[i] * hx2 * T.w[j] * hy2 * T.w[k] * hz2;
            a.out[c][e * NPE + q] = sy[c * NPEP + (q / n) * NX + i] / m;
        }
    }
}

template <int DIM>
struct ConvDispatch {
    template <int P>
    static cudaError_t go(const ConvParams &a, cudaStream_t st)
    {
        if constexpr (DIM == 3 && C3Cfg<P>::SMEM <= 227 * 1024) {
            static const bool v1 = DG_DEV_ENV("DG_CONVECT_V1") != nullptr;
            if (!v1) {
                constexpr int smem3 = C3Cfg<P>::SMEM;
                static int resident = 0;  // persistent: one full wave of CTAs
                if (!resident) {
                    cudaError_t e = cudaFuncSetAttribute(k_convect3<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
                    if (e != cudaSuccess) return e;
                    int dev = 0, nsm = 148, occ = 1;
                    cudaGetDevice(&dev);
                    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_convect3<P>, C3Cfg<P>::NT, smem3) !=
                            cudaSuccess || occ < 1)
                        occ = 1;
                    resident = nsm * occ;
                }
                long long grid = a.g.nel;
                if (grid > resident) grid = resident;
                k_convect3<P><<<(int)grid, C3Cfg<P>::NT, smem3, st>>>(a);
                return cudaGetLastError();
            }
        }
        constexpr int smem = CCfg<DIM, P>::SMEM;
        if constexpr (smem > 227 * 1024) {
            return cudaErrorNotSupported;  // shared-memory tile too large (3-D P=10)
        } else {
        auto kern = k_convect<DIM, P>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        long long grid = a.g.nel;
        if (grid > 148 * 16) grid = 148 * 16;
        kern<<<(int)grid, 256, smem, st>>>(a);
        return cudaGetLastError();
        }
    }
    static cudaError_t run(const ConvParams &a, cudaStream_t st)
    {
        switch (a.g.P) {
        case 1: if constexpr (DG_HAS_P(1)) return go<1>(a, st); else return cudaErrorNotSupported;
        case 2: if constexpr (DG_HAS_P(2)) return go<2>(a, st); else return cudaErrorNotSupported;
        case 3: if constexpr (DG_HAS_P(3)) return go<3>(a, st); else return cudaErrorNotSupported;
        case 4: if constexpr (DG_HAS_P(4)) return go<4>(a, st); else return cudaErrorNotSupported;
        case 5: if constexpr (DG_HAS_P(5)) return go<5>(a, st); else return cudaErrorNotSupported;
        case 6: if constexpr (DG_HAS_P(6)) return go<6>(a, st); else return cudaErrorNotSupported;
        case 7: if constexpr (DG_HAS_P(7)) return go<7>(a, st); else return cudaErrorNotSupported;
        case 8: if constexpr (DG_HAS_P(8)) return go<8>(a, st); else return cudaErrorNotSupported;
        case 9: if constexpr (DG_HAS_P(9)) return go<9>(a, st); else return cudaErrorNotSupported;
        case 10: if constexpr (DG_HAS_P(10)) return go<10>(a, st); else return cudaErrorNotSupported;
        default: return cudaErrorInvalidValue;
        }
    }
};

}  // namespace dg
