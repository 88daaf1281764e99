// stage.cu -- element-local pieces of the config-4 IMEX-RK stage (
// Alg. 3 lines 4-9; DESIGN.md §9 "stage composition").
//
//   k_stage_combine : F_d1 = -M^-1 (A_0 v)            (nodal viscous term, P:693 F_d1 = div nu grad v)
//                     v'   = v + dt a^ex_21 (F_c + F_d1)            (Alg. 3 line 4, F_s = 0)
//                     g    = v' + dt (a^im_21 - a^ex_21) F_d1       (Alg. 3 line 8, v'' = v')
//                     f_H  = g / (dt a^im_22)                       (reading A4: f = lam g)
//   k_dg_div        : weak DG divergence of v' tested with the degree-(P-1) pressure basis
//                     (the rhs of the pressure Poisson problem, Alg. 3 line 5);
//   k_dg_grad       : weak DG gradient of psi tested with the velocity basis (Alg. 3 line 6,
//                     v'' = v' - M^-1 G psi).  -G is the transpose of D.
#include <cstdlib>

#include "dev_common.cuh"

namespace dg {
cudaError_t upload_tables_stage() { return cudaSuccess; }  // tables: upload_tables_stage_interp

// pressure basis (degree P-1 GLL Lagrange) at the velocity GLL nodes of degree P:
// E[i][a] = l^{P-1}_a(xi^P_i), Ed[i][a] = l^{P-1}_a'(xi^P_i) (barycentric, long double)
struct StTab {
    double w[NMAX];             // velocity GLL weights
    double D[NMAX][NMAX];       // velocity differentiation matrix
    double E[NMAX][NMAX - 1];
    double Ed[NMAX][NMAX - 1];
};
static __constant__ StTab c_stab[PMAX + 1];

cudaError_t upload_tables_stage_interp()
{
    static StTab h[PMAX + 1];
    for (int P = 2; P <= PMAX; ++P) {
        const Tab &t = host_tab(P), &tp = host_tab(P - 1);
        const int m = P;  // pressure nodes per direction
        long double bw[NMAX];
        for (int a = 0; a < m; ++a) {
            long double b = 1.0L;
            for (int c = 0; c < m; ++c)
                if (c != a) b *= (long double)tp.xi[a] - (long double)tp.xi[c];
            bw[a] = 1.0L / b;
        }
        for (int i = 0; i <= P; ++i) {
            const long double x = t.xi[i];
            // l_a(x) = prod_{c != a} (x - xp_c) bw_a ;  l_a'(x) = l_a(x) sum_{c != a} 1/(x - xp_c)
            // (evaluated directly; velocity and pressure nodes coincide only at +-1)
            for (int a = 0; a < m; ++a) {
                long double la = bw[a], dla = 0.0L;
                for (int c = 0; c < m; ++c) {
                    if (c == a) continue;
                    long double prod = bw[a];
                    for (int c2 = 0; c2 < m; ++c2)
                        if (c2 != a && c2 != c) prod *= x - (long double)tp.xi[c2];
                    dla += prod;
                    la *= x - (long double)tp.xi[c];
                }
                h[P].E[i][a] = (double)la;
                h[P].Ed[i][a] = (double)dla;
            }
        }
        for (int i = 0; i <= P; ++i) {
            h[P].w[i] = t.w[i];
            for (int j = 0; j <= P; ++j) h[P].D[i][j] = t.D[i][j];
        }
    }
    return cudaMemcpyToSymbol(c_stab, h, sizeof(h));
}

namespace {

__global__ void k_stage_combine(long long ndof, int npe, const double *mass_e, double a_ex, double c_g, double lamH,
                                const double *v, const double *Fc, const double *Av, double *vp, double *fH)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ndof; t += (long long)gridDim.x * blockDim.x) {
        const double fd = -Av[t] / mass_e[t % npe];
        const double vpr = fma(a_ex, Fc[t] + fd, v[t]);
        vp[t] = vpr;
        fH[t] = lamH * fma(c_g, fd, vpr);
    }
}

// out = c * in / m (nodal value of a weak vector; m = GLL-lumped mass of the node)
__global__ void k_scale_minv(long long ndof, int npe, const double *mass_e, double c, const double *in, double *out)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ndof; t += (long long)gridDim.x * blockDim.x)
        out[t] = c * in[t] / mass_e[t % npe];
}

// out = c0 x0 + sum_k c_k y_k  (+ cm * w / m when w != null) -- the stage combinations of the
// IMEX-RK step driver (Alg. 3 lines 4, 6, 8, 11)
__global__ void k_lincomb(long long ndof, int npe, LinComb lc, const double *mass_e, double *out)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ndof; t += (long long)gridDim.x * blockDim.x) {
        double s = lc.x0 ? lc.c0 * lc.x0[t] : 0.0;
        for (int k = 0; k < lc.n; ++k) s = fma(lc.c[k], lc.y[k][t], s);
        if (lc.w) s = fma(lc.cm, lc.w[t] / mass_e[t % npe], s);
        out[t] = s;
    }
}

// projection (Alg. 3 line 6) and its effect on the Helmholtz rhs (line 8):
// v'' = v' - M^-1 G psi ;  f_H -= lam M^-1 G psi
__global__ void k_stage_project(long long ndof, int npe, const double *mass_e, double lamH, const double *gw,
                                double *vp, double *fH)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ndof; t += (long long)gridDim.x * blockDim.x) {
        const double gn = gw[t] / mass_e[t % npe];
        vp[t] -= gn;
        fH[t] = fma(-lamH, gn, fH[t]);
    }
}

// ---------------------------------------------------------------------------
// DG divergence / gradient pair (Alg. 3 lines 5-6).  One CTA per element
// (grid-stride), element data in shared memory, sum-factorised 1-D contractions with the
// pressure basis at the velocity GLL nodes (E, E') or the velocity derivative matrix (D),
// face traces of the neighbours read from global memory (rank halos in the slowest
// direction).  Integrals on the velocity GLL grid; central fluxes; see include/dg.h.
// ---------------------------------------------------------------------------
// out = M (contracted along axis ax) in; element arrays with x fastest, extents ext[0..2]
// (ext[ax] = ni on input, no on output); M is [no][ni] row-major in shared memory.
__device__ __forceinline__ void contract(const double *in, double *out, const double *M, const int (&ext)[3], int ax,
                                         int ni, int no)
{
    int eo[3] = {ext[0], ext[1], ext[2]};
    eo[ax] = no;
    const int tot = eo[0] * eo[1] * eo[2];
    const int st = ax == 0 ? 1 : (ax == 1 ? ext[0] : ext[0] * ext[1]);  // input stride along ax
    for (int q = threadIdx.x; q < tot; q += blockDim.x) {
        const int c0 = q % eo[0], c1 = (q / eo[0]) % eo[1], c2 = q / (eo[0] * eo[1]);
        int ci[3] = {c0, c1, c2};
        const int o = ci[ax];
        ci[ax] = 0;
        const int base = ci[0] + ext[0] * (ci[1] + ext[1] * ci[2]);
        double s = 0.0;
        for (int i = 0; i < ni; ++i) s = fma(M[o * ni + i], in[base + i * st], s);
        out[q] = s;
    }
}

template <int DIM, int P>
struct PV {
    static constexpr int n = P + 1, m = P;
    static constexpr int NV = DIM == 3 ? n * n * n : n * n;   // velocity nodes per element
    static constexpr int NPp = DIM == 3 ? m * m * m : m * m;  // pressure nodes per element
};

// shared tables: ET[a][i] = E[i][a] (m x n), EdT (m x n), Em = E (n x m), DT[j][i] = D[i][j] (n x n), w (n)
template <int P>
__device__ __forceinline__ void load_pv_tables(double *ET, double *EdT, double *Em, double *DT, double *sw)
{
    constexpr int n = P + 1, m = P;
    const StTab &S = c_stab[P];
    const StTab &T = S;
    for (int t = threadIdx.x; t < m * n; t += blockDim.x) {
        const int a = t / n, i = t % n;
        ET[t] = S.E[i][a];
        EdT[t] = S.Ed[i][a];
        Em[i * m + a] = S.E[i][a];
    }
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) DT[t] = T.D[t % n][t / n];
    for (int t = threadIdx.x; t < n; t += blockDim.x) sw[t] = T.w[t];
}

// weak divergence d_a = -sum_q W_q v.grad phi^p_a + sum_F W^F {v}.n [phi^p_a]
template <int DIM, int P>
__global__ void __launch_bounds__(256) k_dg_div(const Geom g, DivGradParams a)
{
    using C = PV<DIM, P>;
    constexpr int n = C::n, m = C::m, NV = C::NV, NPp = C::NPp;
    __shared__ double ET[m * n], EdT[m * n], Em[n * m], DT[n * n], sw[n];
    __shared__ double sv[NV], b1[NV], b2[NV], acc[NPp], fc[DIM == 3 ? n * n : n], fo[DIM == 3 ? n * m : m];
    load_pv_tables<P>(ET, EdT, Em, DT, sw);
    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        __syncthreads();
        for (int q = threadIdx.x; q < NPp; q += blockDim.x) acc[q] = 0.0;
        const int ec[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                           DIM == 3 ? (int)(e / ((long long)g.Nl[0] * g.Nl[1])) : 0};
        for (int c = 0; c < DIM; ++c) {
            __syncthreads();
            for (int q = threadIdx.x; q < NV; q += blockDim.x) {
                const int i = q % n, j = (q / n) % n, k = DIM == 3 ? q / (n * n) : 0;
                double W = sw[i] * sw[j] * g.mfac;
                if (DIM == 3) W *= sw[k];
                sv[q] = W * a.v[c][e * NV + q];
            }
            __syncthreads();
            // volume: contract x, y (, z) with E^T, the direction c with (2/h_c) E'^T
            int ext[3] = {n, n, DIM == 3 ? n : 1};
            const double *src = sv;
            double *bufs[2] = {b1, b2};
            for (int d = 0; d < DIM; ++d) {
                double *dst = bufs[d & 1];
                contract(src, dst, d == c ? EdT : ET, ext, d, n, m);
                __syncthreads();
                ext[d] = m;
                src = dst;
            }
            const double sdc = g.sd[c];
            for (int q = threadIdx.x; q < NPp; q += blockDim.x) acc[q] -= sdc * src[q];
        }
        // faces normal to d: own side 1 is '-' ([phi] = +phi), side 0 is '+' ([phi] = -phi)
        for (int d = 0; d < DIM; ++d) {
            const int o1 = d == 0 ? 1 : 0, o2 = d == 2 ? 1 : 2;
            const int GS[3] = {1, n, n * n};
            const int nt = DIM == 3 ? n * n : n;
            for (int side = 0; side < 2; ++side) {
                __syncthreads();
                int cn[3] = {ec[0], ec[1], ec[2]};
                cn[d] += side ? 1 : -1;
                const double *nb = elem_ptr(g, a.v[d], a.vlo[d], a.vhi[d], cn[0], cn[1], cn[2]);
                const double *ow = a.v[d] + e * NV;
                for (int t = threadIdx.x; t < nt; t += blockDim.x) {
                    const int ta = t % n, tb = DIM == 3 ? t / n : 0;
                    const int off = ta * GS[o1] + (DIM == 3 ? tb * GS[o2] : 0);
                    double Wf = sw[ta] * g.wfac[d];
                    if (DIM == 3) Wf *= sw[tb];
                    fc[t] = Wf * 0.5 * (ow[off + (side ? P : 0) * GS[d]] + nb[off + (side ? 0 : P) * GS[d]]);
                }
                __syncthreads();
                // transverse contractions with E^T: (n [, n]) -> (m [, m]); face array axes (o1, o2)
                int ext[3] = {n, DIM == 3 ? n : 1, 1};
                contract(fc, fo, ET, ext, 0, n, m);
                __syncthreads();
                const double *fr = fo;
                if (DIM == 3) {
                    ext[0] = m;
                    contract(fo, fc, ET, ext, 1, n, m);
                    __syncthreads();
                    fr = fc;
                }
                const int PS[3] = {1, m, m * m};
                const int lay = side ? m - 1 : 0;
                for (int t = threadIdx.x; t < (DIM == 3 ? m * m : m); t += blockDim.x) {
                    const int ta = t % m, tb = DIM == 3 ? t / m : 0;
                    acc[ta * PS[o1] + (DIM == 3 ? tb * PS[o2] : 0) + lay * PS[d]] += (side ? 1.0 : -1.0) * fr[t];
                }
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < NPp; q += blockDim.x) a.out[e * NPp + q] = acc[q];
    }
}

// weak gradient g_{c,i} = -sum_q W_q psi_h d_c phi^v_i + sum_F W^F {psi_h} n_c [phi^v_i]
template <int DIM, int P>
__global__ void __launch_bounds__(256) k_dg_grad(const Geom g, DivGradParams a)
{
    using C = PV<DIM, P>;
    constexpr int n = C::n, m = C::m, NV = C::NV, NPp = C::NPp;
    __shared__ double ET[m * n], EdT[m * n], Em[n * m], DT[n * n], sw[n];
    __shared__ double sp[NV], b1[NV], b2[NV], fc[DIM == 3 ? n * n : n], fo[DIM == 3 ? n * n : n];
    load_pv_tables<P>(ET, EdT, Em, DT, sw);
    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        __syncthreads();
        for (int q = threadIdx.x; q < NPp; q += blockDim.x) sp[q] = a.psi[e * NPp + q];
        __syncthreads();
        const int ec[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                           DIM == 3 ? (int)(e / ((long long)g.Nl[0] * g.Nl[1])) : 0};
        // psi_h at the velocity nodes (b1 or b2)
        int ext[3] = {m, m, DIM == 3 ? m : 1};
        const double *src = sp;
        double *bufs[2] = {b1, b2};
        for (int d = 0; d < DIM; ++d) {
            double *dst = bufs[d & 1];
            contract(src, dst, Em, ext, d, m, n);
            __syncthreads();
            ext[d] = n;
            src = dst;
        }
        double *ph = const_cast<double *>(src);         // psi_h
        double *wph = (ph == b1) ? b2 : b1;             // W psi_h
        for (int q = threadIdx.x; q < NV; q += blockDim.x) {
            const int i = q % n, j = (q / n) % n, k = DIM == 3 ? q / (n * n) : 0;
            double W = sw[i] * sw[j] * g.mfac;
            if (DIM == 3) W *= sw[k];
            wph[q] = W * ph[q];
        }
        __syncthreads();
        for (int c = 0; c < DIM; ++c) {
            // volume: -(2/h_c) D^T along c of W psi_h -> written straight to out[c]
            const int GS[3] = {1, n, n * n};
            const double sdc = g.sd[c];
            for (int q = threadIdx.x; q < NV; q += blockDim.x) {
                const int qc[3] = {q % n, (q / n) % n, DIM == 3 ? q / (n * n) : 0};
                const int i = qc[c], base = q - i * GS[c];
                double s = 0.0;
                for (int r = 0; r < n; ++r) s = fma(DT[i * n + r], wph[base + r * GS[c]], s);
                a.gout[c][e * NV + q] = -sdc * s;
            }
            // faces normal to c
            const int d = c, o1 = d == 0 ? 1 : 0, o2 = d == 2 ? 1 : 2;
            const int PS[3] = {1, m, m * m};
            const int nt = DIM == 3 ? n * n : n, mt = DIM == 3 ? m * m : m;
            for (int side = 0; side < 2; ++side) {
                int cn[3] = {ec[0], ec[1], ec[2]};
                cn[d] += side ? 1 : -1;
                Geom gp = g;  // pressure-mesh element stride
                gp.npe = NPp;
                const double *nb = elem_ptr(gp, a.psi, a.plo, a.phi, cn[0], cn[1], cn[2]);
                __syncthreads();
                // the neighbour's pressure face layer, then its transverse interpolation
                for (int t = threadIdx.x; t < mt; t += blockDim.x) {
                    const int ta = t % m, tb = DIM == 3 ? t / m : 0;
                    fo[t] = nb[ta * PS[o1] + (DIM == 3 ? tb * PS[o2] : 0) + (side ? 0 : m - 1) * PS[d]];
                }
                __syncthreads();
                int ext2[3] = {m, DIM == 3 ? m : 1, 1};
                contract(fo, fc, Em, ext2, 0, m, n);
                __syncthreads();
                const double *fr = fc;
                if (DIM == 3) {
                    ext2[0] = n;
                    contract(fc, fo, Em, ext2, 1, m, n);
                    __syncthreads();
                    fr = fo;
                }
                for (int t = threadIdx.x; t < nt; t += blockDim.x) {
                    const int ta = t % n, tb = DIM == 3 ? t / n : 0;
                    const int off = ta * GS[o1] + (DIM == 3 ? tb * GS[o2] : 0) + (side ? P : 0) * GS[d];
                    double Wf = sw[ta] * g.wfac[d];
                    if (DIM == 3) Wf *= sw[tb];
                    a.gout[c][e * NV + off] += (side ? 1.0 : -1.0) * Wf * 0.5 * (ph[off] + fr[t]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Tiled versions (the ones dispatched): a CTA takes EPC consecutive elements, one thread per
// element line; 1-D transforms with the tables of __constant__ c_stab (uniform operands in
// fully unrolled loops), data exchanged through shared memory, coalesced global loads and
// stores; the neighbours' face layers are gathered into shared memory once per tile.
// ---------------------------------------------------------------------------
template <int DIM, int P>
struct DG2 {
    static constexpr int n = P + 1, m = P;
    static constexpr int NV = DIM == 3 ? n * n * n : n * n;
    static constexpr int NPp = DIM == 3 ? m * m * m : m * m;
    static constexpr int NL = DIM == 3 ? n * n : n;       // velocity lines per direction
    static constexpr int FV = DIM == 3 ? n * n : n;       // velocity face nodes
    static constexpr int FP = DIM == 3 ? m * m : m;       // pressure face nodes
    static constexpr int NT = 256;
    static constexpr int EPC = NT / NL > 16 ? 16 : (NT / NL < 1 ? 1 : NT / NL);
    // shared-memory element slots with an odd x pitch (pit): lines along x, y and z hit distinct
    // banks (an even pitch of 8 doubles put 16 lanes of an x-line pass on one bank pair)
    __host__ __device__ static constexpr int pit(int e) { return e % 2 ? e : e + 1; }
    static constexpr int NVS = DIM == 3 ? pit(n) * n * n : pit(n) * n;  // any array with extents <= n
    static constexpr int NPS = DIM == 3 ? pit(m) * m * m : pit(m) * m;
};

// strides of direction d in an element array with extents (e0, e1, e2), x fastest
__device__ __forceinline__ int gstride(int d, int e0, int e1) { return d == 0 ? 1 : (d == 1 ? e0 : e0 * e1); }
// the same in a shared-memory slot with the odd x pitch
__device__ __forceinline__ int pstride(int d, int e0, int e1)
{
    const int p0 = e0 % 2 ? e0 : e0 + 1;
    return d == 0 ? 1 : (d == 1 ? p0 : p0 * e1);
}
// element-local linear index (x fastest, x extent E0) -> padded slot index
template <int E0>
__device__ __forceinline__ int pidx(int t) { return t % E0 + (E0 % 2 ? E0 : E0 + 1) * (t / E0); }

// weak gradient (velocity layout) of the pressure psi, see k_dg_grad
template <int DIM, int P>
__global__ void __launch_bounds__(256, 3) k_dg_grad2(const Geom g, DivGradParams a)
{
    using C = DG2<DIM, P>;
    constexpr int n = C::n, m = C::m, NV = C::NV, NPp = C::NPp, NL = C::NL, FP = C::FP, NT = C::NT, EPC = C::EPC;
    constexpr int NVS = C::NVS, NPS = C::NPS, PN = C::pit(n), PM = C::pit(m);
    const StTab &S = c_stab[P];
    extern __shared__ double dsm[];
    double *sPs = dsm;                       // [EPC][NPS]
    double *sX = sPs + EPC * NPS;            // [EPC][NVS] (interpolation stages, output staging)
    double *sH = sX + EPC * NVS;             // [EPC][NVS] psi_h
    double *sF = sH + EPC * NVS;             // [EPC][DIM][2][FP] neighbour pressure face layers
    __shared__ const double *sNb[EPC * DIM * 2];  // face-neighbour element pointers of the tile
    const int le = threadIdx.x / NL, ln = threadIdx.x % NL;
    Geom gp = g;
    gp.npe = NPp;
    for (long long e0 = (long long)blockIdx.x * EPC; e0 < g.nel; e0 += (long long)gridDim.x * EPC) {
        const int ne = g.nel - e0 < EPC ? (int)(g.nel - e0) : EPC;
        const bool act = le < ne;
        __syncthreads();
        for (int t = threadIdx.x; t < ne * NPp; t += NT) sPs[(t / NPp) * NPS + pidx<m>(t % NPp)] = a.psi[e0 * NPp + t];
        // the tile's face-neighbour element pointers, once per (element, direction, side)
        for (int t = threadIdx.x; t < ne * DIM * 2; t += NT) {
            const int s = t % 2, d = (t / 2) % DIM, el = t / (2 * DIM);
            const long long e = e0 + el;
            int cn[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                         DIM == 3 ? (int)(e / ((long long)g.Nl[0] * g.Nl[1])) : 0};
            cn[d] += s ? 1 : -1;
            sNb[t] = elem_ptr(gp, a.psi, a.plo, a.phi, cn[0], cn[1], cn[2]);
        }
        __syncthreads();
        // neighbour face layers: element el, direction d, side s (s = 1: the +d neighbour's layer 0)
        for (int t = threadIdx.x; t < ne * DIM * 2 * FP; t += NT) {
            const int f = t % FP, r = t / FP, s = r % 2, d = (r / 2) % DIM;
            const double *nb = sNb[r];
            const int o1 = d == 0 ? 1 : 0, o2 = d == 2 ? 1 : 2;
            const int fa = f % m, fb = DIM == 3 ? f / m : 0;
            sF[t] = nb[fa * gstride(o1, m, m) + (DIM == 3 ? fb * gstride(o2, m, m) : 0) + (s ? 0 : m - 1) * gstride(d, m, m)];
        }
        __syncthreads();
        double v[n], o[n];
        // psi_h = (E (x) E (x) E) psi: x (m^(d-1) lines), y, z
        if (act && ln < (DIM == 3 ? m * m : m)) {
            const int b = le * NPS + ln * PM;
#pragma unroll
            for (int r = 0; r < m; ++r) v[r] = sPs[b + r];
#pragma unroll
            for (int i = 0; i < n; ++i) {
                double s = 0.0;
#pragma unroll
                for (int r = 0; r < m; ++r) s = fma(S.E[i][r], v[r], s);
                sX[le * NVS + ln * PN + i] = s;  // layout (i, b, c): extents (n, m, m)
            }
        }
        __syncthreads();
        if (DIM == 3) {
            if (act && ln < n * m) {  // y lines (i, c) of the (n, m, m) array -> (n, n, m)
                const int i = ln % n, c = ln / n;
#pragma unroll
                for (int r = 0; r < m; ++r) v[r] = sX[le * NVS + i + PN * (r + m * c)];
#pragma unroll
                for (int j = 0; j < n; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int r = 0; r < m; ++r) s = fma(S.E[j][r], v[r], s);
                    o[j] = s;
                }
            }
            __syncthreads();
            if (act && ln < n * m) {
                const int i = ln % n, c = ln / n;
#pragma unroll
                for (int j = 0; j < n; ++j) sX[le * NVS + i + PN * (j + n * c)] = o[j];
            }
            __syncthreads();
            if (act) {  // z lines (i, j) of (n, n, m) -> psi_h (n, n, n)
#pragma unroll
                for (int r = 0; r < m; ++r) v[r] = sX[le * NVS + ln % n + PN * (ln / n + n * r)];
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    double s = 0.0;
#pragma unroll
                    for (int r = 0; r < m; ++r) s = fma(S.E[k][r], v[r], s);
                    sH[le * NVS + ln % n + PN * (ln / n + n * k)] = s;
                }
            }
        } else {
            if (act) {  // y lines (i) of (n, m) -> (n, n)
#pragma unroll
                for (int r = 0; r < m; ++r) v[r] = sX[le * NVS + ln + PN * r];
#pragma unroll
                for (int j = 0; j < n; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int r = 0; r < m; ++r) s = fma(S.E[j][r], v[r], s);
                    sH[le * NVS + ln + PN * j] = s;
                }
            }
        }
        __syncthreads();
        // per direction d: line along d through transverse node (t1, t2) = ln
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
            const int o1 = d == 0 ? 1 : 0, o2 = d == 2 ? 1 : 2;
            const int t1 = ln % n, t2 = DIM == 3 ? ln / n : 0;
            const int GS = pstride(d, n, n);
            if (act) {
                const int base = le * NVS + t1 * pstride(o1, n, n) + (DIM == 3 ? t2 * pstride(o2, n, n) : 0);
                double Wt = S.w[t1] * g.wfac[d];  // transverse weight W^F
                if (DIM == 3) Wt *= S.w[t2];
#pragma unroll
                for (int r = 0; r < n; ++r) v[r] = sH[base + r * GS];
                // neighbour psi_h on the two faces at (t1, t2): (E (x) E) of the face layers
                double nb[2];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const double *F = sF + ((le * DIM + d) * 2 + s) * FP;
                    double acc = 0.0;
                    if (DIM == 3) {
#pragma unroll
                        for (int fb = 0; fb < m; ++fb) {
                            double ra = 0.0;
#pragma unroll
                            for (int fa = 0; fa < m; ++fa) ra = fma(S.E[t1][fa], F[fa + m * fb], ra);
                            acc = fma(S.E[t2][fb], ra, acc);
                        }
                    } else {
#pragma unroll
                        for (int fa = 0; fa < m; ++fa) acc = fma(S.E[t1][fa], F[fa], acc);
                    }
                    nb[s] = acc;
                }
                const double sdc = g.sd[d] * g.h[d] * 0.5;  // (2/h) * (h/2): W = W^F w_r h/2
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    double s = 0.0;
#pragma unroll
                    for (int r = 0; r < n; ++r) s = fma(S.D[r][k] * S.w[r], v[r], s);
                    o[k] = -sdc * Wt * s;
                }
                o[0] -= Wt * 0.5 * (v[0] + nb[0]);
                o[P] += Wt * 0.5 * (v[P] + nb[1]);
#pragma unroll
                for (int k = 0; k < n; ++k) sX[base + k * GS] = o[k];
            }
            __syncthreads();
            for (int t = threadIdx.x; t < ne * NV; t += NT) a.gout[d][e0 * NV + t] = sX[(t / NV) * NVS + pidx<n>(t % NV)];
            __syncthreads();
        }
    }
}

// weak divergence (pressure layout) of the velocity v, see k_dg_div
template <int DIM, int P>
__global__ void __launch_bounds__(256, 3) k_dg_div2(const Geom g, DivGradParams a)
{
    using C = DG2<DIM, P>;
    constexpr int n = C::n, m = C::m, NV = C::NV, NPp = C::NPp, NL = C::NL, FV = C::FV, NT = C::NT, EPC = C::EPC;
    constexpr int NVS = C::NVS, NPS = C::NPS;
    const StTab &S = c_stab[P];
    extern __shared__ double dsm[];
    double *sV = dsm;                        // [EPC][NVS] one velocity component
    double *sX = sV + EPC * NVS;             // [EPC][NVS] work
    double *sY = sX + EPC * NVS;             // [EPC][NVS] work
    double *sO = sY + EPC * NVS;             // [EPC][NPS] accumulated divergence
    double *sF = sO + EPC * NPS;             // [EPC][2][FV] neighbour velocity face layers
    __shared__ long long sNe[EPC * DIM * 2];  // face-neighbour element indices of the tile (-1 - i: halo layer i)
    const int le = threadIdx.x / NL, ln = threadIdx.x % NL;
    for (long long e0 = (long long)blockIdx.x * EPC; e0 < g.nel; e0 += (long long)gridDim.x * EPC) {
        const int ne = g.nel - e0 < EPC ? (int)(g.nel - e0) : EPC;
        const bool act = le < ne;
        __syncthreads();
        for (int t = threadIdx.x; t < ne * NPS; t += NT) sO[t] = 0.0;
        // the tile's face-neighbour elements, once per (element, direction, side): the local
        // element index, or for a slab-boundary layer of a halo mesh the halo's in-layer index
        // encoded as -1 - li (elem_ptr's convention, resolved per component below)
        for (int t = threadIdx.x; t < ne * DIM * 2; t += NT) {
            const int s = t % 2, d = (t / 2) % DIM, el = t / (2 * DIM);
            const long long e = e0 + el;
            int cn[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                         DIM == 3 ? (int)(e / ((long long)g.Nl[0] * g.Nl[1])) : 0};
            cn[d] += s ? 1 : -1;
            // pointer offset from component 0's base; elem_ptr resolves wraps and halo layers
            const double *p0 = elem_ptr(g, a.v[0], a.vlo[0], a.vhi[0], cn[0], cn[1], cn[2]);
            const bool lo = a.vlo[0] && p0 >= a.vlo[0] && p0 < a.vlo[0] + (long long)g.Nl[0] * (DIM == 3 ? g.Nl[1] : 1) * NV;
            const bool hi = a.vhi[0] && p0 >= a.vhi[0] && p0 < a.vhi[0] + (long long)g.Nl[0] * (DIM == 3 ? g.Nl[1] : 1) * NV;
            const long long off = lo ? p0 - a.vlo[0] : (hi ? p0 - a.vhi[0] : p0 - a.v[0]);
            sNe[t] = 2 * off + (lo || hi ? 1 : 0) + (hi ? 0x4000000000000000LL : 0);
        }
#pragma unroll
        for (int c = 0; c < DIM; ++c) {  // unrolled: the extents ex / ey below stay in registers
            const int o1 = c == 0 ? 1 : 0, o2 = c == 2 ? 1 : 2;
            __syncthreads();
            for (int t = threadIdx.x; t < ne * NV; t += NT) sV[(t / NV) * NVS + pidx<n>(t % NV)] = a.v[c][e0 * NV + t];
            for (int t = threadIdx.x; t < ne * 2 * FV; t += NT) {
                const int f = t % FV, s = (t / FV) % 2, el = t / (2 * FV);
                const long long code = sNe[(el * DIM + c) * 2 + s];
                const long long off = (code & 0x3FFFFFFFFFFFFFFFLL) >> 1;
                const double *base = (code & 1) ? ((code & 0x4000000000000000LL) ? a.vhi[c] : a.vlo[c]) : a.v[c];
                const double *nb = base + off;
                const int fa = f % n, fb = DIM == 3 ? f / n : 0;
                sF[t] = nb[fa * gstride(o1, n, n) + (DIM == 3 ? fb * gstride(o2, n, n) : 0) + (s ? 0 : P) * gstride(c, n, n)];
            }
            __syncthreads();
            // c lines: -(2/h_c) E'^T (W v_c) plus the face fluxes at the end layers
            const int t1 = ln % n, t2 = DIM == 3 ? ln / n : 0;
            double v[n], o[n];
            if (act) {
                const int GS = pstride(c, n, n);
                const int tb = t1 * pstride(o1, n, n) + (DIM == 3 ? t2 * pstride(o2, n, n) : 0);
                double Wt = S.w[t1] * g.wfac[c];
                if (DIM == 3) Wt *= S.w[t2];
#pragma unroll
                for (int r = 0; r < n; ++r) v[r] = sV[le * NVS + tb + r * GS];
                const double sdc = g.sd[c] * g.h[c] * 0.5;
#pragma unroll
                for (int q = 0; q < m; ++q) {
                    double s = 0.0;
#pragma unroll
                    for (int r = 0; r < n; ++r) s = fma(S.Ed[r][q] * S.w[r], v[r], s);
                    o[q] = -sdc * Wt * s;
                }
                const double *F0 = sF + (le * 2 + 0) * FV, *F1 = sF + (le * 2 + 1) * FV;
                o[0] -= Wt * 0.5 * (v[0] + F0[ln]);
                o[m - 1] += Wt * 0.5 * (v[P] + F1[ln]);
                // result (q along c; transverse n x n) -> sX with the c extent m
                int ex[3] = {n, n, n};
                ex[c] = m;
                const int ob = t1 * pstride(o1, ex[0], ex[1]) + (DIM == 3 ? t2 * pstride(o2, ex[0], ex[1]) : 0);
#pragma unroll
                for (int q = 0; q < m; ++q) sX[le * NVS + ob + q * pstride(c, ex[0], ex[1])] = o[q];
            }
            __syncthreads();
            // transverse projections with E^T along o1 (then o2): n -> m
            {
                int ex[3] = {n, n, DIM == 3 ? n : 1};
                ex[c] = m;
                // along o1: lines over the other two axes
                const int nl1 = (DIM == 3 ? ex[c] * ex[o2] : ex[c]);
                if (act && ln < nl1) {
                    const int u0 = ln % ex[c], u1 = DIM == 3 ? ln / ex[c] : 0;
                    int ey[3] = {ex[0], ex[1], ex[2]};
                    ey[o1] = m;
                    const int bi = u0 * pstride(c, ex[0], ex[1]) + (DIM == 3 ? u1 * pstride(o2, ex[0], ex[1]) : 0);
                    const int bo = u0 * pstride(c, ey[0], ey[1]) + (DIM == 3 ? u1 * pstride(o2, ey[0], ey[1]) : 0);
#pragma unroll
                    for (int r = 0; r < n; ++r) v[r] = sX[le * NVS + bi + r * pstride(o1, ex[0], ex[1])];
#pragma unroll
                    for (int q = 0; q < m; ++q) {
                        double s = 0.0;
#pragma unroll
                        for (int r = 0; r < n; ++r) s = fma(S.E[r][q], v[r], s);
                        if (DIM == 3) sY[le * NVS + bo + q * pstride(o1, ey[0], ey[1])] = s;
                        else sO[le * NPS + bo + q * pstride(o1, ey[0], ey[1])] += s;
                    }
                }
                if (DIM == 3) {
                    __syncthreads();
                    ex[o1] = m;  // now (m along c, m along o1, n along o2)
                    const int nl2 = ex[c] * ex[o1];
                    if (act && ln < nl2) {
                        const int u0 = ln % ex[c], u1 = ln / ex[c];
                        const int bi = u0 * pstride(c, ex[0], ex[1]) + u1 * pstride(o1, ex[0], ex[1]);
                        const int bo = u0 * pstride(c, m, m) + u1 * pstride(o1, m, m);
#pragma unroll
                        for (int r = 0; r < n; ++r) v[r] = sY[le * NVS + bi + r * pstride(o2, ex[0], ex[1])];
#pragma unroll
                        for (int q = 0; q < m; ++q) {
                            double s = 0.0;
#pragma unroll
                            for (int r = 0; r < n; ++r) s = fma(S.E[r][q], v[r], s);
                            sO[le * NPS + bo + q * pstride(o2, m, m)] += s;
                        }
                    }
                }
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < ne * NPp; t += NT) a.out[e0 * NPp + t] = sO[(t / NPp) * NPS + pidx<m>(t % NPp)];
    }
}

template <int DIM, bool DIV, int P>
cudaError_t dg2_launch(const Geom &g, const DivGradParams &a, cudaStream_t st)
{
    using C = DG2<DIM, P>;
    const int smem = DIV ? (int)sizeof(double) * (3 * C::EPC * C::NVS + C::EPC * C::NPS + C::EPC * 2 * C::FV)
                         : (int)sizeof(double) * (C::EPC * C::NPS + 2 * C::EPC * C::NVS + C::EPC * DIM * 2 * C::FP);
    if (smem > 227 * 1024) return cudaErrorNotSupported;
    static int resident = 0;  // persistent tiles: one full wave of CTAs
    if (!resident) {
        int dev = 0, nsm = 148, occ = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e;
        if (DIV) {
            cudaFuncSetAttribute(k_dg_div2<DIM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dg_div2<DIM, P>, C::NT, smem);
        } else {
            cudaFuncSetAttribute(k_dg_grad2<DIM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dg_grad2<DIM, P>, C::NT, smem);
        }
        if (e != cudaSuccess || occ < 1) occ = 1;
        resident = nsm * occ;
    }
    long long blocks = (g.nel + C::EPC - 1) / C::EPC;
    if (blocks > resident) blocks = resident;
    if (DIV) k_dg_div2<DIM, P><<<(int)blocks, C::NT, smem, st>>>(g, a);
    else k_dg_grad2<DIM, P><<<(int)blocks, C::NT, smem, st>>>(g, a);
    return cudaGetLastError();
}

#ifdef DG_DEVELOPMENT  // first-generation one-CTA-per-element kernels (A/B measurements only)
#define DG_DIVGRAD_V1_CASE(p)                                                                              \
    if (DG_DEV_ENV("DG_DIVGRAD_V1")) {                                                                     \
        if (DIV) k_dg_div<DIM, p><<<(int)blocks, 256, 0, st>>>(g, a);                                     \
        else k_dg_grad<DIM, p><<<(int)blocks, 256, 0, st>>>(g, a);                                        \
        return cudaGetLastError();                                                                         \
    }
#else
#define DG_DIVGRAD_V1_CASE(p)
#endif

template <int DIM, bool DIV>
cudaError_t dg_dispatch(const Geom &g, const DivGradParams &a, cudaStream_t st)
{
    const long long blocks = g.nel < 148LL * 16 ? g.nel : 148LL * 16;
    switch (g.P) {  // g: the VELOCITY geometry (degree P >= 2)
#define DG_CASE(p)                                                                                         \
    case p:                                                                                                \
        if constexpr (DG_HAS_P(p) && (DIM == 2 || 3 * (p + 1) * (p + 1) * (p + 1) * 8 <= 40 * 1024)) {     \
            DG_DIVGRAD_V1_CASE(p)                                                                          \
            return dg2_launch<DIM, DIV, p>(g, a, st);                                                      \
        } else {                                                                                           \
            return cudaErrorNotSupported;                                                                  \
        }
        DG_CASE(2) DG_CASE(3) DG_CASE(4) DG_CASE(5) DG_CASE(6) DG_CASE(7) DG_CASE(8) DG_CASE(9) DG_CASE(10)
#undef DG_CASE
    default:
        return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_stage_combine(const Geom &g, const double *mass_e, double a_ex, double c_g, double lamH,
                                 const double *v, const double *Fc, const double *Av, double *vp, double *fH,
                                 cudaStream_t st)
{
    const long long nd = g.nel * g.npe;
    const long long blocks = (nd + 255) / 256 < 148LL * 6 ? (nd + 255) / 256 : 148LL * 6;
    k_stage_combine<<<(int)blocks, 256, 0, st>>>(nd, g.npe, mass_e, a_ex, c_g, lamH, v, Fc, Av, vp, fH);
    return cudaGetLastError();
}

// one full wave of the 34-40-register streams (6 CTAs of 256 threads per SM)
static int vblocks(long long nd) { return (int)((nd + 255) / 256 < 148LL * 6 ? (nd + 255) / 256 : 148LL * 6); }

cudaError_t launch_scale_minv(const Geom &g, const double *mass_e, double c, const double *in, double *out,
                              cudaStream_t st)
{
    const long long nd = g.nel * g.npe;
    k_scale_minv<<<vblocks(nd), 256, 0, st>>>(nd, g.npe, mass_e, c, in, out);
    return cudaGetLastError();
}

cudaError_t launch_lincomb(const Geom &g, const LinComb &lc, const double *mass_e, double *out, cudaStream_t st)
{
    const long long nd = g.nel * g.npe;
    k_lincomb<<<vblocks(nd), 256, 0, st>>>(nd, g.npe, lc, mass_e, out);
    return cudaGetLastError();
}

cudaError_t launch_stage_project(const Geom &g, const double *mass_e, double lamH, const double *gw, double *vp,
                                 double *fH, cudaStream_t st)
{
    const long long nd = g.nel * g.npe;
    k_stage_project<<<vblocks(nd), 256, 0, st>>>(nd, g.npe, mass_e, lamH, gw, vp, fH);
    return cudaGetLastError();
}

cudaError_t launch_dg_div(const Geom &gv, const DivGradParams &a, cudaStream_t st)
{
    return gv.dim == 3 ? dg_dispatch<3, true>(gv, a, st) : dg_dispatch<2, true>(gv, a, st);
}

cudaError_t launch_dg_grad(const Geom &gv, const DivGradParams &a, cudaStream_t st)
{
    return gv.dim == 3 ? dg_dispatch<3, false>(gv, a, st) : dg_dispatch<2, false>(gv, a, st);
}

}  // namespace dg
