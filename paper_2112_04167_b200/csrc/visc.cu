// visc.cu -- pieces of the variable-viscosity IMEX-RK step (Alg. 3
// lines 4, 7, 8, 11; F_d2 = div(nu grad(v)^T), F_d3 = -grad(nu div v)):
//
//   k_dg_deriv   : velocity-level central-flux DG derivative (reading)
//                    (D_c u)_i = m_i^-1 [ -sum_K sum_q W_q u(x_q) d_c phi_i(x_q)
//                                         + sum_F sum_q W^F_q {u} n_c [phi_i] ]
//                  (GLL_P quadrature; -M D_c is the transpose of M D_c: skew), one CTA per
//                  element, selected directions, overwrite or accumulate;
//   k_visc_model : nu = nu0 + nu1 |v|^2 / v_max^2 at the nodes (Alg. 3 line 7);
//   k_nu_mul     : out = nu (a - b)  (the stress-like products nu D_c v_e, nu div v).
// Explicit terms evaluated once per stage: element-local, HBM/latency-bound, not on the
// per-iteration path.
#include "dev_common.cuh"

namespace dg {
DG_DEFINE_CONST_TABLES(upload_tables_visc)

namespace {

template <int DIM, int P>
__global__ void __launch_bounds__(256) k_dg_deriv(const Geom g, DerivParams a)
{
    constexpr int n = P + 1;
    constexpr int NV = DIM == 3 ? n * n * n : n * n;
    constexpr int NF = DIM == 3 ? n * n : n;
    const DevTab &T = c_tab[P];
    __shared__ double su[NV], swu[NV], DT[n * n], sw[n], fl[2][NF];
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) DT[t] = T.D[t % n][t / n];  // DT[i*n + r] = D[r][i]
    for (int t = threadIdx.x; t < n; t += blockDim.x) sw[t] = T.w[t];
    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        __syncthreads();
        for (int q = threadIdx.x; q < NV; q += blockDim.x) su[q] = a.u[e * NV + q];
        __syncthreads();
        for (int q = threadIdx.x; q < NV; q += blockDim.x) {
            const int i = q % n, j = (q / n) % n, k = DIM == 3 ? q / (n * n) : 0;
            double W = sw[i] * sw[j] * g.mfac;
            if (DIM == 3) W *= sw[k];
            swu[q] = W * su[q];
        }
        const int ec[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                           DIM == 3 ? (int)(e / ((long long)g.Nl[0] * g.Nl[1])) : 0};
        for (int c = 0; c < DIM; ++c) {
            if (!((a.dirs >> c) & 1)) continue;
            const int GS[3] = {1, n, n * n};
            const int o1 = c == 0 ? 1 : 0, o2 = c == 2 ? 1 : 2;
            __syncthreads();  // swu ready / fl free
            // the two neighbours' face layers (minus side: its node P, plus side: its node 0)
            for (int side = 0; side < 2; ++side) {
                int cn[3] = {ec[0], ec[1], ec[2]};
                cn[c] += side ? 1 : -1;
                const double *nb = elem_ptr(g, a.u, a.lo, a.hi, cn[0], cn[1], cn[2]);
                for (int t = threadIdx.x; t < NF; t += blockDim.x) {
                    const int ta = t % n, tb = DIM == 3 ? t / n : 0;
                    fl[side][t] = nb[ta * GS[o1] + (DIM == 3 ? tb * GS[o2] : 0) + (side ? 0 : P) * GS[c]];
                }
            }
            __syncthreads();
            const double sdc = g.sd[c];
            for (int q = threadIdx.x; q < NV; q += blockDim.x) {
                const int qc[3] = {q % n, (q / n) % n, DIM == 3 ? q / (n * n) : 0};
                const int i = qc[c], base = q - i * GS[c];
                // volume: -(u, d_c phi_i) = -(2/h_c) sum_r D[r][i] (W u)_r
                double s = 0.0;
#pragma unroll
                for (int r = 0; r < n; ++r) s = fma(DT[i * n + r], swu[base + r * GS[c]], s);
                double val = -sdc * s;
                // faces normal to c: +-W^F {u} at the face nodes
                if (i == 0 || i == P) {
                    const int side = i == P ? 1 : 0;
                    const int t = qc[o1] + (DIM == 3 ? qc[o2] * n : 0);
                    double Wf = sw[qc[o1]] * g.wfac[c];
                    if (DIM == 3) Wf *= sw[qc[o2]];
                    val += (side ? 1.0 : -1.0) * Wf * 0.5 * (su[q] + fl[side][t]);
                }
                double W = sw[qc[0]] * sw[qc[1]] * g.mfac;
                if (DIM == 3) W *= sw[qc[2]];
                double *o = a.out[c] + e * NV + q;
                const double r = a.scale * val / W;
                *o = a.accumulate ? *o + r : r;
            }
        }
    }
}

__global__ void k_visc_model(long long nd, int dim, const double *vx, const double *vy, const double *vz, double nu0,
                             double c1, double *nu)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nd; t += (long long)gridDim.x * blockDim.x) {
        double s = vx[t] * vx[t] + vy[t] * vy[t];
        if (dim == 3) s = fma(vz[t], vz[t], s);
        nu[t] = fma(c1, s, nu0);
    }
}

__global__ void k_nu_mul(long long nd, const double *nu, const double *x, const double *y, double *out)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nd; t += (long long)gridDim.x * blockDim.x)
        out[t] = nu[t] * (y ? x[t] - y[t] : x[t]);
}

int vgrid(long long nd) { return (int)((nd + 255) / 256 < 148LL * 16 ? (nd + 255) / 256 : 148LL * 16); }

}  // namespace

cudaError_t launch_dg_deriv(const Geom &g, const DerivParams &a, cudaStream_t st)
{
    const long long blocks = g.nel < 148LL * 16 ? g.nel : 148LL * 16;
    switch (g.P) {
#define DG_CASE(p)                                                                                   \
    case p:                                                                                          \
        if constexpr (DG_HAS_P(p)) {                                                                 \
            if (g.dim == 3) k_dg_deriv<3, p><<<(int)blocks, 256, 0, st>>>(g, a);                     \
            else k_dg_deriv<2, p><<<(int)blocks, 256, 0, st>>>(g, a);                                \
            return cudaGetLastError();                                                               \
        } else {                                                                                     \
            return cudaErrorNotSupported;                                                            \
        }
        DG_CASE(1) DG_CASE(2) DG_CASE(3) DG_CASE(4) DG_CASE(5) DG_CASE(6) DG_CASE(7) DG_CASE(8) DG_CASE(9)
        DG_CASE(10)
#undef DG_CASE
    default:
        return cudaErrorInvalidValue;
    }
}

cudaError_t launch_visc_model(const Geom &g, const double *const v[3], double nu0, double nu1, double vmax, double *nu,
                              cudaStream_t st)
{
    const long long nd = g.nel * g.npe;
    k_visc_model<<<vgrid(nd), 256, 0, st>>>(nd, g.dim, v[0], v[1], g.dim == 3 ? v[2] : nullptr, nu0,
                                            nu1 / (vmax * vmax), nu);
    return cudaGetLastError();
}

cudaError_t launch_nu_mul(const Geom &g, const double *nu, const double *x, const double *y, double *out,
                          cudaStream_t st)
{
    const long long nd = g.nel * g.npe;
    k_nu_mul<<<vgrid(nd), 256, 0, st>>>(nd, nu, x, y, out);
    return cudaGetLastError();
}

}  // namespace dg
