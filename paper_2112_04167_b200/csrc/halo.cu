// halo.cu -- face traces of a slab's boundary layers for the multi-rank (and 1-rank halo-mode)
// operator application ("send per face node (u, nu d_n u), 2 FP64 values";
// P:1044 element decomposition with MPI, replaced by NCCL over NVLink).
//
// One thread per face node of the slowest direction S: it reads its S-line of the boundary
// element (n values, coalesced across the face), and writes the trace in the layout of
// dg_internal.h Halo: u at the face node, s = nu (2/h_S) (D u)_node (physical derivative along
// +S) and nu.  The receiving rank's apply / diagonal kernels consume exactly these values
// where they would otherwise compute them from the neighbour element's line.
#include "dev_common.cuh"

namespace dg {

DG_DEFINE_CONST_TABLES(upload_tables_halo)

namespace {

template <int P>
__global__ void __launch_bounds__(256) k_slab_traces(const Geom g, const double *__restrict__ u,
                                                     const double *__restrict__ nu, double nu_const,
                                                     double *__restrict__ slo, double *__restrict__ shi, int with_nu)
{
    constexpr int n = P + 1;
    const DevTab &T = c_tab[P];
    const int S = g.dim - 1;
    const int NF = g.dim == 3 ? n * n : n;                 // face nodes per element = node stride along S
    const long long lay = g.dim == 3 ? (long long)g.Nl[0] * g.Nl[1] : (long long)g.Nl[0];
    const long long F = lay * NF;
    const double sd = g.sd[S];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < 2 * F;
         t += (long long)gridDim.x * blockDim.x) {
        const int side = t >= F;                            // 0: bottom face of layer 0, 1: top of the last
        const long long f = t - side * F;
        const long long fe = f / NF;
        const int in = (int)(f - fe * NF);
        const long long e = fe + (side ? (long long)(g.Nl[S] - 1) * lay : 0);
        const double *pu = u + e * g.npe + in;
        double v[n];
#pragma unroll
        for (int k = 0; k < n; ++k) v[k] = __ldg(pu + k * NF);
        const int node = side ? P : 0;
        double d = 0.0;
#pragma unroll
        for (int j = 0; j < n; ++j) d = fma(T.D[node][j], v[j], d);
        const double nv = nu ? __ldg(nu + e * g.npe + in + node * NF) : nu_const;
        double *o = side ? shi : slo;
        o[f] = v[node];
        o[F + f] = nv * sd * d;
        if (with_nu) o[2 * F + f] = nv;
    }
}

}  // namespace

cudaError_t launch_slab_traces(const Geom &g, const double *u, const double *nu, double nu_const, double *send_lo,
                               double *send_hi, int with_nu, cudaStream_t st)
{
    const int n = g.P + 1;
    const long long F = (g.dim == 3 ? (long long)g.Nl[0] * g.Nl[1] * n * n : (long long)g.Nl[0] * n);
    long long blocks = (2 * F + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    switch (g.P) {
#define DG_TR(p)                                                                                              \
    case p:                                                                                                   \
        if constexpr (DG_HAS_P(p)) {                                                                          \
            k_slab_traces<p><<<(int)blocks, 256, 0, st>>>(g, u, nu, nu_const, send_lo, send_hi, with_nu);    \
            return cudaGetLastError();                                                                        \
        } else {                                                                                              \
            return cudaErrorNotSupported;                                                                     \
        }
        DG_TR(1) DG_TR(2) DG_TR(3) DG_TR(4) DG_TR(5) DG_TR(6) DG_TR(7) DG_TR(8) DG_TR(9) DG_TR(10)
#undef DG_TR
    default:
        return cudaErrorInvalidValue;
    }
}

}  // namespace dg
