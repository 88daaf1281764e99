// stage.cu -- element-local pieces of the config-4 IMEX-RK stage (
// Alg. 3 lines 4-9; DESIGN.md §9 "stage composition").
//
//   k_stage_combine : F_d1 = -M^-1 (A_0 v)            (nodal viscous term, P:693 F_d1 = div nu grad v)
//                     v'   = v + dt a^ex_21 (F_c + F_d1)            (Alg. 3 line 4, F_s = 0)
//                     g    = v' + dt (a^im_21 - a^ex_21) F_d1       (Alg. 3 line 8, v'' = v')
//                     f_H  = g / (dt a^im_22)                       (reading A4: f = lam g)
//   k_div_interp    : the stand-in pressure rhs of Alg. 3 line 5 until the DG divergence
//                      lands: the broken (element-local collocation) divergence
//                     of v' at the velocity GLL nodes, interpolated to the GLL nodes of the
//                     pressure degree P-1, sign-flipped for the positive operator
//                     (-lap psi = -div v').  The mass weighting and mean projection are done
//                     by dg_pcg_solve (reading A8).
#include "dev_common.cuh"

namespace dg {
DG_DEFINE_CONST_TABLES(upload_tables_stage)

// interpolation from the degree-P GLL nodes to the degree-(P-1) GLL nodes:
// I[a][i] = l_i(xi'_a), barycentric form in long double
struct StTab {
    double I[NMAX][NMAX];
};
static __constant__ StTab c_stab[PMAX + 1];

cudaError_t upload_tables_stage_interp()
{
    static StTab h[PMAX + 1];
    for (int P = 2; P <= PMAX; ++P) {
        const Tab &t = host_tab(P), &tp = host_tab(P - 1);
        const int n = P + 1;
        long double bw[NMAX];
        for (int j = 0; j < n; ++j) {
            long double b = 1.0L;
            for (int m = 0; m < n; ++m)
                if (m != j) b *= (long double)t.xi[j] - (long double)t.xi[m];
            bw[j] = 1.0L / b;
        }
        for (int a = 0; a < P; ++a) {
            const long double x = tp.xi[a];
            int hit = -1;
            for (int j = 0; j < n; ++j)
                if (x == (long double)t.xi[j]) hit = j;
            long double den = 0.0L, num[NMAX];
            for (int j = 0; j < n; ++j) {
                num[j] = hit >= 0 ? (j == hit ? 1.0L : 0.0L) : bw[j] / (x - (long double)t.xi[j]);
                den += num[j];
            }
            for (int j = 0; j < n; ++j) h[P].I[a][j] = hit >= 0 ? (double)num[j] : (double)(num[j] / den);
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

// one CTA per element: div at the velocity nodes in shared memory, then three (two)
// interpolation passes P -> P-1
template <int DIM, int P>
__global__ void __launch_bounds__(256) k_div_interp(const Geom g, const double *v0, const double *v1, const double *v2,
                                                     double *fp)
{
    constexpr int n = P + 1, m = P;  // velocity / pressure nodes per direction
    constexpr int NPE = DIM == 3 ? n * n * n : n * n;
    constexpr int MPE = DIM == 3 ? m * m * m : m * m;
    const DevTab &T = c_tab[P];
    const StTab &S = c_stab[P];
    __shared__ double sv[3][NPE];
    __shared__ double sa[NPE], sb[NPE];
    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        for (int q = threadIdx.x; q < NPE; q += blockDim.x) {
            sv[0][q] = v0[e * NPE + q];
            sv[1][q] = v1[e * NPE + q];
            if (DIM == 3) sv[2][q] = v2[e * NPE + q];
        }
        __syncthreads();
        for (int q = threadIdx.x; q < NPE; q += blockDim.x) {
            const int i = q % n, j = (q / n) % n, k = DIM == 3 ? q / (n * n) : 0;
            double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
            for (int r = 0; r < n; ++r) {
                d0 = fma(T.D[i][r], sv[0][q + (r - i)], d0);
                d1 = fma(T.D[j][r], sv[1][q + (r - j) * n], d1);
                if (DIM == 3) d2 = fma(T.D[k][r], sv[2][q + (r - k) * n * n], d2);
            }
            sa[q] = g.sd[0] * d0 + g.sd[1] * d1 + (DIM == 3 ? g.sd[2] * d2 : 0.0);
        }
        __syncthreads();
        // x: sa[k][j][i] -> sb[k][j][a]
        for (int q = threadIdx.x; q < (DIM == 3 ? n * n * m : n * m); q += blockDim.x) {
            const int a = q % m, r = q / m;  // r = j + n k
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < n; ++i) s = fma(S.I[a][i], sa[r * n + i], s);
            sb[r * m + a] = s;
        }
        __syncthreads();
        // y: sb[k][j][a] -> sa[k][b][a]
        for (int q = threadIdx.x; q < (DIM == 3 ? n * m * m : m * m); q += blockDim.x) {
            const int a = q % m, b = (q / m) % m, k = q / (m * m);
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < n; ++j) s = fma(S.I[b][j], sb[(k * n + j) * m + a], s);
            sa[(k * m + b) * m + a] = s;
        }
        __syncthreads();
        if (DIM == 3) {  // z: sa[k][b][a] -> out[c][b][a]
            for (int q = threadIdx.x; q < MPE; q += blockDim.x) {
                const int ab = q % (m * m), c = q / (m * m);
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < n; ++k) s = fma(S.I[c][k], sa[k * m * m + ab], s);
                fp[e * MPE + q] = -s;
            }
        } else {
            for (int q = threadIdx.x; q < MPE; q += blockDim.x) fp[e * MPE + q] = -sa[q];
        }
        __syncthreads();
    }
}

template <int DIM>
cudaError_t div_dispatch(const Geom &g, const double *v0, const double *v1, const double *v2, double *fp,
                         cudaStream_t st)
{
    const long long blocks = g.nel < 148LL * 16 ? g.nel : 148LL * 16;
    switch (g.P) {
#define DG_CASE(p)                                                                          \
    case p:                                                                                 \
        if constexpr (DG_HAS_P(p) && (DIM == 2 || 5 * (p + 1) * (p + 1) * (p + 1) * 8 <= 48 * 1024)) { \
            k_div_interp<DIM, p><<<(int)blocks, 256, 0, st>>>(g, v0, v1, v2, fp);           \
            return cudaGetLastError();                                                      \
        } else {                                                                            \
            return cudaErrorNotSupported;                                                   \
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
    const long long blocks = (nd + 255) / 256 < 148LL * 16 ? (nd + 255) / 256 : 148LL * 16;
    k_stage_combine<<<(int)blocks, 256, 0, st>>>(nd, g.npe, mass_e, a_ex, c_g, lamH, v, Fc, Av, vp, fH);
    return cudaGetLastError();
}

cudaError_t launch_div_interp(const Geom &g, const double *v0, const double *v1, const double *v2, double *fp,
                              cudaStream_t st)
{
    return g.dim == 3 ? div_dispatch<3>(g, v0, v1, v2, fp, st) : div_dispatch<2>(g, v0, v1, v2, fp, st);
}

}  // namespace dg
