// stab.cu -- divergence / mass-flux stabilisation of the projection step (
// PAPER.md:1040 "for pressure robustness a divergence/mass-flux stabilization is added as
// proposed in [Joshi 2016, Akbas 2018]"; reading A26 in DESIGN.md §2):
//
//   (M + a_D K_D + a_C K_C) v^ = M v'',
//   (K_D v)_{c,I} = sum_K sum_q W_q (div v)(x_q) d_c phi_I(x_q)     (broken divergence, GLL_P)
//   (K_C v)_{c,I} = sum_{F normal to c} sum_q W^F_q [v_c] [phi_I]     (normal-velocity jumps)
//
// solved by Jacobi-preconditioned CG over the dim velocity components at once.
//
// k_stab_apply: one CTA per element (grid-stride over a resident grid): the element's velocity
// components are staged in shared memory, every node computes a_D W_q div_q (dim n-term
// derivative dot products), then every (component, node) its row: m_I v + the D^T contraction
// of a_D W div along the component's direction + a_C W_perp [v_c] at the two faces normal to
// it (the neighbour's face value from global memory / the rank halo layer), with the CG dot
// epilogue p.q.  Once per stage (a few CG iterations at the convective CFL): HBM-bound.
// The Jacobi diagonal is a per-node table (uniform mesh, constant coefficients): z = D^-1 r is
// never stored.
#include "dev_common.cuh"

namespace dg {

DG_DEFINE_CONST_TABLES(upload_tables_stab)

namespace {

// grid-stride DOF loops track the node index q = i mod npe incrementally (no 64-bit division)
struct NodeQ {
    int q, step, npe;
    __device__ __forceinline__ NodeQ(long long i0, long long stride, int npe_)
        : q((int)(i0 % npe_)), step((int)(stride % npe_)), npe(npe_) {}
    __device__ __forceinline__ void next()
    {
        q += step;
        if (q >= npe) q -= npe;
    }
};

template <int K>
__device__ __forceinline__ void write_partials_s(double (&v)[K], double *partial)
{
    __shared__ double red[32 * K];
    block_sum<K>(v, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) partial[blockIdx.x * K + k] = v[k];
}

template <int DIM, int P>
__global__ void __launch_bounds__(256, 6) k_stab_apply(const Geom g, StabParams a)
{
    constexpr int n = P + 1, NPE = DIM == 3 ? n * n * n : n * n;
    const DevTab &T = c_tab[P];
    __shared__ double sv[DIM][NPE];
    __shared__ double swd[NPE];
    __shared__ double sD[n][n], sw[n];  // per-thread row indices: shared, not the constant bank
    double dot = 0.0;
    if (a.s && a.s->done) return;
    for (int q = threadIdx.x; q < n * n; q += blockDim.x) {
        sD[q / n][q % n] = T.D[q / n][q % n];
        if (q < n) sw[q] = T.w[q];
    }
    for (long long e = blockIdx.x; e < g.nel; e += gridDim.x) {
        for (int q = threadIdx.x; q < DIM * NPE; q += blockDim.x) {
            const int c = q / NPE, I = q - c * NPE;
            sv[c][I] = __ldg(a.in[c] + e * NPE + I);
        }
        __syncthreads();
        for (int q = threadIdx.x; q < NPE; q += blockDim.x) {
            const int qc[3] = {q % n, (q / n) % n, DIM == 3 ? q / (n * n) : 0};
            double div = 0.0, W = g.mfac;
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
                const int GS = d == 0 ? 1 : (d == 1 ? n : n * n);
                const int base = q - qc[d] * GS;
                double t = 0.0;
#pragma unroll
                for (int j = 0; j < n; ++j) t = fma(sD[qc[d]][j], sv[d][base + j * GS], t);
                div = fma(g.sd[d], t, div);
                W *= sw[qc[d]];
            }
            swd[q] = a.aD * W * div;
        }
        __syncthreads();
        const int ec[3] = {(int)(e % g.Nl[0]), (int)((e / g.Nl[0]) % g.Nl[1]),
                           DIM == 3 ? (int)(e / ((long long)g.Nl[0] * g.Nl[1])) : 0};
        for (int q = threadIdx.x; q < DIM * NPE; q += blockDim.x) {
            const int c = q / NPE, I = q - c * NPE;
            const int qc[3] = {I % n, (I / n) % n, DIM == 3 ? I / (n * n) : 0};
            const int GS = c == 0 ? 1 : (c == 1 ? n : n * n);
            const int i = qc[c], base = I - i * GS;
            double m = g.mfac;
#pragma unroll
            for (int d = 0; d < DIM; ++d) m *= sw[qc[d]];
            const double vi = sv[c][I];
            double t = 0.0;  // sum_k (2/h_c) D[k][i] (a_D W div)(k along c)
#pragma unroll
            for (int k = 0; k < n; ++k) t = fma(sD[k][i], swd[base + k * GS], t);
            double acc = fma(g.sd[c], t, m * vi);
            if (i == P || i == 0) {  // [v_c][phi_I] on the face normal to c through I
                int cn[3] = {ec[0], ec[1], ec[2]};
                cn[c] += i == P ? 1 : -1;
                const double *nb = elem_ptr(g, a.in[c], a.lo[c], a.hi[c], cn[0], cn[1], cn[2]);
                const double vn = __ldg(nb + base + (i == P ? 0 : P * GS));
                const double Wp = m / (sw[i] * 0.5 * g.h[c]);
                acc = fma(a.aC * Wp, vi - vn, acc);
            }
            a.out[c][e * NPE + I] = acc;
            dot = fma(vi, acc, dot);
        }
        __syncthreads();
    }
    if (a.partial) {
        double v[2] = {dot, 0.0};
        write_partials_s<2>(v, a.partial);
    }
}

// r = M x - q (x = v'', q = A x), partials [r . D^-1 r, sum (r/m)^2] and [0, sum x^2]
__global__ void __launch_bounds__(256) k_stab_init(StabVec a)
{
    double v[2] = {0.0, 0.0}, f[2] = {0.0, 0.0};
    for (int c = 0; c < a.dim; ++c) {
        const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
        NodeQ nq(i0, st, a.npe);
        for (long long i = i0; i < a.ndof; i += st, nq.next()) {
            const int q = nq.q;
            const double x = a.x[c][i];
            const double r = fma(__ldg(a.mass_e + q), x, -a.q[c * a.ndof + i]);
            a.r[c * a.ndof + i] = r;
            const double mi = __ldg(a.mass_e + a.npe + q);
            v[0] = fma(r * r, __ldg(a.dinv + c * a.npe + q), v[0]);
            v[1] = fma(r * mi, r * mi, v[1]);
            f[1] = fma(x, x, f[1]);
        }
    }
    write_partials_s<2>(v, a.partial);
    write_partials_s<2>(f, a.partial2);
}

// p = D^-1 r + beta p
__global__ void __launch_bounds__(256) k_stab_pupd(StabVec a)
{
    if (a.s->done) return;
    const double beta = a.s->beta;
    for (int c = 0; c < a.dim; ++c) {
        const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
        NodeQ nq(i0, st, a.npe);
        const double *dv = a.dinv + c * a.npe;
        double *p = a.p + c * a.ndof;
        const double *r = a.r + c * a.ndof;
        for (long long i = i0; i < a.ndof; i += st, nq.next()) p[i] = fma(beta, p[i], __ldg(dv + nq.q) * r[i]);
    }
}

// x += alpha p ; r -= alpha q ; partials r . D^-1 r, sum (r/m)^2
__global__ void __launch_bounds__(256) k_stab_update(StabVec a)
{
    if (a.s->done) return;
    const double alpha = a.s->alpha;
    double v[2] = {0.0, 0.0};
    for (int c = 0; c < a.dim; ++c) {
        const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
        NodeQ nq(i0, st, a.npe);
        for (long long i = i0; i < a.ndof; i += st, nq.next()) {
            const int q = nq.q;
            const long long k = c * a.ndof + i;
            a.x[c][i] = fma(alpha, a.p[k], a.x[c][i]);
            const double r = fma(-alpha, a.q[k], a.r[k]);
            a.r[k] = r;
            const double mi = __ldg(a.mass_e + a.npe + q);
            v[0] = fma(r * r, __ldg(a.dinv + c * a.npe + q), v[0]);
            v[1] = fma(r * mi, r * mi, v[1]);
        }
    }
    write_partials_s<2>(v, a.partial);
}

// partials [sum m |v|^2, sum m] (the RMS velocity of reading A26)
__global__ void __launch_bounds__(256) k_stab_u2(StabVec a)
{
    double v[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeQ nq(i0, st, a.npe);
    for (long long i = i0; i < a.ndof; i += st, nq.next()) {
        const double m = __ldg(a.mass_e + nq.q);
        double s2 = 0.0;
        for (int c = 0; c < a.dim; ++c) s2 = fma(a.x[c][i], a.x[c][i], s2);
        v[0] = fma(m, s2, v[0]);
        v[1] += m;
    }
    write_partials_s<2>(v, a.partial);
}

}  // namespace

int stab_grid() { return 148 * 4; }

cudaError_t launch_stab_apply(const Geom &g, const StabParams &a, cudaStream_t st, int *grid)
{
    // one resident wave of CTAs (one element per CTA in flight: more CTAs per SM hide the load
    // latency of the next element); the partial-sum count stays <= 148 * 6
    int nsm = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const long long cap = (long long)nsm * 6;
    const long long blocks = g.nel < cap ? g.nel : cap;
    if (grid) *grid = (int)blocks;
    switch (g.P) {
#define DG_SA(p)                                                                                       \
    case p:                                                                                            \
        if constexpr (DG_HAS_P(p)) {                                                                   \
            if (g.dim == 3) {                                                                          \
                if constexpr (4 * (p + 1) * (p + 1) * (p + 1) * 8 <= 48 * 1024)                        \
                    k_stab_apply<3, p><<<(int)blocks, 256, 0, st>>>(g, a);                             \
                else                                                                                   \
                    return cudaErrorNotSupported;                                                      \
            } else {                                                                                   \
                k_stab_apply<2, p><<<(int)blocks, 256, 0, st>>>(g, a);                                 \
            }                                                                                          \
            return cudaGetLastError();                                                                 \
        } else {                                                                                       \
            return cudaErrorNotSupported;                                                              \
        }
        DG_SA(1) DG_SA(2) DG_SA(3) DG_SA(4) DG_SA(5) DG_SA(6) DG_SA(7) DG_SA(8) DG_SA(9) DG_SA(10)
#undef DG_SA
    default:
        return cudaErrorInvalidValue;
    }
}

cudaError_t launch_stab_vec(int op, const StabVec &a, cudaStream_t st)
{
    const int G = stab_grid();
    switch (op) {
    case STAB_INIT: k_stab_init<<<G, 256, 0, st>>>(a); break;
    case STAB_PUPD: k_stab_pupd<<<148 * 8, 256, 0, st>>>(a); break;
    case STAB_UPDATE: k_stab_update<<<G, 256, 0, st>>>(a); break;
    case STAB_U2: k_stab_u2<<<G, 256, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace dg
