// vec.cu -- PCG vector kernels, deterministic reductions, scalar finalisation, and small
// mesh utilities (coords, mass, field checks).  All HBM-bound streaming kernels with a
// fixed grid of 148 x 8 CTAs (grid-stride), per-CTA partial sums written in a fixed
// order and reduced by one CTA in a fixed order (bitwise reproducible).
//
// Jacobi-PCG (north star; Alg. 3 lines 5/9 solves; stopping rule P:1070 read as
// ||M^-1 r||_2 <= tol ||f||_2, reading A7; lam = 0 null-space handling, reading A8).
#include <cmath>

#include "dev_common.cuh"

namespace dg {

DG_DEFINE_CONST_TABLES(upload_tables_vec)

// one full wave of 256-thread CTAs: 6 per SM for the 40-register reduction kernels, 8 per SM
// for the <= 32-register streams (a partial second wave costs up to the whole first one)
int vec_grid() { return 148 * 6; }
int vec_grid_wide() { return 148 * 8; }

namespace {

// Grid-stride loops over the DOFs of a slab track the node index q = i mod npe incrementally
// (no 64-bit division per DOF); the mesh's mass table holds m_q at [0, npe) and 1/m_q at
// [npe, 2 npe) (no double division per DOF).
struct NodeIdx {
    int q, step, npe;
    __device__ __forceinline__ NodeIdx(long long i0, long long stride, int npe_)
        : q((int)(i0 % npe_)), step((int)(stride % npe_)), npe(npe_) {}
    __device__ __forceinline__ void next()
    {
        q += step;
        if (q >= npe) q -= npe;
    }
};

template <int K>
__device__ __forceinline__ void write_partials(double (&v)[K], double *partial)
{
    __shared__ double red[32 * K];
    block_sum<K>(v, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) partial[blockIdx.x * K + k] = v[k];
}

__global__ void k_mass_moments(long long ndof, int npe, const double *__restrict__ f,
                               const double *__restrict__ me, double *partial)
{
    double v[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        const double m = __ldg(me + nq.q);
        v[0] = fma(m, f[i], v[0]);
        v[1] += m;
    }
    write_partials<2>(v, partial);
}

// partials: sum |u| and 0 (an all-zero initial guess skips the initial-residual apply)
__global__ void k_abssum(long long ndof, const double *__restrict__ u, double *partial)
{
    double v[2] = {0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x)
        v[0] += fabs(u[i]);
    write_partials<2>(v, partial);
}

__global__ void __launch_bounds__(256, 8) k_pcg_init(long long ndof, int npe, const double *__restrict__ f, const double *__restrict__ Ar,
                           double *__restrict__ r, const double *__restrict__ me, const PcgScal *s, double *partial)
{
    const double fmean = s->fmean;
    double v[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        const double m = __ldg(me + nq.q);
        const double fp = f[i] - fmean;
        const double ri = fma(m, fp, -Ar[i]);
        r[i] = ri;
        v[0] += ri;
        v[1] = fma(fp, fp, v[1]);
    }
    write_partials<2>(v, partial);
}

// lam > 0 (no mean projection) in one pass: r = M f - A u (Ar null: zero guess), z = D^-1 r
// (z null with a dinv table: z is applied on the fly later), partials [r.z, sum (r/m)^2] and
// [0, sum f^2] (the latter -> FIN_INIT, the former -> FIN_INIT2)
__global__ void __launch_bounds__(256) k_pcg_init_fused(long long ndof, int npe, const double *__restrict__ f,
                                                        const double *__restrict__ Ar, double *__restrict__ r,
                                                        const double *__restrict__ dinv, int dinv_table,
                                                        double *__restrict__ z, const double *__restrict__ me,
                                                        double *partial, double *partial2)
{
    double v[2] = {0.0, 0.0}, w[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        const double fi = f[i];
        const double ri = Ar ? fma(__ldg(me + nq.q), fi, -Ar[i]) : __ldg(me + nq.q) * fi;
        r[i] = ri;
        const double zi = (dinv_table ? __ldg(dinv + nq.q) : dinv[i]) * ri;
        if (z) z[i] = zi;
        v[0] = fma(ri, zi, v[0]);
        const double rm = ri * __ldg(me + npe + nq.q);
        v[1] = fma(rm, rm, v[1]);
        w[1] = fma(fi, fi, w[1]);
    }
    write_partials<2>(v, partial);
    write_partials<2>(w, partial2);
}

__global__ void k_pcg_init2(long long ndof, int npe, double *__restrict__ r, const double *__restrict__ dinv,
                            double *__restrict__ z, const double *__restrict__ me, const PcgScal *s, double *partial)
{
    const double rmean = s->qmean;  // FIN_INIT stores the mean of r here (lam == 0), else 0
    double v[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        const double ri = r[i] - rmean;
        r[i] = ri;
        const double zi = dinv[i] * ri;
        z[i] = zi;
        v[0] = fma(ri, zi, v[0]);
        const double rm = ri * __ldg(me + npe + nq.q);
        v[1] = fma(rm, rm, v[1]);
    }
    write_partials<2>(v, partial);
}

__global__ void k_pcg_update(long long ndof, int npe, double *__restrict__ x, double *__restrict__ r,
                             const double *__restrict__ p, const double *__restrict__ q,
                             const double *__restrict__ dinv, double *__restrict__ z, const double *__restrict__ me,
                             const PcgScal *s, double *partial)
{
    if (s->done) return;
    const double alpha = s->alpha, qmean = s->qmean;
    double v[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        x[i] = fma(alpha, p[i], x[i]);
        const double ri = fma(-alpha, q[i] - qmean, r[i]);
        r[i] = ri;
        const double zi = dinv[i] * ri;
        z[i] = zi;
        v[0] = fma(ri, zi, v[0]);
        const double rm = ri * __ldg(me + npe + nq.q);
        v[1] = fma(rm, rm, v[1]);
    }
    write_partials<2>(v, partial);
}

// split single-rank step, x update deferred by one iteration (saves a read and a write of
// p and x in the update pass): x += alpha_{k-1} p_{k-1}, then p_k = z_k + beta_{k-1} p_{k-1}
__global__ void k_pcg_pupd_x(long long ndof, double *__restrict__ x, double *__restrict__ p,
                             const double *__restrict__ z, const PcgScal *s)
{
    if (s->done) return;
    const double alpha = s->alpha, beta = s->beta;  // alpha = beta = 0 before the first iteration
    if (alpha == 0.0 && beta == 0.0) {               // p = z; p_old is not read (not initialised)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x)
            p[i] = z[i];
        return;
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x) {
        const double pi = p[i];
        x[i] = fma(alpha, pi, x[i]);
        p[i] = fma(beta, pi, z[i]);
    }
}

// r -= alpha (q - qmean) ; z = dinv r ; partials r.z, sum (r/m)^2   (x deferred, see above)
__global__ void k_pcg_update_nox(long long ndof, int npe, double *__restrict__ r, const double *__restrict__ q,
                                 const double *__restrict__ dinv, double *__restrict__ z,
                                 const double *__restrict__ me, const PcgScal *s, double *partial)
{
    if (s->done) return;
    const double alpha = s->alpha, qmean = s->qmean;
    double v[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        const double ri = fma(-alpha, q[i] - qmean, r[i]);
        r[i] = ri;
        const double zi = dinv[i] * ri;
        z[i] = zi;
        v[0] = fma(ri, zi, v[0]);
        const double rm = ri * __ldg(me + npe + nq.q);
        v[1] = fma(rm, rm, v[1]);
    }
    write_partials<2>(v, partial);
}

// constant-nu split step on a uniform periodic mesh: diag(A) is the same for every element, so
// z = D^-1 r is never stored -- dinv_t[q] (the first element's diagonal inverse) is applied on
// the fly: the update reads r, q and writes r (24 B/DOF), the p update reads x, p, r (40 B/DOF)
__global__ void __launch_bounds__(256, 8) k_pcg_update_t(long long ndof, int npe, double *__restrict__ r, const double *__restrict__ q,
                               const double *__restrict__ dinv_t, const double *__restrict__ me, const PcgScal *s,
                               double *partial)
{
    if (s->done) return;
    const double alpha = s->alpha, qmean = s->qmean;
    double v[2] = {0.0, 0.0};
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        const double ri = fma(-alpha, q[i] - qmean, r[i]);
        r[i] = ri;
        v[0] = fma(ri * __ldg(dinv_t + nq.q), ri, v[0]);
        const double rm = ri * __ldg(me + npe + nq.q);
        v[1] = fma(rm, rm, v[1]);
    }
    write_partials<2>(v, partial);
}

__global__ void k_pcg_pupd_xt(long long ndof, int npe, double *__restrict__ x, double *__restrict__ p,
                              const double *__restrict__ r, const double *__restrict__ dinv_t, const PcgScal *s)
{
    if (s->done) return;
    const double alpha = s->alpha, beta = s->beta;
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    NodeIdx nq(i0, st, npe);
    if (alpha == 0.0 && beta == 0.0) {  // before the first iteration: p = D^-1 r, p_old not read
        for (long long i = i0; i < ndof; i += st, nq.next()) p[i] = r[i] * __ldg(dinv_t + nq.q);
        return;
    }
    for (long long i = i0; i < ndof; i += st, nq.next()) {
        const double pi = p[i];
        x[i] = fma(alpha, pi, x[i]);
        p[i] = fma(beta, pi, r[i] * __ldg(dinv_t + nq.q));
    }
}

// the deferred last x update: x += alpha_k p_k once the loop stopped after an update pass
__global__ void k_pcg_xfinal(long long ndof, double *__restrict__ x, const double *__restrict__ p, const PcgScal *s)
{
    if (s->iter < 1 || (s->status != PCG_ST_CONV && s->status != PCG_ST_MAXIT)) return;
    const double alpha = s->alpha;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x)
        x[i] = fma(alpha, p[i], x[i]);
}

// p = z + beta p (multi-rank path, where the apply prologue is not used)
__global__ void k_pcg_pupd(long long ndof, double *__restrict__ p, const double *__restrict__ z, const PcgScal *s)
{
    if (s->done) return;
    const double beta = s->beta;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x)
        p[i] = fma(beta, p[i], z[i]);
}

// partial p.q and sum q (multi-rank path)
__global__ void k_dot_pq(long long ndof, const double *__restrict__ p, const double *__restrict__ q,
                         const PcgScal *s, double *partial)
{
    if (s->done) return;
    double v[2] = {0.0, 0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x) {
        v[0] = fma(p[i], q[i], v[0]);
        v[1] += q[i];
    }
    write_partials<2>(v, partial);
}

__global__ void k_shift(long long ndof, double *x, const double *shift)
{
    const double sh = *shift;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x)
        x[i] -= sh;
}

__global__ void k_recip(long long ndof, const double *d, double *dinv)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ndof; i += (long long)gridDim.x * blockDim.x)
        dinv[i] = 1.0 / d[i];
}

// single-CTA deterministic reduction of partial[G][K] -> sums[K]
__global__ void k_reduce(const double *partial, int G, int K, double *sums, const PcgScal *s)
{
    if (s && s->done) return;
    __shared__ double red[32 * 4];
    for (int k0 = 0; k0 < K; k0 += 2) {
        double v[2] = {0.0, 0.0};
        for (int gi = threadIdx.x; gi < G; gi += blockDim.x) {
            v[0] += partial[gi * K + k0];
            if (k0 + 1 < K) v[1] += partial[gi * K + k0 + 1];
        }
        block_sum<2>(v, red);
        if (threadIdx.x == 0) {
            sums[k0] = v[0];
            if (k0 + 1 < K) sums[k0 + 1] = v[1];
        }
    }
}

__device__ void finalize(int mode, const double *sums, PcgScal *s, double *hist, double *aux)
{
    switch (mode) {
    case FIN_FMEAN:
        s->sum_m = sums[1];
        s->fmean = (s->lam == 0.0) ? sums[0] / sums[1] : 0.0;
        aux[0] = s->fmean;
        break;
    case FIN_INIT:
        s->fnorm2 = sums[1];
        s->qmean = (s->lam == 0.0) ? sums[0] / (double)s->ndof_global : 0.0;
        break;
    case FIN_INIT2:
        s->rz = sums[0];
        s->res2 = sums[1];
        s->beta = 0.0;
        s->qmean = 0.0;
        s->iter = 0;
        s->done = 0;
        s->status = PCG_ST_RUN;
        if (!(sums[1] > s->tol2 * s->fnorm2)) { s->done = 1; s->status = PCG_ST_CONV; }
        else if (s->maxit <= 0) { s->done = 1; s->status = PCG_ST_MAXIT; }
        break;
    case FIN_ALPHA: {
        if (s->done) return;
        const double pq = sums[0];
        s->pq = pq;
        if (!(pq > 0.0) || !isfinite(pq) || !isfinite(s->rz)) {
            s->done = 1;
            s->status = PCG_ST_BREAKDOWN;
            return;
        }
        s->alpha = s->rz / pq;
        s->qmean = (s->lam == 0.0) ? sums[1] / (double)s->ndof_global : 0.0;
        break;
    }
    case FIN_BETA: {
        if (s->done) return;
        const double rz_new = sums[0];
        s->beta = rz_new / s->rz;
        if (s->iter < s->hist_cap) {  // Lanczos history of the first hist_cap iterations
            hist[2 * s->iter + 0] = s->alpha;
            hist[2 * s->iter + 1] = s->beta;
        }
        s->rz = rz_new;
        s->res2 = sums[1];
        s->iter += 1;
        if (!isfinite(rz_new) || !isfinite(sums[1])) { s->done = 1; s->status = PCG_ST_BREAKDOWN; }
        else if (sums[1] <= s->tol2 * s->fnorm2) { s->done = 1; s->status = PCG_ST_CONV; }
        else if (s->iter >= s->maxit) { s->done = 1; s->status = PCG_ST_MAXIT; }
        break;
    }
    case FIN_UMEAN:
        aux[0] = sums[0] / sums[1];
        break;
    case FIN_ABSSUM:
        aux[0] = sums[0];
        break;
    case FIN_NUMEAN:  // sum m nu / sum m
        s->nu_eff = sums[0] / sums[1];
        break;
    }
}

// reduce + finalize in one launch (single-rank path)
__global__ void k_reduce_fin(const double *partial, int G, int K, double *sums, int mode, PcgScal *s, double *hist,
                             double *aux)
{
    if (s->done && (mode == FIN_ALPHA || mode == FIN_BETA)) return;
    __shared__ double red[32 * 4];
    for (int k0 = 0; k0 < K; k0 += 2) {
        double v[2] = {0.0, 0.0};
        for (int gi = threadIdx.x; gi < G; gi += blockDim.x) {
            v[0] += partial[gi * K + k0];
            if (k0 + 1 < K) v[1] += partial[gi * K + k0 + 1];
        }
        block_sum<2>(v, red);
        if (threadIdx.x == 0) {
            sums[k0] = v[0];
            if (k0 + 1 < K) sums[k0 + 1] = v[1];
        }
    }
    if (threadIdx.x == 0) finalize(mode, sums, s, hist, aux);
}

__global__ void k_finalize(int mode, const double *sums, PcgScal *s, double *hist, double *aux)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) finalize(mode, sums, s, hist, aux);
}

__global__ void __launch_bounds__(256, 8) k_coords(int dim, int n, int npe, int Nl0, int Nl1, long long nel, long long el_off0, int N0, int N1,
                         double h0, double h1, double h2, long long ndof, double *xyz, int P)
{
    const DevTab &T = c_tab[P];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nel * npe; t += (long long)gridDim.x * blockDim.x) {
        const long long e = t / npe + el_off0;  // global element index
        const int q = (int)(t % npe);
        const long long ex = e % N0, ey = (e / N0) % N1, ez = e / ((long long)N0 * N1);
        const int i = q % n, j = (q / n) % n, k = q / (n * n);
        xyz[t] = ex * h0 + (T.xi[i] + 1.0) * 0.5 * h0;
        xyz[ndof + t] = ey * h1 + (T.xi[j] + 1.0) * 0.5 * h1;
        if (dim == 3) xyz[2 * ndof + t] = ez * h2 + (T.xi[k] + 1.0) * 0.5 * h2;
    }
}

__global__ void k_mass(int dim, int n, int npe, long long ndof, double h0, double h1, double h2, double *mass, int P)
{
    const DevTab &T = c_tab[P];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ndof; t += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(t % npe);
        const int i = q % n, j = (q / n) % n, k = q / (n * n);
        double m = T.w[i] * 0.5 * h0 * T.w[j] * 0.5 * h1;
        if (dim == 3) m *= T.w[k] * 0.5 * h2;
        mass[t] = m;
    }
}

__global__ void k_check(long long n, const double *x, int positive, int *bad)
{
    int b = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = x[i];
        if (!isfinite(v) || (positive && !(v > 0.0))) b = 1;
    }
    if (b) atomicOr(bad, 1);
}

inline long long nd(const Geom &g) { return g.nel * g.npe; }

}  // namespace

cudaError_t launch_mass_moments(const Geom &g, const double *f, const double *mass_e, double *partial, cudaStream_t st)
{
    k_mass_moments<<<vec_grid(), 256, 0, st>>>(nd(g), g.npe, f, mass_e, partial);
    return cudaGetLastError();
}

cudaError_t launch_abssum(const Geom &g, const double *u, double *partial, cudaStream_t st)
{
    k_abssum<<<vec_grid(), 256, 0, st>>>(nd(g), u, partial);
    return cudaGetLastError();
}

cudaError_t launch_pcg_init(const Geom &g, const double *f, const double *Ar, double *r, const double *mass_e,
                            const PcgScal *s, double *partial, cudaStream_t st)
{
    k_pcg_init<<<vec_grid(), 256, 0, st>>>(nd(g), g.npe, f, Ar, r, mass_e, s, partial);
    return cudaGetLastError();
}

cudaError_t launch_pcg_init_fused(const Geom &g, const double *f, const double *Ar, double *r, const double *dinv,
                                  int dinv_table, double *z, const double *mass_e, double *partial, double *partial2,
                                  cudaStream_t st)
{
    k_pcg_init_fused<<<vec_grid(), 256, 0, st>>>(nd(g), g.npe, f, Ar, r, dinv, dinv_table, z, mass_e, partial, partial2);
    return cudaGetLastError();
}

cudaError_t launch_pcg_init2(const Geom &g, double *r, const double *dinv, double *z, const double *mass_e,
                             const PcgScal *s, double *partial, cudaStream_t st)
{
    k_pcg_init2<<<vec_grid(), 256, 0, st>>>(nd(g), g.npe, r, dinv, z, mass_e, s, partial);
    return cudaGetLastError();
}

cudaError_t launch_pcg_update(const Geom &g, double *x, double *r, const double *p, const double *q,
                              const double *dinv, double *z, const double *mass_e, const PcgScal *s, double *partial,
                              cudaStream_t st)
{
    k_pcg_update<<<vec_grid(), 256, 0, st>>>(nd(g), g.npe, x, r, p, q, dinv, z, mass_e, s, partial);
    return cudaGetLastError();
}

cudaError_t launch_pcg_pupd(const Geom &g, double *p, const double *z, const PcgScal *s, cudaStream_t st)
{
    k_pcg_pupd<<<vec_grid_wide(), 256, 0, st>>>(nd(g), p, z, s);
    return cudaGetLastError();
}

cudaError_t launch_pcg_pupd_x(const Geom &g, double *x, double *p, const double *z, const PcgScal *s, cudaStream_t st)
{
    k_pcg_pupd_x<<<vec_grid_wide(), 256, 0, st>>>(nd(g), x, p, z, s);
    return cudaGetLastError();
}

cudaError_t launch_pcg_update_nox(const Geom &g, double *r, const double *q, const double *dinv, double *z,
                                  const double *mass_e, const PcgScal *s, double *partial, cudaStream_t st)
{
    k_pcg_update_nox<<<vec_grid(), 256, 0, st>>>(nd(g), g.npe, r, q, dinv, z, mass_e, s, partial);
    return cudaGetLastError();
}

cudaError_t launch_pcg_update_t(const Geom &g, double *r, const double *q, const double *dinv_t,
                                const double *mass_e, const PcgScal *s, double *partial, cudaStream_t st)
{
    k_pcg_update_t<<<vec_grid_wide(), 256, 0, st>>>(nd(g), g.npe, r, q, dinv_t, mass_e, s, partial);
    return cudaGetLastError();
}

cudaError_t launch_pcg_pupd_xt(const Geom &g, double *x, double *p, const double *r, const double *dinv_t,
                               const PcgScal *s, cudaStream_t st)
{
    k_pcg_pupd_xt<<<vec_grid_wide(), 256, 0, st>>>(nd(g), g.npe, x, p, r, dinv_t, s);
    return cudaGetLastError();
}

cudaError_t launch_pcg_xfinal(const Geom &g, double *x, const double *p, const PcgScal *s, cudaStream_t st)
{
    k_pcg_xfinal<<<vec_grid_wide(), 256, 0, st>>>(nd(g), x, p, s);
    return cudaGetLastError();
}

cudaError_t launch_dot_pq(const Geom &g, const double *p, const double *q, const PcgScal *s, double *partial,
                          cudaStream_t st)
{
    k_dot_pq<<<vec_grid(), 256, 0, st>>>(nd(g), p, q, s, partial);
    return cudaGetLastError();
}

cudaError_t launch_shift(const Geom &g, double *x, const double *shift, cudaStream_t st)
{
    k_shift<<<vec_grid_wide(), 256, 0, st>>>(nd(g), x, shift);
    return cudaGetLastError();
}

cudaError_t launch_recip(const Geom &g, const double *d, double *dinv, cudaStream_t st)
{
    k_recip<<<vec_grid_wide(), 256, 0, st>>>(nd(g), d, dinv);
    return cudaGetLastError();
}

cudaError_t launch_reduce_s(const double *partial, int G, int K, double *sums, const PcgScal *s, cudaStream_t st)
{
    k_reduce<<<1, 256, 0, st>>>(partial, G, K, sums, s);
    return cudaGetLastError();
}

cudaError_t launch_reduce(const double *partial, int G, int K, double *sums, cudaStream_t st)
{
    return launch_reduce_s(partial, G, K, sums, nullptr, st);
}

cudaError_t launch_reduce_fin(const double *partial, int G, int K, double *sums, int mode, PcgScal *s, double *hist,
                              double *aux, cudaStream_t st)
{
    k_reduce_fin<<<1, 256, 0, st>>>(partial, G, K, sums, mode, s, hist, aux);
    return cudaGetLastError();
}

cudaError_t launch_finalize(int mode, const double *sums, PcgScal *s, double *hist, double *aux, cudaStream_t st)
{
    k_finalize<<<1, 32, 0, st>>>(mode, sums, s, hist, aux);
    return cudaGetLastError();
}

cudaError_t launch_coords(const Geom &g, long long el_offset, double *xyz, cudaStream_t st)
{
    k_coords<<<vec_grid(), 256, 0, st>>>(g.dim, g.n, g.npe, g.Nl[0], g.Nl[1], g.nel, el_offset, g.N[0], g.N[1],
                                         g.h[0], g.h[1], g.h[2], nd(g), xyz, g.P);
    return cudaGetLastError();
}

cudaError_t launch_mass(const Geom &g, double *mass, cudaStream_t st)
{
    k_mass<<<vec_grid(), 256, 0, st>>>(g.dim, g.n, g.npe, nd(g), g.h[0], g.h[1], g.h[2], mass, g.P);
    return cudaGetLastError();
}

cudaError_t launch_check_field(long long n, const double *x, int positive, int *bad, cudaStream_t st)
{
    k_check<<<vec_grid(), 256, 0, st>>>(n, x, positive, bad);
    return cudaGetLastError();
}

}  // namespace dg
