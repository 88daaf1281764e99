// schwarz.cu -- two-level additive Schwarz preconditioner for the SIP system (SURVEY §8(f)
// NEXT-4; "Krylov-accelerated Schwarz/multigrid methods ... for solving the
// implicit pressure and diffusion problems").  Reading (both sides):
//
//     B r = sum_K R_K^T A_KK^-1 R_K r  +  P_1 A_c^+ P_1^T r,      A_c = P_1^T A P_1,
//
// non-overlapping element subdomains plus the continuous vertex-based Q1 coarse space on the
// same mesh.  B200 design (constant nu, uniform periodic mesh, N_d >= 2, N_d <= 64):
//
// * Element blocks by fast diagonalisation.  For constant nu the element block is a
//   Kronecker sum (pin Q7): A_KK = lam M(x)M(x)M + K_x(x)M(x)M + M(x)K_y(x)M + M(x)M(x)K_z
//   with the 1-D own-element line block K_d = nu (2/h_d) Kref (tables.cpp) and the GLL mass
//   M_d = diag(w h_d/2).  With K_d S_d = M_d S_d L_d, S_d^T M_d S_d = I (host, long double
//   Jacobi eigen-solver):  A_KK^-1 = (S(x)S(x)S) diag(1/(lam + L_x + L_y + L_z)) (S(x)S(x)S)^T,
//   i.e. 2 dim sum-factorised n x n contractions per element -- no face data, no halo.  The
//   kernel fuses it with the PCG residual update (r -= alpha (q - qbar)), the stopping-rule
//   and r.z partial sums and the Q1 restriction of r (2^dim hat moments per element).
// * Coarse space solve by diagonalisation.  For continuous Q1 functions every SIP face term
//   carries a jump and vanishes, and GLL_P quadrature integrates Q1 products exactly
//   (P >= 2), so A_c = lam Mc(x)Mc(x)Mc + nu (Kc(x)Mc(x)Mc + ...) with the periodic 1-D
//   circulants Kc = circ(2, -1)/h, Mc = circ(2 m00, m01) (m_ab by GLL quadrature of the
//   hats).  A real orthonormal Fourier basis diagonalises every symmetric circulant:
//   x_c = F diag(1/mu) F^T r_c, F = F_z(x)F_y(x)F_x, mu = 0 (lam = 0 constant mode) -> 0
//   (the pseudo-inverse).  Three small kernels (plane: gather + x,y transforms; column:
//   z transform, 1/mu, r_c.x_c partial (Parseval), inverse z; plane: inverse y, x).
// * The prolongation P_1 x_c is never stored: the PCG direction update p = z_b + P_1 x_c +
//   beta p evaluates the trilinear hats on the fly from the element's 2^dim vertex values
//   (L2-resident), and r.z = r.z_b + r_c.x_c.
#include <algorithm>
#include <cstdint>
#include <cmath>
#include <vector>

#include "dev_common.cuh"

namespace dg {

namespace {

// Cyclic Jacobi eigen-decomposition of a symmetric n x n matrix (long double, n <= NMAX):
// A = V diag(ev) V^T, columns of V orthonormal.
void jacobi_eig(int n, long double A[NMAX][NMAX], long double V[NMAX][NMAX], long double ev[NMAX])
{
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) V[i][j] = i == j ? 1.0L : 0.0L;
    for (int sweep = 0; sweep < 100; ++sweep) {
        long double off = 0.0L, tot = 0.0L;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                tot += A[i][j] * A[i][j];
                if (i != j) off += A[i][j] * A[i][j];
            }
        if (off <= 1e-36L * tot) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                if (fabsl(A[p][q]) < 1e-300L) continue;
                const long double th = (A[q][q] - A[p][p]) / (2.0L * A[p][q]);
                const long double t = (th >= 0 ? 1.0L : -1.0L) / (fabsl(th) + sqrtl(th * th + 1.0L));
                const long double c = 1.0L / sqrtl(t * t + 1.0L), s = t * c;
                for (int k = 0; k < n; ++k) {  // A <- J^T A J
                    const long double akp = A[k][p], akq = A[k][q];
                    A[k][p] = c * akp - s * akq;
                    A[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    const long double apk = A[p][k], aqk = A[q][k];
                    A[p][k] = c * apk - s * aqk;
                    A[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const long double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
    }
    for (int i = 0; i < n; ++i) ev[i] = A[i][i];
}

const long double PI_L = 3.14159265358979323846264338327950288L;

}  // namespace

bool schwarz_supported(const Geom &g, const char **why)
{
    for (int d = 0; d < g.dim; ++d) {
        if (g.N[d] < 2) {
            *why = "the Schwarz preconditioner needs N_d >= 2 (an N_d = 1 element is its own face neighbour)";
            return false;
        }
        if (g.N[d] > SW_NCMAX) {
            *why = "the Schwarz coarse solve supports N_d <= 64";
            return false;
        }
    }
    if (g.P < 2) {
        *why = "the Schwarz coarse operator needs P >= 2 (exact GLL quadrature of Q1 products)";
        return false;
    }
    return true;
}

void build_sw_tab(const Geom &g, double nu, SwTab *t, std::vector<double> &F)
{
    const int n = g.n, P = g.P;
    const Tab &T = host_tab(P);
    *t = SwTab{};
    t->nu = nu;
    for (int d = 0; d < 3; ++d) t->Nc[d] = d < g.dim ? g.N[d] : 1;
    for (int i = 0; i < n; ++i) {
        t->hat[0][i] = 0.5 * (1.0 - T.xi[i]);
        t->hat[1][i] = 0.5 * (1.0 + T.xi[i]);
    }
    for (int d = 0; d < g.dim; ++d) {
        // generalised eigenproblem K S = M S L via M^-1/2 K M^-1/2 (M = diag(w h/2))
        long double A[NMAX][NMAX], V[NMAX][NMAX], ev[NMAX], ms[NMAX];
        for (int i = 0; i < n; ++i) ms[i] = sqrtl((long double)T.w[i] * 0.5L * (long double)g.h[d]);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                A[i][j] = (long double)nu * (2.0L / (long double)g.h[d]) * (long double)T.Kref[i][j] / (ms[i] * ms[j]);
        // A is centro-symmetric (Kref and the GLL weights are): its eigenvectors are taken in the
        // even / odd subspaces separately, so that S[P-i][k] = +S[i][k] for the even modes
        // k < he and -S[i][k] for the odd modes k >= he (the block kernel's even-odd transforms)
        const int he = (n + 1) / 2, ho = n / 2, P = n - 1;
        long double Be[NMAX][NMAX] = {}, Bo[NMAX][NMAX] = {};  // basis columns (n x he, n x ho)
        const long double r2 = 1.0L / sqrtl(2.0L);
        for (int c = 0; c < he; ++c) {
            if (c == P - c) Be[c][c] = 1.0L;
            else Be[c][c] = Be[P - c][c] = r2;
        }
        for (int c = 0; c < ho; ++c) {
            Bo[c][c] = r2;
            Bo[P - c][c] = -r2;
        }
        auto sub = [&](long double (&Bm)[NMAX][NMAX], int m, int k0) {
            long double As[NMAX][NMAX], Vs[NMAX][NMAX], es[NMAX];
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b) {
                    long double acc = 0.0L;
                    for (int i = 0; i < n; ++i)
                        for (int j = 0; j < n; ++j) acc += Bm[i][a] * A[i][j] * Bm[j][b];
                    As[a][b] = acc;
                }
            jacobi_eig(m, As, Vs, es);
            for (int kk = 0; kk < m; ++kk) {
                ev[k0 + kk] = es[kk];
                for (int i = 0; i < n; ++i) {
                    long double acc = 0.0L;
                    for (int a = 0; a < m; ++a) acc += Bm[i][a] * Vs[a][kk];
                    V[i][k0 + kk] = acc;
                }
            }
        };
        sub(Be, he, 0);
        if (ho > 0) sub(Bo, ho, he);
        for (int i = 0; i < n; ++i) {
            t->Lam[d][i] = (double)ev[i];
            for (int k = 0; k < n; ++k) t->S[d][i * n + k] = (double)(V[i][k] / ms[i]);
        }
    }
    // coarse: 1-D circulant symbols and real orthonormal Fourier bases
    F.assign(3 * SW_NCMAX * SW_NCMAX, 0.0);
    for (int d = 0; d < 3; ++d) {
        const int N = t->Nc[d];
        double *Fd = F.data() + (size_t)d * SW_NCMAX * SW_NCMAX;  // Fd[j * N + col]
        if (d >= g.dim) {  // absent direction: identity, Kc = 0, Mc = 1
            Fd[0] = 1.0;
            t->eK[d][0] = 0.0;
            t->eM[d][0] = 1.0;
            continue;
        }
        const long double h = g.h[d];
        long double m00 = 0.0L, m01 = 0.0L;
        for (int k = 0; k < n; ++k) {
            m00 += (long double)T.w[k] * 0.5L * h * t->hat[0][k] * t->hat[0][k];
            m01 += (long double)T.w[k] * 0.5L * h * t->hat[0][k] * t->hat[1][k];
        }
        for (int col = 0; col < N; ++col) {
            // column col: k = 0 constant; (2k-1, 2k) = cos, sin of frequency k; N even: k = N/2
            int k;
            int kind;  // 0 const, 1 cos, 2 sin, 3 alternating
            if (col == 0) { k = 0; kind = 0; }
            else if (N % 2 == 0 && col == N - 1) { k = N / 2; kind = 3; }
            else { k = (col + 1) / 2; kind = (col % 2) ? 1 : 2; }
            const long double th = 2.0L * PI_L * k / N;
            t->eK[d][col] = (double)((2.0L - 2.0L * cosl(th)) / h);
            t->eM[d][col] = (double)(2.0L * m00 + 2.0L * m01 * cosl(th));
            if (k == 0) t->eK[d][col] = 0.0;
            for (int j = 0; j < N; ++j) {
                long double v;
                if (kind == 0) v = 1.0L / sqrtl((long double)N);
                else if (kind == 3) v = ((j % 2) ? -1.0L : 1.0L) / sqrtl((long double)N);
                else if (kind == 1) v = sqrtl(2.0L / N) * cosl(th * j);
                else v = sqrtl(2.0L / N) * sinl(th * j);
                Fd[j * N + col] = (double)v;
            }
        }
    }
}

namespace {

// ---------------------------------------------------------------------------
// element blocks: fast-diagonalisation solve fused with the PCG residual update.
// One thread per element line: a CTA takes EPC = 256 / n^(dim-1) consecutive elements
// (coalesced loads/stores of their contiguous nodal data), the 1-D transforms run along
// x, y (, z) with the line in registers and the n x n tables in the kernel's parameter
// space (uniform operands: no table loads), lines exchanged through shared memory
// (strides n, n^2 doubles: conflict-free for odd n).  The last direction does forward,
// 1/(lam + L) and backward in the same thread.
// ---------------------------------------------------------------------------
template <int n>
struct SwLine {
    double S[3][n * n];  // S_d[i*n + k]
    double L[3][n];
    double hat[2][n];
};

template <int DIM, int n>
struct SwCfg {
    static constexpr int NPE = DIM == 3 ? n * n * n : n * n;
    static constexpr int NL = DIM == 3 ? n * n : n;  // lines per element per direction
    static constexpr int NT = 256;
    // elements per CTA tile: <= 32 and the block kernel's dynamic shared memory (3 tiles,
    // 2 node tables, x moments) within 110 KB (two CTAs per SM at the largest degrees)
    static constexpr int epc(int e) { return (e > 1 && (3 * e * NPE + 2 * NPE + 2 * e * NL) * 8 > 110000) ? epc(e - 1) : e; }
    static constexpr int EPC0 = epc(NT / NL > 32 ? 32 : (NT / NL < 1 ? 1 : NT / NL));
    // even tiles when npe is odd: 16-byte aligned tile starts (measured: n = 7, 4 vs 5
    // elements per tile, 365 vs 370 us per Schwarz Poisson iteration on config 4)
    static constexpr int EPC = (NPE % 2 == 1 && EPC0 % 2 == 1 && EPC0 > 1) ? EPC0 - 1 : EPC0;
    static constexpr int NC = 1 << DIM;
};

// forward (TR: out[k] = sum_m S[m][k] v[m]) or backward (out[i] = sum_m S[i][m] v[m])
template <int n, bool TR>
__device__ __forceinline__ void line_xform(const double (&S)[n * n], const double (&v)[n], double (&o)[n])
{
#pragma unroll
    for (int k = 0; k < n; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < n; ++m) acc = fma(TR ? S[m * n + k] : S[k * n + m], v[m], acc);
        o[k] = acc;
    }
}

// even-odd forms of the S transforms (S[P-i][k] = +-S[i][k] for the even / odd modes, see
// build_sw_tab): half the FMAs of line_xform
template <int n>
__device__ __forceinline__ void eo_fwd(const double (&S)[n * n], const double (&v)[n], double (&o)[n])
{
    constexpr int h = n / 2, he = (n + 1) / 2, P = n - 1;
    double sp[h > 0 ? h : 1], sm[h > 0 ? h : 1];
#pragma unroll
    for (int i = 0; i < h; ++i) {
        sp[i] = v[i] + v[P - i];
        sm[i] = v[i] - v[P - i];
    }
#pragma unroll
    for (int k = 0; k < he; ++k) {
        double acc = (n % 2) ? S[h * n + k] * v[h] : 0.0;
#pragma unroll
        for (int i = 0; i < h; ++i) acc = fma(S[i * n + k], sp[i], acc);
        o[k] = acc;
    }
#pragma unroll
    for (int k = he; k < n; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < h; ++i) acc = fma(S[i * n + k], sm[i], acc);
        o[k] = acc;
    }
}

template <int n>
__device__ __forceinline__ void eo_bwd(const double (&S)[n * n], const double (&t)[n], double (&o)[n])
{
    constexpr int h = n / 2, he = (n + 1) / 2, P = n - 1;
#pragma unroll
    for (int i = 0; i < h; ++i) {
        double e = 0.0, q = 0.0;
#pragma unroll
        for (int k = 0; k < he; ++k) e = fma(S[i * n + k], t[k], e);
#pragma unroll
        for (int k = he; k < n; ++k) q = fma(S[i * n + k], t[k], q);
        o[i] = e + q;
        o[P - i] = e - q;
    }
    if (n % 2) {
        double e = 0.0;
#pragma unroll
        for (int k = 0; k < he; ++k) e = fma(S[h * n + k], t[k], e);
        o[h] = e;
    }
}

template <int DIM, int n>
struct SwBlkSmem {  // dynamic shared memory layout of k_sw_block (doubles)
    using C = SwCfg<DIM, n>;
    static constexpr int T = C::EPC * C::NPE;
    static constexpr int R = 0, Q = T, A = 2 * T, INV = 3 * T, MI = INV + C::NPE, X = MI + C::NPE;
    static constexpr int TOTAL = X + 2 * C::EPC * C::NL;
    static constexpr int BYTES = TOTAL * 8;
};

__device__ __forceinline__ void cp_async8(double *dst, const double *src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(double *dst, const double *src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Per tile: [wait for the tile's r (, q) in sR (, sQ)] -> r update in place (+ global store,
// stopping-rule partial) -> x forward (sR -> sA) and x hat moments -> [sR, sQ free: the next
// tile's cp.async prefetch is issued] -> corner moments, y forward, z forward / scale / backward
// (r.z_b = sum t^2 / (lam + L) in the same thread), y backward, x backward -> store z.
template <int DIM, int n>
__global__ void __launch_bounds__(256) k_sw_block(SwBlockParams a, const __grid_constant__ SwLine<n> L)
{
    using C = SwCfg<DIM, n>;
    using SM = SwBlkSmem<DIM, n>;
    constexpr int NPE = C::NPE, NL = C::NL, NT = C::NT, EPC = C::EPC, NC = C::NC;
    extern __shared__ double smem[];
    double *sR = smem + SM::R, *sQ = smem + SM::Q, *sA = smem + SM::A, *sInv = smem + SM::INV,
           *sMi = smem + SM::MI, *sx = smem + SM::X;
    __shared__ double red[8][2];
    // tables are built for nu = 1: K = nu (2/h) Kref scales the eigenvalues only
    const double nu_eff = a.nu_eff ? *a.nu_eff : a.nu;
    for (int t = threadIdx.x; t < NPE; t += NT) {
        const int i = t % n, j = (t / n) % n, k = DIM == 3 ? t / (n * n) : 0;
        double ls = L.L[0][i] + L.L[1][j];
        if (DIM == 3) ls += L.L[2][k];
        const double den = fma(nu_eff, ls, a.lam);
        sInv[t] = 1.0 / den;
        sMi[t] = 1.0 / a.mass_e[t];
    }
    const PcgScal *s = a.s;
    if (a.mode == SW_UPDATE && s->done) return;
    double alpha = 0.0, shift = 0.0;
    if (a.mode == SW_UPDATE) {
        alpha = s->alpha;
        shift = s->qmean;  // r -= alpha (q - qmean)
    } else if (a.mode == SW_INIT) {
        shift = s->qmean;  // FIN_INIT stores the mean of r here (lam == 0), else 0
    }
    const double *__restrict__ rsrc = a.mode == SW_APPLY ? a.rin : a.r;
    // 16-byte copies when every tile start is 16-byte aligned (even EPC npe, aligned sources)
    const bool c16 = (EPC * NPE) % 2 == 0 && (reinterpret_cast<uintptr_t>(rsrc) & 15) == 0 &&
                     (a.mode != SW_UPDATE || (reinterpret_cast<uintptr_t>(a.q) & 15) == 0);
    auto prefetch = [&](long long e0n) {
        const long long g0 = e0n * NPE;
        const int cnt = (int)((a.nel - e0n < EPC ? a.nel - e0n : EPC) * NPE);
        if (c16) {
            for (int t2 = threadIdx.x; t2 < cnt / 2; t2 += NT) {
                cp_async16(sR + 2 * t2, rsrc + g0 + 2 * t2);
                if (a.mode == SW_UPDATE) cp_async16(sQ + 2 * t2, a.q + g0 + 2 * t2);
            }
            if ((cnt & 1) && threadIdx.x == 0) {
                cp_async8(sR + cnt - 1, rsrc + g0 + cnt - 1);
                if (a.mode == SW_UPDATE) cp_async8(sQ + cnt - 1, a.q + g0 + cnt - 1);
            }
        } else {
            for (int t = threadIdx.x; t < cnt; t += NT) {
                cp_async8(sR + t, rsrc + g0 + t);
                if (a.mode == SW_UPDATE) cp_async8(sQ + t, a.q + g0 + t);
            }
        }
        cp_async_commit();
    };
    double acc_rz = 0.0, acc_res = 0.0;
    const int le = threadIdx.x / NL, ln = threadIdx.x % NL;
    const long long stride = (long long)gridDim.x * EPC;
    if ((long long)blockIdx.x * EPC < a.nel) prefetch((long long)blockIdx.x * EPC);
    for (long long e0 = (long long)blockIdx.x * EPC; e0 < a.nel; e0 += stride) {
        const int ne = a.nel - e0 < EPC ? (int)(a.nel - e0) : EPC;
        const bool act = le < ne;
        cp_async_wait_all();
        __syncthreads();  // the tile has landed; the previous tile's sA readers are done
        {
            const long long g0 = e0 * NPE;
            int tn = threadIdx.x % NPE;
            for (int t = threadIdx.x; t < ne * NPE; t += NT) {
                double ri = sR[t];
                if (a.mode == SW_UPDATE) ri = fma(-alpha, sQ[t] - shift, ri);
                else if (a.mode == SW_INIT) ri -= shift;
                if (a.mode != SW_APPLY) {
                    a.r[g0 + t] = ri;
                    sR[t] = ri;
                }
                const double rm = ri * sMi[tn];
                acc_res = fma(rm, rm, acc_res);
                tn += NT % NPE;
                if (tn >= NPE) tn -= NPE;
            }
        }
        __syncthreads();
        double v[n], o[n];
        // x forward (line j,k = ln), plus the two x hat moments of the line
        if (act) {
            const int b = le * NPE + ln * n;
#pragma unroll
            for (int m = 0; m < n; ++m) v[m] = sR[b + m];
            double h0 = 0.0, h1 = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                h0 = fma(L.hat[0][m], v[m], h0);
                h1 = fma(L.hat[1][m], v[m], h1);
            }
            sx[(le * NL + ln) * 2 + 0] = h0;
            sx[(le * NL + ln) * 2 + 1] = h1;
            eo_fwd<n>(L.S[0], v, o);
#pragma unroll
            for (int m = 0; m < n; ++m) sA[b + m] = o[m];
        }
        __syncthreads();
        if (e0 + stride < a.nel) prefetch(e0 + stride);  // sR, sQ are free now
        // corner moments rc_el[c][e] = sum_{j,k} hat_cy(j) hat_cz(k) xmoment_cx(j,k)
        if (threadIdx.x < ne * NC) {
            const int el = threadIdx.x / NC, c = threadIdx.x % NC;
            const double *xm = sx + el * NL * 2 + (c & 1);
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < (DIM == 3 ? n : 1); ++k) {
                double accj = 0.0;
#pragma unroll
                for (int j = 0; j < n; ++j) accj = fma(L.hat[(c >> 1) & 1][j], xm[2 * (j + n * k)], accj);
                acc = DIM == 3 ? fma(L.hat[(c >> 2) & 1][k], accj, acc) : accj;
            }
            a.rc_el[(long long)c * a.nel + e0 + el] = acc;
        }
        if (DIM == 3) {
            // y forward (line i,k)
            if (act) {
                const int i = ln % n, k = ln / n, b = le * NPE + i + n * n * k;
#pragma unroll
                for (int m = 0; m < n; ++m) v[m] = sA[b + m * n];
                eo_fwd<n>(L.S[1], v, o);
#pragma unroll
                for (int m = 0; m < n; ++m) sA[b + m * n] = o[m];
            }
            __syncthreads();
            // z forward, scale, z backward (line i,j); r.z_b = sum t^2 / (lam + L)
            if (act) {
                const int b = le * NPE + ln;
#pragma unroll
                for (int m = 0; m < n; ++m) v[m] = sA[b + m * n * n];
                eo_fwd<n>(L.S[2], v, o);
#pragma unroll
                for (int m = 0; m < n; ++m) {
                    const double oi = o[m] * sInv[ln + m * n * n];
                    acc_rz = fma(oi, o[m], acc_rz);
                    o[m] = oi;
                }
                eo_bwd<n>(L.S[2], o, v);
#pragma unroll
                for (int m = 0; m < n; ++m) sA[b + m * n * n] = v[m];
            }
            __syncthreads();
            // y backward
            if (act) {
                const int i = ln % n, k = ln / n, b = le * NPE + i + n * n * k;
#pragma unroll
                for (int m = 0; m < n; ++m) v[m] = sA[b + m * n];
                eo_bwd<n>(L.S[1], v, o);
#pragma unroll
                for (int m = 0; m < n; ++m) sA[b + m * n] = o[m];
            }
            __syncthreads();
        } else {
            // y forward, scale, y backward (line i)
            if (act) {
                const int b = le * NPE + ln;
#pragma unroll
                for (int m = 0; m < n; ++m) v[m] = sA[b + m * n];
                eo_fwd<n>(L.S[1], v, o);
#pragma unroll
                for (int m = 0; m < n; ++m) {
                    const double oi = o[m] * sInv[ln + m * n];
                    acc_rz = fma(oi, o[m], acc_rz);
                    o[m] = oi;
                }
                eo_bwd<n>(L.S[1], o, v);
#pragma unroll
                for (int m = 0; m < n; ++m) sA[b + m * n] = v[m];
            }
            __syncthreads();
        }
        // x backward
        if (act) {
            const int b = le * NPE + ln * n;
#pragma unroll
            for (int m = 0; m < n; ++m) v[m] = sA[b + m];
            eo_bwd<n>(L.S[0], v, o);
#pragma unroll
            for (int m = 0; m < n; ++m) sA[b + m] = o[m];
        }
        __syncthreads();
        {
            const long long g0 = e0 * NPE;
            for (int t = threadIdx.x; t < ne * NPE; t += NT) a.z[g0 + t] = sA[t];
        }
    }
    cp_async_wait_all();
    // partials: r.z_b, sum (r/m)^2 (fixed-order CTA reduction)
    acc_rz = warp_sum(acc_rz);
    acc_res = warp_sum(acc_res);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) {
        red[wid][0] = acc_rz;
        red[wid][1] = acc_res;
    }
    __syncthreads();
    if (threadIdx.x == 0 && a.partial) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < NT / 32; ++w) {
            t0 += red[w][0];
            t1 += red[w][1];
        }
        a.partial[blockIdx.x * 2 + 0] = t0;
        a.partial[blockIdx.x * 2 + 1] = t1;
    }
}

// ---------------------------------------------------------------------------
// coarse solve
// ---------------------------------------------------------------------------
// vertex (vx, vy, vz) gathers corner c = a + 2b + 4cc of element (vx - a, vy - b, vz - cc)
__device__ __forceinline__ double gather_vertex(const double *rc_el, long long nel, int dim, const int *Nc, int vx,
                                                int vy, int vz)
{
    double acc = 0.0;
    const int NC = 1 << dim;
#pragma unroll 8
    for (int c = 0; c < NC; ++c) {
        int ex = vx - (c & 1), ey = vy - ((c >> 1) & 1), ez = vz - ((c >> 2) & 1);
        if (ex < 0) ex += Nc[0];
        if (ey < 0) ey += Nc[1];
        if (ez < 0) ez += Nc[2];
        const long long e = (long long)ex + (long long)Nc[0] * (ey + (long long)Nc[1] * ez);
        acc += rc_el[(long long)c * nel + e];
    }
    return acc;
}

// plane vz: gather (single rank) or read rc, then transform along x and y (forward, F^T)
__global__ void k_sw_cfwd(SwCoarseParams a)
{
    if (a.done && *a.done) return;
    extern __shared__ double sm[];
    const SwTab *T = a.T;
    const int Nx = T->Nc[0], Ny = T->Nc[1];
    double *pl = sm, *tmp = sm + Nx * Ny, *Fx = tmp + Nx * Ny, *Fy = Fx + Nx * Nx;
    const int vz = blockIdx.x;
    for (int q = threadIdx.x; q < Nx * Nx; q += blockDim.x) Fx[q] = a.F[q];
    for (int q = threadIdx.x; q < Ny * Ny; q += blockDim.x) Fy[q] = a.F[SW_NCMAX * SW_NCMAX + q];
    for (int q = threadIdx.x; q < Nx * Ny; q += blockDim.x) {
        const int vx = q % Nx, vy = q / Nx;
        pl[q] = a.rc_el ? gather_vertex(a.rc_el, a.nel, a.dim, T->Nc, vx, vy, vz) : a.rc[(long long)vz * Nx * Ny + q];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < Nx * Ny; q += blockDim.x) {  // x: tmp[vy][kx] = sum_vx F[vx][kx] pl[vy][vx]
        const int kx = q % Nx, vy = q / Nx;
        double acc = 0.0;
        for (int j = 0; j < Nx; ++j) acc = fma(Fx[j * Nx + kx], pl[vy * Nx + j], acc);
        tmp[q] = acc;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < Nx * Ny; q += blockDim.x) {  // y
        const int kx = q % Nx, ky = q / Nx;
        double acc = 0.0;
        for (int j = 0; j < Ny; ++j) acc = fma(Fy[j * Ny + ky], tmp[j * Nx + kx], acc);
        a.chat[(long long)vz * Nx * Ny + q] = acc;
    }
}

// 32 columns (ky, kx) per CTA (blockDim 32 x 8): z transform, 1/mu, Parseval partial, inverse z
__global__ void k_sw_cz(SwCoarseParams a)
{
    if (a.done && *a.done) return;
    extern __shared__ double sm[];
    const SwTab *T = a.T;
    const int Nx = T->Nc[0], Ny = T->Nc[1], Nz = T->Nc[2], NP = Nx * Ny;
    double *col = sm, *hat = sm + 32 * Nz, *Fz = hat + 32 * Nz;
    __shared__ double red[32];
    for (int q = threadIdx.y * 32 + threadIdx.x; q < Nz * Nz; q += 32 * blockDim.y) Fz[q] = a.F[2 * SW_NCMAX * SW_NCMAX + q];
    const int p = blockIdx.x * 32 + threadIdx.x;  // plane index ky * Nx + kx
    const double nu_eff = a.nu_eff ? *a.nu_eff : a.nu;
    for (int vz = threadIdx.y; vz < Nz; vz += blockDim.y) col[vz * 32 + threadIdx.x] = p < NP ? a.chat[(long long)vz * NP + p] : 0.0;
    __syncthreads();
    double dot = 0.0;
    const int kx = p % Nx, ky = p / Nx;
    for (int kz = threadIdx.y; kz < Nz; kz += blockDim.y) {
        double acc = 0.0;
        for (int j = 0; j < Nz; ++j) acc = fma(Fz[j * Nz + kz], col[j * 32 + threadIdx.x], acc);
        double inv = 0.0;
        if (p < NP) {
            const double mx = T->eM[0][kx], my = T->eM[1][ky], mz = T->eM[2][kz];
            const double mu = a.lam * mx * my * mz +
                              nu_eff * (T->eK[0][kx] * my * mz + mx * T->eK[1][ky] * mz + mx * my * T->eK[2][kz]);
            inv = mu > 0.0 ? 1.0 / mu : 0.0;
        }
        dot = fma(acc * inv, acc, dot);
        hat[kz * 32 + threadIdx.x] = acc * inv;
    }
    __syncthreads();
    for (int vz = threadIdx.y; vz < Nz; vz += blockDim.y) {
        double acc = 0.0;
        for (int k = 0; k < Nz; ++k) acc = fma(Fz[vz * Nz + k], hat[k * 32 + threadIdx.x], acc);
        if (p < NP) a.chat[(long long)vz * NP + p] = acc;
    }
    // partial r_c . x_c = sum chat^2 / mu (orthonormal F)
    dot = warp_sum(dot);
    if (threadIdx.x == 0) red[threadIdx.y] = dot;
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0 && a.partial) {
        double t = 0.0;
        for (int w = 0; w < (int)blockDim.y; ++w) t += red[w];
        a.partial[(a.pslot + blockIdx.x) * 2 + 0] = a.count_dot ? t : 0.0;
        a.partial[(a.pslot + blockIdx.x) * 2 + 1] = 0.0;
    }
}

// plane vz: inverse y then x transform -> x_c
__global__ void k_sw_cinv(SwCoarseParams a)
{
    if (a.done && *a.done) return;
    extern __shared__ double sm[];
    const SwTab *T = a.T;
    const int Nx = T->Nc[0], Ny = T->Nc[1];
    double *pl = sm, *tmp = sm + Nx * Ny, *Fx = tmp + Nx * Ny, *Fy = Fx + Nx * Nx;
    const int vz = blockIdx.x;
    for (int q = threadIdx.x; q < Nx * Nx; q += blockDim.x) Fx[(q % Nx) * Nx + q / Nx] = a.F[q];  // transposed
    for (int q = threadIdx.x; q < Ny * Ny; q += blockDim.x) Fy[q] = a.F[SW_NCMAX * SW_NCMAX + q];
    for (int q = threadIdx.x; q < Nx * Ny; q += blockDim.x) pl[q] = a.chat[(long long)vz * Nx * Ny + q];
    __syncthreads();
    for (int q = threadIdx.x; q < Nx * Ny; q += blockDim.x) {  // y: tmp[vy][kx] = sum_ky F[vy][ky] pl[ky][kx]
        const int kx = q % Nx, vy = q / Nx;
        double acc = 0.0;
        for (int k = 0; k < Ny; ++k) acc = fma(Fy[vy * Ny + k], pl[k * Nx + kx], acc);
        tmp[q] = acc;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < Nx * Ny; q += blockDim.x) {  // x
        const int vx = q % Nx, vy = q / Nx;
        double acc = 0.0;
        for (int k = 0; k < Nx; ++k) acc = fma(Fx[k * Nx + vx], tmp[vy * Nx + k], acc);
        a.xc[(long long)vz * Nx * Ny + q] = acc;
    }
}

// multi-rank: vertex values of the local element layers (partial sums on the two boundary
// vertex layers; the caller zeroes rc and all-reduces it)
__global__ void k_sw_cgather_local(SwCoarseParams a, int S, int off, int nl)
{
    if (a.done && *a.done) return;
    const SwTab *T = a.T;
    const int *Nc = T->Nc;
    const int NC = 1 << a.dim;
    const long long lay = S == 2 ? (long long)Nc[0] * Nc[1] : (long long)Nc[0];
    const long long tot = lay * (nl + 1);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
        const int vs = off + (int)(q / lay);        // global vertex layer (may be == N_S: wraps)
        const long long in = q % lay;
        int v[3] = {(int)(in % Nc[0]), S == 2 ? (int)(in / Nc[0]) : vs, S == 2 ? vs : 0};
        double acc = 0.0;
        for (int c = 0; c < NC; ++c) {
            int ec[3] = {v[0] - (c & 1), v[1] - ((c >> 1) & 1), v[2] - ((c >> 2) & 1)};
            const int ls = ec[S] - off;             // local layer of the slowest direction
            if (ls < 0 || ls >= nl) continue;
            ec[S] = ls;
            for (int d = 0; d < S; ++d)
                if (ec[d] < 0) ec[d] += Nc[d];
            const long long e = (long long)ec[0] + (long long)Nc[0] * (ec[1] + (long long)(S == 2 ? Nc[1] : 0) * ec[2]);
            acc += a.rc_el[(long long)c * a.nel + e];
        }
        v[S] = vs % Nc[S];
        a.rc[(long long)v[0] + (long long)Nc[0] * (v[1] + (long long)Nc[1] * v[2])] += acc;
    }
}

// ---------------------------------------------------------------------------
// p = z_b + P_1 x_c + beta p  (and the deferred x += alpha p_old): a CTA takes EPC
// consecutive elements, the 2^dim vertex values of each in shared memory, coalesced
// streaming of x, z, p
// ---------------------------------------------------------------------------
template <int DIM, int n>
__global__ void __launch_bounds__(256, 4) k_sw_pupd(SwPupdParams a, const __grid_constant__ SwLine<n> L)
{
    using C = SwCfg<DIM, n>;
    constexpr int NPE = C::NPE, NT = C::NT, EPC = C::EPC, NC = C::NC;
    __shared__ double sxv[EPC][NC], sh[2][n];
    const SwTab *T = a.T;
    if (threadIdx.x < n) {
        sh[0][threadIdx.x] = L.hat[0][threadIdx.x];
        sh[1][threadIdx.x] = L.hat[1][threadIdx.x];
    }
    double alpha = 0.0, beta = 0.0;
    if (a.s) {
        if (a.s->done) return;
        alpha = a.s->alpha;
        beta = a.s->beta;
    }
    const int N0 = T->Nc[0], N1 = T->Nc[1], N2 = T->Nc[2];
    // p is updated in place (a.p_old == a.p or null): distinct streams z_b, p, x
    const bool upd = a.p_old != nullptr;
    const double *__restrict__ zb = a.zb;
    double *__restrict__ p = a.p;
    double *__restrict__ x = a.x;
    for (long long e0 = (long long)blockIdx.x * EPC; e0 < a.nel; e0 += (long long)gridDim.x * EPC) {
        const int ne = a.nel - e0 < EPC ? (int)(a.nel - e0) : EPC;
        __syncthreads();
        if (threadIdx.x < ne * NC) {
            const int el = threadIdx.x / NC, c = threadIdx.x % NC;
            const long long eg = e0 + el + a.el_off;  // global element (slab offset)
            int vx = (int)(eg % N0) + (c & 1), vy = (int)((eg / N0) % N1) + ((c >> 1) & 1),
                vz = DIM == 3 ? (int)(eg / ((long long)N0 * N1)) + ((c >> 2) & 1) : 0;
            if (vx >= N0) vx -= N0;
            if (vy >= N1) vy -= N1;
            if (vz >= N2) vz -= N2;
            sxv[el][c] = a.xc[(long long)vx + (long long)N0 * (vy + (long long)N1 * vz)];
        }
        __syncthreads();
        // all loads of the tile first (up to 3 PER doubles in flight per thread), then the
        // interpolation and the stores
        const long long g0 = e0 * NPE;
        const int cnt = ne * NPE;
        constexpr int PER = (EPC * NPE + NT - 1) / NT;
        constexpr int CH = PER < 4 ? PER : 4;  // loads in flight per chunk (register budget)
#pragma unroll 1
        for (int q0 = 0; q0 < PER; q0 += CH) {
            double rz[CH], rp[CH], rx[CH];
#pragma unroll
            for (int qq = 0; qq < CH; ++qq) {
                const int t = threadIdx.x + (q0 + qq) * NT;
                if (q0 + qq < PER && t < cnt) {
                    rz[qq] = zb[g0 + t];
                    rp[qq] = upd ? p[g0 + t] : 0.0;
                    rx[qq] = (upd && x) ? x[g0 + t] : 0.0;
                }
            }
#pragma unroll
            for (int qq = 0; qq < CH; ++qq) {
                const int t = threadIdx.x + (q0 + qq) * NT;
                if (q0 + qq < PER && t < cnt) {
                    const int el = t / NPE, tn = t - el * NPE;
                    // trilinear (bilinear) interpolation of the element's vertex values at node tn
                    const int i = tn % n, j = (tn / n) % n;
                    const double hx0 = sh[0][i], hx1 = sh[1][i], hy0 = sh[0][j], hy1 = sh[1][j];
                    const double *xv = sxv[el];
                    double zc = hy0 * fma(hx1, xv[1], hx0 * xv[0]) + hy1 * fma(hx1, xv[3], hx0 * xv[2]);
                    if (DIM == 3) {
                        const int k = tn / (n * n);
                        const double zc1 = hy0 * fma(hx1, xv[5], hx0 * xv[4]) + hy1 * fma(hx1, xv[7], hx0 * xv[6]);
                        zc = fma(sh[1][k], zc1, sh[0][k] * zc);
                    }
                    if (upd) {
                        if (x) x[g0 + t] = fma(alpha, rp[qq], rx[qq]);
                        p[g0 + t] = fma(beta, rp[qq], rz[qq] + zc);
                    } else {
                        p[g0 + t] = rz[qq] + zc;
                    }
                }
            }
        }
    }
}

template <int n>
SwLine<n> make_line(const SwTab &h)
{
    SwLine<n> L;
    for (int d = 0; d < 3; ++d) {
        for (int q = 0; q < n * n; ++q) L.S[d][q] = h.S[d][q];
        for (int q = 0; q < n; ++q) L.L[d][q] = h.Lam[d][q];
    }
    for (int q = 0; q < n; ++q) {
        L.hat[0][q] = h.hat[0][q];
        L.hat[1][q] = h.hat[1][q];
    }
    return L;
}

// CTAs of one full wave: SMs x resident CTAs per SM (at least one wave of 148)
template <class F>
int resident_ctas(F kern, int threads, int smem)
{
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
    return nsm * occ;
}

template <int DIM>
struct SwDispatch {
    template <int P>
    static cudaError_t block_p(const SwBlockParams &a, const SwTab &h, cudaStream_t st, int *grid)
    {
        constexpr int EPC = SwCfg<DIM, P + 1>::EPC;
        constexpr int smem = SwBlkSmem<DIM, P + 1>::BYTES;
        static int resident = 0;  // one wave of persistent CTAs (a partial second wave would
        if (!resident) {          // double the tail)
            cudaFuncSetAttribute(k_sw_block<DIM, P + 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            resident = resident_ctas(k_sw_block<DIM, P + 1>, 256, smem);
        }
        long long g = (a.nel + EPC - 1) / EPC;
        if (g > resident) g = resident;
        if (g < 1) g = 1;
        *grid = (int)g;
        k_sw_block<DIM, P + 1><<<(int)g, 256, smem, st>>>(a, make_line<P + 1>(h));
        return cudaGetLastError();
    }
    template <int P>
    static cudaError_t pupd_p(const SwPupdParams &a, const SwTab &h, cudaStream_t st)
    {
        constexpr int EPC = SwCfg<DIM, P + 1>::EPC;
        static int resident = 0;
        if (!resident) resident = resident_ctas(k_sw_pupd<DIM, P + 1>, 256, 0);
        long long g = (a.nel + EPC - 1) / EPC;
        if (g > resident) g = resident;
        if (g < 1) g = 1;
        k_sw_pupd<DIM, P + 1><<<(int)g, 256, 0, st>>>(a, make_line<P + 1>(h));
        return cudaGetLastError();
    }
#define DG_SW_CASES(fn, ...)                                                                                     \
    switch (P) {                                                                                                 \
    case 2: if constexpr (DG_HAS_P(2)) return fn<2>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 3: if constexpr (DG_HAS_P(3)) return fn<3>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 4: if constexpr (DG_HAS_P(4)) return fn<4>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 5: if constexpr (DG_HAS_P(5)) return fn<5>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 6: if constexpr (DG_HAS_P(6)) return fn<6>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 7: if constexpr (DG_HAS_P(7)) return fn<7>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 8: if constexpr (DG_HAS_P(8)) return fn<8>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 9: if constexpr (DG_HAS_P(9)) return fn<9>(__VA_ARGS__); else return cudaErrorNotSupported;             \
    case 10: if constexpr (DG_HAS_P(10)) return fn<10>(__VA_ARGS__); else return cudaErrorNotSupported;          \
    default: return cudaErrorInvalidValue;                                                                       \
    }
    static cudaError_t block(int P, const SwBlockParams &a, const SwTab &h, cudaStream_t st, int *grid)
    {
        DG_SW_CASES(block_p, a, h, st, grid)
    }
    static cudaError_t pupd(int P, const SwPupdParams &a, const SwTab &h, cudaStream_t st)
    {
        DG_SW_CASES(pupd_p, a, h, st)
    }
#undef DG_SW_CASES
};

}  // namespace

cudaError_t launch_sw_block(const Geom &g, const SwTab &h, const SwBlockParams &a, cudaStream_t st, int *grid)
{
    return g.dim == 3 ? SwDispatch<3>::block(g.P, a, h, st, grid) : SwDispatch<2>::block(g.P, a, h, st, grid);
}

cudaError_t launch_sw_pupd(const Geom &g, const SwTab &h, const SwPupdParams &a, cudaStream_t st)
{
    return g.dim == 3 ? SwDispatch<3>::pupd(g.P, a, h, st) : SwDispatch<2>::pupd(g.P, a, h, st);
}

int sw_cz_grid(const SwTab &h) { return (h.Nc[0] * h.Nc[1] + 31) / 32; }

cudaError_t launch_sw_coarse(const SwCoarseParams &a, const SwTab &h, int stage, cudaStream_t st)
{
    const int Nx = h.Nc[0], Ny = h.Nc[1], Nz = h.Nc[2];
    const size_t plane_smem = sizeof(double) * (2 * (size_t)Nx * Ny + (size_t)Nx * Nx + (size_t)Ny * Ny);
    static bool attr = false;
    if (!attr) {
        const int mx = (int)(sizeof(double) * (2 * SW_NCMAX * SW_NCMAX + 2 * SW_NCMAX * SW_NCMAX));
        cudaFuncSetAttribute(k_sw_cfwd, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_sw_cinv, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_sw_cz, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * (64 * SW_NCMAX + SW_NCMAX * SW_NCMAX)));
        attr = true;
    }
    // one thread per plane entry (latency-bound small transforms), one per column entry
    const int pt = std::min(1024, std::max(128, ((Nx * Ny + 31) / 32) * 32));
    const int cy = std::min(32, Nz);
    switch (stage) {
    case 0: k_sw_cfwd<<<Nz, pt, plane_smem, st>>>(a); break;
    case 1: k_sw_cz<<<sw_cz_grid(h), dim3(32, cy), sizeof(double) * (64 * (size_t)Nz + (size_t)Nz * Nz), st>>>(a); break;
    case 2: k_sw_cinv<<<Nz, pt, plane_smem, st>>>(a); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_sw_gather_local(const SwCoarseParams &a, int S, int off, int nl, cudaStream_t st)
{
    k_sw_cgather_local<<<148, 256, 0, st>>>(a, S, off, nl);
    return cudaGetLastError();
}

}  // namespace dg
