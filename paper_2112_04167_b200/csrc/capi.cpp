// capi.cpp -- the C-ABI of libdgsip.so (include/dg.h): mesh/workspace ownership, kernel
// orchestration on the caller's stream, the Jacobi-PCG driver with device-resident
// scalars, NCCL halo exchange / allreduce for slab-partitioned meshes, and error plumbing.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "dg_internal.h"

namespace dg {

thread_local std::string g_err;
thread_local char g_last_kernel[160] = "";

char *last_apply_kernel() { return g_last_kernel; }

dg_status set_error(dg_status s, const std::string &msg)
{
    g_err = msg;
    return s;
}

cudaError_t upload_tables()
{
    cudaError_t e;
    if ((e = upload_tables_vec()) != cudaSuccess) return e;
    if ((e = upload_tables_apply2()) != cudaSuccess) return e;
    if ((e = upload_tables_apply3()) != cudaSuccess) return e;
    if ((e = upload_tables_stage()) != cudaSuccess) return e;
    if ((e = upload_tables_stage_interp()) != cudaSuccess) return e;
    if ((e = upload_tables_visc()) != cudaSuccess) return e;
    if ((e = upload_tables_halo()) != cudaSuccess) return e;
    if ((e = upload_tables_stab()) != cudaSuccess) return e;
    return upload_tables_convect();
}

// ---------------------------------------------------------------------------
// NCCL, loaded on demand (single-rank meshes never need it)
// ---------------------------------------------------------------------------
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char *(*GetErrorString)(ncclResult_t);
    bool ok = false;
    std::string why;
};

static NcclApi *nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *env = getenv("DG_NCCL_LIB");
        const char *cands[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
        void *h = nullptr;
        for (const char *c : cands)
            if ((h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            api.why = std::string("cannot dlopen NCCL (set DG_NCCL_LIB): ") + dlerror();
            return;
        }
#define LOAD(field, sym)                                                      \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym));         \
    if (!api.field) {                                                         \
        api.why = "NCCL symbol missing: " sym;                                \
        return;                                                               \
    }
        LOAD(GetUniqueId, "ncclGetUniqueId");
        LOAD(CommInitRank, "ncclCommInitRank");
        LOAD(CommDestroy, "ncclCommDestroy");
        LOAD(Send, "ncclSend");
        LOAD(Recv, "ncclRecv");
        LOAD(AllReduce, "ncclAllReduce");
        LOAD(GroupStart, "ncclGroupStart");
        LOAD(GroupEnd, "ncclGroupEnd");
        LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
        api.ok = true;
    });
    return &api;
}

// ---------------------------------------------------------------------------
// Lanczos estimate of cond(D^-1 A) from the CG coefficients (tridiagonal, Sturm bisection)
// ---------------------------------------------------------------------------
static int sturm_count(const std::vector<double> &a, const std::vector<double> &b, double x)
{
    int cnt = 0;
    double d = 1.0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double bb = i ? b[i - 1] * b[i - 1] : 0.0;
        d = (a[i] - x) - (i ? bb / d : 0.0);
        if (d == 0.0) d = -1e-300;
        if (d < 0.0) ++cnt;
    }
    return cnt;
}

static double lanczos_kappa(const double *hist, int k)
{
    if (k < 2) return NAN;
    std::vector<double> a(k), b(k - 1);
    for (int j = 0; j < k; ++j) {
        const double al = hist[2 * j], be_prev = j ? hist[2 * (j - 1) + 1] : 0.0, al_prev = j ? hist[2 * (j - 1)] : 1.0;
        a[j] = 1.0 / al + (j ? be_prev / al_prev : 0.0);
        if (j < k - 1) b[j] = std::sqrt(std::max(hist[2 * j + 1], 0.0)) / al;
    }
    double lo = 1e300, hi = -1e300;
    for (int j = 0; j < k; ++j) {
        const double r = (j ? std::fabs(b[j - 1]) : 0.0) + (j < k - 1 ? std::fabs(b[j]) : 0.0);
        lo = std::min(lo, a[j] - r);
        hi = std::max(hi, a[j] + r);
    }
    auto kth = [&](int idx) {  // idx-th smallest eigenvalue (0-based)
        double l = lo, h = hi;
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (l + h);
            if (sturm_count(a, b, mid) > idx) h = mid;
            else l = mid;
        }
        return 0.5 * (l + h);
    };
    const double emin = kth(0), emax = kth(k - 1);
    return emin > 0.0 ? emax / emin : NAN;
}

}  // namespace dg

using namespace dg;

// ---------------------------------------------------------------------------
// mesh
// ---------------------------------------------------------------------------
struct dg_mesh {
    Geom g{};
    int rank = 0, nranks = 1, device = 0;
    long long el_off = 0, ndof = 0, ndof_global = 0, layer = 0;  // layer: doubles per slab layer
    cudaStream_t st = nullptr;
    // PCG workspace
    double *r = nullptr, *q = nullptr, *pa = nullptr, *pb = nullptr, *dinv = nullptr, *z = nullptr;
    double *partial = nullptr;
    int partial_cap = 0;  // in doubles
    double *sums = nullptr, *aux = nullptr, *mass_e = nullptr, *hist = nullptr;
    int hist_cap = 0;
    PcgScal *scal = nullptr, *hscal = nullptr;
    // halos: multi-rank slabs, or the 1-rank halo mode (dg_mesh_create with nranks == 1 and an
    // NCCL id: the slab-boundary faces go through a self send/recv instead of the local wrap)
    bool halo = false;
    long long F = 0;  // face nodes of one slab layer (trace arrays hold 3 F doubles)
    double *ts_lo = nullptr, *ts_hi = nullptr, *tr_lo = nullptr, *tr_hi = nullptr;  // face traces
    cudaStream_t cs_comm = nullptr;                                                   // exchange stream
    cudaStream_t cs_cap = nullptr;  // non-blocking stream the PCG iteration graphs are captured on
    // the last PCG iteration graph and what it was captured for (reused by the next solve with the
    // same key: the stage's repeated solves skip the instantiation)
    struct GraphKey {
        int flags = -1;
        const double *u = nullptr, *nu = nullptr;
        double lam = 0.0, nu_const = 0.0;
        bool operator==(const GraphKey &o) const
        {
            return flags == o.flags && u == o.u && nu == o.nu && lam == o.lam && nu_const == o.nu_const;
        }
    } gkey;
    cudaGraphExec_t gexec = nullptr;
    long long gexec_launches = 0;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    double *h_lo = nullptr, *h_hi = nullptr, *hn_lo = nullptr, *hn_hi = nullptr;       // element layers
    double *hv_lo[3] = {nullptr, nullptr, nullptr}, *hv_hi[3] = {nullptr, nullptr, nullptr};
    ncclComm_t comm = nullptr;
    // host-variant staging
    double *st_a = nullptr, *st_b = nullptr, *st_c = nullptr;
    // pipelined host apply: copy streams and per-chunk events (created on first use)
    cudaStream_t cs_in = nullptr, cs_out = nullptr;
    std::vector<cudaEvent_t> ev;
    // IMEX stage workspace (velocity mesh: F_c[0..dim), A v; pressure mesh: rhs)
    double *sf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    std::vector<double *> rk;  // IMEX-RK step workspace (velocity fields)
    int *d_flag = nullptr;
    long long launches = 0;
    // two-level Schwarz preconditioner (schwarz.cu): tables for sw_nu, coarse workspace
    int pc = DG_PC_JACOBI;
    SwTab *d_sw = nullptr;
    SwTab h_sw{};
    double *d_swF = nullptr, *rc_el = nullptr, *chat = nullptr, *xc = nullptr, *rc = nullptr;
    double sw_nu = -1.0;
    bool sw_coarse_on = true;
    // D^-1 cache: `dinv` is reserved for the Jacobi preconditioner and written only by
    // pcg_impl; (dinv_lam, dinv_nu) name the constant-nu operator it holds (-1: invalid).  Any
    // other writer of `dinv` (or a stream change) must reset both to -1.
    double dinv_lam = -1.0, dinv_nu = -1.0;
    // divergence / mass-flux stabilisation (stab.cu; dg_mesh_set_div_stab): zeta_D, zeta_C, the
    // CG workspace [r | p | q | v''] of dim * ndof doubles each and the Jacobi table [dim][npe]
    double stab_zD = 0.0, stab_zC = 0.0;
    double *stab_ws = nullptr, *stab_dinv = nullptr;
    double stab_dinv_aD = -1.0, stab_dinv_aC = -1.0;
};

#define CK(call)                                                                                         \
    do {                                                                                                 \
        cudaError_t _e = (call);                                                                         \
        if (_e != cudaSuccess)                                                                           \
            return set_error(_e == cudaErrorNotSupported ? DG_EUNSUPPORTED : DG_ECUDA,                  \
                             std::string(#call) + ": " + cudaGetErrorString(_e));                        \
    } while (0)

#define CKN(call)                                                                                        \
    do {                                                                                                 \
        ncclResult_t _r = (call);                                                                        \
        if (_r != ncclSuccess) return set_error(DG_ENCCL, std::string(#call) + ": " + nccl()->GetErrorString(_r)); \
    } while (0)

namespace {

long long nbricks(const Geom &g) { return (long long)g.nbk[0] * g.nbk[1] * g.nbk[2]; }

dg_status alloc(void **p, size_t bytes)
{
    if (cudaMalloc(p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return set_error(DG_ENOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    }
    return DG_OK;
}

#define CKS(x)                        \
    do {                              \
        dg_status _s = (x);           \
        if (_s != DG_OK) return _s;   \
    } while (0)

// PCG workspace (x, r, p_a, p_b, q, z, D^-1 and the alpha/beta history): allocated once by
// dg_mesh_create, so dg_pcg_solve never allocates.  All-or-nothing: on a partial failure
// every buffer is released again and nulled (the mesh creation then fails).
dg_status alloc_workspace(dg_mesh *m)
{
    const size_t b = sizeof(double) * (size_t)m->ndof;
    double **bufs[] = {&m->r, &m->q, &m->pa, &m->pb, &m->dinv, &m->z};
    dg_status s = DG_OK;
    for (double **p : bufs)
        if ((s = alloc((void **)p, b)) != DG_OK) break;
    if (s == DG_OK) s = alloc((void **)&m->hist, sizeof(double) * 2 * (size_t)PCG_HIST_CAP);
    if (s != DG_OK) {
        for (double **p : bufs) {
            if (*p) cudaFree(*p);
            *p = nullptr;
        }
        if (m->hist) cudaFree(m->hist);
        m->hist = nullptr;
        return s;
    }
    m->hist_cap = PCG_HIST_CAP;
    return DG_OK;
}

dg_status ensure_halos(dg_mesh *m, bool vel)
{
    if (!m->halo) return DG_OK;
    const size_t b = sizeof(double) * (size_t)m->layer;
    if (!m->h_lo) {
        CKS(alloc((void **)&m->h_lo, b));
        CKS(alloc((void **)&m->h_hi, b));
        CKS(alloc((void **)&m->hn_lo, b));
        CKS(alloc((void **)&m->hn_hi, b));
    }
    if (vel && !m->hv_lo[0])
        for (int c = 0; c < 3; ++c) {
            CKS(alloc((void **)&m->hv_lo[c], b));
            CKS(alloc((void **)&m->hv_hi[c], b));
        }
    return DG_OK;
}

// Exchange the first/last slab layers of `field` with the neighbouring ranks (periodic ring):
// lo <- last layer of rank-1, hi <- first layer of rank+1.  Sends are posted as
// (last -> next, first -> prev) and receives as (lo <- prev, hi <- next), so that with two
// ranks (prev == next) the in-order matching per peer still pairs them correctly.
dg_status exchange(dg_mesh *m, const double *field, double *lo, double *hi)
{
    NcclApi *nc = nccl();
    const int R = m->nranks, prev = (m->rank - 1 + R) % R, next = (m->rank + 1) % R;
    const int S = m->g.dim - 1;
    const double *first = field, *last = field + (size_t)(m->g.Nl[S] - 1) * m->layer;
    CKN(nc->GroupStart());
    CKN(nc->Send(last, (size_t)m->layer, ncclDouble, next, m->comm, m->st));
    CKN(nc->Send(first, (size_t)m->layer, ncclDouble, prev, m->comm, m->st));
    CKN(nc->Recv(lo, (size_t)m->layer, ncclDouble, prev, m->comm, m->st));
    CKN(nc->Recv(hi, (size_t)m->layer, ncclDouble, next, m->comm, m->st));
    CKN(nc->GroupEnd());
    return DG_OK;
}

dg_status allreduce(dg_mesh *m, double *buf, int count)
{
    if (!m->halo) return DG_OK;
    CKN(nccl()->AllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, m->comm, m->st));
    return DG_OK;
}

dg_status check_common(dg_mesh *m, double lam, const double *nu, double nu_const)
{
    if (!m) return set_error(DG_EINVAL, "null mesh");
    if (!(lam >= 0.0) || !std::isfinite(lam)) return set_error(DG_EINVAL, "lambda must be finite and >= 0");
    if (!nu && !(nu_const > 0.0 && std::isfinite(nu_const)))
        return set_error(DG_EINVAL, "nu_const must be finite and > 0 when nu == NULL");
    return DG_OK;
}

dg_status run_apply(dg_mesh *m, double lam, const double *nu, double nu_const, const double *u, double *out,
                    const Halo &halo, const DotEpi &epi, const PProl &pro, int *grid_out = nullptr, int zlo = 0,
                    int zhi = -1)
{
    ApplyParams a{};
    a.g = m->g;
    a.lam = lam;
    a.nu_const = nu_const;
    a.u = u;
    a.nu = nu;
    a.out = out;
    a.halo = halo;
    if (m->halo) {
        a.halo.tr_lo = m->tr_lo;
        a.halo.tr_hi = m->tr_hi;
    }
    a.epi = epi;
    a.pro = pro;
    a.b0 = 0;
    a.b1 = nbricks(a.g);
    a.zlo = zlo;
    a.zhi = zhi;
    const bool varnu = nu != nullptr;
    int grid = 0;
    const int mode = pro.on ? 1 : (epi.partial ? 2 : 0);
    const cudaError_t e = m->g.dim == 3 ? launch_apply3(a, varnu, mode, &grid, 0, m->st)
                                        : launch_apply2(a, varnu, mode, &grid, 0, m->st);
    CK(e);
    if (grid_out) *grid_out = grid;
    m->launches += 1;
    return DG_OK;
}

// Face-trace exchange: on the exchange stream, after the work already enqueued on
// the mesh stream, compute the (u, s = nu d_S u[, nu]) traces of the slab's two boundary faces
// and swap them with the neighbouring ranks (grouped NCCL send/recv; the ring order pairs the
// two messages correctly also for two ranks, where prev == next, and for the 1-rank halo mode,
// where both peers are this rank).  ev_b marks the received halo (tr_lo, tr_hi).  nu_too: also
// the nu traces (once per solve / per standalone call); otherwise the nu part of the halo
// buffers is kept from the last exchange.
dg_status trace_exchange(dg_mesh *m, const double *u, const double *nu, double nu_const, bool nu_too)
{
    NcclApi *nc = nccl();
    CK(cudaEventRecord(m->ev_a, m->st));
    CK(cudaStreamWaitEvent(m->cs_comm, m->ev_a, 0));
    CK(launch_slab_traces(m->g, u, nu, nu_const, m->ts_lo, m->ts_hi, nu_too ? 1 : 0, m->cs_comm));
    m->launches += 1;
    const int R = m->nranks, prev = (m->rank - 1 + R) % R, next = (m->rank + 1) % R;
    const size_t cnt = (size_t)(nu_too ? 3 : 2) * (size_t)m->F;
    CKN(nc->GroupStart());
    CKN(nc->Send(m->ts_hi, cnt, ncclDouble, next, m->comm, m->cs_comm));
    CKN(nc->Send(m->ts_lo, cnt, ncclDouble, prev, m->comm, m->cs_comm));
    CKN(nc->Recv(m->tr_lo, cnt, ncclDouble, prev, m->comm, m->cs_comm));
    CKN(nc->Recv(m->tr_hi, cnt, ncclDouble, next, m->comm, m->cs_comm));
    CKN(nc->GroupEnd());
    CK(cudaEventRecord(m->ev_b, m->cs_comm));
    return DG_OK;
}

// q = A u over the slab with the face-trace halo.  Single rank: one launch.  Halo meshes: the
// trace exchange runs on the exchange stream, then one launch (by default; with the layer
// split -- DG_OVERLAP_MIN_LAYERS -- the interior layers [2, Nl - 2) are applied during the
// exchange and the two boundary layer pairs [0, 2) and [Nl - 2, Nl) after it).
// partial != null: dot epilogue (MODE 2/3), the launches' block partials back to back; *G =
// their total count.  nu_traced: the nu halo of this nu is already in place (PCG iterations).
dg_status halo_apply(dg_mesh *m, double lam, const double *nu, double nu_const, const double *u, double *out,
                     double *partial, int *G, const int *done, bool nu_traced)
{
    DotEpi epi;
    epi.partial = partial;
    PProl pro;
    pro.done = done;
    int g1 = 0, g2 = 0, g3 = 0;
    if (!m->halo) {
        CKS(run_apply(m, lam, nu, nu_const, u, out, Halo{}, epi, pro, &g1));
        if (G) *G = g1;
        return DG_OK;
    }
    CKS(trace_exchange(m, u, nu, nu_const, !nu_traced));
    const Geom &g = m->g;
    const int Nl = g.Nl[g.dim - 1];
// The interior / boundary layer split (overlap of the trace exchange with the interior layers)
// costs more than it hides with these persistent kernels: three launches and 2-layer segments
// (pipeline fill, segment-end z traces, a partial last round) -- measured on the c5 per-rank
// slab model, apply 0.333 / 0.211 / 0.150 ms with the split vs 0.292 / 0.171 / 0.110 ms as one
// launch after the exchange for 32 / 16 / 8 layers (bench.py `halo.slab_model`).  Kept
// selectable for builds with -DDG_OVERLAP_MIN_LAYERS=<n>.
#ifndef DG_OVERLAP_MIN_LAYERS
#define DG_OVERLAP_MIN_LAYERS (1 << 30)
#endif
    bool ranges = g.dim == 3 && apply3_ranges_ok(g) && Nl >= DG_OVERLAP_MIN_LAYERS && Nl >= 6 && Nl % 2 == 0 &&
                  (!partial || apply3_split_pcg_ok(g, nu));
    if (ranges) {  // (the layer-range kernels exist for most (P, nu) pairs; otherwise one launch)
        const dg_status st = run_apply(m, lam, nu, nu_const, u, out, Halo{}, epi, pro, &g1, 2, Nl - 2);
        if (st == DG_EUNSUPPORTED) ranges = false;  // nothing was enqueued
        else if (st != DG_OK) return st;
    }
    if (ranges) {
        CK(cudaStreamWaitEvent(m->st, m->ev_b, 0));
        if (partial) epi.partial = partial + 2 * g1;
        CKS(run_apply(m, lam, nu, nu_const, u, out, Halo{}, epi, pro, &g2, 0, 2));
        if (partial) epi.partial = partial + 2 * (g1 + g2);
        CKS(run_apply(m, lam, nu, nu_const, u, out, Halo{}, epi, pro, &g3, Nl - 2, Nl));
    } else {
        CK(cudaStreamWaitEvent(m->st, m->ev_b, 0));
        CKS(run_apply(m, lam, nu, nu_const, u, out, Halo{}, epi, pro, &g1));
    }
    if (G) *G = g1 + g2 + g3;
    return DG_OK;
}

dg_status apply_impl(dg_mesh *m, double lam, const double *nu, double nu_const, const double *u, double *out)
{
    return halo_apply(m, lam, nu, nu_const, u, out, nullptr, nullptr, nullptr, false);
}

// the nu face traces for the diagonal and the PCG iterations of one solve
dg_status nu_halo(dg_mesh *m, const double *nu, double nu_const)
{
    if (!m->halo || !nu) return DG_OK;  // constant nu: the kernels use nu_const
    CKS(trace_exchange(m, nu, nu, nu_const, true));  // (the u part of this exchange is unused)
    CK(cudaStreamWaitEvent(m->st, m->ev_b, 0));
    return DG_OK;
}

dg_status diag_impl(dg_mesh *m, double lam, const double *nu, double nu_const, double *diag, bool nu_traced = false)
{
    if (!nu_traced) CKS(nu_halo(m, nu, nu_const));
    Halo h;
    if (m->halo) {
        h.tr_lo = m->tr_lo;
        h.tr_hi = m->tr_hi;
    }
    CK(m->g.dim == 3 ? launch_diag3(m->g, lam, nu, nu_const, h, diag, m->st)
                     : launch_diag2(m->g, lam, nu, nu_const, h, diag, m->st));
    m->launches += 1;
    return DG_OK;
}

// reduce partial[G][2] -> sums[2] (+ allreduce) -> finalize(mode)
dg_status reduce_fin(dg_mesh *m, int G, int mode, const double *partial = nullptr)
{
    if (!partial) partial = m->partial;
    if (!m->halo) {
        CK(launch_reduce_fin(partial, G, 2, m->sums, mode, m->scal, m->hist, m->aux, m->st));
        m->launches += 1;
    } else {
        CK(launch_reduce_s(partial, G, 2, m->sums,
                           (mode == FIN_ALPHA || mode == FIN_BETA) ? m->scal : nullptr, m->st));
        CKS(allreduce(m, m->sums, 2));
        CK(launch_finalize(mode, m->sums, m->scal, m->hist, m->aux, m->st));
        m->launches += 2;
    }
    return DG_OK;
}

// ---------------------------------------------------------------------------
// two-level Schwarz preconditioner (schwarz.cu)
// ---------------------------------------------------------------------------
dg_status sw_check(const dg_mesh *m, const double *nu)
{
    (void)nu;  // variable nu: the preconditioner uses the mass-weighted mean viscosity
    const char *why = nullptr;
    if (!schwarz_supported(m->g, &why)) return set_error(DG_EUNSUPPORTED, why);
    return DG_OK;
}

dg_status ensure_sw(dg_mesh *m, double nu_const)
{
    const Geom &g = m->g;
    const long long NV = (long long)g.N[0] * g.N[1] * (g.dim == 3 ? g.N[2] : 1);
    if (!m->d_sw) {
        CKS(alloc((void **)&m->d_sw, sizeof(SwTab)));
        CKS(alloc((void **)&m->d_swF, sizeof(double) * 3 * SW_NCMAX * SW_NCMAX));
        CKS(alloc((void **)&m->rc_el, sizeof(double) * (size_t)g.nel * (g.dim == 3 ? 8 : 4)));
        CKS(alloc((void **)&m->chat, sizeof(double) * (size_t)NV));
        CKS(alloc((void **)&m->xc, sizeof(double) * (size_t)NV));
        if (m->halo) CKS(alloc((void **)&m->rc, sizeof(double) * (size_t)NV));
    }
    (void)nu_const;  // the tables are built once for nu = 1 (nu scales eigenvalues / symbols only)
    if (m->sw_nu != 1.0) {
        std::vector<double> F;
        build_sw_tab(g, 1.0, &m->h_sw, F);
        CK(cudaMemcpyAsync(m->d_sw, &m->h_sw, sizeof(SwTab), cudaMemcpyHostToDevice, m->st));
        CK(cudaMemcpyAsync(m->d_swF, F.data(), sizeof(double) * F.size(), cudaMemcpyHostToDevice, m->st));
        CK(cudaStreamSynchronize(m->st));  // F is a host temporary
        m->sw_nu = 1.0;
    }
    return DG_OK;
}

// coarse part: x_c = A_c^+ P_1^T r from the element moments rc_el; r_c.x_c partials written
// to partial[pslot + b] (b < sw_cz_grid) when `partial` is set
dg_status sw_coarse(dg_mesh *m, double lam, double nu, const double *nu_eff, double *partial, int pslot,
                    const int *done = nullptr)
{
    const Geom &g = m->g;
    SwCoarseParams c;
    c.done = done;
    c.nu = nu;
    c.nu_eff = nu_eff;
    c.T = m->d_sw;
    c.F = m->d_swF;
    c.dim = g.dim;
    c.lam = lam;
    c.chat = m->chat;
    c.xc = m->xc;
    c.partial = partial;
    c.pslot = pslot;
    c.count_dot = m->rank == 0;
    c.nel = g.nel;
    if (!m->halo) {
        c.rc_el = m->rc_el;
    } else {
        const long long NV = (long long)g.N[0] * g.N[1] * (g.dim == 3 ? g.N[2] : 1);
        CK(cudaMemsetAsync(m->rc, 0, sizeof(double) * (size_t)NV, m->st));
        SwCoarseParams gl = c;
        gl.rc_el = m->rc_el;
        gl.rc = m->rc;
        const int S = g.dim - 1;
        const long long lay_el = S == 2 ? (long long)g.N[0] * g.N[1] : (long long)g.N[0];
        CK(launch_sw_gather_local(gl, S, (int)(m->el_off / lay_el), g.Nl[S], m->st));
        m->launches += 1;
        CKS(allreduce(m, m->rc, (int)NV));
        c.rc = m->rc;
    }
    for (int stage = 0; stage < 3; ++stage) CK(launch_sw_coarse(c, m->h_sw, stage, m->st));
    m->launches += 3;
    return DG_OK;
}

// z = B r (block part into z, rc_el moments; then the coarse solve and z += P_1 x_c)
dg_status sw_apply_impl(dg_mesh *m, double lam, double nu, const double *r, double *z)
{
    SwBlockParams b;
    b.T = m->d_sw;
    b.lam = lam;
    b.nu = nu;
    b.mode = SW_APPLY;
    b.nel = m->g.nel;
    b.rin = r;
    b.z = z;
    b.rc_el = m->rc_el;
    b.mass_e = m->mass_e;
    int grid = 0;
    CK(launch_sw_block(m->g, m->h_sw, b, m->st, &grid));
    m->launches += 1;
    CKS(sw_coarse(m, lam, nu, nullptr, nullptr, 0));
    SwPupdParams p;
    p.T = m->d_sw;
    p.nel = m->g.nel;
    p.el_off = m->el_off;
    p.zb = z;
    p.xc = m->xc;
    p.p = z;
    CK(launch_sw_pupd(m->g, m->h_sw, p, m->st));
    m->launches += 1;
    return DG_OK;
}

// PCG preconditioner step (mode SW_INIT or SW_UPDATE): r update, z_b, moments, coarse solve,
// r.z and residual partials -> reduce_fin(fin)
dg_status sw_pcg_step(dg_mesh *m, double lam, int mode, int fin)
{
    SwBlockParams b;
    b.T = m->d_sw;
    b.lam = lam;
    b.nu_eff = &m->scal->nu_eff;
    b.mode = mode;
    b.nel = m->g.nel;
    b.r = m->r;
    b.q = m->q;
    b.z = m->z;
    b.rc_el = m->rc_el;
    b.mass_e = m->mass_e;
    b.s = m->scal;
    b.partial = m->partial;
    int grid = 0;
    CK(launch_sw_block(m->g, m->h_sw, b, m->st, &grid));
    m->launches += 1;
    if (!m->sw_coarse_on) return reduce_fin(m, grid, fin);  // element blocks only (x_c = 0)
    CKS(sw_coarse(m, lam, 1.0, &m->scal->nu_eff, m->partial, grid, mode == SW_UPDATE ? &m->scal->done : nullptr));
    return reduce_fin(m, grid + sw_cz_grid(m->h_sw), fin);
}

dg_status pcg_impl(dg_mesh *m, double lam, const double *nu, double nu_const, const double *f, double tol,
                   int maxit, double *u, dg_solve_info *info)
{
    const Geom &g = m->g;
    const int VG = vec_grid();

    // scalars
    PcgScal s0{};
    s0.lam = lam;
    s0.tol2 = tol * tol;
    s0.ndof_global = m->ndof_global;
    s0.maxit = maxit;
    s0.hist_cap = m->hist_cap;
    s0.nu_eff = nu ? 1.0 : nu_const;
    CK(cudaMemcpyAsync(m->scal, &s0, sizeof(s0), cudaMemcpyHostToDevice, m->st));

    // preconditioner: two-level Schwarz (dg_mesh_set_precond) or Jacobi
    const bool sw = m->pc == DG_PC_SCHWARZ2;
    if (sw) {
        CKS(sw_check(m, nu));
        CKS(ensure_sw(m, nu_const));
        double nu_bar = nu_const;
        if (nu) {  // variable nu: blocks and coarse operator with the mass-weighted mean viscosity
            CK(launch_mass_moments(g, nu, m->mass_e, m->partial, m->st));
            m->launches += 1;
            CKS(reduce_fin(m, VG, FIN_NUMEAN));
            CK(cudaMemcpyAsync(m->hscal, m->scal, sizeof(PcgScal), cudaMemcpyDeviceToHost, m->st));
            CK(cudaStreamSynchronize(m->st));
            nu_bar = m->hscal->nu_eff;
        }
        // the Q1 coarse space pays while diffusion dominates at the element scale (measured:
        // lam h^2 / nu <= ~50); above, the element blocks alone are better
        double h2 = 1e300;
        for (int d = 0; d < g.dim; ++d) h2 = std::min(h2, g.h[d] * g.h[d]);
        m->sw_coarse_on = lam * h2 <= 50.0 * nu_bar;
        if (!m->sw_coarse_on) CK(cudaMemsetAsync(m->xc, 0, sizeof(double) * (size_t)g.N[0] * g.N[1] *
                                                              (g.dim == 3 ? g.N[2] : 1), m->st));
    }
    // halo meshes: the nu face traces once per solve (the diagonal and every apply of the
    // iterations read them; the per-iteration exchanges carry only u and s)
    CKS(nu_halo(m, nu, nu_const));
    // Jacobi preconditioner: D^-1 straight from the closed-form kernel where it applies
    bool self = false;
    for (int d = 0; d < g.dim; ++d) self = self || g.N[d] == 1;
    if (sw) {
    } else if (!self && !nu && m->dinv_lam == lam && m->dinv_nu == nu_const) {
        // constant nu: D^-1 depends on (lam, nu) and the geometry only -- kept from the last
        // solve with the same pair (e.g. the three velocity components of a stage)
    } else if (!self) {
        Halo hd;
        if (m->halo) {
            hd.tr_lo = m->tr_lo;
            hd.tr_hi = m->tr_hi;
        }
        CK(g.dim == 3 ? launch_diag3(g, lam, nu, nu_const, hd, m->dinv, m->st, 1)
                      : launch_diag2(g, lam, nu, nu_const, hd, m->dinv, m->st, 1));
        m->launches += 1;
        m->dinv_lam = nu ? -1.0 : lam;
        m->dinv_nu = nu ? -1.0 : nu_const;
    } else {
        CKS(diag_impl(m, lam, nu, nu_const, m->q, true));
        CK(launch_recip(g, m->q, m->dinv, m->st));
        m->launches += 1;
        m->dinv_lam = m->dinv_nu = -1.0;
    }
    // split PCG step (pupd kernel + apply with the dot epilogue) where the v5 / v6 applies run:
    // measured faster than the fused prologue of v5; halo meshes too (the apply
    // overlaps the face-trace exchange with the interior layers)
    const bool split_ok = g.dim == 3 && apply3_split_pcg_ok(g, nu);
    const bool split = !sw && split_ok && !DG_DEV_ENV("DG_PCG_FUSED");
    // constant nu on the uniform periodic mesh (N_d >= 2: the closed-form diagonal): the first
    // element's D^-1 serves every element
    const bool table = split && !nu && !self && !DG_DEV_ENV("DG_PCG_NOTABLE");
    // r = M (f - fmean) - A u; an all-zero guess (one reduction and a host read instead of an
    // operator application) takes A u = 0
    CK(launch_abssum(g, u, m->partial, m->st));
    m->launches += 1;
    CKS(reduce_fin(m, VG, FIN_ABSSUM));
    CK(cudaMemcpyAsync(&m->hscal->rz, m->aux, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    CK(cudaStreamSynchronize(m->st));
    const double usum = m->hscal->rz;
    if (usum != 0.0) CKS(halo_apply(m, lam, nu, nu_const, u, m->q, nullptr, nullptr, nullptr, true));
    if (lam > 0.0 && !sw) {
        // no mean projection: r, z (or nothing with the D^-1 table) and both partial sets in one pass
        CK(launch_pcg_init_fused(g, f, usum != 0.0 ? m->q : nullptr, m->r, m->dinv, table ? 1 : 0,
                                 table ? nullptr : m->z, m->mass_e, m->partial, m->partial + 2 * VG, m->st));
        m->launches += 1;
        CKS(reduce_fin(m, VG, FIN_INIT, m->partial + 2 * VG));
        CKS(reduce_fin(m, VG, FIN_INIT2));
    } else {
        // f mean (lam == 0) and total mass
        CK(launch_mass_moments(g, f, m->mass_e, m->partial, m->st));
        m->launches += 1;
        CKS(reduce_fin(m, VG, FIN_FMEAN));
        if (usum == 0.0) CK(cudaMemsetAsync(m->q, 0, sizeof(double) * (size_t)m->ndof, m->st));
        CK(launch_pcg_init(g, f, m->q, m->r, m->mass_e, m->scal, m->partial, m->st));
        m->launches += 1;
        CKS(reduce_fin(m, VG, FIN_INIT));
        if (sw) {
            CKS(sw_pcg_step(m, lam, SW_INIT, FIN_INIT2));
        } else {
            CK(launch_pcg_init2(g, m->r, m->dinv, m->z, m->mass_e, m->scal, m->partial, m->st));
            m->launches += 1;
            CKS(reduce_fin(m, VG, FIN_INIT2));
        }
    }
    // the split p updates treat alpha = beta = 0 (before the first iteration) as p = z without
    // reading p; the other variants read p_old from the start
    if (!split) CK(cudaMemsetAsync(m->pa, 0, sizeof(double) * (size_t)m->ndof, m->st));

    double *p_old = m->pa, *p_new = m->pb;
    // one CG iteration, enqueued on the mesh stream (the fused variant swaps p_old / p_new)
    auto iteration = [&]() -> dg_status {
        if (sw) {
            // x += alpha p, p = z_b + P_1 x_c + beta p (in place) ; q = A p ; Schwarz step
            SwPupdParams pp;
            pp.T = m->d_sw;
            pp.nel = g.nel;
            pp.el_off = m->el_off;
            pp.zb = m->z;
            pp.xc = m->xc;
            pp.p_old = p_old;
            pp.p = p_old;
            pp.x = u;
            pp.s = m->scal;
            CK(launch_sw_pupd(g, m->h_sw, pp, m->st));
            m->launches += 1;
            if (split_ok) {
                int grid = 0;
                CKS(halo_apply(m, lam, nu, nu_const, p_old, m->q, m->partial, &grid, &m->scal->done, true));
                CKS(reduce_fin(m, grid, FIN_ALPHA));
            } else {
                CKS(halo_apply(m, lam, nu, nu_const, p_old, m->q, nullptr, nullptr, nullptr, true));
                CK(launch_dot_pq(g, p_old, m->q, m->scal, m->partial, m->st));
                m->launches += 1;
                CKS(reduce_fin(m, VG, FIN_ALPHA));
            }
            CKS(sw_pcg_step(m, lam, SW_UPDATE, FIN_BETA));
        } else if (split) {
            // x += alpha p, p = z + beta p (in place; x deferred by one iteration) ;
            // q = A p with the dot epilogue (apply MODE 2) ; r, z update.  Constant nu: z is
            // never stored (the diagonal is one [npe] table, applied on the fly)
            if (table) CK(launch_pcg_pupd_xt(g, u, p_old, m->r, m->dinv, m->scal, m->st));
            else CK(launch_pcg_pupd_x(g, u, p_old, m->z, m->scal, m->st));
            m->launches += 1;
            int grid = 0;
            CKS(halo_apply(m, lam, nu, nu_const, p_old, m->q, m->partial, &grid, &m->scal->done, true));
            CKS(reduce_fin(m, grid, FIN_ALPHA));
            if (table) CK(launch_pcg_update_t(g, m->r, m->q, m->dinv, m->mass_e, m->scal, m->partial, m->st));
            else CK(launch_pcg_update_nox(g, m->r, m->q, m->dinv, m->z, m->mass_e, m->scal, m->partial, m->st));
            m->launches += 1;
            CKS(reduce_fin(m, table ? vec_grid_wide() : VG, FIN_BETA));
        } else if (!m->halo) {
            // q = A p with p = dinv r + beta p_old (prologue), partials p.q, sum q (epilogue)
            PProl pro;
            pro.on = true;
            pro.z = m->z;
            pro.p_old = p_old;
            pro.p_out = p_new;
            pro.beta = &m->scal->beta;
            pro.done = &m->scal->done;
            DotEpi epi;
            epi.partial = m->partial;
            int grid = 0;
            CKS(run_apply(m, lam, nu, nu_const, nullptr, m->q, Halo{}, epi, pro, &grid));
            CKS(reduce_fin(m, grid, FIN_ALPHA));
            CK(launch_pcg_update(g, u, m->r, p_new, m->q, m->dinv, m->z, m->mass_e, m->scal, m->partial, m->st));
            m->launches += 1;
            CKS(reduce_fin(m, VG, FIN_BETA));
            std::swap(p_old, p_new);
        } else {
            // unfused: p = dinv r + beta p ; halo(p) ; q = A p ; p.q
            CK(launch_pcg_pupd(g, p_old, m->z, m->scal, m->st));
            m->launches += 1;
            CKS(halo_apply(m, lam, nu, nu_const, p_old, m->q, nullptr, nullptr, nullptr, true));
            CK(launch_dot_pq(g, p_old, m->q, m->scal, m->partial, m->st));
            m->launches += 1;
            CKS(reduce_fin(m, VG, FIN_ALPHA));
            CK(launch_pcg_update(g, u, m->r, p_old, m->q, m->dinv, m->z, m->mass_e, m->scal, m->partial, m->st));
            m->launches += 1;
            CKS(reduce_fin(m, VG, FIN_BETA));
        }
        return DG_OK;
    };
    // Single-rank meshes replay the iterations as a CUDA graph (captured once per solve: two
    // iterations for the fused variant, whose p buffers alternate): the launch-bound small
    // configurations lose most of their per-kernel launch overhead.  Halo meshes enqueue the
    // iterations directly (their exchange runs on a second stream).
    const bool use_graph = !m->halo;
    const int gper = (!sw && !split && !m->halo) ? 2 : 1;
    dg_mesh::GraphKey key;
    key.flags = (sw ? 1 : 0) | (split ? 2 : 0) | (table ? 4 : 0) | (split_ok ? 8 : 0) | (m->sw_coarse_on ? 16 : 0);
    key.u = u;
    key.nu = nu;
    key.lam = lam;
    key.nu_const = nu_const;
    auto capture = [&]() -> dg_status {
        if (m->gexec) cudaGraphExecDestroy(m->gexec);
        m->gexec = nullptr;
        m->gkey = dg_mesh::GraphKey{};
        // captured on the mesh's private non-blocking stream (the caller's stream may be the
        // legacy default stream, which cannot be captured); replayed on the caller's stream
        cudaGraph_t gr = nullptr;
        const long long l0 = m->launches;
        cudaStream_t user = m->st;
        CK(cudaStreamBeginCapture(m->cs_cap, cudaStreamCaptureModeRelaxed));
        m->st = m->cs_cap;
        dg_status cs = DG_OK;
        for (int k = 0; k < gper && cs == DG_OK; ++k) cs = iteration();
        m->st = user;
        const cudaError_t ce = cudaStreamEndCapture(m->cs_cap, &gr);
        if (cs != DG_OK) {
            if (gr) cudaGraphDestroy(gr);
            return cs;
        }
        CK(ce);
        const cudaError_t ie = cudaGraphInstantiate(&m->gexec, gr, 0);
        cudaGraphDestroy(gr);
        CK(ie);
        m->gexec_launches = m->launches - l0;  // kernels per graph replay (none ran during capture)
        m->launches = l0;
        m->gkey = key;
        return DG_OK;
    };
    // iterations are enqueued in chunks between host convergence checks; after the first chunk
    // the next one is sized from the observed residual reduction per iteration (launches past
    // convergence exit at their first instruction but still cost a few microseconds each)
    int chunk = 4, prev_iter = -1;
    double prev_res2 = 0.0;
    for (;;) {
        CK(cudaMemcpyAsync(m->hscal, m->scal, sizeof(PcgScal), cudaMemcpyDeviceToHost, m->st));
        CK(cudaStreamSynchronize(m->st));
        if (m->hscal->done) break;
        {
            const PcgScal &hs = *m->hscal;
            int next = std::min(chunk * 2, 32);
            if (prev_iter >= 0 && hs.iter > prev_iter && hs.res2 > 0.0 && prev_res2 > hs.res2) {
                const double rate = std::log(hs.res2 / prev_res2) / (hs.iter - prev_iter);  // < 0
                const double need = std::log(hs.tol2 * hs.fnorm2 / hs.res2) / rate;
                if (std::isfinite(need) && need > 0.0) next = std::max(2, std::min(64, (int)std::ceil(1.1 * need) + 1));
            }
            if (prev_iter >= 0) chunk = next;
            prev_iter = hs.iter;
            prev_res2 = hs.res2;
        }
        // long runs replay the captured iteration graph (captured when a chunk of >= 8
        // iterations is due, or reused from an earlier solve with the same key); short solves
        // do not pay for the instantiation
        key.flags = (key.flags & 31) | (p_old == m->pa ? 32 : 0);  // the fused variant's p parity
        const bool have = use_graph && m->gexec && m->gkey == key;
        if (use_graph && !have && chunk >= 8) CKS(capture());
        if (use_graph && m->gexec && m->gkey == key) {
            for (int it = 0; it < chunk; it += gper) {
                CK(cudaGraphLaunch(m->gexec, m->st));
                m->launches += m->gexec_launches;
            }
        } else {
            for (int it = 0; it < chunk; ++it) CKS(iteration());
        }
    }
    if (split || sw) {  // the deferred x update of the last iteration
        CK(launch_pcg_xfinal(g, u, p_old, m->scal, m->st));
        m->launches += 1;
    }
    // lam == 0: zero mass-weighted mean of u
    if (lam == 0.0) {
        CK(launch_mass_moments(g, u, m->mass_e, m->partial, m->st));
        m->launches += 1;
        CKS(reduce_fin(m, VG, FIN_UMEAN));
        CK(launch_shift(g, u, m->aux, m->st));
        m->launches += 1;
    }
    CK(cudaMemcpyAsync(m->hscal, m->scal, sizeof(PcgScal), cudaMemcpyDeviceToHost, m->st));
    CK(cudaStreamSynchronize(m->st));
    const PcgScal hs = *m->hscal;
    if (info) {
        info->iters = hs.iter;
        info->rel_res = hs.fnorm2 > 0 ? std::sqrt(hs.res2 / hs.fnorm2) : std::sqrt(hs.res2);
        info->removed_mean = hs.fmean;
        info->f_norm = std::sqrt(hs.fnorm2);
        info->kappa_est = NAN;
        if (hs.iter >= 2) {
            const int k = std::min(hs.iter, m->hist_cap);
            std::vector<double> hh(2 * (size_t)k);
            CK(cudaMemcpy(hh.data(), m->hist, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost));
            info->kappa_est = lanczos_kappa(hh.data(), k);
        }
    }
    if (hs.status == PCG_ST_BREAKDOWN) return set_error(DG_EBREAKDOWN, "PCG breakdown (p.Ap <= 0 or non-finite)");
    if (hs.status == PCG_ST_MAXIT)
        return set_error(DG_ENOTCONV, "PCG reached maxit=" + std::to_string(maxit) + ", rel_res=" +
                                          std::to_string(hs.fnorm2 > 0 ? std::sqrt(hs.res2 / hs.fnorm2) : 0.0));
    return DG_OK;
}

dg_status stage(dg_mesh *m, double **buf, size_t bytes)
{
    if (*buf) return DG_OK;
    return alloc((void **)buf, bytes);
}

dg_status check_pair(const dg_mesh *mv, const dg_mesh *mp)
{
    const Geom &g = mv->g, &gp = mp->g;
    if (gp.dim != g.dim || gp.P != g.P - 1 || mp->nranks != mv->nranks || mp->rank != mv->rank)
        return set_error(DG_EINVAL, "pressure mesh must match the velocity mesh with degree P-1 (P:1036)");
    for (int d = 0; d < 3; ++d)
        if (gp.N[d] != g.N[d] || gp.h[d] != g.h[d]) return set_error(DG_EINVAL, "pressure mesh geometry differs");
    if (g.P < 2) return set_error(DG_EINVAL, "the velocity degree must be >= 2 (pressure degree P-1 >= 1)");
    return DG_OK;
}

// weak DG divergence of v (velocity mesh) into div (pressure mesh), on mv's stream
dg_status div_impl(dg_mesh *mv, const double *const v[3], double *div)
{
    DivGradParams a;
    for (int c = 0; c < mv->g.dim; ++c) a.v[c] = v[c];
    if (mv->halo) {
        CKS(ensure_halos(mv, true));
        for (int c = 0; c < mv->g.dim; ++c) {
            CKS(exchange(mv, v[c], mv->hv_lo[c], mv->hv_hi[c]));
            a.vlo[c] = mv->hv_lo[c];
            a.vhi[c] = mv->hv_hi[c];
        }
    }
    a.out = div;
    CK(launch_dg_div(mv->g, a, mv->st));
    mv->launches += 1;
    return DG_OK;
}

// weak DG gradient of psi (pressure mesh) into grad[c] (velocity mesh), on mv's stream
dg_status grad_impl(dg_mesh *mp, dg_mesh *mv, const double *psi, double *const grad[3])
{
    DivGradParams a;
    a.psi = psi;
    if (mp->halo) {
        cudaStream_t s0 = mp->st;
        mp->st = mv->st;
        dg_status s = ensure_halos(mp, false);
        if (s == DG_OK) s = exchange(mp, psi, mp->h_lo, mp->h_hi);
        mp->st = s0;
        if (s != DG_OK) return s;
        a.plo = mp->h_lo;
        a.phi = mp->h_hi;
    }
    for (int c = 0; c < mv->g.dim; ++c) a.gout[c] = grad[c];
    CK(launch_dg_grad(mv->g, a, mv->st));
    mv->launches += 1;
    return DG_OK;
}

// ---------------------------------------------------------------------------
// divergence / mass-flux stabilisation (stab.cu, reading A26)
// ---------------------------------------------------------------------------
dg_status stab_apply_impl(dg_mesh *m, const double *const in[3], double *const out[3], double aD, double aC,
                          double *partial, const PcgScal *s, int *grid = nullptr)
{
    StabParams a;
    const int dim = m->g.dim;
    for (int c = 0; c < dim; ++c) {
        a.in[c] = in[c];
        a.out[c] = out[c];
        if (m->halo) {
            CKS(exchange(m, in[c], m->hv_lo[c], m->hv_hi[c]));
            a.lo[c] = m->hv_lo[c];
            a.hi[c] = m->hv_hi[c];
        }
    }
    a.aD = aD;
    a.aC = aC;
    a.partial = partial;
    a.s = s;
    CK(launch_stab_apply(m->g, a, m->st, grid));
    m->launches += 1;
    return DG_OK;
}

// v^ = (M + a_D K_D + a_C K_C)^-1 M v'' in place (v), a_D = dt zeta_D U h / (P+1),
// a_C = dt zeta_C U with U the RMS of v''; v'' is kept in the workspace's last block
dg_status stab_solve_impl(dg_mesh *m, double dt, double zD, double zC, double *const v[3], double tol, int maxit,
                          dg_solve_info *info, double *coef)
{
    if (!m->stab_ws) return set_error(DG_EINVAL, "divergence stabilisation workspace missing: call dg_mesh_set_div_stab first");
    const Geom &g = m->g;
    const int dim = g.dim, npe = g.npe;
    const long long nd = m->ndof;
    StabVec sv;
    sv.dim = dim;
    sv.npe = npe;
    sv.ndof = nd;
    for (int c = 0; c < dim; ++c) sv.x[c] = v[c];
    sv.r = m->stab_ws;
    sv.p = m->stab_ws + dim * nd;
    sv.q = m->stab_ws + 2 * dim * nd;
    double *vkeep = m->stab_ws + 3 * dim * nd;
    sv.dinv = m->stab_dinv;
    sv.mass_e = m->mass_e;
    sv.s = m->scal;
    sv.partial = m->partial;
    const int G = stab_grid();
    sv.partial2 = m->partial + 2 * G;
    for (int c = 0; c < dim; ++c)
        CK(cudaMemcpyAsync(vkeep + c * nd, v[c], sizeof(double) * (size_t)nd, cudaMemcpyDeviceToDevice, m->st));
    // U^2 = sum m |v''|^2 / sum m (one device reduction, read by the host for the coefficients)
    PcgScal s0{};
    s0.lam = 1.0;  // no null space
    s0.tol2 = tol * tol;
    s0.ndof_global = m->ndof_global * dim;
    s0.maxit = maxit;
    s0.hist_cap = m->hist_cap;
    CK(cudaMemcpyAsync(m->scal, &s0, sizeof(s0), cudaMemcpyHostToDevice, m->st));
    CK(launch_stab_vec(STAB_U2, sv, m->st));
    m->launches += 1;
    CKS(reduce_fin(m, G, FIN_NUMEAN));
    CK(cudaMemcpyAsync(m->hscal, m->scal, sizeof(PcgScal), cudaMemcpyDeviceToHost, m->st));
    CK(cudaStreamSynchronize(m->st));
    const double U = std::sqrt(std::max(m->hscal->nu_eff, 0.0));
    double hh = 1.0;
    for (int d = 0; d < dim; ++d) hh *= g.h[d];
    hh = std::pow(hh, 1.0 / dim);
    const double aD = dt * zD * U * hh / (g.P + 1), aC = dt * zC * U;
    if (coef) {
        coef[0] = aD;
        coef[1] = aC;
        coef[2] = U;
    }
    // Jacobi table 1/diag, diag_{c,I} = m_I + W_perp [a_D (2/h_c) sum_k w_k D_ki^2 + a_C (i in {0, P})]
    if (aD != m->stab_dinv_aD || aC != m->stab_dinv_aC) {
        const Tab &t = host_tab(g.P);
        const int n = g.n;
        std::vector<double> tab((size_t)dim * npe);
        for (int c = 0; c < dim; ++c)
            for (int I = 0; I < npe; ++I) {
                const int qc[3] = {I % n, (I / n) % n, dim == 3 ? I / (n * n) : 0};
                double mI = g.mfac;
                for (int d = 0; d < dim; ++d) mI *= t.w[qc[d]];
                const int i = qc[c];
                const double Wp = mI / (t.w[i] * 0.5 * g.h[c]);
                double kd = 0.0;
                for (int k = 0; k < n; ++k) kd += t.w[k] * t.D[k][i] * t.D[k][i];
                const double dg = mI + Wp * (aD * g.sd[c] * kd + ((i == 0 || i == g.P) ? aC : 0.0));
                tab[(size_t)c * npe + I] = 1.0 / dg;
            }
        CK(cudaMemcpyAsync(m->stab_dinv, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice, m->st));
        CK(cudaStreamSynchronize(m->st));  // tab is a host temporary
        m->stab_dinv_aD = aD;
        m->stab_dinv_aC = aC;
    }
    // r = M v'' - A v'' ; z = D^-1 r (never stored)
    {
        double *qq[3] = {sv.q, sv.q + nd, sv.q + 2 * nd};
        const double *xx[3] = {v[0], v[1], dim == 3 ? v[2] : nullptr};
        CKS(stab_apply_impl(m, xx, qq, aD, aC, nullptr, nullptr));
    }
    CK(launch_stab_vec(STAB_INIT, sv, m->st));
    m->launches += 1;
    CKS(reduce_fin(m, G, FIN_INIT, sv.partial2));   // fnorm2 = ||v''||^2
    CKS(reduce_fin(m, G, FIN_INIT2));                // r.z, ||M^-1 r||^2, convergence test
    CK(cudaMemsetAsync(sv.p, 0, sizeof(double) * (size_t)dim * nd, m->st));
    for (;;) {
        CK(cudaMemcpyAsync(m->hscal, m->scal, sizeof(PcgScal), cudaMemcpyDeviceToHost, m->st));
        CK(cudaStreamSynchronize(m->st));
        if (m->hscal->done) break;
        for (int it = 0; it < 8; ++it) {
            CK(launch_stab_vec(STAB_PUPD, sv, m->st));
            const double *pp[3] = {sv.p, sv.p + nd, dim == 3 ? sv.p + 2 * nd : nullptr};
            double *qq[3] = {sv.q, sv.q + nd, dim == 3 ? sv.q + 2 * nd : nullptr};
            int GA = 0;
            CKS(stab_apply_impl(m, pp, qq, aD, aC, m->partial, m->scal, &GA));
            CKS(reduce_fin(m, GA, FIN_ALPHA));
            CK(launch_stab_vec(STAB_UPDATE, sv, m->st));
            CKS(reduce_fin(m, G, FIN_BETA));
            m->launches += 2;
        }
    }
    const PcgScal hs = *m->hscal;
    if (info) {
        info->iters = hs.iter;
        info->rel_res = hs.fnorm2 > 0 ? std::sqrt(hs.res2 / hs.fnorm2) : std::sqrt(hs.res2);
        info->removed_mean = 0.0;
        info->f_norm = std::sqrt(hs.fnorm2);
        info->kappa_est = NAN;
    }
    if (hs.status == PCG_ST_BREAKDOWN) return set_error(DG_EBREAKDOWN, "stabilisation CG breakdown");
    if (hs.status == PCG_ST_MAXIT) return set_error(DG_ENOTCONV, "stabilisation CG reached maxit");
    return DG_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char *dg_last_error(void) { return g_err.c_str(); }

const char *dg_last_apply_kernel(void) { return g_last_kernel; }

const char *dg_version(void) { return "dgsip 0.1 (sm_100a, fp64)"; }

dg_status dg_nccl_unique_id(unsigned char out[128])
{
    if (!out) return set_error(DG_EINVAL, "null output");
    NcclApi *nc = nccl();
    if (!nc->ok) return set_error(DG_ENCCL, nc->why);
    ncclUniqueId id;
    CKN(nc->GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return DG_OK;
}

dg_status dg_mesh_create(int dim, const int N[3], const double L[3], int P, int rank, int nranks,
                         const unsigned char *nccl_uid, void *cuda_stream, dg_mesh **out)
{
    if (!out || !N || !L) return set_error(DG_EINVAL, "null argument");
    *out = nullptr;
    if (dim != 2 && dim != 3) return set_error(DG_EINVAL, "dim must be 2 or 3");
    if (P < 1 || P > PMAX) return set_error(DG_EINVAL, "P must be in [1, 10]");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(DG_EINVAL, "bad rank / nranks");
    for (int d = 0; d < dim; ++d) {
        if (N[d] < 1) return set_error(DG_EINVAL, "N[d] must be >= 1");
        if (!(L[d] > 0.0) || !std::isfinite(L[d])) return set_error(DG_EINVAL, "L[d] must be > 0");
    }
    const int S = dim - 1;
    if (N[S] % nranks != 0) return set_error(DG_EINVAL, "N of the slowest direction must be divisible by nranks");
    if (nranks > 1 && !nccl_uid) return set_error(DG_EINVAL, "nccl_uid required when nranks > 1");

    dg_mesh *m = new dg_mesh();
    Geom &g = m->g;
    g.dim = dim;
    g.P = P;
    g.n = P + 1;
    g.npe = dim == 3 ? g.n * g.n * g.n : g.n * g.n;
    for (int d = 0; d < 3; ++d) {
        g.N[d] = d < dim ? N[d] : 1;
        g.Nl[d] = g.N[d];
        g.h[d] = d < dim ? L[d] / N[d] : 1.0;
        g.tau[d] = (double)(P + 1) * (P + 1) / g.h[d];
        g.sd[d] = 2.0 / g.h[d];
    }
    g.mfac = 1.0;
    for (int d = 0; d < dim; ++d) g.mfac *= 0.5 * g.h[d];
    for (int d = 0; d < 3; ++d)
        for (int k = 0; k < NMAX; ++k) g.wsd[d][k] = k <= P ? host_tab(P).w[k] * g.sd[d] : 0.0;
    for (int d = 0; d < 3; ++d) {
        g.wfac[d] = 1.0;
        for (int d2 = 0; d2 < dim; ++d2)
            if (d2 != d) g.wfac[d] *= 0.5 * g.h[d2];
    }
    g.Nl[S] = g.N[S] / nranks;
    g.nel = (long long)g.Nl[0] * g.Nl[1] * g.Nl[2];
    for (int d = 0; d < 3; ++d) {  // brick shape is chosen per launch by the apply dispatch
        g.B[d] = 1;
        g.nbk[d] = g.Nl[d];
    }
    m->rank = rank;
    m->nranks = nranks;
    m->st = (cudaStream_t)cuda_stream;
    m->ndof = g.nel * g.npe;
    m->ndof_global = m->ndof * nranks;
    m->layer = (S == 2 ? (long long)g.Nl[0] * g.Nl[1] : (long long)g.Nl[0]) * g.npe;
    m->el_off = (long long)rank * g.nel;

    auto fail = [&](dg_status s) {
        dg_mesh_destroy(m);
        return s;
    };
    cudaGetDevice(&m->device);
    {
        static std::mutex mu;
        static std::vector<int> done;
        std::lock_guard<std::mutex> lk(mu);
        if (std::find(done.begin(), done.end(), m->device) == done.end()) {
            cudaError_t e = upload_tables();
            if (e != cudaSuccess) return fail(set_error(DG_ECUDA, std::string("table upload: ") + cudaGetErrorString(e)));
            done.push_back(m->device);
        }
    }
    // block-partial capacity: every persistent / reduction grid is at most 16 resident CTAs per SM
    // (the apply grids at most 8, the vector reductions 6-8), plus the coarse-solve slots
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
    const int pcap = 2 * (std::max(nsm, 148) * 16 + SW_NCMAX * SW_NCMAX / 32) + 64;
    dg_status s;
    if ((s = alloc_workspace(m)) != DG_OK) return fail(s);
    if ((s = alloc((void **)&m->partial, sizeof(double) * pcap)) != DG_OK) return fail(s);
    m->partial_cap = pcap;
    if ((s = alloc((void **)&m->sums, sizeof(double) * 8)) != DG_OK) return fail(s);
    if ((s = alloc((void **)&m->aux, sizeof(double) * 8)) != DG_OK) return fail(s);
    if ((s = alloc((void **)&m->scal, sizeof(PcgScal))) != DG_OK) return fail(s);
    if ((s = alloc((void **)&m->mass_e, sizeof(double) * 2 * g.npe)) != DG_OK) return fail(s);  // m, 1/m
    if ((s = alloc((void **)&m->d_flag, sizeof(int))) != DG_OK) return fail(s);
    if (cudaMallocHost((void **)&m->hscal, sizeof(PcgScal)) != cudaSuccess)
        return fail(set_error(DG_ENOMEM, "cudaMallocHost failed"));
    {
        // element-local mass table m_q = prod_d w h_d/2 (uniform mesh)
        Geom g1 = g;
        g1.nel = 1;
        cudaError_t e = launch_mass(g1, m->mass_e, m->st);
        if (e == cudaSuccess) e = launch_recip(g1, m->mass_e, m->mass_e + g.npe, m->st);
        if (e != cudaSuccess) return fail(set_error(DG_ECUDA, cudaGetErrorString(e)));
        m->launches += 2;
    }
    if (cudaStreamCreateWithFlags(&m->cs_cap, cudaStreamNonBlocking) != cudaSuccess)
        return fail(set_error(DG_ECUDA, "capture stream creation failed"));
    // halo meshes (nranks > 1, or the 1-rank halo mode: an NCCL id with nranks == 1): the
    // communicator, the exchange stream and events, the face-trace buffers and the element-layer
    // buffers of the once-per-stage kernels -- all allocated here, none in the hot calls
    m->halo = nranks > 1 || nccl_uid != nullptr;
    if (m->halo) {
        NcclApi *nc = nccl();
        if (!nc->ok) return fail(set_error(DG_ENCCL, nc->why));
        ncclUniqueId id;
        std::memcpy(&id, nccl_uid, 128);
        ncclResult_t r = nc->CommInitRank(&m->comm, nranks, id, rank);
        if (r != ncclSuccess) return fail(set_error(DG_ENCCL, std::string("ncclCommInitRank: ") + nc->GetErrorString(r)));
        m->F = (dim == 3 ? (long long)g.Nl[0] * g.Nl[1] * g.n * g.n : (long long)g.Nl[0] * g.n);
        const size_t tb = sizeof(double) * 3 * (size_t)m->F;
        double **tbufs[] = {&m->ts_lo, &m->ts_hi, &m->tr_lo, &m->tr_hi};
        for (double **p : tbufs)
            if ((s = alloc((void **)p, tb)) != DG_OK) return fail(s);
        if ((s = ensure_halos(m, true)) != DG_OK) return fail(s);
        if (cudaStreamCreateWithFlags(&m->cs_comm, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&m->ev_a, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&m->ev_b, cudaEventDisableTiming) != cudaSuccess)
            return fail(set_error(DG_ECUDA, "exchange stream / event creation failed"));
    }
    *out = m;
    return DG_OK;
}

void dg_mesh_destroy(dg_mesh *m)
{
    if (!m) return;
    if (m->st) cudaStreamSynchronize(m->st);
    else cudaDeviceSynchronize();
    double *bufs[] = {m->r,    m->q,    m->pa,    m->pb,     m->dinv,   m->z,    m->partial,
                      m->sums, m->aux,  m->mass_e, m->hist,  m->h_lo,   m->h_hi, m->hn_lo,
                      m->hn_hi, m->st_a, m->st_b,  m->st_c,  m->sf[0], m->sf[1], m->sf[2], m->sf[3],
                      m->sf[4], m->sf[5], m->d_swF, m->rc_el, m->chat, m->xc, m->rc,
                      m->ts_lo, m->ts_hi, m->tr_lo, m->tr_hi, m->stab_ws, m->stab_dinv};
    for (double *b : bufs)
        if (b) cudaFree(b);
    for (int c = 0; c < 3; ++c) {
        if (m->hv_lo[c]) cudaFree(m->hv_lo[c]);
        if (m->hv_hi[c]) cudaFree(m->hv_hi[c]);
    }
    if (m->scal) cudaFree(m->scal);
    if (m->d_sw) cudaFree(m->d_sw);
    if (m->d_flag) cudaFree(m->d_flag);
    if (m->hscal) cudaFreeHost(m->hscal);
    if (m->cs_comm) cudaStreamSynchronize(m->cs_comm);
    if (m->comm) nccl()->CommDestroy(m->comm);
    if (m->ev_a) cudaEventDestroy(m->ev_a);
    if (m->ev_b) cudaEventDestroy(m->ev_b);
    if (m->cs_comm) cudaStreamDestroy(m->cs_comm);
    if (m->gexec) cudaGraphExecDestroy(m->gexec);
    if (m->cs_cap) cudaStreamDestroy(m->cs_cap);
    for (cudaEvent_t e : m->ev) cudaEventDestroy(e);
    for (double *b : m->rk) cudaFree(b);
    if (m->cs_in) cudaStreamDestroy(m->cs_in);
    if (m->cs_out) cudaStreamDestroy(m->cs_out);
    delete m;
}

dg_status dg_mesh_set_stream(dg_mesh *m, void *cuda_stream)
{
    if (!m) return set_error(DG_EINVAL, "null mesh");
    if (m->st != (cudaStream_t)cuda_stream) {
        // work on the old stream must finish before the new one may overwrite the cached D^-1
        if (m->st) cudaStreamSynchronize(m->st);
        m->dinv_lam = m->dinv_nu = -1.0;
    }
    m->st = (cudaStream_t)cuda_stream;
    return DG_OK;
}

long long dg_mesh_local_ndof(const dg_mesh *m) { return m ? m->ndof : -1; }
long long dg_mesh_local_elements(const dg_mesh *m) { return m ? m->g.nel : -1; }
long long dg_mesh_element_offset(const dg_mesh *m) { return m ? m->el_off : -1; }
long long dg_mesh_launch_count(const dg_mesh *m) { return m ? m->launches : -1; }

dg_status dg_mesh_node_coords(const dg_mesh *m, double *xyz)
{
    if (!m || !xyz) return set_error(DG_EINVAL, "null argument");
    CK(launch_coords(m->g, m->el_off, xyz, m->st));
    const_cast<dg_mesh *>(m)->launches += 1;
    return DG_OK;
}

dg_status dg_mesh_mass(const dg_mesh *m, double *mass)
{
    if (!m || !mass) return set_error(DG_EINVAL, "null argument");
    CK(launch_mass(m->g, mass, m->st));
    const_cast<dg_mesh *>(m)->launches += 1;
    return DG_OK;
}

dg_status dg_helmholtz_apply(dg_mesh *m, double lam, const double *nu, double nu_const, const double *u, double *out)
{
    CKS(check_common(m, lam, nu, nu_const));
    if (!u || !out) return set_error(DG_EINVAL, "null field pointer");
    if (u == out) return set_error(DG_EINVAL, "u and out must not alias");
    return apply_impl(m, lam, nu, nu_const, u, out);
}

dg_status dg_helmholtz_diag(dg_mesh *m, double lam, const double *nu, double nu_const, double *diag)
{
    CKS(check_common(m, lam, nu, nu_const));
    if (!diag) return set_error(DG_EINVAL, "null field pointer");
    return diag_impl(m, lam, nu, nu_const, diag);
}

dg_status dg_pcg_solve(dg_mesh *m, double lam, const double *nu, double nu_const, const double *f, double tol,
                       int maxit, double *u, dg_solve_info *info)
{
    CKS(check_common(m, lam, nu, nu_const));
    if (!f || !u) return set_error(DG_EINVAL, "null field pointer");
    if (!(tol > 0.0)) return set_error(DG_EINVAL, "tol must be > 0");
    if (maxit < 1) return set_error(DG_EINVAL, "maxit must be >= 1");
    return pcg_impl(m, lam, nu, nu_const, f, tol, maxit, u, info);
}

dg_status dg_mesh_set_precond(dg_mesh *m, int precond)
{
    if (!m) return set_error(DG_EINVAL, "null mesh");
    if (precond != DG_PC_JACOBI && precond != DG_PC_SCHWARZ2) return set_error(DG_EINVAL, "unknown preconditioner");
    if (precond == DG_PC_SCHWARZ2) {
        const char *why = nullptr;
        if (!schwarz_supported(m->g, &why)) return set_error(DG_EUNSUPPORTED, why);
    }
    m->pc = precond;
    return DG_OK;
}

int dg_mesh_get_precond(const dg_mesh *m) { return m ? m->pc : -1; }

dg_status dg_schwarz_apply(dg_mesh *m, double lam, double nu_const, const double *r, double *z)
{
    CKS(check_common(m, lam, nullptr, nu_const));
    if (!r || !z) return set_error(DG_EINVAL, "null field pointer");
    if (r == z) return set_error(DG_EINVAL, "r and z must not alias");
    CKS(sw_check(m, nullptr));
    CKS(ensure_sw(m, nu_const));
    return sw_apply_impl(m, lam, nu_const, r, z);
}

dg_status dg_convect_rhs(dg_mesh *m, const double *const v[3], double *const out[3])
{
    if (!m || !v || !out) return set_error(DG_EINVAL, "null argument");
    const int dim = m->g.dim;
    for (int c = 0; c < dim; ++c) {
        if (!v[c] || !out[c]) return set_error(DG_EINVAL, "null component pointer");
        for (int c2 = 0; c2 < dim; ++c2)
            if (out[c] == v[c2]) return set_error(DG_EINVAL, "out must not alias v");
    }
    ConvParams a{};
    a.g = m->g;
    for (int c = 0; c < 3; ++c) {
        a.v[c] = c < dim ? v[c] : nullptr;
        a.out[c] = c < dim ? out[c] : nullptr;
    }
    if (m->halo) {
        CKS(ensure_halos(m, true));
        for (int c = 0; c < dim; ++c) {
            CKS(exchange(m, v[c], m->hv_lo[c], m->hv_hi[c]));
            a.lo[c] = m->hv_lo[c];
            a.hi[c] = m->hv_hi[c];
        }
    }
    CK(launch_convect_k(a, m->st));
    m->launches += 1;
    return DG_OK;
}

// Host-buffer apply.  Single-rank 3-D meshes with even N (the v5 kernel) are pipelined over
// C slabs of element layers: the H2D copies of u (and nu) run on one copy stream, the apply
// of slab k starts as soon as slabs k-1, k, k+1 have landed (slab 0, which needs the last
// slab across the periodic seam, goes last) and its result is copied back on a second copy
// stream, so both PCIe directions and the kernel overlap.  Otherwise: copy, apply, copy.
dg_status dg_helmholtz_apply_host(dg_mesh *m, double lam, const double *nu_host, double nu_const,
                                  const double *u_host, double *out_host)
{
    CKS(check_common(m, lam, nu_host, nu_const));
    if (!u_host || !out_host) return set_error(DG_EINVAL, "null field pointer");
    const size_t b = sizeof(double) * (size_t)m->ndof;
    CKS(stage(m, &m->st_a, b));
    CKS(stage(m, &m->st_b, b));
    if (nu_host) CKS(stage(m, &m->st_c, b));
    const Geom &g = m->g;
    int C = 0;
    if (!m->halo && g.dim == 3 && apply3_ranges_ok(g)) {
        const int nbz = g.Nl[2] / 2;
        for (int c = 16; c >= 3; --c)
            if (nbz % c == 0) {
                C = c;
                break;
            }
    }
    if (C == 0) {
        CK(cudaMemcpyAsync(m->st_a, u_host, b, cudaMemcpyHostToDevice, m->st));
        if (nu_host) CK(cudaMemcpyAsync(m->st_c, nu_host, b, cudaMemcpyHostToDevice, m->st));
        CKS(apply_impl(m, lam, nu_host ? m->st_c : nullptr, nu_const, m->st_a, m->st_b));
        CK(cudaMemcpyAsync(out_host, m->st_b, b, cudaMemcpyDeviceToHost, m->st));
        CK(cudaStreamSynchronize(m->st));
        return DG_OK;
    }
    if (!m->cs_in) {
        CK(cudaStreamCreateWithFlags(&m->cs_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&m->cs_out, cudaStreamNonBlocking));
    }
    while ((int)m->ev.size() < 2 * C + 2) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        m->ev.push_back(e);
    }
    cudaEvent_t *ein = m->ev.data(), *ecmp = m->ev.data() + C, e0 = m->ev[2 * C], e1 = m->ev[2 * C + 1];
    const int lay = g.Nl[2] / C;  // element layers per slab (even)
    const size_t cb = b / C, cn = (size_t)m->ndof / C;
    // staging buffers may still be read by earlier work on the mesh stream
    CK(cudaEventRecord(e0, m->st));
    CK(cudaStreamWaitEvent(m->cs_in, e0, 0));
    CK(cudaStreamWaitEvent(m->cs_out, e0, 0));
    for (int k = 0; k < C; ++k) {
        CK(cudaMemcpyAsync(m->st_a + k * cn, u_host + k * cn, cb, cudaMemcpyHostToDevice, m->cs_in));
        if (nu_host) CK(cudaMemcpyAsync(m->st_c + k * cn, nu_host + k * cn, cb, cudaMemcpyHostToDevice, m->cs_in));
        CK(cudaEventRecord(ein[k], m->cs_in));
    }
    for (int q = 1; q <= C; ++q) {
        const int k = q % C;                          // 1, 2, ..., C-1, then 0
        CK(cudaStreamWaitEvent(m->st, ein[k == C - 1 ? 0 : (k + 1) % C], 0));
        CK(cudaStreamWaitEvent(m->st, ein[k], 0));
        CKS(run_apply(m, lam, nu_host ? m->st_c : nullptr, nu_const, m->st_a, m->st_b, Halo{}, DotEpi{}, PProl{},
                      nullptr, k * lay, (k + 1) * lay));
        CK(cudaEventRecord(ecmp[k], m->st));
        CK(cudaStreamWaitEvent(m->cs_out, ecmp[k], 0));
        CK(cudaMemcpyAsync(out_host + k * cn, m->st_b + k * cn, cb, cudaMemcpyDeviceToHost, m->cs_out));
    }
    CK(cudaEventRecord(e1, m->cs_out));
    CK(cudaStreamWaitEvent(m->st, e1, 0));
    CK(cudaStreamSynchronize(m->st));
    return DG_OK;
}

dg_status dg_pcg_solve_host(dg_mesh *m, double lam, const double *nu_host, double nu_const, const double *f_host,
                            double tol, int maxit, double *u_host, dg_solve_info *info)
{
    CKS(check_common(m, lam, nu_host, nu_const));
    if (!f_host || !u_host) return set_error(DG_EINVAL, "null field pointer");
    if (!(tol > 0.0)) return set_error(DG_EINVAL, "tol must be > 0");
    if (maxit < 1) return set_error(DG_EINVAL, "maxit must be >= 1");
    const size_t b = sizeof(double) * (size_t)m->ndof;
    CKS(stage(m, &m->st_a, b));
    CKS(stage(m, &m->st_b, b));
    if (nu_host) CKS(stage(m, &m->st_c, b));
    CK(cudaMemcpyAsync(m->st_a, f_host, b, cudaMemcpyHostToDevice, m->st));
    CK(cudaMemcpyAsync(m->st_b, u_host, b, cudaMemcpyHostToDevice, m->st));
    if (nu_host) CK(cudaMemcpyAsync(m->st_c, nu_host, b, cudaMemcpyHostToDevice, m->st));
    dg_status s = pcg_impl(m, lam, nu_host ? m->st_c : nullptr, nu_const, m->st_a, tol, maxit, m->st_b, info);
    if (s != DG_OK && s != DG_ENOTCONV) return s;
    CK(cudaMemcpyAsync(u_host, m->st_b, b, cudaMemcpyDeviceToHost, m->st));
    CK(cudaStreamSynchronize(m->st));
    return s;
}

dg_status dg_imex_stage(dg_mesh *mv, dg_mesh *mp, double dt, double a_ex21, double a_im21, double a_im22,
                        double nu, const double *const v[3], double *const vout[3], double *psi, double tol,
                        int maxit, dg_stage_info *info)
{
    if (!mv || !mp || !v || !vout || !psi) return set_error(DG_EINVAL, "null argument");
    const Geom &g = mv->g, &gp = mp->g;
    const int dim = g.dim;
    CKS(check_pair(mv, mp));
    if (!(dt > 0.0) || !(a_im22 > 0.0) || !std::isfinite(a_ex21) || !std::isfinite(a_im21) ||
        !(nu > 0.0 && std::isfinite(nu)))
        return set_error(DG_EINVAL, "need dt > 0, a_im22 > 0, finite a_ex21/a_im21, nu > 0");
    if (!(tol > 0.0) || maxit < 1) return set_error(DG_EINVAL, "need tol > 0 and maxit >= 1");
    for (int c = 0; c < dim; ++c) {
        if (!v[c] || !vout[c]) return set_error(DG_EINVAL, "null component pointer");
        for (int c2 = 0; c2 < dim; ++c2)
            if (vout[c] == v[c2]) return set_error(DG_EINVAL, "vout must not alias v");
    }
    cudaStream_t mp_stream = mp->st;
    mp->st = mv->st;  // the whole stage runs on the velocity mesh's stream
    struct Restore {
        dg_mesh *m;
        cudaStream_t s;
        ~Restore() { m->st = s; }
    } restore{mp, mp_stream};
    const size_t bv = sizeof(double) * (size_t)mv->ndof, bp = sizeof(double) * (size_t)mp->ndof;
    for (int c = 0; c <= dim; ++c) CKS(stage(mv, &mv->sf[c], bv));
    for (int c = 4; c < 4 + dim - 1; ++c) CKS(stage(mv, &mv->sf[c], bv));
    CKS(stage(mp, &mp->sf[0], bp));
    double *Fc[3] = {mv->sf[0], mv->sf[1], dim == 3 ? mv->sf[2] : nullptr};
    double *Av = mv->sf[dim];
    // line 4 (explicit part): F_c(v) (LLF DG) ...
    CKS(dg_convect_rhs(mv, v, Fc));
    const double lamH = 1.0 / (dt * a_im22);
    for (int c = 0; c < dim; ++c) {
        // ... and F_d1(v) = -M^-1 A_0 v; v' (line 4), and the Helmholtz rhs from g (line 8);
        // Fc[c] is overwritten by f_H = lam g
        CKS(apply_impl(mv, 0.0, nullptr, nu, v[c], Av));
        CK(launch_stage_combine(g, mv->mass_e, dt * a_ex21, dt * (a_im21 - a_ex21), lamH, v[c], Fc[c], Av, vout[c],
                                Fc[c], mv->st));
        mv->launches += 1;
    }
    // line 4's explicit viscous part in rotational form (constant nu):
    // F_d + F_d3 = F_d1 - nu grad div v  ->  v' -= dt a_ex21 nu M^-1 G M_p^-1 D v.  In line 8
    // the -a_ex21 F_d3 term adds it back, so f_H = lam g is unchanged.
    double *gw[3] = {Av, mv->sf[4], mv->sf[5]};
    {
        const double *vin[3] = {v[0], v[1], dim == 3 ? v[2] : nullptr};
        CKS(div_impl(mv, vin, mp->sf[0]));
        CK(launch_scale_minv(gp, mp->mass_e, 1.0, mp->sf[0], mp->sf[0], mv->st));
        mv->launches += 1;
        CKS(grad_impl(mp, mv, mp->sf[0], gw));
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = vout[c];
            lc.c0 = 1.0;
            lc.w = gw[c];
            lc.cm = -dt * a_ex21 * nu;
            CK(launch_lincomb(g, lc, mv->mass_e, vout[c], mv->st));
            mv->launches += 1;
        }
    }
    // line 5: -lap psi = -div v' on the P-1 mesh: b = -D v' (weak DG divergence), f = M_p^-1 b
    CKS(div_impl(mv, vout, mp->sf[0]));
    CK(launch_scale_minv(gp, mp->mass_e, -1.0, mp->sf[0], mp->sf[0], mv->st));
    mv->launches += 1;
    CK(cudaMemsetAsync(psi, 0, bp, mv->st));
    dg_solve_info ip{};
    dg_status s = pcg_impl(mp, 0.0, nullptr, 1.0, mp->sf[0], tol, maxit, psi, &ip);
    if (info) info->pressure = ip;
    if (s != DG_OK) return s;
    // line 6: v'' = v' - M^-1 G psi (weak DG gradient), and line 8's rhs follows (f_H -= lam M^-1 G psi)
    CKS(grad_impl(mp, mv, psi, gw));
    for (int c = 0; c < dim; ++c) {
        CK(launch_stage_project(g, mv->mass_e, lamH, gw[c], vout[c], Fc[c], mv->st));
        mv->launches += 1;
    }
    // divergence / mass-flux stabilisation of v'' (reading A26; dg_mesh_set_div_stab),
    // and line 8's rhs follows: f_H += lam (v^ - v'')
    if (mv->stab_zD > 0.0 || mv->stab_zC > 0.0) {
        dg_solve_info is{};
        s = stab_solve_impl(mv, dt, mv->stab_zD, mv->stab_zC, vout, tol, maxit, &is, nullptr);
        if (info) info->stab = is;
        if (s != DG_OK) return s;
        const double *vkeep = mv->stab_ws + 3 * (long long)dim * mv->ndof;
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = Fc[c];
            lc.c0 = 1.0;
            lc.c[lc.n] = lamH;
            lc.y[lc.n++] = vout[c];
            lc.c[lc.n] = -lamH;
            lc.y[lc.n++] = vkeep + c * mv->ndof;
            CK(launch_lincomb(g, lc, mv->mass_e, Fc[c], mv->st));
            mv->launches += 1;
        }
    }
    // line 9: v_i - dt a_ii div(nu grad v_i) = g_i per component, from the guess v''
    for (int c = 0; c < dim; ++c) {
        dg_solve_info iv{};
        s = pcg_impl(mv, lamH, nullptr, nu, Fc[c], tol, maxit, vout[c], &iv);
        if (info) info->velocity[c] = iv;
        if (s != DG_OK) return s;
    }
    return DG_OK;
}

dg_status dg_imex_rk_step(dg_mesh *mv, dg_mesh *mp, const dg_tableau *tab, double dt, double nu,
                          double *const v[3], double *psi, double tol, int maxit, dg_step_info *info)
{
    if (!mv || !mp || !tab || !v || !psi) return set_error(DG_EINVAL, "null argument");
    CKS(check_pair(mv, mp));
    const int S = tab->s, dim = mv->g.dim;
    if (S < 2 || S > DG_RK_MAX_STAGES) return set_error(DG_EINVAL, "tableau: 2 <= s <= DG_RK_MAX_STAGES");
    if (tab->a_im[0][0] != 0.0 || tab->c[0] != 0.0)
        return set_error(DG_EINVAL, "tableau: the first stage must be explicit (a_im[0][0] = c[0] = 0)");
    for (int i = 0; i < S; ++i) {
        if (!(tab->a_im[i][i] >= 0.0)) return set_error(DG_EINVAL, "tableau: a_im[i][i] must be >= 0");
        for (int j = i; j < S; ++j)
            if (tab->a_ex[i][j] != 0.0 || (j > i && tab->a_im[i][j] != 0.0))
                return set_error(DG_EINVAL, "tableau: a_ex strictly lower, a_im lower triangular");
    }
    if (!(dt > 0.0) || !(nu > 0.0 && std::isfinite(nu)) || !(tol > 0.0) || maxit < 1)
        return set_error(DG_EINVAL, "need dt > 0, nu > 0, tol > 0, maxit >= 1");
    for (int c = 0; c < dim; ++c)
        if (!v[c]) return set_error(DG_EINVAL, "null component pointer");
    cudaStream_t mp_stream = mp->st;
    mp->st = mv->st;
    struct Restore {
        dg_mesh *m;
        cudaStream_t s;
        ~Restore() { m->st = s; }
    } restore{mp, mp_stream};
    const Geom &g = mv->g, &gp = mp->g;
    const size_t bv = sizeof(double) * (size_t)mv->ndof;
    const int need = (3 * S + 2) * dim;
    while ((int)mv->rk.size() < need) {
        double *b = nullptr;
        CKS(alloc((void **)&b, bv));
        mv->rk.push_back(b);
    }
    CKS(stage(mp, &mp->sf[0], sizeof(double) * (size_t)mp->ndof));
    auto Fc = [&](int i, int c) { return mv->rk[(i * dim + c)]; };
    auto Fd = [&](int i, int c) { return mv->rk[(S + i) * dim + c]; };
    auto Fg = [&](int i, int c) { return mv->rk[(2 * S + i) * dim + c]; };  // nu grad(div u_i)
    auto VP = [&](int c) { return mv->rk[3 * S * dim + c]; };
    auto TM = [&](int c) { return mv->rk[(3 * S + 1) * dim + c]; };
    dg_step_info inf{};
    // stage forces: F_c, F_d1 = -M^-1 A_0 u and the grad-div term nu grad(div u)
    // = nu M^-1 G M_p^-1 D u with the DG pair (constant nu: F_d2 = -F_d3 = nu grad div u)
    auto forces = [&](int i, double *const *u) -> dg_status {
        double *out[3] = {Fc(i, 0), Fc(i, 1), dim == 3 ? Fc(i, 2) : nullptr};
        const double *uin[3] = {u[0], u[1], dim == 3 ? u[2] : nullptr};
        CKS(dg_convect_rhs(mv, uin, out));
        for (int c = 0; c < dim; ++c) {
            CKS(apply_impl(mv, 0.0, nullptr, nu, u[c], TM(c)));
            LinComb lc;
            lc.w = TM(c);
            lc.cm = -1.0;
            CK(launch_lincomb(g, lc, mv->mass_e, Fd(i, c), mv->st));
            mv->launches += 1;
        }
        double *tmg[3] = {TM(0), TM(1), dim == 3 ? TM(2) : nullptr};
        CKS(div_impl(mv, uin, mp->sf[0]));
        CK(launch_scale_minv(gp, mp->mass_e, 1.0, mp->sf[0], mp->sf[0], mv->st));
        mv->launches += 1;
        CKS(grad_impl(mp, mv, mp->sf[0], tmg));
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.w = TM(c);
            lc.cm = nu;
            CK(launch_lincomb(g, lc, mv->mass_e, Fg(i, c), mv->st));
            mv->launches += 1;
        }
        return DG_OK;
    };
    CKS(forces(0, v));  // stage 1: v_1 = v
    double *vp[3] = {VP(0), VP(1), dim == 3 ? VP(2) : nullptr};
    double *tm[3] = {TM(0), TM(1), dim == 3 ? TM(2) : nullptr};
    for (int i = 1; i < S; ++i) {
        // line 4: v'_i = v + dt sum_j a_ex[i][j] (F_c + F_d + F_d3)_j, with (constant nu)
        // F_d + F_d3 = F_d1 - nu grad div u_j: the rotational, divergence-free form
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = v[c];
            lc.c0 = 1.0;
            for (int j = 0; j < i; ++j) {
                if (tab->a_ex[i][j] == 0.0) continue;
                lc.c[lc.n] = dt * tab->a_ex[i][j];
                lc.y[lc.n++] = Fc(j, c);
                lc.c[lc.n] = dt * tab->a_ex[i][j];
                lc.y[lc.n++] = Fd(j, c);
                lc.c[lc.n] = -dt * tab->a_ex[i][j];
                lc.y[lc.n++] = Fg(j, c);
            }
            CK(launch_lincomb(g, lc, mv->mass_e, vp[c], mv->st));
            mv->launches += 1;
        }
        // lines 5-6: pressure Poisson with the weak DG divergence, v'' = v' - M^-1 G psi
        CKS(div_impl(mv, vp, mp->sf[0]));
        CK(launch_scale_minv(gp, mp->mass_e, -1.0, mp->sf[0], mp->sf[0], mv->st));
        mv->launches += 1;
        // first implicit stage from psi = 0, later stages from the previous stage's psi''
        // (psi''_i ~ dt sum_j a_ij p_j changes smoothly from stage to stage)
        if (i == 1) CK(cudaMemsetAsync(psi, 0, sizeof(double) * (size_t)mp->ndof, mv->st));
        dg_solve_info ip{};
        dg_status st = pcg_impl(mp, 0.0, nullptr, 1.0, mp->sf[0], tol, maxit, psi, &ip);
        inf.pressure_iters += ip.iters;
        if (st != DG_OK) {
            if (info) *info = inf;
            return st;
        }
        CKS(grad_impl(mp, mv, psi, tm));
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = vp[c];
            lc.c0 = 1.0;
            lc.w = tm[c];
            lc.cm = -1.0;
            CK(launch_lincomb(g, lc, mv->mass_e, vp[c], mv->st));
            mv->launches += 1;
        }
        if (mv->stab_zD > 0.0 || mv->stab_zC > 0.0) {  // P:1040, reading A26
            dg_solve_info is{};
            st = stab_solve_impl(mv, dt, mv->stab_zD, mv->stab_zC, vp, tol, maxit, &is, nullptr);
            inf.stab_iters += is.iters;
            if (st != DG_OK) {
                if (info) *info = inf;
                return st;
            }
        }
        // lines 8-9: g_i = v'' + dt sum_j [(a_im - a_ex)[i][j] F_d1,j - a_ex[i][j] F_d3,j],
        // F_d3,j = -nu grad div u_j ;  v_i - dt a_ii nu lap v_i = g_i
        const double aii = tab->a_im[i][i];
        const double lam = aii > 0.0 ? 1.0 / (dt * aii) : 1.0;
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = vp[c];
            lc.c0 = lam;
            for (int j = 0; j < i; ++j) {
                const double cj = tab->a_im[i][j] - tab->a_ex[i][j];
                if (cj != 0.0) {
                    lc.c[lc.n] = lam * dt * cj;
                    lc.y[lc.n++] = Fd(j, c);
                }
                if (tab->a_ex[i][j] != 0.0) {
                    lc.c[lc.n] = lam * dt * tab->a_ex[i][j];
                    lc.y[lc.n++] = Fg(j, c);
                }
            }
            CK(launch_lincomb(g, lc, mv->mass_e, tm[c], mv->st));  // f = lam g_i
            mv->launches += 1;
            if (aii > 0.0) {
                dg_solve_info iv{};
                st = pcg_impl(mv, lam, nullptr, nu, tm[c], tol, maxit, vp[c], &iv);
                inf.velocity_iters += iv.iters;
                if (st != DG_OK) {
                    if (info) *info = inf;
                    return st;
                }
            } else {
                CK(cudaMemcpyAsync(vp[c], tm[c], bv, cudaMemcpyDeviceToDevice, mv->st));
            }
        }
        CKS(forces(i, vp));
        inf.stages += 1;
    }
    // line 11: v = v_s + dt sum_i [(b_ex - a_ex[s])_i F_c,i + (b_im - a_im[s])_i F_d1,i]
    for (int c = 0; c < dim; ++c) {
        LinComb lc;
        lc.x0 = vp[c];
        lc.c0 = 1.0;
        for (int j = 0; j < S; ++j) {
            const double ce = tab->b_ex[j] - tab->a_ex[S - 1][j], ci = tab->b_im[j] - tab->a_im[S - 1][j];
            if (ce != 0.0) {
                lc.c[lc.n] = dt * ce;
                lc.y[lc.n++] = Fc(j, c);
            }
            if (ci != 0.0) {
                lc.c[lc.n] = dt * ci;
                lc.y[lc.n++] = Fd(j, c);
            }
        }
        CK(launch_lincomb(g, lc, mv->mass_e, v[c], mv->st));
        mv->launches += 1;
    }
    CK(cudaStreamSynchronize(mv->st));
    if (info) *info = inf;
    return DG_OK;
}

dg_status dg_mesh_set_div_stab(dg_mesh *mv, double zeta_D, double zeta_C)
{
    if (!mv) return set_error(DG_EINVAL, "null mesh");
    if (!(zeta_D >= 0.0) || !(zeta_C >= 0.0) || !std::isfinite(zeta_D) || !std::isfinite(zeta_C))
        return set_error(DG_EINVAL, "zeta_D, zeta_C must be finite and >= 0");
    if ((zeta_D > 0.0 || zeta_C > 0.0) && !mv->stab_ws) {
        CKS(alloc((void **)&mv->stab_ws, sizeof(double) * 4 * (size_t)mv->g.dim * (size_t)mv->ndof));
        CKS(alloc((void **)&mv->stab_dinv, sizeof(double) * (size_t)mv->g.dim * (size_t)mv->g.npe));
    }
    mv->stab_zD = zeta_D;
    mv->stab_zC = zeta_C;
    return DG_OK;
}

dg_status dg_div_stab_apply(dg_mesh *m, double a_D, double a_C, const double *const v[3], double *const out[3])
{
    if (!m || !v || !out) return set_error(DG_EINVAL, "null argument");
    for (int c = 0; c < m->g.dim; ++c) {
        if (!v[c] || !out[c]) return set_error(DG_EINVAL, "null component pointer");
        for (int c2 = 0; c2 < m->g.dim; ++c2)
            if (out[c] == v[c2]) return set_error(DG_EINVAL, "out must not alias v");
    }
    if (!(a_D >= 0.0) || !(a_C >= 0.0)) return set_error(DG_EINVAL, "a_D, a_C must be >= 0");
    return stab_apply_impl(m, v, out, a_D, a_C, nullptr, nullptr);
}

dg_status dg_div_stab_solve(dg_mesh *m, double dt, double zeta_D, double zeta_C, double *const v[3], double tol,
                            int maxit, double coef[3], dg_solve_info *info)
{
    if (!m || !v) return set_error(DG_EINVAL, "null argument");
    for (int c = 0; c < m->g.dim; ++c)
        if (!v[c]) return set_error(DG_EINVAL, "null component pointer");
    if (!(dt > 0.0) || !(zeta_D >= 0.0) || !(zeta_C >= 0.0) || !(tol > 0.0) || maxit < 1)
        return set_error(DG_EINVAL, "dt > 0, zeta >= 0, tol > 0, maxit >= 1 required");
    return stab_solve_impl(m, dt, zeta_D, zeta_C, v, tol, maxit, info, coef);
}

dg_status dg_derivative(dg_mesh *m, const double *u, double *const out[3])
{
    if (!m || !u || !out) return set_error(DG_EINVAL, "null argument");
    DerivParams a;
    a.u = u;
    a.dirs = 0;
    for (int c = 0; c < m->g.dim; ++c)
        if (out[c]) {
            if (out[c] == u) return set_error(DG_EINVAL, "out must not alias u");
            a.out[c] = out[c];
            a.dirs |= 1 << c;
        }
    if (m->halo) {
        CKS(ensure_halos(m, true));
        CKS(exchange(m, u, m->hv_lo[0], m->hv_hi[0]));
        a.lo = m->hv_lo[0];
        a.hi = m->hv_hi[0];
    }
    CK(launch_dg_deriv(m->g, a, m->st));
    m->launches += 1;
    return DG_OK;
}

dg_status dg_imex_rk_step_vv(dg_mesh *mv, dg_mesh *mp, const dg_tableau *tab, double dt, const dg_visc_model *visc,
                             const double *const *fs, int final_projection, double *const v[3], double *psi,
                             double tol, int maxit, dg_step_info *info)
{
    if (!mv || !mp || !tab || !visc || !v || !psi) return set_error(DG_EINVAL, "null argument");
    CKS(check_pair(mv, mp));
    const int S = tab->s, dim = mv->g.dim;
    if (S < 2 || S > DG_RK_MAX_STAGES) return set_error(DG_EINVAL, "tableau: 2 <= s <= DG_RK_MAX_STAGES");
    if (tab->a_im[0][0] != 0.0 || tab->c[0] != 0.0)
        return set_error(DG_EINVAL, "tableau: the first stage must be explicit (a_im[0][0] = c[0] = 0)");
    for (int i = 0; i < S; ++i) {
        if (!(tab->a_im[i][i] >= 0.0)) return set_error(DG_EINVAL, "tableau: a_im[i][i] must be >= 0");
        for (int j = i; j < S; ++j)
            if (tab->a_ex[i][j] != 0.0 || (j > i && tab->a_im[i][j] != 0.0))
                return set_error(DG_EINVAL, "tableau: a_ex strictly lower, a_im lower triangular");
    }
    if (!(dt > 0.0) || !(visc->nu0 > 0.0) || !(visc->nu1 >= 0.0) || !(visc->vmax > 0.0) || !std::isfinite(visc->nu0) ||
        !std::isfinite(visc->nu1) || !(tol > 0.0) || maxit < 1)
        return set_error(DG_EINVAL, "need dt > 0, nu0 > 0, nu1 >= 0, vmax > 0, tol > 0, maxit >= 1");
    for (int c = 0; c < dim; ++c)
        if (!v[c]) return set_error(DG_EINVAL, "null component pointer");
    if (fs)
        for (int k = 0; k < S * dim; ++k)
            if (!fs[k]) return set_error(DG_EINVAL, "null forcing pointer");
    cudaStream_t mp_stream = mp->st;
    mp->st = mv->st;
    struct Restore {
        dg_mesh *m;
        cudaStream_t s;
        ~Restore() { m->st = s; }
    } restore{mp, mp_stream};
    const Geom &g = mv->g, &gp = mp->g;
    const size_t bv = sizeof(double) * (size_t)mv->ndof;
    const int need = 4 * S * dim + 2 * dim + 2 + dim * dim;
    while ((int)mv->rk.size() < need) {
        double *b = nullptr;
        CKS(alloc((void **)&b, bv));
        mv->rk.push_back(b);
    }
    CKS(stage(mp, &mp->sf[0], sizeof(double) * (size_t)mp->ndof));
    auto Fc = [&](int i, int c) { return mv->rk[(i * dim + c)]; };
    auto Fd1 = [&](int i, int c) { return mv->rk[(S + i) * dim + c]; };
    auto Fd3 = [&](int i, int c) { return mv->rk[(2 * S + i) * dim + c]; };
    auto Fd23 = [&](int i, int c) { return mv->rk[(3 * S + i) * dim + c]; };  // F_d2 + F_d3
    auto VP = [&](int c) { return mv->rk[4 * S * dim + c]; };
    auto TM = [&](int c) { return mv->rk[(4 * S + 1) * dim + c]; };
    double *NU = mv->rk[(4 * S + 2) * dim], *WK = mv->rk[(4 * S + 2) * dim + 1];
    auto DV = [&](int e, int c) { return mv->rk[(4 * S + 2) * dim + 2 + e * dim + c]; };  // D_c v_e
    const bool multi = mv->halo;
    if (multi) CKS(ensure_halos(mv, true));
    dg_step_info inf{};
    // D_c u for the selected directions (overwrite or accumulate scale * D_c u)
    auto deriv = [&](const double *u, double *const *out, int dirs, int acc, double scale) -> dg_status {
        DerivParams a;
        a.u = u;
        if (multi) {
            CKS(exchange(mv, u, mv->hv_lo[0], mv->hv_hi[0]));
            a.lo = mv->hv_lo[0];
            a.hi = mv->hv_hi[0];
        }
        for (int c = 0; c < 3; ++c) a.out[c] = out[c];
        a.dirs = dirs;
        a.accumulate = acc;
        a.scale = scale;
        CK(launch_dg_deriv(g, a, mv->st));
        mv->launches += 1;
        return DG_OK;
    };
    // stage forces at (u, nu): F_c (LLF), F_d1 = -M^-1 A_0(nu) u (SIP, lam = 0),
    // F_d3 = -D(nu div u), F_d2 + F_d3 = sum_e D_e(nu D_c u_e) + F_d3, div u = sum_e D_e u_e
    auto forces = [&](int i, double *const *u, const double *nu) -> dg_status {
        double *out[3] = {Fc(i, 0), Fc(i, 1), dim == 3 ? Fc(i, 2) : nullptr};
        const double *uin[3] = {u[0], u[1], dim == 3 ? u[2] : nullptr};
        CKS(dg_convect_rhs(mv, uin, out));
        for (int c = 0; c < dim; ++c) {
            CKS(apply_impl(mv, 0.0, nu, 0.0, u[c], TM(c)));
            LinComb lc;
            lc.w = TM(c);
            lc.cm = -1.0;
            CK(launch_lincomb(g, lc, mv->mass_e, Fd1(i, c), mv->st));
            mv->launches += 1;
        }
        for (int e = 0; e < dim; ++e) {
            double *o[3] = {DV(e, 0), DV(e, 1), dim == 3 ? DV(e, 2) : nullptr};
            CKS(deriv(u[e], o, (1 << dim) - 1, 0, 1.0));
        }
        LinComb ld;
        for (int e = 0; e < dim; ++e) {
            ld.c[ld.n] = 1.0;
            ld.y[ld.n++] = DV(e, e);
        }
        CK(launch_lincomb(g, ld, mv->mass_e, WK, mv->st));  // div u
        CK(launch_nu_mul(g, nu, WK, nullptr, WK, mv->st));   // nu div u
        mv->launches += 2;
        double *f3[3] = {Fd3(i, 0), Fd3(i, 1), dim == 3 ? Fd3(i, 2) : nullptr};
        CKS(deriv(WK, f3, (1 << dim) - 1, 0, -1.0));
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = Fd3(i, c);
            lc.c0 = 1.0;
            CK(launch_lincomb(g, lc, mv->mass_e, Fd23(i, c), mv->st));
            mv->launches += 1;
            for (int e = 0; e < dim; ++e) {
                CK(launch_nu_mul(g, nu, DV(e, c), nullptr, WK, mv->st));  // nu D_c u_e
                mv->launches += 1;
                double *o[3] = {nullptr, nullptr, nullptr};
                o[e] = Fd23(i, c);
                CKS(deriv(WK, o, 1 << e, 1, 1.0));
            }
        }
        return DG_OK;
    };
    // lines 5-6 (and 13-14): lap psi = div w (weak DG divergence, SIP Poisson on mp from psi = 0),
    // w <- w - M^-1 G psi
    auto project = [&](double *const *w, bool warm) -> dg_status {
        CKS(div_impl(mv, w, mp->sf[0]));
        CK(launch_scale_minv(gp, mp->mass_e, -1.0, mp->sf[0], mp->sf[0], mv->st));
        mv->launches += 1;
        // stages i > 2 start from the previous stage's psi''; the first stage and the
        // final projection (a small correction) from 0
        if (!warm) CK(cudaMemsetAsync(psi, 0, sizeof(double) * (size_t)mp->ndof, mv->st));
        dg_solve_info ip{};
        const dg_status st = pcg_impl(mp, 0.0, nullptr, 1.0, mp->sf[0], tol, maxit, psi, &ip);
        inf.pressure_iters += ip.iters;
        if (st != DG_OK) return st;
        double *tm[3] = {TM(0), TM(1), dim == 3 ? TM(2) : nullptr};
        CKS(grad_impl(mp, mv, psi, tm));
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = w[c];
            lc.c0 = 1.0;
            lc.w = tm[c];
            lc.cm = -1.0;
            CK(launch_lincomb(g, lc, mv->mass_e, w[c], mv->st));
            mv->launches += 1;
        }
        if (mv->stab_zD > 0.0 || mv->stab_zC > 0.0) {  // P:1040, reading A26
            dg_solve_info is{};
            const dg_status ss = stab_solve_impl(mv, dt, mv->stab_zD, mv->stab_zC, w, tol, maxit, &is, nullptr);
            inf.stab_iters += is.iters;
            if (ss != DG_OK) return ss;
        }
        return DG_OK;
    };
    auto fsp = [&](int j, int c) { return fs ? fs[j * dim + c] : nullptr; };
    auto fail = [&](dg_status st) {
        if (info) *info = inf;
        return st;
    };
    // stage 1: v_1 = v, nu_1 = nu(v)
    {
        const double *vv[3] = {v[0], v[1], dim == 3 ? v[2] : nullptr};
        CK(launch_visc_model(g, vv, visc->nu0, visc->nu1, visc->vmax, NU, mv->st));
        mv->launches += 1;
        dg_status st = forces(0, v, NU);
        if (st != DG_OK) return fail(st);
    }
    double *vp[3] = {VP(0), VP(1), dim == 3 ? VP(2) : nullptr};
    double *tm[3] = {TM(0), TM(1), dim == 3 ? TM(2) : nullptr};
    for (int i = 1; i < S; ++i) {
        // line 4: v'_i = v + dt [sum_j a_ex[i][j] (F_c + F_d + F_d3)_j + sum_{j<=i} a_im[i][j] F_s,j],
        // F_d + F_d3 = F_d1 + (F_d2 + F_d3) + F_d3
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = v[c];
            lc.c0 = 1.0;
            for (int j = 0; j < i; ++j) {
                const double a = dt * tab->a_ex[i][j];
                if (a == 0.0) continue;
                const double *ys[4] = {Fc(j, c), Fd1(j, c), Fd23(j, c), Fd3(j, c)};
                for (const double *y : ys) {
                    lc.c[lc.n] = a;
                    lc.y[lc.n++] = y;
                }
            }
            for (int j = 0; j <= i && fs; ++j)
                if (tab->a_im[i][j] != 0.0) {
                    lc.c[lc.n] = dt * tab->a_im[i][j];
                    lc.y[lc.n++] = fsp(j, c);
                }
            CK(launch_lincomb(g, lc, mv->mass_e, vp[c], mv->st));
            mv->launches += 1;
        }
        dg_status st = project(vp, i > 1);  // lines 5-6
        if (st != DG_OK) return fail(st);
        // line 7: nu_i = nu(v''_i)
        {
            const double *vv[3] = {vp[0], vp[1], dim == 3 ? vp[2] : nullptr};
            CK(launch_visc_model(g, vv, visc->nu0, visc->nu1, visc->vmax, NU, mv->st));
            mv->launches += 1;
        }
        // lines 8-9: g_i = v'' + dt sum_j [(a_im - a_ex)[i][j] F_d1,j - a_ex[i][j] F_d3,j];
        // v_i - dt a_ii div(nu_i grad v_i) = g_i  (lam = 1/(dt a_ii), f = lam g_i; Jacobi-PCG
        // with the nu_i field), from the guess v''_i
        const double aii = tab->a_im[i][i];
        const double lam = aii > 0.0 ? 1.0 / (dt * aii) : 1.0;
        for (int c = 0; c < dim; ++c) {
            LinComb lc;
            lc.x0 = vp[c];
            lc.c0 = lam;
            for (int j = 0; j < i; ++j) {
                const double cj = tab->a_im[i][j] - tab->a_ex[i][j];
                if (cj != 0.0) {
                    lc.c[lc.n] = lam * dt * cj;
                    lc.y[lc.n++] = Fd1(j, c);
                }
                if (tab->a_ex[i][j] != 0.0) {
                    lc.c[lc.n] = -lam * dt * tab->a_ex[i][j];
                    lc.y[lc.n++] = Fd3(j, c);
                }
            }
            CK(launch_lincomb(g, lc, mv->mass_e, tm[c], mv->st));
            mv->launches += 1;
            if (aii > 0.0) {
                dg_solve_info iv{};
                st = pcg_impl(mv, lam, NU, 0.0, tm[c], tol, maxit, vp[c], &iv);
                inf.velocity_iters += iv.iters;
                if (st != DG_OK) return fail(st);
            } else {
                CK(cudaMemcpyAsync(vp[c], tm[c], bv, cudaMemcpyDeviceToDevice, mv->st));
            }
        }
        st = forces(i, vp, NU);
        if (st != DG_OK) return fail(st);
        inf.stages += 1;
    }
    // line 11: v = v_s + dt sum_i [(b_ex - a_ex[s])_i (F_c + F_d2 + F_d3)_i
    //                              + (b_im - a_im[s])_i (F_d1 + F_s)_i]
    for (int c = 0; c < dim; ++c) {
        LinComb lc;
        lc.x0 = vp[c];
        lc.c0 = 1.0;
        for (int j = 0; j < S; ++j) {
            const double ce = tab->b_ex[j] - tab->a_ex[S - 1][j], ci = tab->b_im[j] - tab->a_im[S - 1][j];
            if (ce != 0.0) {
                lc.c[lc.n] = dt * ce;
                lc.y[lc.n++] = Fc(j, c);
                lc.c[lc.n] = dt * ce;
                lc.y[lc.n++] = Fd23(j, c);
            }
            if (ci != 0.0) {
                lc.c[lc.n] = dt * ci;
                lc.y[lc.n++] = Fd1(j, c);
                if (fs) {
                    lc.c[lc.n] = dt * ci;
                    lc.y[lc.n++] = fsp(j, c);
                }
            }
        }
        CK(launch_lincomb(g, lc, mv->mass_e, v[c], mv->st));
        mv->launches += 1;
    }
    // lines 12-15: final projection
    if (final_projection) {
        const dg_status st = project(v, false);
        if (st != DG_OK) return fail(st);
    }
    CK(cudaStreamSynchronize(mv->st));
    if (info) *info = inf;
    return DG_OK;
}

dg_status dg_divergence(dg_mesh *mv, dg_mesh *mp, const double *const v[3], double *div_weak)
{
    if (!mv || !mp || !v || !div_weak) return set_error(DG_EINVAL, "null argument");
    CKS(check_pair(mv, mp));
    for (int c = 0; c < mv->g.dim; ++c)
        if (!v[c]) return set_error(DG_EINVAL, "null component pointer");
    return div_impl(mv, v, div_weak);
}

dg_status dg_gradient(dg_mesh *mp, dg_mesh *mv, const double *psi, double *const grad_weak[3])
{
    if (!mv || !mp || !psi || !grad_weak) return set_error(DG_EINVAL, "null argument");
    CKS(check_pair(mv, mp));
    for (int c = 0; c < mv->g.dim; ++c)
        if (!grad_weak[c] || grad_weak[c] == psi) return set_error(DG_EINVAL, "null or aliased component pointer");
    return grad_impl(mp, mv, psi, grad_weak);
}

dg_status dg_gll_tables(int P, double *xi, double *w, double *D)
{
    if (P < 1 || P > PMAX) return set_error(DG_EINVAL, "P must be in [1, 10]");
    if (!xi || !w || !D) return set_error(DG_EINVAL, "null argument");
    const Tab &t = host_tab(P);
    for (int i = 0; i <= P; ++i) {
        xi[i] = t.xi[i];
        w[i] = t.w[i];
        for (int j = 0; j <= P; ++j) D[i * (P + 1) + j] = t.D[i][j];
    }
    return DG_OK;
}

dg_status dg_check_field(dg_mesh *m, const double *x, int positive)
{
    if (!m || !x) return set_error(DG_EINVAL, "null argument");
    CK(cudaMemsetAsync(m->d_flag, 0, sizeof(int), m->st));
    CK(launch_check_field(m->ndof, x, positive, m->d_flag, m->st));
    m->launches += 1;
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, m->d_flag, sizeof(int), cudaMemcpyDeviceToHost, m->st));
    CK(cudaStreamSynchronize(m->st));
    if (bad) return set_error(DG_EINVAL, positive ? "field has non-finite or non-positive entries"
                                                  : "field has non-finite entries");
    return DG_OK;
}

}  // extern "C"
