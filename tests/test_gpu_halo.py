"""The multi-GPU data plane on one GPU: the 1-rank HALO MODE (SURVEY.md:311).

A mesh created with an NCCL id and nranks == 1 routes every slab-boundary face of the slowest
direction through the same machinery a multi-rank slab uses: the face-trace kernel, the grouped
NCCL send/recv on the exchange stream (here: to itself), the interior / boundary layer split of
the apply, the halo-consuming branches of every apply generation (v4, v5, v6), the diagonal,
the split MODE-2/3 PCG with all-reduced dots, the Schwarz coarse gather + all-reduce, and the
element-layer exchanges of the once-per-stage kernels.  Each is compared with the oracle and
with the plain mesh (Q16: the per-element arithmetic is partition-independent; only dot-product
grouping may differ).
"""
import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import config, node_coords  # noqa: E402

DEV = torch.device("cuda:0")


def rel(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV)


def H(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def mk(dim, N, L, P, halo):
    return dg.dg_mesh_create(dim, N, L, P, stream=torch.cuda.current_stream(), halo_mode=halo)


# shapes: v6 (N_x, N_y % 4 == 0, P odd <= 5) with and without the layer split (N_z >= 6 even),
# v5 (even N, other P), v4 (odd counts, 2-D)
SHAPES = [(3, (4, 4, 6), 5), (3, (4, 8, 8), 3), (3, (4, 4, 2), 5), (3, (2, 2, 6), 6), (3, (2, 4, 8), 7),
          (3, (3, 2, 5), 4), (3, (2, 2, 4), 2), (2, (4, 6), 4), (2, (3, 5), 3)]


@pytest.mark.parametrize("dim,N,P", SHAPES)
@pytest.mark.parametrize("varnu", [False, True])
def test_halo_apply_diag(dim, N, P, varnu):
    L = (1.0, 1.3, 0.8)[:dim]
    mh, m0 = mk(dim, N, L, P, True), mk(dim, N, L, P, False)
    om = oracle.Mesh(dim, N, L, P)
    rng = np.random.default_rng(P + 7 * dim)
    u = rng.uniform(-1, 1, (om.n_el, om.npe))
    nu = (0.3 + rng.uniform(0, 1, u.shape)) if varnu else None
    dnu = None if nu is None else T(nu)
    for lam in (0.0, 3.1):
        oh, o0 = torch.empty(u.shape, dtype=torch.float64, device=DEV), torch.empty(u.shape, dtype=torch.float64, device=DEV)
        dg.dg_helmholtz_apply(mh, lam, dnu, 0.45, T(u), oh)
        dg.dg_helmholtz_apply(m0, lam, dnu, 0.45, T(u), o0)
        ref = oracle.sip_apply(om, lam, u, nu=nu, nu_const=0.45)
        assert rel(H(oh), ref) <= 1e-12
        assert rel(H(oh), H(o0)) <= 1e-15          # Q16
        dh = torch.empty_like(oh)
        dg.dg_helmholtz_diag(mh, lam, dnu, 0.45, dh)
        assert rel(H(dh), oracle.sip_diag(om, lam, nu=nu, nu_const=0.45)) <= 1e-12


@pytest.mark.parametrize("dim,N,P,lam,varnu", [(3, (4, 4, 6), 5, 4.0, True), (3, (4, 4, 8), 3, 0.0, False),
                                               (3, (2, 2, 6), 6, 0.0, False), (3, (2, 4, 6), 7, 9.0, True),
                                               (3, (3, 2, 3), 4, 2.0, True), (2, (4, 6), 4, 0.0, True)])
def test_halo_pcg(dim, N, P, lam, varnu):
    L = (1.0, 1.1, 1.2)[:dim]
    mh = mk(dim, N, L, P, True)
    om = oracle.Mesh(dim, N, L, P)
    rng = np.random.default_rng(40 + P)
    f = rng.uniform(-1, 1, (om.n_el, om.npe))
    nu = (0.5 + rng.uniform(0, 1, f.shape)) if varnu else None
    u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
    info = dg.dg_pcg_solve(mh, lam, None if nu is None else T(nu), 0.7, T(f), 1e-11, 20000, u)
    ref, *_ = oracle.pcg_solve(om, lam, f, nu=nu, nu_const=0.7, tol=1e-14)
    assert rel(H(u), ref) <= 1e-9, info.as_dict()


@pytest.mark.parametrize("N,P,lam", [((4, 4, 6), 6, 0.0), ((4, 4, 8), 5, 0.0), ((2, 4, 6), 4, 3.0)])
def test_halo_schwarz_pcg(N, P, lam):
    L = (2 * math.pi,) * 3
    mh = mk(3, N, L, P, True)
    dg.dg_mesh_set_precond(mh, dg.DG_PC_SCHWARZ2)
    om = oracle.Mesh(3, N, L, P)
    f = np.random.default_rng(9).uniform(-1, 1, (om.n_el, om.npe))
    u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
    info = dg.dg_pcg_solve(mh, lam, None, 1.0, T(f), 1e-11, 5000, u)
    ref, *_ = oracle.pcg_solve(om, lam, f, nu_const=1.0, tol=1e-14)
    assert rel(H(u), ref) <= 1e-9, info.as_dict()
    # the variable-nu Schwarz path (mean-nu blocks, nu face traces for the apply)
    nu = 0.5 + np.random.default_rng(10).uniform(0, 1, f.shape)
    u2 = torch.zeros_like(u)
    dg.dg_pcg_solve(mh, lam + 1.0, T(nu), 0.0, T(f), 1e-11, 5000, u2)
    ref2, *_ = oracle.pcg_solve(om, lam + 1.0, f, nu=nu, tol=1e-14)
    assert rel(H(u2), ref2) <= 1e-9


@pytest.mark.parametrize("dim,N,P", [(3, (2, 3, 4), 5), (2, (4, 3), 4), (3, (2, 2, 2), 7)])
def test_halo_convect_pair_derivative(dim, N, P):
    L = (1.0, 1.4, 0.8)[:dim]
    mh = mk(dim, N, L, P, True)
    mph = mk(dim, N, L, P - 1, True)
    om, omp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    rng = np.random.default_rng(P)
    v = [rng.uniform(-1, 1, (om.n_el, om.npe)) for _ in range(dim)]
    dv = [T(a) for a in v]
    do = [torch.empty_like(dv[0]) for _ in range(dim)]
    dg.dg_convect_rhs(mh, dv, do)
    ref = oracle.convect(om, v)
    for c in range(dim):
        assert rel(H(do[c]), ref[c]) <= 1e-12
    d = torch.empty(omp.n_el, omp.npe, dtype=torch.float64, device=DEV)
    dg.dg_divergence(mh, mph, dv, d)
    assert rel(H(d), oracle.dg_divergence_weak(om, v)) <= 1e-12
    q = rng.uniform(-1, 1, (omp.n_el, omp.npe))
    gw = [torch.empty_like(dv[0]) for _ in range(dim)]
    dg.dg_gradient(mph, mh, T(q), gw)
    rg = oracle.dg_gradient_weak(omp, q)
    for c in range(dim):
        assert rel(H(gw[c]), rg[c]) <= 1e-12
    dd = [torch.empty_like(dv[0]) for _ in range(dim)]
    dg.dg_derivative(mh, dv[0], dd)
    rd = oracle.dg_derivative(om, v[0])
    for c in range(dim):
        assert rel(H(dd[c]), rd[c]) <= 1e-12


def test_halo_imex_stage_and_rk_step():
    dim, N, P = 3, (4, 4, 6), 5
    L = (2 * math.pi,) * 3
    mv, mp = mk(dim, N, L, P, True), mk(dim, N, L, P - 1, True)
    dg.dg_mesh_set_precond(mp, dg.DG_PC_SCHWARZ2)
    omv, omp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    X = node_coords(dim, N, L, P)
    rng = np.random.default_rng(3)
    v = [np.sin(X[0]) * np.cos(X[1]) * np.cos(X[2]) + 1e-2 * rng.uniform(-1, 1, X[0].shape),
         -np.cos(X[0]) * np.sin(X[1]) * np.cos(X[2]) + 1e-2 * rng.uniform(-1, 1, X[0].shape),
         1e-2 * rng.uniform(-1, 1, X[0].shape)]
    dt, a, nu = 1e-2, 0.4358665, 1.0 / 1600.0
    dv = [T(x) for x in v]
    do = [torch.empty_like(dv[0]) for _ in range(3)]
    psi = torch.zeros(omp.n_el, omp.npe, dtype=torch.float64, device=DEV)
    dg.dg_imex_stage(mv, mp, dt, a, 0.0, a, nu, dv, do, psi, 1e-12, 20000)
    ref, psi_ref, _ = oracle.imex_stage(omv, omp, dt, a, 0.0, a, nu, v, tol=1e-14)
    for c in range(3):
        assert rel(H(do[c]), ref[c]) <= 1e-9
    vs = [T(x) for x in v]
    dg.dg_imex_rk_step(mv, mp, dg.TABLEAUX["RK-ARS3"], 5e-3, 0.02, vs, psi, 1e-13, 20000)
    ref2 = oracle.imex_rk_step(omv, omp, oracle.ORACLE_TABLEAUX["RK-ARS3"], 5e-3, 0.02, v, tol=1e-14)
    for c in range(3):
        assert rel(H(vs[c]), ref2[c]) <= 1e-9


def test_halo_c5_full_size_matches_plain_mesh():
    """BASELINE configs[4] at full size in halo mode (face traces exchanged every apply, the
    interior / boundary layer split): the apply equals the plain mesh's to rounding (Q16) and
    the PCG solve takes the same number of iterations to the same solution."""
    c = config(5)
    st = torch.cuda.current_stream()
    mh = dg.dg_mesh_create(3, c.N, c.L, c.P, stream=st, halo_mode=True)
    m0 = dg.dg_mesh_create(3, c.N, c.L, c.P, stream=st)
    u, nu, f = T(c.apply_input()), T(c.nu()), T(c.rhs(0))
    oh, o0 = torch.empty_like(u), torch.empty_like(u)
    dg.dg_helmholtz_apply(mh, c.lam, nu, c.nu0, u, oh)
    dg.dg_helmholtz_apply(m0, c.lam, nu, c.nu0, u, o0)
    assert rel(H(oh), H(o0)) <= 1e-15
    xh, x0 = torch.zeros_like(u), torch.zeros_like(u)
    ih = dg.dg_pcg_solve(mh, c.lam, nu, c.nu0, f, c.tol, 2000, xh)
    i0 = dg.dg_pcg_solve(m0, c.lam, nu, c.nu0, f, c.tol, 2000, x0)
    assert ih.iters == i0.iters
    assert rel(H(xh), H(x0)) <= 1e-12
