"""GPU parity of the two-level additive Schwarz preconditioner
against the oracle's plain definition (oracle.Schwarz2: dense element blocks extracted from
the oracle's own operator, dense Q1 prolongation, numpy pseudo-inverse of P^T A P), and of
Schwarz-preconditioned solves against the oracle's exact discrete solutions.

Tolerances: the preconditioner is a linear operator applied once -> relative L2 <= 1e-12
(the 'operator application' bar of north_star); solves converged to 1e-11 -> <= 1e-9.
"""
import math

import numpy as np
import pytest

import oracle
from workloads import config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2112_04167_b200 as dg  # noqa: E402

DEV = torch.device("cuda:0")
TWO_PI = 2 * math.pi


def rel(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV)


def H(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def meshes(dim, N, L, P):
    return dg.dg_mesh_create(dim, N, L, P, stream=torch.cuda.current_stream()), oracle.Mesh(dim, N, L, P)


CASES = [
    (2, (5, 4), (1.0, 1.3), 3, 0.7, 1.3),      # ragged 2-D, odd N, lam > 0
    (2, (2, 2), (TWO_PI, TWO_PI), 6, 0.0, 1.0),  # N = 2: both faces to the same neighbour; Poisson
    (3, (3, 2, 4), (1.0, 0.8, 1.2), 4, 0.0, 1.0),
    (3, (2, 3, 2), (TWO_PI,) * 3, 2, 229.4, 1.0 / 1600),
    (3, (4, 4, 4), (TWO_PI,) * 3, 6, 0.0, 1.0),
    (3, (3, 3, 3), (1.0, 1.0, 1.0), 7, 5.0, 0.3),
]


@pytest.mark.parametrize("dim,N,L,P,lam,nu", CASES)
def test_schwarz_apply_matches_oracle(dim, N, L, P, lam, nu):
    m, om = meshes(dim, N, L, P)
    r = np.random.default_rng(P + 10 * dim).uniform(-1, 1, (om.n_el, om.npe))
    if lam == 0.0:
        r -= r.mean()  # a residual of the Poisson system is orthogonal to the constants (A8)
    z = torch.empty(om.n_el, om.npe, dtype=torch.float64, device=DEV)
    dg.dg_schwarz_apply(m, lam, nu, T(r), z)
    ref = oracle.Schwarz2(om, lam, nu_const=nu)(r)
    assert rel(H(z), ref) <= 1e-12


@pytest.mark.parametrize("dim,N,L,P,lam,nu", CASES)
def test_schwarz_pcg_matches_oracle_solution(dim, N, L, P, lam, nu):
    m, om = meshes(dim, N, L, P)
    dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    assert dg.dg_mesh_get_precond(m) == dg.DG_PC_SCHWARZ2
    f = np.random.default_rng(7 + P).uniform(-1, 1, (om.n_el, om.npe))
    u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
    info = dg.dg_pcg_solve(m, lam, None, nu, T(f), 1e-11, 2000, u)
    ref, *_ = oracle.pcg_solve(om, lam, f, nu_const=nu, tol=1e-14)
    assert rel(H(u), ref) <= 1e-9, info.as_dict()
    assert info.rel_res <= 1e-11


def test_schwarz_pcg_iterates_match_oracle_pcg():
    # the k-th iterate of the GPU Schwarz-PCG equals the oracle's plain preconditioned CG with
    # the same B after the same k iterations (maxit stop; deferred x update included)
    dim, N, L, P = 3, (3, 4, 3), (1.0, 1.2, 0.9), 3
    m, om = meshes(dim, N, L, P)
    dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    f = np.random.default_rng(5).uniform(-1, 1, (om.n_el, om.npe))
    B = oracle.Schwarz2(om, 0.0)
    for k in (1, 2, 5):
        u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
        info = dg.dg_pcg_solve(m, 0.0, None, 1.0, T(f), 1e-30, k, u, raise_on_notconv=False)
        assert info.iters == k
        ref, it = oracle.pcg_precond(om, 0.0, f, B, tol=1e-30, maxit=k)
        assert it == k
        assert rel(H(u), ref) <= 1e-10, k


def test_schwarz_poisson_iterations_h_robust():
    # two-level Schwarz: the iteration count of the P = 6 Poisson problem does not grow with
    # the element count (Jacobi-PCG roughly doubles per refinement)
    its = []
    for Ne in (8, 16):
        m = dg.dg_mesh_create(3, (Ne,) * 3, (TWO_PI,) * 3, 6, stream=torch.cuda.current_stream())
        dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
        f = np.random.default_rng(Ne).uniform(-1, 1, (Ne ** 3, 343))
        u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
        info = dg.dg_pcg_solve(m, 0.0, None, 1.0, T(f), 1e-10, 2000, u)
        its.append(info.iters)
    assert its[1] <= 1.25 * its[0] + 3 and its[1] <= 150, its


def test_schwarz_c4_poisson_full_size_residual():
    """Config-4 pressure Poisson (32^3, P_p = 6, lam = 0) with the Schwarz preconditioner at the
    config tolerance: residual recomputed with the ORACLE's operator on sampled elements."""
    c = config(4)
    N, P = c.N, c.P_p
    m = dg.dg_mesh_create(3, N, c.L, P, stream=torch.cuda.current_stream())
    om = oracle.Mesh(3, N, c.L, P)
    dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    f = np.random.default_rng(404).uniform(-1, 1, (om.n_el, om.npe))
    u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
    info = dg.dg_pcg_solve(m, 0.0, None, 1.0, T(f), c.tol, 2000, u)
    assert info.rel_res <= c.tol and info.iters <= 150, info.as_dict()
    mass = oracle.mass(om)
    fp = f - (mass * f).sum() / mass.sum()
    uh = H(u)
    rng = np.random.default_rng(9)
    el = np.sort(rng.choice(om.n_el, 256, replace=False))
    au = oracle.sip_apply(om, 0.0, uh, nu_const=1.0, elems=el)
    res = (mass[el] * fp[el] - au) / mass[el]
    assert np.linalg.norm(res) / np.linalg.norm(fp[el]) <= 20 * c.tol
    assert abs((mass * uh).sum()) <= 1e-10 * np.abs(uh).max() * mass.sum()


def test_schwarz_rejections():
    m = dg.dg_mesh_create(3, (1, 2, 2), (1.0,) * 3, 3, stream=torch.cuda.current_stream())
    with pytest.raises(dg.DGError) as e:
        dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    assert e.value.status == dg.DG_EUNSUPPORTED
    m = dg.dg_mesh_create(3, (2, 2, 2), (1.0,) * 3, 3, stream=torch.cuda.current_stream())
    with pytest.raises(dg.DGError):
        dg.dg_mesh_set_precond(m, 7)


@pytest.mark.parametrize("dim,N,P,lam", [(3, (8, 8, 8), 4, 0.0), (3, (4, 4, 4), 7, 256.0), (2, (6, 5), 6, 3.0)])
def test_schwarz_variable_nu_solve_matches_oracle(dim, N, P, lam):
    # variable nu: blocks and coarse operator with the mass-weighted mean nu (a spectrally
    # equivalent preconditioner); the solution is the exact discrete one of the nu-field system
    L = (1.0, 1.0, 1.0)[:dim]
    m, om = meshes(dim, N, L, P)
    dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    from workloads import node_coords

    X = node_coords(dim, N, L, P)
    nu = 0.01 * (1.5 + 0.5 * np.sin(2 * np.pi * X[0]) * np.cos(2 * np.pi * X[1]))
    f = np.random.default_rng(31).uniform(-1, 1, (om.n_el, om.npe))
    u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
    info = dg.dg_pcg_solve(m, lam, T(nu), 0.0, T(f), 1e-11, 5000, u)
    ref, it_j, *_ = oracle.pcg_solve(om, lam, f, nu=nu, tol=1e-14)
    assert rel(H(u), ref) <= 1e-9, info.as_dict()
    if lam == 0.0:  # diffusion-dominated: clearly fewer iterations than Jacobi
        m2 = dg.dg_mesh_create(dim, N, L, P, stream=torch.cuda.current_stream())
        u2 = torch.zeros_like(u)
        info_j = dg.dg_pcg_solve(m2, lam, T(nu), 0.0, T(f), 1e-11, 5000, u2)
        assert info.iters < 0.6 * info_j.iters, (info.iters, info_j.iters)


def test_schwarz_c3_poisson_full_size():
    """Config-3 pressure Poisson (16^3, P_p = 6, lam = 0) with the Schwarz preconditioner at the
    config tolerance, checked with the ORACLE's full operator: ||M^-1 (M f' - A u)|| / ||f'||."""
    c = config(3)
    m = dg.dg_mesh_create(3, c.N, c.L, c.P_p, stream=torch.cuda.current_stream())
    om = oracle.Mesh(3, c.N, c.L, c.P_p)
    dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    f = c.poisson_rhs_raw()
    u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
    info = dg.dg_pcg_solve(m, 0.0, None, 1.0, T(f), c.tol, 2000, u)
    mass = oracle.mass(om)
    fp = f - (mass * f).sum() / mass.sum()
    uh = H(u)
    r = mass * fp - oracle.sip_apply(om, 0.0, uh, nu_const=1.0)
    res = np.linalg.norm(r / mass) / np.linalg.norm(fp)
    assert res <= 1.1 * c.tol, (res, info.as_dict())
    assert info.iters <= 120, info.as_dict()


def test_schwarz_max_coarse_grid_c5_mesh():
    """The largest coarse grid (N_d = 64: config-5 mesh, 56.6 M DOF, P = 5) with constant nu:
    Poisson to 1e-10, residual recomputed with the ORACLE's operator on sampled elements."""
    c = config(5)
    m = dg.dg_mesh_create(3, c.N, c.L, c.P, stream=torch.cuda.current_stream())
    om = oracle.Mesh(3, c.N, c.L, c.P)
    dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    f = c.rhs(0)
    u = torch.zeros(f.shape, dtype=torch.float64, device=DEV)
    info = dg.dg_pcg_solve(m, 0.0, None, 1.0, T(f), 1e-10, 2000, u)
    assert info.rel_res <= 1e-10 and info.iters <= 150, info.as_dict()
    mass = oracle.mass(om)
    fbar = (mass * f).sum() / mass.sum()
    uh = H(u)
    el = np.sort(np.random.default_rng(3).choice(om.n_el, 128, replace=False))
    au = oracle.sip_apply(om, 0.0, uh, nu_const=1.0, elems=el)
    res = (mass[el] * (f[el] - fbar) - au) / mass[el]
    assert np.linalg.norm(res) / np.linalg.norm(f[el] - fbar) <= 20 * 1e-10
