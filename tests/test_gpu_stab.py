"""GPU parity of the divergence / mass-flux stabilisation (
reading A26) through the C-ABI: operator (<= 1e-12), coefficients, solve (<= 1e-9 vs the
oracle's CG to 1e-14), the stabilised IMEX stage / RK step vs the oracle composition, and the
NEXT-1 pin: the discrete divergence (broken divergence + normal jumps) of the projected
velocity drops when the stabilisation follows the projection, and tends to 0 as zeta grows."""
import math

import numpy as np
import pytest

import oracle
from oracle.stab import div_measures, div_stab_apply, div_stab_solve

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import node_coords  # noqa: E402

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


SHAPES = [(3, (2, 3, 2), 3), (3, (3, 2, 4), 5), (3, (1, 2, 2), 4), (3, (2, 2, 2), 7), (2, (4, 3), 5), (2, (1, 2), 3)]


@pytest.mark.parametrize("dim,N,P", SHAPES)
@pytest.mark.parametrize("halo", [False, True])
def test_stab_apply(dim, N, P, halo):
    L = (1.0, 1.3, 0.8)[:dim]
    m = dg.dg_mesh_create(dim, N, L, P, stream=torch.cuda.current_stream(), halo_mode=halo)
    om = oracle.Mesh(dim, N, L, P)
    rng = np.random.default_rng(P)
    v = [rng.uniform(-1, 1, (om.n_el, om.npe)) for _ in range(dim)]
    out = [torch.empty(om.n_el, om.npe, dtype=torch.float64, device=DEV) for _ in range(dim)]
    dg.dg_div_stab_apply(m, 0.37, 1.9, [T(x) for x in v], out)
    ref = div_stab_apply(om, v, 0.37, 1.9)
    for c in range(dim):
        assert rel(H(out[c]), ref[c]) <= 1e-12, c


@pytest.mark.parametrize("dim,N,P", [(3, (2, 3, 2), 3), (3, (2, 2, 4), 4), (2, (4, 3), 5)])
@pytest.mark.parametrize("halo", [False, True])
def test_stab_solve(dim, N, P, halo):
    L = (1.0, 1.3, 0.8)[:dim]
    m = dg.dg_mesh_create(dim, N, L, P, stream=torch.cuda.current_stream(), halo_mode=halo)
    dg.dg_mesh_set_div_stab(m, 1.0, 1.0)
    om = oracle.Mesh(dim, N, L, P)
    rng = np.random.default_rng(11 + P)
    v = [1.0 + rng.uniform(-1, 1, (om.n_el, om.npe)) for _ in range(dim)]
    dv = [T(x) for x in v]
    dt = 0.05
    info, coef = dg.dg_div_stab_solve(m, dt, 1.3, 0.7, dv, tol=1e-12)
    ref, it, (aD, aC, U) = div_stab_solve(om, v, dt, 1.3, 0.7, tol=1e-14)
    assert abs(coef[0] - aD) <= 1e-13 * aD and abs(coef[1] - aC) <= 1e-13 * aC and abs(coef[2] - U) <= 1e-13 * U
    for c in range(dim):
        assert rel(H(dv[c]), ref[c]) <= 1e-9, (c, info.as_dict(), it)
    assert info.iters > 0 and info.rel_res <= 1e-12


def test_stabilised_projection_reduces_the_discrete_divergence():
    """NEXT-1 pin (SURVEY.md:807): v'' = v' - M^-1 G psi from the DG pair and the SIP Poisson
    solve on the P-1 mesh, then the stabilisation; the penalised divergence measures of v''
    (broken divergence, normal jumps) fall with zeta and tend to 0."""
    dim, N, P = 3, (3, 3, 4), 4
    L = (2 * math.pi,) * 3
    st = torch.cuda.current_stream()
    mv = dg.dg_mesh_create(dim, N, L, P, stream=st)
    mp = dg.dg_mesh_create(dim, N, L, P - 1, stream=st)
    dg.dg_mesh_set_div_stab(mv, 1.0, 1.0)
    om = oracle.Mesh(dim, N, L, P)
    rng = np.random.default_rng(2)
    v = [rng.uniform(-1, 1, (om.n_el, om.npe)) for _ in range(dim)]
    dv = [T(x) for x in v]
    d = torch.empty(mp.n_el, mp.npe, dtype=torch.float64, device=DEV)
    dg.dg_divergence(mv, mp, dv, d)
    mpm = torch.empty_like(d)
    dg.dg_mesh_mass(mp, mpm)
    psi = torch.zeros_like(d)
    dg.dg_pcg_solve(mp, 0.0, None, 1.0, -d / mpm, 1e-12, 20000, psi)
    gw = [torch.empty_like(dv[0]) for _ in range(dim)]
    dg.dg_gradient(mp, mv, psi, gw)
    mvm = torch.empty_like(dv[0])
    dg.dg_mesh_mass(mv, mvm)
    vpp = [dv[c] - gw[c] / mvm for c in range(dim)]
    d0 = sum(div_measures(om, v))
    d1 = sum(div_measures(om, [H(x) for x in vpp]))
    assert d1 < d0                                   # the projection alone reduces it
    prev = d1
    for zeta in (1.0, 10.0, 1e3):
        w = [x.clone() for x in vpp]
        dg.dg_div_stab_solve(mv, 0.1, zeta, zeta, w, tol=1e-13, maxit=20000)
        dz = sum(div_measures(om, [H(x) for x in w]))
        assert dz < prev, (zeta, dz, prev)
        prev = dz
    assert prev < 0.05 * d1


def test_stabilised_imex_stage_and_rk_step_vs_oracle():
    dim, N, P = 3, (2, 2, 4), 4
    L = (2 * math.pi,) * 3
    st = torch.cuda.current_stream()
    mv = dg.dg_mesh_create(dim, N, L, P, stream=st)
    mp = dg.dg_mesh_create(dim, N, L, P - 1, stream=st)
    dg.dg_mesh_set_div_stab(mv, 1.0, 1.0)
    omv, omp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    X = node_coords(dim, N, L, P)
    rng = np.random.default_rng(44)
    v = [np.sin(X[0]) * np.cos(X[1]) * np.cos(X[2]) + 1e-2 * rng.uniform(-1, 1, X[0].shape),
         -np.cos(X[0]) * np.sin(X[1]) * np.cos(X[2]) + 1e-2 * rng.uniform(-1, 1, X[0].shape),
         1e-2 * rng.uniform(-1, 1, X[0].shape)]
    dt, a, nu = 5e-2, 0.4358665, 1.0 / 100.0
    dv = [T(x) for x in v]
    do = [torch.empty_like(dv[0]) for _ in range(3)]
    psi = torch.zeros(omp.n_el, omp.npe, dtype=torch.float64, device=DEV)
    info = dg.dg_imex_stage(mv, mp, dt, a, 0.0, a, nu, dv, do, psi, 1e-13, 20000)
    assert info.stab.iters > 0
    ref, _, _ = oracle.imex_stage(omv, omp, dt, a, 0.0, a, nu, v, tol=1e-14, stab=(1.0, 1.0))
    for c in range(3):
        assert rel(H(do[c]), ref[c]) <= 1e-9, (c, info.as_dict())
    vs = [T(x) for x in v]
    si = dg.dg_imex_rk_step(mv, mp, dg.TABLEAUX["RK-CB3e"], dt, nu, vs, psi, 1e-13, 20000)
    assert si.stab_iters > 0
    ref2 = oracle.imex_rk_step(omv, omp, oracle.ORACLE_TABLEAUX["RK-CB3e"], dt, nu, v, tol=1e-14, stab=(1.0, 1.0))
    for c in range(3):
        assert rel(H(vs[c]), ref2[c]) <= 1e-9
