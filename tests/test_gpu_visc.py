"""GPU parity of the variable-viscosity pieces: the central-flux DG
derivative and one dg_imex_rk_step_vv step (nu(v) of P:1222, forcing, final projection) vs the
oracle on identical inputs; temporal order of RK-ARS3 on the VVP manufactured solution."""
import numpy as np
import pytest

import oracle
from workloads import node_coords
from workloads.inputs import vvp_exact, vvp_forcing

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2112_04167_b200 as dg  # noqa: E402

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


@pytest.mark.parametrize("dim,N,P", [(3, (3, 2, 4), 4), (2, (5, 3), 7), (3, (1, 2, 2), 3), (3, (4, 4, 4), 10)])
def test_dg_derivative_matches_oracle(dim, N, P):
    L = (1.0, 1.3, 0.8)[:dim]
    m = dg.dg_mesh_create(dim, N, L, P, stream=torch.cuda.current_stream())
    om = oracle.Mesh(dim, N, L, P)
    u = np.random.default_rng(P).uniform(-1, 1, (om.n_el, om.npe))
    out = [torch.empty(om.n_el, om.npe, dtype=torch.float64, device=DEV) for _ in range(dim)]
    dg.dg_derivative(m, T(u), out)
    ref = oracle.dg_derivative(om, u)
    for c in range(dim):
        assert rel(H(out[c]), ref[c]) <= 1e-12, c


@pytest.mark.parametrize("name,dim,N,P,forced,fp", [("RK-ARS3", 3, (2, 3, 2), 4, True, True),
                                                    ("RK-CB3e", 2, (4, 3), 5, False, True),
                                                    ("RK-ARS3", 3, (2, 2, 4), 3, True, False)])
def test_imex_rk_step_vv_matches_oracle(name, dim, N, P, forced, fp):
    L = (1.0, 1.0, 1.0)[:dim]
    mv = dg.dg_mesh_create(dim, N, L, P, stream=torch.cuda.current_stream())
    mp = dg.dg_mesh_create(dim, N, L, P - 1, stream=torch.cuda.current_stream())
    omv, omp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    X = node_coords(dim, N, L, P)
    rng = np.random.default_rng(11)
    if dim == 3:
        v, _ = vvp_exact(X, 0.05)
    else:
        v = [1.0 + np.sin(2 * np.pi * X[0]) * np.cos(2 * np.pi * X[1]),
             1.0 - np.cos(2 * np.pi * X[0]) * np.sin(2 * np.pi * X[1])]
    v = [a + 1e-3 * rng.uniform(-1, 1, a.shape) for a in v]
    visc = (0.01, 0.02, 2.0)
    dt = 4e-3
    tab = dg.TABLEAUX[name]
    fs = None
    if forced:
        fs = [[f + 0.1 * rng.uniform(-1, 1, f.shape) for f in (vvp_forcing(X, dt * c, *visc[:2]) if dim == 3
                                                               else [np.cos(2 * np.pi * X[1]), np.sin(2 * np.pi * X[0])])]
              for c in tab["c"]]
    dv = [T(a) for a in v]
    psi = torch.zeros(omp.n_el, omp.npe, dtype=torch.float64, device=DEV)
    info = dg.dg_imex_rk_step_vv(mv, mp, tab, dt, visc, dv, psi, 1e-13, 20000,
                                 fs=None if fs is None else [[T(a) for a in row] for row in fs], final_projection=fp)
    ref = oracle.imex_rk_step_vv(omv, omp, oracle.ORACLE_TABLEAUX[name], dt, visc, v, fs=fs, final_projection=fp,
                                 tol=1e-14)
    for cc in range(dim):
        assert rel(H(dv[cc]), ref[cc]) <= 1e-9, (cc, info.as_dict())
    assert info.stages == len(tab["c"]) - 1 and info.velocity_iters > 0


def test_imex_rk_step_vv_rejects_bad_model():
    mv = dg.dg_mesh_create(3, (2, 2, 2), (1.0,) * 3, 3, stream=torch.cuda.current_stream())
    mp = dg.dg_mesh_create(3, (2, 2, 2), (1.0,) * 3, 2, stream=torch.cuda.current_stream())
    v = [torch.zeros(8, 64, dtype=torch.float64, device=DEV) for _ in range(3)]
    psi = torch.zeros(8, 27, dtype=torch.float64, device=DEV)
    with pytest.raises(dg.DGError) as e:
        dg.dg_imex_rk_step_vv(mv, mp, dg.TABLEAUX["RK-ARS3"], 1e-2, (0.0, 0.01, 2.0), v, psi, 1e-10, 100)
    assert e.value.status == dg.DG_EINVAL


def test_vvp_ars3_third_order():
    """VVP: nu0 = nu1 = 0.01, T = 0.25; RK-ARS3 velocity RMS error at T for
    dt = 2^-5..2^-7 shows order ~3 (spatial error of 4^3 elements at P = 8 far below)."""
    import sys

    sys.path.insert(0, ".")
    from tools.vvp_eoc import run

    errs, eoc = run("RK-ARS3", N=4, P=8, ks=(5, 6, 7))
    assert errs[-1] < 1e-4, errs
    assert all(e >= 2.7 for e in eoc), (errs, eoc)
