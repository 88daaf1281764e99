"""Small invocations of every kernel family (for compute-sanitizer memcheck / racecheck runs):
apply (v4/v5/v6 dispatch), diag, Jacobi- and Schwarz-PCG, convect (2-D and 3-D), DG pair,
DG derivative, IMEX stage and steps (constant and variable viscosity)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_04167_b200 as dg  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
rng = np.random.default_rng(0)


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


for dim, N, P in ((3, (4, 4, 2), 5), (3, (2, 2, 2), 6), (3, (3, 2, 3), 3), (2, (4, 3), 4)):
    m = dg.dg_mesh_create(dim, N, (1.0,) * dim, P, stream=st)
    u = T(rng.uniform(-1, 1, (m.n_el, m.npe)))
    nu = T(0.5 + rng.uniform(0, 1, (m.n_el, m.npe)))
    out = torch.empty_like(u)
    dg.dg_helmholtz_apply(m, 2.0, nu, 0.0, u, out)
    dg.dg_helmholtz_apply(m, 2.0, None, 0.7, u, out)
    dg.dg_helmholtz_diag(m, 2.0, nu, 0.0, out)
    x = torch.zeros_like(u)
    dg.dg_pcg_solve(m, 2.0, nu, 0.0, u, 1e-8, 200, x, raise_on_notconv=False)
    dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
    x.zero_()
    dg.dg_pcg_solve(m, 0.0, None, 1.0, u, 1e-8, 200, x, raise_on_notconv=False)
    x.zero_()
    dg.dg_pcg_solve(m, 3.0, nu, 0.0, u, 1e-8, 200, x, raise_on_notconv=False)
    dg.dg_schwarz_apply(m, 0.5, 1.0, u, out)
    v = [T(rng.uniform(-1, 1, (m.n_el, m.npe))) for _ in range(dim)]
    o = [torch.empty_like(u) for _ in range(dim)]
    dg.dg_convect_rhs(m, v, o)
    dg.dg_derivative(m, u, o)
    mp = dg.dg_mesh_create(dim, N, (1.0,) * dim, P - 1, stream=st)
    psi = torch.zeros(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
    dg.dg_imex_rk_step(m, mp, dg.TABLEAUX["RK-ARS3"], 1e-3, 0.01, v, psi, 1e-8, 500)
    dg.dg_mesh_set_precond(m, dg.DG_PC_JACOBI)
    dg.dg_imex_rk_step_vv(m, mp, dg.TABLEAUX["RK-CB3e"], 1e-3, (0.01, 0.01, 2.0), v, psi, 1e-8, 500,
                          fs=[[torch.ones_like(u) for _ in range(dim)] for _ in range(4)])
torch.cuda.synchronize()
print("sanitize_small ok")
