"""Temporal convergence of dg_imex_rk_step_vv on the 3-D vortex with solution-dependent viscosity,
case VVP: nu(v) = nu0 + nu1 (|v|/2)^2, nu0 = nu1 = 0.01 (Re ~ 133), exact
solution and manufactured forcing of eq. var-visc-test, periodic unit cube (one period; the
paper's [-1/2,1/2]^3 shifted), final time T = 0.25, final projection on."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import node_coords  # noqa: E402
from workloads.inputs import vvp_exact, vvp_forcing  # noqa: E402


def run(name, N=4, P=8, ks=(5, 6, 7), nu0=0.01, nu1=0.01, T=0.25, tol=1e-12):
    dev = torch.device("cuda")
    st = torch.cuda.current_stream()
    L = (1.0, 1.0, 1.0)
    mv = dg.dg_mesh_create(3, (N,) * 3, L, P, stream=st)
    mp = dg.dg_mesh_create(3, (N,) * 3, L, P - 1, stream=st)
    if N >= 2:
        dg.dg_mesh_set_precond(mp, dg.DG_PC_SCHWARZ2)
    X = node_coords(3, (N,) * 3, L, P)
    tab = dg.TABLEAUX[name]
    cs = tab["c"]
    errs = []
    for k in ks:
        dt = 2.0 ** -k
        v = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in vvp_exact(X, 0.0)[0]]
        psi = torch.zeros(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
        for n in range(int(round(T / dt))):
            t = n * dt
            fs = [[torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in vvp_forcing(X, t + c * dt, nu0, nu1)]
                  for c in cs]
            dg.dg_imex_rk_step_vv(mv, mp, tab, dt, (nu0, nu1, 2.0), v, psi, tol, 20000, fs=fs)
        ve = vvp_exact(X, T)[0]
        err = math.sqrt(sum(float(((v[c].cpu().numpy() - ve[c]) ** 2).mean()) for c in range(3)) / 3)
        errs.append(err)
    eoc = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    return errs, eoc


if __name__ == "__main__":
    for name in sys.argv[1:] or ("RK-ARS3",):
        errs, eoc = run(name)
        print(name, ["%.3e" % e for e in errs], ["%.2f" % x for x in eoc], flush=True)
