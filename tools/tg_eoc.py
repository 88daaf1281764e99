"""Temporal convergence of dg_imex_rk_step on the 2D traveling Taylor-Green vortex (TGP,
PAPER.md:1094-1125): nu = 0.02, domain [-1/2,1/2]^2 (here [0,1]^2 shifted), T = 0.25."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import node_coords  # noqa: E402


def tg(X, t, nu):
    x, y = X[0] - 0.5, X[1] - 0.5  # [0,1]^2 -> [-1/2,1/2]^2
    e = math.exp(-8 * math.pi ** 2 * nu * t)
    vx = 1 + np.sin(2 * np.pi * (x - t)) * np.cos(2 * np.pi * (y - 0.125 - t)) * e
    vy = 1 - np.cos(2 * np.pi * (x - t)) * np.sin(2 * np.pi * (y - 0.125 - t)) * e
    return vx, vy


def run(name, N=8, P=8, ks=(5, 6, 7, 8), nu=0.02, T=0.25, stab=None):
    """stab = (zeta_D, zeta_C): divergence / mass-flux stabilisation after every projection
    (reading A26); None: off."""
    dev = torch.device("cuda")
    st = torch.cuda.current_stream()
    mv = dg.dg_mesh_create(2, (N, N), (1.0, 1.0), P, stream=st)
    mp = dg.dg_mesh_create(2, (N, N), (1.0, 1.0), P - 1, stream=st)
    if stab is not None:
        dg.dg_mesh_set_div_stab(mv, *stab)
    X = node_coords(2, (N, N), (1.0, 1.0), P)
    errs = []
    for k in ks:
        dt = 2.0 ** -k
        v0 = tg(X, 0.0, nu)
        v = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in v0]
        psi = torch.zeros(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
        for _ in range(int(round(T / dt))):
            dg.dg_imex_rk_step(mv, mp, dg.TABLEAUX[name], dt, nu, v, psi, 1e-13, 20000)
        ve = tg(X, T, nu)
        err = math.sqrt(sum(float(((v[c].cpu().numpy() - ve[c]) ** 2).mean()) for c in range(2)) / 2)
        errs.append(err if math.isfinite(err) else float("inf"))
    eoc = [math.log2(errs[i] / errs[i + 1]) if math.isfinite(errs[i]) and errs[i + 1] > 0 else float("nan")
           for i in range(len(errs) - 1)]
    return errs, eoc


if __name__ == "__main__":
    for stab in (None, (1.0, 1.0)):
        for name in ("RK-ARS3", "RK-CB3e", "RK-CB2", "RK-TR"):
            try:
                errs, eoc = run(name, stab=stab)
            except Exception as e:  # a diverging run may fail inside a solve
                print(name, "stab" if stab else "nostab", "failed:", str(e)[:100], flush=True)
                continue
            print(name, "stab" if stab else "nostab", ["%.3e" % e for e in errs], ["%.2f" % x for x in eoc], flush=True)
