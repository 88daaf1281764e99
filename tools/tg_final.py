"""TGP with the non-stiffly-accurate tableaux RK-CB2 / RK-CB3e: does the
final projection (Alg. 3 lines 12-15, skipped for constant nu at P:801) decide stability?
Runs dg_imex_rk_step_vv with nu1 = 0 (constant nu = 0.02) with and without the final projection,
and dg_imex_rk_step (constant-nu driver) for reference.  python tools/tg_final.py [P]"""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_04167_b200 as dg  # noqa: E402
from tools.tg_eoc import tg  # noqa: E402
from workloads import node_coords  # noqa: E402


def run(name, mode, N=8, P=8, ks=(5, 6, 7, 8), nu=0.02, T=0.25):
    dev = torch.device("cuda")
    st = torch.cuda.current_stream()
    mv = dg.dg_mesh_create(2, (N, N), (1.0, 1.0), P, stream=st)
    mp = dg.dg_mesh_create(2, (N, N), (1.0, 1.0), P - 1, stream=st)
    X = node_coords(2, (N, N), (1.0, 1.0), P)
    errs = []
    for k in ks:
        dt = 2.0 ** -k
        v = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in tg(X, 0.0, nu)]
        psi = torch.zeros(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
        try:
            for _ in range(int(round(T / dt))):
                if mode == "const":
                    dg.dg_imex_rk_step(mv, mp, dg.TABLEAUX[name], dt, nu, v, psi, 1e-13, 20000)
                else:
                    dg.dg_imex_rk_step_vv(mv, mp, dg.TABLEAUX[name], dt, (nu, 0.0, 1.0), v, psi, 1e-13, 20000,
                                          final_projection=(mode == "final"))
            ve = tg(X, T, nu)
            err = math.sqrt(sum(float(((v[c].cpu().numpy() - ve[c]) ** 2).mean()) for c in range(2)) / 2)
        except Exception:
            err = float("inf")
        errs.append(err if math.isfinite(err) else float("inf"))
    return errs


if __name__ == "__main__":
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    for name in ("RK-CB3e", "RK-CB2", "RK-ARS3"):
        for mode in ("const", "vv-nofinal", "final"):
            errs = run(name, mode, P=P)
            print(name, mode, ["%.3e" % e for e in errs], flush=True)
