"""Probe: config-4 Poisson (P_p = 6) and velocity Helmholtz (P = 7) solves with Jacobi vs the
two-level Schwarz preconditioner -- iterations and CUDA-event time per solve."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import config  # noqa: E402

c = config(4)
st = torch.cuda.current_stream()
dev = torch.device("cuda:0")
out = {}
reps = int(os.environ.get("REPS", "3"))
for name, P, lam, nu in (("poisson", c.P_p, 0.0, 1.0), ("helmholtz", c.P, c.lam, c.nu0)):
    m = dg.dg_mesh_create(3, c.N, c.L, P, stream=st)
    f = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (m.n_el, m.npe))).to(dev)
    for pc in (dg.DG_PC_JACOBI, dg.DG_PC_SCHWARZ2):
        if os.environ.get("ONLY_SW") and pc == dg.DG_PC_JACOBI:
            continue
        dg.dg_mesh_set_precond(m, pc)
        ts = []
        for k in range(reps + 1):
            u = torch.zeros_like(f)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(st)
            info = dg.dg_pcg_solve(m, lam, None, nu, f, c.tol, 20000, u)
            b.record(st)
            torch.cuda.synchronize()
            if k:
                ts.append(a.elapsed_time(b))
        out["%s_%s" % (name, "jacobi" if pc == 0 else "schwarz")] = {
            "iters": info.iters, "ms": float(np.median(ts)), "us_per_iter": 1e3 * float(np.median(ts)) / info.iters,
            "kappa": info.kappa_est}
print(json.dumps(out, indent=1))
