"""A/B timing of the config-4 constant-nu applies (P = 6 pressure, P = 7 velocity) and of one
Jacobi Poisson solve / Schwarz Poisson solve (MODE-2 applies): DG_LIBRARY=<so> python tools/ab_c4.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_04167_b200 as dg
from workloads import config

c = config(4)
st = torch.cuda.current_stream()
res = []
for P in (6, 7):
    m = dg.dg_mesh_create(3, c.N, c.L, P, stream=st)
    u = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (m.n_el, m.npe))).cuda()
    out = torch.empty_like(u)
    for _ in range(3):
        dg.dg_helmholtz_apply(m, 0.0, None, 1.0, u, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20):
        dg.dg_helmholtz_apply(m, 0.0, None, 1.0, u, out)
    b.record(st)
    torch.cuda.synchronize()
    res.append("P%d apply %.1f us (%s)" % (P, a.elapsed_time(b) / 20 * 1e3, dg.dg_last_apply_kernel().split(' ')[0]))
    print(res[-1], flush=True)
    if P == 6:
        dg.dg_mesh_set_precond(m, dg.DG_PC_SCHWARZ2)
        f = u - u.mean()
        ts = []
        for k in range(3):
            x = torch.zeros_like(u)
            torch.cuda.synchronize()
            a.record(st)
            info = dg.dg_pcg_solve(m, 0.0, None, 1.0, f, 1e-10, 5000, x)
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res.append("schwarz poisson %.2f ms %d it (%.1f us/it)" % (min(ts[1:]), info.iters, min(ts[1:]) / info.iters * 1e3))
print(os.environ.get("DG_LIBRARY", "default").split('/')[-1], " | ".join(res))
