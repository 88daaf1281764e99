"""Setup vs per-iteration cost of the c5 PCG solve: times dg_pcg_solve capped at k iterations.
    python tools/pcg_breakdown.py [cfg]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_04167_b200 as dg
from workloads import config

c = config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
m = dg.dg_mesh_create(c.dim, c.N[: c.dim], c.L[: c.dim], c.P, stream=st)
nu = c.nu()
nu = None if nu is None else torch.from_numpy(nu).to(dev)
f = torch.from_numpy(c.rhs()).to(dev) if hasattr(c, "rhs") else torch.from_numpy(c.apply_input()).to(dev)
for k in (1, 2, 4, 8, 12, 16, 18, 5000):
    ts = []
    for rep in range(4):
        x = torch.zeros_like(f)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        info = dg.dg_pcg_solve(m, c.lam, nu, c.nu0, f, c.tol if k == 5000 else 1e-30, k, x, raise_on_notconv=False)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print("maxit %5d iters %3d  ms %.3f (min %.3f)" % (k, info.iters, statistics.median(ts[1:]), min(ts[1:])))
