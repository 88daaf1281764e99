"""A/B timing of the variable-nu P = 7 apply and Jacobi Helmholtz solve on 16^3 elements (the VVP step's
velocity solves): DG_LIBRARY=<so> [DG_SMEM_BUDGET_KB=..] python tools/ab_p7nu.py [N]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_04167_b200 as dg

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
P = 7
st = torch.cuda.current_stream()
m = dg.dg_mesh_create(3, (N,) * 3, (1.0,) * 3, P, stream=st)
rng = np.random.default_rng(3)
u = torch.from_numpy(rng.uniform(-1, 1, (m.n_el, m.npe))).cuda()
nu = torch.from_numpy(rng.uniform(0.01, 0.02, (m.n_el, m.npe))).cuda()
out = torch.empty_like(u)
lam = 128.0 / 0.4358665215
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    dg.dg_helmholtz_apply(m, lam, nu, 0.0, u, out)
torch.cuda.synchronize()
a.record(st)
for _ in range(20):
    dg.dg_helmholtz_apply(m, lam, nu, 0.0, u, out)
b.record(st)
torch.cuda.synchronize()
res = ["apply %.1f us (%s)" % (a.elapsed_time(b) / 20 * 1e3, dg.dg_last_apply_kernel())]
ts = []
for k in range(4):
    x = torch.zeros_like(u)
    torch.cuda.synchronize()
    a.record(st)
    info = dg.dg_pcg_solve(m, lam, nu, 0.0, u, 1e-10, 5000, x)
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
res.append("helmholtz %.3f ms %d it (%.1f us/it) (%s)" % (min(ts[1:]), info.iters, min(ts[1:]) / info.iters * 1e3,
                                                          dg.dg_last_apply_kernel()))
print(os.environ.get("DG_LIBRARY", "default").split('/')[-1], os.environ.get("DG_SMEM_BUDGET_KB", "-"), " | ".join(res),
      "chk %.12e" % float(x.double().abs().sum()))
