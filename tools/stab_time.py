"""Timing of the divergence / mass-flux stabilisation on the config-4 velocity (32^3, P = 7)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_04167_b200 as dg
from workloads import config

c = config(4)
st = torch.cuda.current_stream()
m = dg.dg_mesh_create(3, c.N, c.L, c.P, stream=st)
dg.dg_mesh_set_div_stab(m, 1.0, 1.0)
v0 = [torch.from_numpy(a).cuda() for a in c.tg_velocity()]
out = [torch.empty_like(v0[0]) for _ in range(3)]
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    dg.dg_div_stab_apply(m, 1e-4, 1e-3, v0, out)
torch.cuda.synchronize()
a.record(st)
for _ in range(10):
    dg.dg_div_stab_apply(m, 1e-4, 1e-3, v0, out)
b.record(st)
torch.cuda.synchronize()
ta = a.elapsed_time(b) / 10
for k in range(2):
    v = [x.clone() for x in v0]
    torch.cuda.synchronize()
    a.record(st)
    info, coef = dg.dg_div_stab_solve(m, 1e-2, 1.0, 1.0, v, tol=1e-10)
    b.record(st)
    torch.cuda.synchronize()
print("stab apply %.1f us (%.2f TB/s at 48 B/DOF)  solve %.2f ms, %d it, coef %s" % (ta * 1e3, 3 * m.ndof * 16 / (ta * 1e-3) / 1e12, a.elapsed_time(b), info.iters, coef))
