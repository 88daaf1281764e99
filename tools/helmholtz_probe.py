import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2112_04167_b200 as dg
from workloads import config
c = config(4)
st = torch.cuda.current_stream()
m = dg.dg_mesh_create(3, c.N, c.L, c.P, stream=st)
f = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (m.n_el, m.npe))).cuda()
for k in range(3):
    u = torch.zeros_like(f)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(st)
    info = dg.dg_pcg_solve(m, c.lam, None, c.nu0, f, c.tol, 200, u)
    b.record(st); torch.cuda.synchronize()
    print("solve ms", a.elapsed_time(b), info.iters)
