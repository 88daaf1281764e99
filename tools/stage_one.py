"""Two config-4 IMEX stages (Schwarz Poisson), as bench.py's stage leg: for launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_04167_b200 as dg
from workloads import config
from workloads.inputs import GAMMA_SDIRK3

c4 = config(4)
st = torch.cuda.current_stream()
dev = torch.device("cuda:0")
mv = dg.dg_mesh_create(3, c4.N, c4.L, c4.P, stream=st)
mp = dg.dg_mesh_create(3, c4.N, c4.L, c4.P_p, stream=st)
v = [torch.from_numpy(a).to(dev) for a in c4.tg_velocity()]
vo = [torch.empty_like(v[0]) for _ in range(3)]
psi = torch.empty(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
dg.dg_mesh_set_precond(mp, dg.DG_PC_SCHWARZ2)
g = GAMMA_SDIRK3
for k in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    info = dg.dg_imex_stage(mv, mp, 1e-2, g, 0.0, g, c4.nu0, v, vo, psi, c4.tol, 20000)
    b.record(st)
    torch.cuda.synchronize()
    print("stage %.2f ms" % a.elapsed_time(b), info.as_dict())
