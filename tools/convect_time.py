"""Time the LLF convection (dg_convect_rhs) on the config-4 velocity mesh: python tools/convect_time.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_04167_b200 as dg
from workloads import config

c4 = config(4)
st = torch.cuda.current_stream()
dev = torch.device("cuda:0")
mv = dg.dg_mesh_create(3, c4.N, c4.L, c4.P, stream=st)
v = [torch.from_numpy(a).to(dev) for a in c4.tg_velocity()]
out = [torch.empty_like(v[0]) for _ in range(3)]
for _ in range(2):
    dg.dg_convect_rhs(mv, v, out)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    dg.dg_convect_rhs(mv, v, out)
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("%s convect ms median %.3f  checksum %.12e" % (os.environ.get("DG_LIBRARY", "default").split("/")[-1],
      statistics.median(ts), sum(float(o.abs().sum()) for o in out)))
