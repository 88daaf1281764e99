"""A/B timing of the c5 apply for alternative builds: DG_LIBRARY=<so> python tools/ab_apply.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_04167_b200 as dg
from workloads import config

c = config(int(os.environ.get("AB_CFG", "5")))
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
m = dg.dg_mesh_create(c.dim, c.N[: c.dim], c.L[: c.dim], c.P, stream=st)
u = torch.from_numpy(c.apply_input()).to(dev)
nu = c.nu()
nu = None if nu is None else torch.from_numpy(nu).to(dev)
out = torch.empty_like(u)
for _ in range(5):
    dg.dg_helmholtz_apply(m, c.lam, nu, c.nu0, u, out)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    dg.dg_helmholtz_apply(m, c.lam, nu, c.nu0, u, out)
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("%s apply ms median %.4f min %.4f  checksum %.12e" % (os.environ.get("DG_LIBRARY", "default"), statistics.median(ts), min(ts), float(out.double().abs().sum())))
