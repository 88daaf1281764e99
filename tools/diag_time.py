"""Time the Jacobi diagonal (dg_helmholtz_diag) on a BASELINE workload: python tools/diag_time.py [cfg]"""
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
d = torch.empty(dg.dg_mesh_local_ndof(m), dtype=torch.float64, device=dev)
for _ in range(3):
    dg.dg_helmholtz_diag(m, c.lam, nu, c.nu0, d)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    dg.dg_helmholtz_diag(m, c.lam, nu, c.nu0, d)
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("%s diag ms median %.4f  checksum %.15e" % (os.environ.get("DG_LIBRARY", "default"), statistics.median(ts), float(d.abs().sum())))
