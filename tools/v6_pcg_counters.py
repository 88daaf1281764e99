"""Per-role cycle counters of the fused PCG apply (MODE 1) on c5 (DG_V5_DEBUG build, DG_APPLY_IMPL
selects the kernel)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import config  # noqa: E402

lib = ctypes.CDLL(dg.library_path())
buf = (ctypes.c_ulonglong * 16)()
c = config(5)
m = dg.dg_mesh_create(3, c.N, c.L, c.P, stream=torch.cuda.current_stream())
f = torch.from_numpy(c.rhs(0)).cuda()
nu = torch.from_numpy(c.nu()).cuda()
x = torch.zeros_like(f)
dg.dg_pcg_solve(m, c.lam, nu, c.nu0, f, 1e-10, 100, x)
lib.dg_debug_counters(buf, 1)
x.zero_()
info = dg.dg_pcg_solve(m, c.lam, nu, c.nu0, f, 1e-10, 100, x)
lib.dg_debug_counters(buf, 1)
v = list(buf)
nb = max(v[5], 1)
print("iters", info.iters, "bricks", nb)
names = ["cons_wait_full", "cons_brick_compute", "prod_wait_empty", "prod_traces", "prod_tma_issue", "-",
         "cons_x_pass", "cons_y_pass", "cons_z_pass", "prod_x", "prod_y"]
for i, nm in enumerate(names):
    if nm != "-":
        print("%-20s %10.0f cycles/brick" % (nm, v[i] / nb))
