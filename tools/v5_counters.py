"""Run the c5 apply a few times with the DG_V5_DEBUG build and print per-role cycle shares."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import config  # noqa: E402

lib = ctypes.CDLL(dg.library_path())
buf = (ctypes.c_ulonglong * 16)()
c = config(5)
m = dg.dg_mesh_create(3, c.N, c.L, c.P, stream=torch.cuda.current_stream())
u = torch.from_numpy(c.apply_input()).cuda()
nu = torch.from_numpy(c.nu()).cuda()
out = torch.empty_like(u)
for _ in range(3):
    dg.dg_helmholtz_apply(m, c.lam, nu, c.nu0, u, out)
lib.dg_debug_counters(buf, 1)
reps = 10
for _ in range(reps):
    dg.dg_helmholtz_apply(m, c.lam, nu, c.nu0, u, out)
lib.dg_debug_counters(buf, 1)
v = list(buf)
nb = max(v[5], 1)
print("bricks", nb / reps)
names = ["cons_wait_full", "cons_brick_compute", "prod_wait_empty", "prod_traces", "prod_tma_issue", "-",
         "cons_x_pass", "cons_y_pass", "cons_z_pass", "prod_x", "prod_y"]
for i, nm in enumerate(names):
    if nm == "-":
        continue
    print("%-20s %10.0f cycles/brick" % (nm, v[i] / nb))
