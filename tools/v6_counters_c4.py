"""Per-role cycle counters of the v6 apply on the config-4 pressure mesh (P = 6, constant nu),
DG_V5_DEBUG build: DG_LIBRARY=<so> python tools/v6_counters_c4.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_04167_b200 as dg
from workloads import config

lib = ctypes.CDLL(dg.library_path())
buf = (ctypes.c_ulonglong * 16)()
c = config(4)
m = dg.dg_mesh_create(3, c.N, c.L, 6, stream=torch.cuda.current_stream())
u = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (m.n_el, m.npe))).cuda()
out = torch.empty_like(u)
for _ in range(3):
    dg.dg_helmholtz_apply(m, 0.0, None, 1.0, u, out)
lib.dg_debug_counters(buf, 1)
reps = 10
for _ in range(reps):
    dg.dg_helmholtz_apply(m, 0.0, None, 1.0, u, out)
lib.dg_debug_counters(buf, 1)
v = list(buf)
nb = max(v[5], 1)
print("bricks", nb / reps, dg.dg_last_apply_kernel())
names = ["cons_wait_full", "cons_brick_compute", "trace_wait_empty", "traces", "tma_wait_empty", "-",
         "cons_x_pass", "cons_y_pass", "cons_z_pass"]
for i, nm in enumerate(names):
    if nm != "-":
        print("%-20s %10.0f cycles/brick" % (nm, v[i] / nb))
