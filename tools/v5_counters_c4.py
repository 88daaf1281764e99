"""DG_V5_DEBUG build: per-role cycle shares of the v5 apply on the config-4 pressure mesh (32^3,
P = 6, constant nu) and velocity mesh (P = 7)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import config  # noqa: E402

lib = ctypes.CDLL(dg.library_path())
buf = (ctypes.c_ulonglong * 16)()
c = config(4)
names = ["cons_wait_full", "cons_brick_compute", "prod_wait_empty", "prod_traces", "prod_tma_issue", "-",
         "cons_x_pass", "cons_y_pass", "cons_z_pass", "prod_x", "prod_y"]
for P in (6, 7):
    m = dg.dg_mesh_create(3, c.N, c.L, P, stream=torch.cuda.current_stream())
    u = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (m.n_el, m.npe))).cuda()
    out = torch.empty_like(u)
    for _ in range(3):
        dg.dg_helmholtz_apply(m, 0.0, None, 1.0, u, out)
    torch.cuda.synchronize()
    lib.dg_debug_counters(buf, 1)
    reps = 10
    for _ in range(reps):
        dg.dg_helmholtz_apply(m, 0.0, None, 1.0, u, out)
    lib.dg_debug_counters(buf, 1)
    v = list(buf)
    nb = max(v[5], 1)
    print("P", P, dg.dg_last_apply_kernel(), "bricks", nb / reps)
    for i, nm in enumerate(names):
        if nm != "-":
            print("  %-20s %10.0f cycles/brick" % (nm, v[i] / nb))
