"""Two applies of a BASELINE workload (the second is the one ncu measures): used by bench.py
to read the DRAM traffic of the dispatched apply kernel for the current build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import config  # noqa: E402

c = config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
dev = torch.device("cuda:0")
m = dg.dg_mesh_create(c.dim, c.N[: c.dim], c.L[: c.dim], c.P, stream=torch.cuda.current_stream())
u = torch.from_numpy(c.apply_input()).to(dev)
nu = c.nu()
nu = None if nu is None else torch.from_numpy(nu).to(dev)
out = torch.empty_like(u)
for _ in range(2):
    dg.dg_helmholtz_apply(m, c.lam, nu, c.nu0, u, out)
torch.cuda.synchronize()
print(dg.dg_last_apply_kernel())
