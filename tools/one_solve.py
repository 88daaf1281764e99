"""Two c5 PCG solves (the second one is what a launch list looks at)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2112_04167_b200 as dg  # noqa: E402
from workloads import config  # noqa: E402

c = config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
dev = torch.device("cuda:0")
m = dg.dg_mesh_create(c.dim, c.N[: c.dim], c.L[: c.dim], c.P, stream=torch.cuda.current_stream())
f = torch.from_numpy(c.rhs(0)).to(dev)
nu = c.nu()
nu = None if nu is None else torch.from_numpy(nu).to(dev)
for _ in range(2):
    x = torch.zeros_like(f)
    info = dg.dg_pcg_solve(m, c.lam, nu, c.nu0, f, c.tol, 5000, x)
torch.cuda.synchronize()
print(info.as_dict())
