"""The bench's slab model alone (per-rank c5 work for N = 2, 4, 8 in the 1-rank halo mode)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_04167_b200 as dg
import bench
from workloads import config
c = config(5)
st = torch.cuda.current_stream()
u = torch.from_numpy(c.apply_input()).cuda()
nu = torch.from_numpy(c.nu()).cuda()
r = bench.run_slab_model(dg, torch, st, c, u, nu, 0.512, 24.45 / 18)
print(os.environ.get("DG_LIBRARY", "default").split("/")[-1], {k: (round(v["apply_ms"], 4), round(v["pcg_ms_per_iter"], 4), round(v["apply_eff_model"], 3), round(v["pcg_eff_model"], 3)) for k, v in r.items()})
