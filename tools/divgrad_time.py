"""Time the DG divergence / gradient pair (dg_divergence, dg_gradient) on the config-4 meshes
(P = 7 velocity, P = 6 pressure): python tools/divgrad_time.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_04167_b200 as dg
from workloads import config

c4 = config(4)
st = torch.cuda.current_stream()
dev = torch.device("cuda:0")
mv = dg.dg_mesh_create(3, c4.N, c4.L, c4.P, stream=st)
mp = dg.dg_mesh_create(3, c4.N, c4.L, c4.P_p, stream=st)
v = [torch.from_numpy(a).to(dev) for a in c4.tg_velocity()]
d = torch.empty(mp.n_el, mp.npe, dtype=torch.float64, device=dev)
gout = [torch.empty_like(v[0]) for _ in range(3)]
res = {}
for name, fn in (("div", lambda: dg.dg_divergence(mv, mp, v, d)), ("grad", lambda: dg.dg_gradient(mp, mv, d, gout))):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[name] = statistics.median(ts)
    # algorithmic bytes: three velocity components and one pressure field
    byt = 8 * (3 * mv.ndof + mp.ndof)
    print("%s %.1f us  %.0f GB/s  checksum %.12e" % (name, res[name] * 1e3, byt / (res[name] * 1e-3) / 1e9,
          float(d.abs().sum()) if name == "div" else sum(float(g.abs().sum()) for g in gout)))
