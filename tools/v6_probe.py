"""Tiny v6 apply probes (run with a short timeout on the GPU box)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2112_04167_b200 as dg  # noqa: E402

for N, P, varnu in [((4, 4, 2), 3, False), ((4, 4, 2), 3, True), ((4, 4, 4), 5, True), ((8, 8, 6), 5, True)]:
    m = dg.dg_mesh_create(3, N, (1.0, 1.1, 1.2), P, stream=torch.cuda.current_stream())
    om = oracle.Mesh(3, N, (1.0, 1.1, 1.2), P)
    rng = np.random.default_rng(1)
    u = rng.uniform(-1, 1, (om.n_el, om.npe))
    nu = 0.5 + rng.uniform(0, 1, (om.n_el, om.npe)) if varnu else None
    out = torch.empty(u.shape, dtype=torch.float64, device="cuda")
    print("launch", N, P, varnu, flush=True)
    dg.dg_helmholtz_apply(m, 2.0, None if nu is None else torch.from_numpy(nu).cuda(), 0.7,
                          torch.from_numpy(u).cuda(), out)
    torch.cuda.synchronize()
    ref = oracle.sip_apply(om, 2.0, u, nu=nu, nu_const=0.7)
    print("  rel err", np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref), flush=True)
