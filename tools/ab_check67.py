import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle, paper_2112_04167_b200 as dg
for N, P in [((4, 6, 2), 6), ((8, 2, 3), 6), ((4, 4, 3), 6), ((4, 2, 3), 7), ((8, 4, 2), 7)]:
    L = (1.0, 1.7, 0.6)
    m = dg.dg_mesh_create(3, N, L, P, stream=torch.cuda.current_stream()); om = oracle.Mesh(3, N, L, P)
    u = np.random.default_rng(P).uniform(-1, 1, (om.n_el, om.npe))
    for lam in (0.0, 2.3):
        out = torch.empty(u.shape, dtype=torch.float64, device="cuda")
        dg.dg_helmholtz_apply(m, lam, None, 0.37, torch.from_numpy(u).cuda(), out)
        ref = oracle.sip_apply(om, lam, u, nu=None, nu_const=0.37)
        e = np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref)
        print(N, P, lam, "%.2e" % e, dg.dg_last_apply_kernel(), "OK" if e < 1e-12 else "FAIL")
