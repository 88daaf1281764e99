"""Iteration counts of the two-level Schwarz PCG with delta-node overlapping element boxes
(design study for the Poisson preconditioner; CPU, oracle operator).

Box of element K: in every direction the node indices -delta .. n-1+delta (negative ones in
the left neighbour, >= n in the right one), a tensor-product set of (n + 2 delta)^3 nodes.
A_box = the rows / columns of those nodes of the assembled SIP matrix (oracle operator on unit
vectors); identical for every element on the uniform periodic mesh with N_d >= 3.
"""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402


def box_index(mesh, delta):
    """[n_el, (n+2 delta)^dim] global node index of every box node."""
    dim, n, N = mesh.dim, mesh.n, mesh.N
    m = n + 2 * delta
    a = np.arange(-delta, n + delta)
    eoff = np.where(a < 0, -1, np.where(a >= n, 1, 0))
    loc = a - eoff * n
    out = np.zeros((mesh.n_el, m ** dim), dtype=np.int64)
    for e in range(mesh.n_el):
        ec = oracle._elem_coords(mesh, e)
        if dim == 3:
            K, J, I = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
            ex = (ec[0] + eoff[I]) % N[0]
            ey = (ec[1] + eoff[J]) % N[1]
            ez = (ec[2] + eoff[K]) % N[2]
            el = ex + N[0] * (ey + N[1] * ez)
            node = loc[I] + n * (loc[J] + n * loc[K])
        else:
            J, I = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
            ex = (ec[0] + eoff[I]) % N[0]
            ey = (ec[1] + eoff[J]) % N[1]
            el = ex + N[0] * ey
            node = loc[I] + n * loc[J]
        out[e] = (el * mesh.npe + node).reshape(-1)
    return out


def box_matrix(mesh, lam, idx):
    nb = idx.shape[0]
    B = np.zeros((nb, nb))
    for j in range(nb):
        u = np.zeros(mesh.ndof)
        u[idx[j]] = 1.0
        B[:, j] = oracle.sip_apply(mesh, lam, u).reshape(-1)[idx]
    return B


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--N", type=int, default=8)
    ap.add_argument("--P", type=int, default=6)
    ap.add_argument("--deltas", default="0,1,2")
    ap.add_argument("--tol", type=float, default=1e-10)
    a = ap.parse_args()
    dim = a.dim
    mesh = oracle.Mesh(dim, (a.N,) * dim, (2 * np.pi,) * dim, a.P)
    rng = np.random.default_rng(1)
    f = rng.uniform(-1, 1, (mesh.n_el, mesh.npe))
    t0 = time.time()
    Ac, Pm = oracle.q1_coarse_operator(mesh, 0.0)
    Acp = np.linalg.pinv(Ac, rcond=1e-13)
    print("coarse %.1fs" % (time.time() - t0), flush=True)
    u0, itj = oracle.pcg_precond(mesh, 0.0, f, lambda r: r / np.maximum(oracle.sip_diag(mesh, 0.0).reshape(-1), 1e-300),
                                 tol=a.tol)
    print("jacobi its", itj, flush=True)
    for delta in [int(x) for x in a.deltas.split(",")]:
        idx = box_index(mesh, delta)
        t0 = time.time()
        Binv = np.linalg.inv(box_matrix(mesh, 0.0, idx[0]))
        for coarse in (True,):
            def B(r):
                r = np.asarray(r).reshape(-1)
                y = r[idx] @ Binv.T                      # every box, same matrix
                z = np.zeros(mesh.ndof)
                np.add.at(z, idx.reshape(-1), y.reshape(-1))
                if coarse:
                    z += Pm @ (Acp @ (Pm.T @ r))
                return z
            u, it = oracle.pcg_precond(mesh, 0.0, f, B, tol=a.tol)
            print("delta %d coarse %s: %d its (%.1fs), |u - u_jac| %.2e" %
                  (delta, coarse, it, time.time() - t0, np.abs(u - u0).max()), flush=True)


if __name__ == "__main__":
    main()
