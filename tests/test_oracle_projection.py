"""Pins of the projection step (Alg. 3 lines 5-6; SIP pressure Poisson on the
degree P-1 mesh) as the oracle composes it in oracle.imex_stage:

    psi = K^+ (-D v),   v'' = v - M^-1 G psi

with D = dg_divergence_weak, G = dg_gradient_weak, K = the SIP Laplacian of the pressure mesh
(sip_dense, lam = 0) and M the lumped velocity mass.  Facts the mathematics fixes:

* G = -D^T (the central-flux pair is adjoint; pinned elsewhere on dense assemblies, restated
  here only as the premise of the next two);
* the compatible Laplacian C = -D M^-1 G = D M^-1 D^T is symmetric positive semi-definite;
* the SIP operator dominates it on the range of D: the largest eigenvalue of K^+ C is exactly 1
  (attained by the smooth modes, where both are the same discrete Laplacian), so the
  projection is non-expansive in the M-norm -- it cannot amplify the velocity (DESIGN.md §9:
  the TGP instability of RK-CB2 / RK-CB3e is therefore not the projection's);
* a discretely solenoidal field (D v = 0) is left unchanged, and the projected field of any v has
  zero mean pressure-space divergence residual K psi + D v = 0 up to the constant mode.
"""
import numpy as np
import pytest

import oracle


def _assemble(dim, N, P):
    mv, mp = oracle.Mesh(dim, N, (1.0, 1.3, 0.8)[:dim], P), oracle.Mesh(dim, N, (1.0, 1.3, 0.8)[:dim], P - 1)
    nv, npp = mv.ndof, mp.ndof
    shp = (mv.n_el, mv.npe)
    D = np.zeros((npp, dim * nv))
    for c in range(dim):
        for j in range(nv):
            v = [np.zeros(shp) for _ in range(dim)]
            v[c].reshape(-1)[j] = 1.0
            D[:, c * nv + j] = oracle.dg_divergence_weak(mv, v).reshape(-1)
    G = np.zeros((dim * nv, npp))
    for j in range(npp):
        psi = np.zeros((mp.n_el, mp.npe))
        psi.reshape(-1)[j] = 1.0
        g = oracle.dg_gradient_weak(mp, psi)
        for c in range(dim):
            G[c * nv:(c + 1) * nv, j] = np.asarray(g[c]).reshape(-1)
    K = oracle.sip_dense(mp, 0.0)
    m = np.concatenate([oracle.mass(mv).reshape(-1)] * dim)
    return D, G, K, m


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 3), (2, (2, 3), 4), (3, (2, 2, 1), 2)])
def test_projection_is_non_expansive(dim, N, P):
    D, G, K, m = _assemble(dim, N, P)
    assert np.abs(G + D.T).max() <= 1e-12 * max(1.0, np.abs(D).max())
    C = D @ (D.T / m[:, None])                       # D M^-1 D^T
    assert np.abs(C - C.T).max() <= 1e-12 * np.abs(C).max()
    assert np.linalg.eigvalsh(0.5 * (C + C.T)).min() >= -1e-10 * np.abs(C).max()
    Kp = np.linalg.pinv(K, rcond=1e-12)
    lam = np.abs(np.linalg.eigvals(Kp @ C)).max()
    assert abs(lam - 1.0) <= 1e-8, lam
    # the projection matrix of oracle.imex_stage and its M-norm
    Pm = np.eye(D.shape[1]) - (G @ (Kp @ (-D))) / m[:, None]
    s = np.sqrt(m)
    assert np.linalg.norm(s[:, None] * Pm / s[None, :], 2) <= 1.0 + 1e-8


def test_projection_keeps_solenoidal_fields_and_solves_the_poisson_problem():
    dim, N, P = 2, (3, 2), 3
    D, G, K, m = _assemble(dim, N, P)
    Kp = np.linalg.pinv(K, rcond=1e-12)
    # a discretely solenoidal field: project a random field onto null(D)
    rng = np.random.default_rng(7)
    Z = np.linalg.svd(D)[2][np.linalg.matrix_rank(D):].T
    v0 = Z @ rng.standard_normal(Z.shape[1])
    assert np.abs(D @ v0).max() <= 1e-11 * np.abs(v0).max()
    v1 = v0 - (G @ (Kp @ (-D @ v0))) / m
    assert np.abs(v1 - v0).max() <= 1e-11 * np.abs(v0).max()
    # any field: psi solves K psi = -D v up to the constant pressure mode
    v = rng.standard_normal(D.shape[1])
    psi = Kp @ (-D @ v)
    res = K @ psi + D @ v
    ones = np.ones(K.shape[0]) / np.sqrt(K.shape[0])
    res -= ones * (ones @ res)
    assert np.abs(res).max() <= 1e-10 * np.abs(D @ v).max()
