"""Pins for the NEXT-1 / NEXT-3 oracle pieces against a brute-force dense assembly.

``oracle.dg_divergence_weak``, ``oracle.dg_gradient_weak`` and ``oracle.dg_derivative`` are
element-local tensor contractions; ``oracle.dense_pair`` writes the same operators (PAPER.md
Alg. 3 lines 5-6; pressure degree P-1; readings DESIGN.md §9) as explicit
all-(row, column, quadrature point) sums with the basis evaluated at every point by the product
formula -- no factorisation, no sparsity logic (as ``sip_dense`` for the SIP operator).  A
dropped face term, a wrong sign or side, a transposed operand or a lost neighbour pairing
(N = 1 self-neighbour, N = 2 double adjacency, reading A15) fails one of these.
"""
import numpy as np
import pytest

import oracle
from oracle.dense_pair import deriv_dense, div_dense, grad_dense

CASES = [(2, (2, 2), 3), (2, (2, 2), 4), (2, (3, 2), 2), (2, (1, 2), 3), (3, (2, 2, 2), 2), (3, (2, 2, 2), 3),
         (3, (1, 2, 2), 2)]


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.mark.parametrize("dim,N,P", CASES)
def test_divergence_matches_dense(dim, N, P):
    L = (1.0, 1.3, 0.7)[:dim]
    mv = oracle.Mesh(dim, N, L, P)
    rng = np.random.default_rng(10 + P)
    v = [rng.uniform(-1, 1, (mv.n_el, mv.npe)) for _ in range(dim)]
    D = div_dense(mv)
    ref = D @ np.concatenate([x.reshape(-1) for x in v])
    got = oracle.dg_divergence_weak(mv, v).reshape(-1)
    assert rel(got, ref) < 1e-13


@pytest.mark.parametrize("dim,N,P", CASES)
def test_gradient_matches_dense(dim, N, P):
    L = (1.0, 1.3, 0.7)[:dim]
    mp = oracle.Mesh(dim, N, L, P - 1)
    rng = np.random.default_rng(20 + P)
    psi = rng.uniform(-1, 1, (mp.n_el, mp.npe))
    G = grad_dense(mp)
    ref = (G @ psi.reshape(-1)).reshape(dim, -1)
    got = oracle.dg_gradient_weak(mp, psi)
    for c in range(dim):
        assert rel(got[c], ref[c]) < 1e-13, c


@pytest.mark.parametrize("dim,N,P", CASES)
def test_dense_pair_adjoint(dim, N, P):
    """The two independently assembled dense operators satisfy G = -D^T (central fluxes,
    exact quadrature), so the oracle's pair is adjoint by construction of both."""
    L = (1.0, 1.3, 0.7)[:dim]
    D = div_dense(oracle.Mesh(dim, N, L, P))
    G = grad_dense(oracle.Mesh(dim, N, L, P - 1))
    assert np.abs(G + D.T).max() < 1e-13 * np.abs(D).max()


@pytest.mark.parametrize("dim,N,P", CASES)
def test_derivative_matches_dense(dim, N, P):
    L = (1.0, 1.3, 0.7)[:dim]
    m = oracle.Mesh(dim, N, L, P)
    rng = np.random.default_rng(30 + P)
    u = rng.uniform(-1, 1, (m.n_el, m.npe))
    Ds = deriv_dense(m)
    got = oracle.dg_derivative(m, u)
    for c in range(dim):
        assert rel(got[c], Ds[c] @ u.reshape(-1)) < 1e-13, c


@pytest.mark.parametrize("dim,N,P", [(2, (2, 2), 3), (3, (2, 2, 2), 2)])
def test_dense_derivative_skew_and_exact(dim, N, P):
    """M D_c is skew (central fluxes) and D_c reproduces derivatives of continuous periodic
    trigonometric fields spectrally -- properties of the definition, checked on the dense form."""
    L = (2 * np.pi,) * dim
    m = oracle.Mesh(dim, N, L, P)
    mi = oracle.mass(m).reshape(-1)
    for Dc in deriv_dense(m):
        MD = mi[:, None] * Dc
        assert np.abs(MD + MD.T).max() < 1e-13 * np.abs(MD).max()
        assert np.abs(Dc @ np.ones(m.ndof)).max() < 1e-12
