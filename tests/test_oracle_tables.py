"""Pins for the oracle's 1-D tables.

GLL points are named by PAPER.md:1035 ("tensor-product Lagrange polynomials based on GLL
points"); collocation differentiation on them by PAPER.md:1082-1084.  Values are pinned
to the worked example in tests/golden/ (SPEC.md:111,121), to closed forms, and to
library routines (numpy Legendre roots, numpy leggauss) -- never to the oracle itself.
"""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "gll_p3_unit_interval.txt")


def test_gll_p3_worked_example():
    ref = np.loadtxt(GOLD)
    xi, w = oracle.gll(3)
    np.testing.assert_allclose((xi + 1) / 2, ref[:, 0], rtol=0, atol=1e-15)
    np.testing.assert_allclose(w / 2, ref[:, 1], rtol=0, atol=1e-15)


@pytest.mark.parametrize("P", range(1, 17))
def test_gll_closed_forms(P):
    xi, w = oracle.gll(P)
    assert xi[0] == -1.0 and xi[-1] == 1.0
    assert np.all(np.diff(xi) > 0)
    # interior nodes = roots of P_P' (library: numpy Legendre class)
    if P > 1:
        r = np.sort(np.real(np.polynomial.legendre.Legendre.basis(P).deriv().roots()))
        np.testing.assert_allclose(xi[1:-1], r, atol=5e-14)
    # sum w = 2, w_0 = 2/(P(P+1)), symmetry
    assert abs(w.sum() - 2.0) < 1e-14
    assert abs(w[0] - 2.0 / (P * (P + 1))) < 1e-15
    np.testing.assert_allclose(w, w[::-1], atol=1e-15)
    np.testing.assert_allclose(xi, -xi[::-1], atol=1e-15)
    # exact for polynomials of degree <= 2P-1
    for k in range(0, 2 * P):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, xi ** k) - exact) < 2e-14, (P, k)
    # and NOT exact at degree 2P (GLL with P+1 points); x^{2P} even
    assert abs(np.dot(w, xi ** (2 * P)) - 2.0 / (2 * P + 1)) > 1e-13


@pytest.mark.parametrize("Q", range(1, 19))
def test_gauss_vs_numpy_leggauss(Q):
    z, w = oracle.gauss(Q)
    zr, wr = np.polynomial.legendre.leggauss(Q)
    np.testing.assert_allclose(z, zr, atol=2e-15)
    np.testing.assert_allclose(w, wr, atol=2e-15)


@pytest.mark.parametrize("P", [1, 2, 3, 5, 7, 8, 10])
def test_lagrange_product_formula(P):
    xi, _ = oracle.gll(P)
    # cardinality l_j(xi_i) = delta_ij, exactly (a zero factor / an all-ones product)
    D = np.zeros((P + 1, P + 1))
    for i, x in enumerate(xi):
        l, dl = oracle.lagrange(P, xi, x)
        assert np.array_equal(l, np.eye(P + 1)[i])
        D[i] = dl
    # D 1 = 0 ; D xi^k = k xi^(k-1) for k <= P ; D_00 = -P(P+1)/4 = -D_PP
    assert np.abs(D.sum(axis=1)).max() < 1e-12 * max(1.0, np.abs(D).max())
    for k in range(1, P + 1):
        np.testing.assert_allclose(D @ xi ** k, k * xi ** (k - 1), atol=1e-11 * P * P)
    assert abs(D[0, 0] + P * (P + 1) / 4.0) < 1e-12 * P * P
    assert abs(D[P, P] - P * (P + 1) / 4.0) < 1e-12 * P * P
    # partition of unity / derivative sum at an off-node point
    l, dl = oracle.lagrange(P, xi, 0.123456)
    assert abs(l.sum() - 1.0) < 1e-13 and abs(dl.sum()) < 1e-11
    # closed-form off-diagonal entries D_ij = P_P(xi_i)/(P_P(xi_j)(xi_i-xi_j)) (textbook, Canuto)
    LP = np.polynomial.legendre.Legendre.basis(P)(xi)
    for i in range(P + 1):
        for j in range(P + 1):
            if i != j:
                assert abs(D[i, j] - LP[i] / (LP[j] * (xi[i] - xi[j]))) < 1e-11 * P * P
