"""Pins for the oracle's LLF DG convective tendency.

F_c = -div(v v) (term split of §3.2), discretised by DG-SEM "with consistent
integration and local Lax-Friedrichs fluxes for convection".  The
quadrature rule (Gauss, Q = floor(3P/2)+1; reading A13) and the LLF constant (Lambda =
2 max|v.n|; reading A12) are readings the paper does not fix: their parity is "unpinned" by
the paper.  The pins below hold for any consistent, conservative LLF DG scheme with exact
integration of polynomial fluxes:
  * constant v  ->  F_c = 0;
  * conservation: sum_I m_I F_c,I = 0 for every component (test function 1);
  * polynomial v in Q_P on interior elements: M F_c = int -div(v v_c) phi_I exactly
    (reference moments by numpy Gauss quadrature + an independent numpy basis);
  * Taylor-Green closed form: -(v.grad)v -> (-1/2 sin 2x, -1/2 sin 2y) (2-D) at rate ~P.
"""
import math

import numpy as np
import pytest

import oracle

TWO_PI = 2 * math.pi


def coords(m):
    xi, _ = oracle.gll(m.P)
    out = []
    for d in range(m.dim):
        h = m.L[d] / m.N[d]
        c1 = np.arange(m.N[d])[:, None] * h + (xi[None, :] + 1) * h / 2
        shape = [1] * (2 * m.dim)
        shape[m.dim - 1 - d] = m.N[d]
        shape[2 * m.dim - 1 - d] = m.n
        full = np.broadcast_to(c1.reshape(shape), tuple(m.N[: m.dim][::-1]) + (m.n,) * m.dim)
        out.append(np.ascontiguousarray(full).reshape(m.n_el, m.npe))
    return out


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 3), (3, (2, 2, 2), 2), (2, (1, 2), 4)])
def test_constant_velocity_gives_zero(dim, N, P):
    m = oracle.Mesh(dim, N, [TWO_PI] * 3, P)
    v = [np.full(m.ndof, c) for c in (0.7, -1.3, 0.4)[:dim]]
    out = oracle.convect(m, v)
    for o in out:
        assert np.abs(o).max() < 1e-13


@pytest.mark.parametrize("dim,N,P", [(2, (3, 3), 3), (3, (2, 3, 2), 2), (2, (2, 1), 5)])
def test_conservation(dim, N, P):
    m = oracle.Mesh(dim, N, [1.0, 1.7, 0.6], P)
    rng = np.random.default_rng(3)
    v = [rng.uniform(-1, 1, m.ndof) for _ in range(dim)]
    out = oracle.convect(m, v)
    mass = oracle.mass(m)
    for o in out:
        tot = np.sum(mass * o)
        scale = np.sum(mass * np.abs(o))
        assert abs(tot) < 1e-13 * scale


def lagrange_np(nodes, j):
    """Independent Lagrange basis polynomial (numpy Polynomial from roots)."""
    others = np.delete(nodes, j)
    p = np.polynomial.Polynomial.fromroots(others)
    return p / p(nodes[j])


@pytest.mark.parametrize("P", [2, 3])
def test_polynomial_exactness_3d(P):
    """Interior element, v in Q_P globally continuous: LLF dissipation vanishes ([v] = 0) and
    Gauss Q = floor(3P/2)+1 integrates (v v) . grad phi exactly, so M F_c = int -div(v v_c) phi_I."""
    N = 3
    L = [1.0, 1.2, 0.9]
    m = oracle.Mesh(3, (N, N, N), L, P)
    X = coords(m)
    rng = np.random.default_rng(21)
    Pol = np.polynomial.Polynomial
    # separable polynomial components, degree P per direction
    comps = []
    for c in range(3):
        comps.append([Pol(rng.uniform(-1, 1, P + 1)) for _ in range(3)])
    cen = [l / 2 for l in L]

    def val(c, x, y, z):
        a = comps[c]
        return a[0](x - cen[0]) * a[1](y - cen[1]) * a[2](z - cen[2])

    v = [val(c, X[0], X[1], X[2]) for c in range(3)]
    e = 1 + N * (1 + N * 1)  # the interior element (1,1,1)
    out = oracle.convect(m, v, elems=[e])
    mass = oracle.mass(m)[e]
    xi, _ = oracle.gll(P)
    basis = [lagrange_np(xi, j) for j in range(P + 1)]
    # exact moments with a high-order numpy Gauss rule on element (1,1,1)
    zg, wg = np.polynomial.legendre.leggauss(3 * P + 4)
    h = [L[d] / N for d in range(3)]
    xs = [h[d] * 1 + (zg + 1) * h[d] / 2 for d in range(3)]
    Xg, Yg, Zg = np.meshgrid(xs[0], xs[1], xs[2], indexing="ij")
    Wg = np.einsum("i,j,k->ijk", wg, wg, wg) * np.prod(h) / 8

    def dval(c, d, x, y, z):
        a = comps[c]
        fs = [a[0], a[1], a[2]]
        fs = [fs[k].deriv() if k == d else fs[k] for k in range(3)]
        return fs[0](x - cen[0]) * fs[1](y - cen[1]) * fs[2](z - cen[2])

    V = [val(c, Xg, Yg, Zg) for c in range(3)]
    for c in range(3):
        g = np.zeros_like(Xg)
        for d in range(3):  # -d_d(v_d v_c)
            g -= dval(d, d, Xg, Yg, Zg) * V[c] + V[d] * dval(c, d, Xg, Yg, Zg)
        ref = np.zeros(m.npe)
        for k in range(P + 1):
            for j in range(P + 1):
                for i in range(P + 1):
                    phi = (basis[i](zg)[:, None, None] * basis[j](zg)[None, :, None] * basis[k](zg)[None, None, :])
                    ref[i + (P + 1) * (j + (P + 1) * k)] = np.sum(Wg * g * phi)
        got = mass * out[c][0]
        assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max(), c


def test_taylor_green_limit_2d():
    """v = (sin x cos y, -cos x sin y) -> F_c = (-1/2 sin 2x, -1/2 sin 2y); rate ~ P."""
    P = 4
    errs = []
    Ns = (4, 8, 16)
    for N in Ns:
        m = oracle.Mesh(2, (N, N), [TWO_PI] * 3, P)
        X = coords(m)
        v = [np.sin(X[0]) * np.cos(X[1]), -np.cos(X[0]) * np.sin(X[1])]
        out = oracle.convect(m, v)
        ex = [-0.5 * np.sin(2 * X[0]), -0.5 * np.sin(2 * X[1])]
        errs.append(max(math.sqrt(np.mean((out[c] - ex[c]) ** 2)) for c in range(2)))
    eoc = [math.log(errs[i] / errs[i + 1]) / math.log(2) for i in range(len(errs) - 1)]
    assert eoc[-1] > P - 0.3, (errs, eoc)


def test_taylor_green_3d_closed_form():
    """BASELINE configs[3] velocity: F_c -> (-1/2 sin2x cos^2 z, -1/2 sin2y cos^2 z, 0)."""
    P, N = 4, 4
    m = oracle.Mesh(3, (N, N, N), [TWO_PI] * 3, P)
    X = coords(m)
    v = [np.sin(X[0]) * np.cos(X[1]) * np.cos(X[2]), -np.cos(X[0]) * np.sin(X[1]) * np.cos(X[2]),
         np.zeros_like(X[0])]
    elems = [0, 5, 21, 42, 63]
    out = oracle.convect(m, v, elems=elems)
    ex = [-0.5 * np.sin(2 * X[0]) * np.cos(X[2]) ** 2, -0.5 * np.sin(2 * X[1]) * np.cos(X[2]) ** 2,
          np.zeros_like(X[0])]
    for c in range(3):
        assert np.abs(out[c] - ex[c][elems]).max() < 2e-2
