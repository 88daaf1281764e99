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


def _poly_exactness_err(P, Q=None):
    """max_c |M F_c - int -div(v v_c) phi_I| / max |ref| on the interior element of a 3^3 mesh
    for a globally continuous v in Q_P (oracle with Q Gauss points per direction)."""
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
    out = oracle.convect(m, v, elems=[e], Q=Q)
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
    worst = 0.0
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
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    return worst


@pytest.mark.parametrize("P", [2, 3])
def test_polynomial_exactness_3d(P):
    """Interior element, v in Q_P globally continuous: LLF dissipation vanishes ([v] = 0) and
    Gauss Q = floor(3P/2)+1 integrates (v v) . grad phi exactly, so M F_c = int -div(v v_c) phi_I."""
    assert _poly_exactness_err(P) < 1e-12


@pytest.mark.parametrize("P", [2, 3, 4])
def test_gauss_count_is_the_smallest_exact_rule(P):
    """Reading A13 pinned as 'consistent integration' = the smallest exact Gauss rule: the
    integrands (v v_c) d_e phi (degree 3P-1 along e, 3P across) and (v.n) v_c phi on faces
    (degree 3P) need 2Q - 1 >= 3P.  The oracle's default Q = floor(3P/2)+1 is exact, one
    point more changes nothing beyond rounding, one point fewer is not exact."""
    Q = (3 * P) // 2 + 1
    assert 2 * Q - 1 >= 3 * P > 2 * (Q - 1) - 1
    assert _poly_exactness_err(P) < 1e-12
    assert _poly_exactness_err(P, Q=Q) < 1e-12
    assert _poly_exactness_err(P, Q=Q + 1) < 1e-12
    assert _poly_exactness_err(P, Q=Q - 1) > 1e-8


@pytest.mark.parametrize("P,seed", [(2, 1), (3, 2), (4, 3)])
def test_llf_flux_constant_states(P, seed):
    """Reading A12 pinned on a two-element mesh (N = (2,1,1)) with constant, different states
    v^0, v^1: every face integrand is then constant, so the node at the middle of element 0's
    +x face gives the numerical flux exactly, h_c = f_c(v^0) - F_c,I w_P h/2 (the volume term
    integrates to f(v^0) times the face moment of phi_I and the face term subtracts h times the
    same moment).  Compared with the local Lax-Friedrichs flux of f(v) = (v.n) v written from
    its definition: 1/2 (f^- + f^+) + 1/2 Lambda (v^- - v^+), Lambda = the larger spectral
    radius of the flux Jacobian J = (v.n) I + v n^T on the two sides (numpy.linalg.eigvals)."""
    rng = np.random.default_rng(seed)
    L = [1.3, 0.8, 1.1]
    m = oracle.Mesh(3, (2, 1, 1), L, P)
    v0, v1 = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
    v0[0], v1[0] = 0.35, -0.9   # |v.n| differs on the two sides (tests the max)
    v = [np.concatenate([np.full(m.npe, v0[c]), np.full(m.npe, v1[c])]) for c in range(3)]
    out = oracle.convect(m, v)
    n_ = np.array([1.0, 0.0, 0.0])

    def f(w):
        return np.dot(w, n_) * w

    def rho(w):
        J = np.dot(w, n_) * np.eye(3) + np.outer(w, n_)
        return np.abs(np.linalg.eigvals(J)).max()

    lam = max(rho(v0), rho(v1))
    h_ref = 0.5 * (f(v0) + f(v1)) + 0.5 * lam * (v0 - v1)     # face +x of element 0: '-' = v0
    h_ref_w = 0.5 * (f(v1) + f(v0)) + 0.5 * lam * (v1 - v0)   # face -x of element 0: '-' = v1
    _, w = oracle.gll(P)
    hx = L[0] / 2
    mid = P // 2
    I_p = P + (P + 1) * (mid + (P + 1) * mid)   # node (P, mid, mid) of element 0
    I_m = 0 + (P + 1) * (mid + (P + 1) * mid)   # node (0, mid, mid)
    for c in range(3):
        h_got = f(v0)[c] - out[c][0, I_p] * w[P] * hx / 2
        assert abs(h_got - h_ref[c]) < 1e-13 * (1 + abs(h_ref[c])), (c, h_got, h_ref[c])
        # -x face of element 0 (outward normal -x): M F = (h(v1, v0) - f(v0)) * moment
        h_got_w = f(v0)[c] + out[c][0, I_m] * w[0] * hx / 2
        assert abs(h_got_w - h_ref_w[c]) < 1e-13 * (1 + abs(h_ref_w[c])), (c, h_got_w, h_ref_w[c])
    # a dissipation constant without the factor 2 (max |v.n|) would miss by
    # 1/2 max|v.n| |v0 - v1| -- far outside the tolerance above
    assert 0.5 * max(abs(v0[0]), abs(v1[0])) * np.abs(v0 - v1).max() > 1e-3


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
