"""Pins of the oracle's IMEX-RK stage pieces (Alg. 3 lines 4-9,
P:818-861): the DG divergence / gradient pair of the projection step and the stage."""
import numpy as np
import pytest

import oracle
from workloads import node_coords


def _poly(dim, X):
    """Polynomial velocity of degree <= 2 per direction and its exact divergence."""
    x, y = X[0], X[1]
    z = X[2] if dim == 3 else 0.0 * x
    v = [x ** 2 * y + 0.3 * z, x * y ** 2 - z ** 2 * x, x * y * z + z ** 2][:dim]
    div = 4.0 * x * y + ((x * y + 2.0 * z) if dim == 3 else 0.0)
    return v, div


def _interior(mesh):
    """Elements whose closure avoids the periodic seam (global polynomials are continuous there)."""
    out = []
    for e in range(mesh.n_el):
        ec = oracle._elem_coords(mesh, e)
        if all(0 < c < mesh.N[k] - 1 for k, c in enumerate(ec)):
            out.append(e)
    return out


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 3), (3, (2, 2, 3), 3), (2, (2, 3), 5), (3, (1, 2, 2), 2)])
def test_dg_divergence_gradient_adjoint(dim, N, P):
    """q . D v = -v . G q for all v, q (central fluxes, exact GLL_P quadrature): -G = D^T."""
    L = (1.0, 1.3, 0.8)[:dim]
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    rng = np.random.default_rng(P)
    v = [rng.uniform(-1, 1, (mv.n_el, mv.npe)) for _ in range(dim)]
    q = rng.uniform(-1, 1, (mp.n_el, mp.npe))
    d = oracle.dg_divergence_weak(mv, v)
    g = oracle.dg_gradient_weak(mp, q)
    lhs = float(np.sum(q * d))
    rhs = -sum(float(np.sum(v[c] * g[c])) for c in range(dim))
    assert abs(lhs - rhs) <= 1e-13 * (np.abs(q * d).sum() + 1.0)


@pytest.mark.parametrize("dim,N,P", [(2, (4, 3), 3), (3, (3, 3, 4), 3), (2, (3, 4), 5), (3, (3, 3, 3), 2)])
def test_dg_divergence_gradient_polynomial_exactness(dim, N, P):
    """For continuous polynomial fields of degree <= P-1 the pair is exact on interior elements:
    D v = (phi^p, div v) evaluated with GLL_P quadrature, M^-1 G psi = grad psi at the nodes."""
    L = (1.0, 1.3, 0.8)[:dim]
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    X = node_coords(dim, N, L, P)
    x, y = X[0], X[1]
    z = X[2] if dim == 3 else 0.0 * x
    if P >= 3:
        v = [x ** 2 * y + 0.3 * z, x * y ** 2 - z ** 2 * x, x * y * z + z ** 2][:dim]
        divv = 4.0 * x * y + ((x * y + 2.0 * z) if dim == 3 else 0.0)
    else:
        v = [x * y + z, y * z + x, x * z + y][:dim]
        divv = y + z + (x if dim == 3 else 0.0)
    d = oracle.dg_divergence_weak(mv, v)
    _, wv, E, _, _ = oracle._pv_tables(P)
    n = P + 1
    h = [L[k] / N[k] for k in range(dim)]
    W = np.ones((n,) * dim)
    for k in range(dim):
        shp = [1] * dim
        shp[dim - 1 - k] = n
        W = W * (wv * 0.5 * h[k]).reshape(shp)
    Xp = node_coords(dim, N, L, P - 1)
    xp, yp = Xp[0], Xp[1]
    zp = Xp[2] if dim == 3 else 0.0 * xp
    psi = (xp ** 2 * yp + (zp * xp if dim == 3 else 0.0)) if P >= 3 else xp * yp + (zp if dim == 3 else 0.0)
    gexact = ([2 * x * y + (z if dim == 3 else 0.0), x ** 2, x][:dim] if P >= 3 else [y, x + 0.0 * x, 1.0 + 0.0 * x][:dim])
    g = oracle.dg_gradient_weak(mp, psi)
    m = oracle.mass(mv)
    inner = _interior(mv)
    assert inner
    for e in inner:
        t = W * divv[e].reshape((n,) * dim)
        for k in range(dim):
            t = oracle._apply_1d(E.T, t, dim - 1 - k)
        assert np.abs(d[e] - t.reshape(-1)).max() <= 1e-12 * max(np.abs(t).max(), 1e-300)
        for c in range(dim):
            assert np.abs(g[c][e] / m[e] - gexact[c][e]).max() <= 1e-12 * max(np.abs(gexact[c]).max(), 1.0)


def test_dg_divergence_gradient_constants():
    """Constant fields on a periodic mesh: D v = 0 and G psi = 0."""
    dim, N, L, P = 3, (2, 3, 2), (1.0, 1.3, 0.8), 3
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    v = [np.full((mv.n_el, mv.npe), c) for c in (0.7, -0.2, 0.4)]
    assert np.abs(oracle.dg_divergence_weak(mv, v)).max() < 1e-14
    g = oracle.dg_gradient_weak(mp, np.full((mp.n_el, mp.npe), 2.5))
    assert max(np.abs(x).max() for x in g) < 1e-13


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 3), (3, (2, 2, 2), 3)])
def test_stage_keeps_a_uniform_flow(dim, N, P):
    """v = const: F_c = 0 (Q15), F_d1 = 0 (A 1 = 0 at lam = 0, Q4), div v' = 0 so psi = 0, and
    (lam M + A_0) u = lam M v has the unique solution u = v: the stage returns v."""
    L = (1.0, 1.3, 0.8)[:dim]
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    v = [np.full((mv.n_el, mv.npe), c) for c in (0.7, -0.2, 0.4)[:dim]]
    out, psi, vp = oracle.imex_stage(mv, mp, 1e-2, 0.4358665, 0.0, 0.4358665, 1e-2, v)
    for c in range(dim):
        assert np.abs(vp[c] - v[c]).max() < 1e-13
        assert np.abs(out[c] - v[c]).max() < 1e-12
    assert np.abs(psi).max() < 1e-12


def test_stage_viscous_decay_of_a_shear_mode():
    """v = (sin y, 0): F_c = 0 (v.grad v = 0 and the LLF flux of a y-dependent x-velocity
    across x-faces is continuous), div v = 0.  Line 4 gives v' = (1 - dt a nu) sin y, line 8
    (a_im21 = 0) adds the explicit diffusion back, g = sin y, and line 9 is the implicit
    diffusion step: the result approaches sin(y) / (1 + dt a nu) as h -> 0."""
    dim, P = 2, 6
    N, L = (2, 8), (2 * np.pi, 2 * np.pi)
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    X = node_coords(dim, N, L, P)
    v = [np.sin(X[1]), 0.0 * X[0]]
    dt, a, nu = 0.1, 0.5, 0.3
    out, psi, _ = oracle.imex_stage(mv, mp, dt, a, 0.0, a, nu, v)
    expect = np.sin(X[1]) / (1.0 + dt * a * nu)
    assert np.abs(out[0] - expect).max() < 1e-5
    assert np.abs(out[1]).max() < 1e-9
    assert np.abs(psi).max() < 1e-6


@pytest.mark.parametrize("name", ["RK-CB3e", "RK-ARS3"])
def test_oracle_tableaux_consistency(name):
    """Row sums of both tableaux give the same nodes c (CK structure); b sums to 1;
    the explicit part is strictly lower triangular and a_im[0][0] = 0."""
    t = oracle.ORACLE_TABLEAUX[name]
    A_im, A_ex = np.array(t["a_im"]), np.array(t["a_ex"])
    assert np.allclose(A_im.sum(1), A_ex.sum(1), atol=1e-15)
    assert abs(sum(t["b_im"]) - 1) < 1e-15 and abs(sum(t["b_ex"]) - 1) < 1e-15
    assert np.allclose(np.triu(A_ex), 0) and A_im[0, 0] == 0 and np.allclose(np.triu(A_im, 1), 0)


@pytest.mark.parametrize("name", ["RK-CB3e", "RK-ARS3"])
def test_rk_step_keeps_a_uniform_flow(name):
    """v = const is an exact steady solution: every stage force vanishes, the step returns v."""
    dim, N, L, P = 2, (3, 2), (1.0, 1.3), 3
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    v = [np.full((mv.n_el, mv.npe), c) for c in (0.7, -0.2)]
    out = oracle.imex_rk_step(mv, mp, oracle.ORACLE_TABLEAUX[name], 0.05, 0.02, v)
    for c in range(dim):
        assert np.abs(out[c] - v[c]).max() < 1e-12


@pytest.mark.parametrize("name,z", [("RK-CB3e", -0.3), ("RK-ARS3", -0.7)])
def test_rk_step_shear_mode_is_the_dirk_stability_function(name, z):
    """v = (sin(2 pi y / L_y) mode of the discrete operator, 0): F_c = 0, div v = 0, so one step
    is the implicit (DIRK) tableau applied to u' = mu u on the mode's discrete eigenvalue mu:
    u^{n+1} = R(dt mu) u^n with R(z) = 1 + z b^T (I - z A)^{-1} 1 (Alg. 3 lines 4, 8, 9, 11)."""
    dim, N, L, P = 2, (2, 4), (1.0, 1.0), 5
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    # the discrete y-mode: eigenvector of M^-1 A_0 restricted to fields constant in x
    X = node_coords(dim, N, L, P)
    u0 = np.sin(2 * np.pi * X[1])
    nu = 0.02
    A = oracle.sip_dense(mv, 0.0, nu_const=nu)
    m = oracle.mass(mv).reshape(-1)
    w, V = np.linalg.eigh(A / np.sqrt(np.outer(m, m)))
    # component of u0 along its dominant eigenvector (symmetric scaling M^-1/2 A M^-1/2)
    y = np.sqrt(m) * u0.reshape(-1)
    k = int(np.argmax(np.abs(V.T @ y)))
    sel = np.abs(w - w[k]) <= 1e-9 * w[k]  # the eigenvalue is degenerate (x and y modes, sin and cos)
    ev = V[:, sel] @ (V[:, sel].T @ y) / np.sqrt(m)   # u0's component in the eigenspace of M^-1 A
    mu = -w[k]
    ev = ev.reshape(mv.n_el, mv.npe) / np.abs(ev).max()
    dt = z / mu
    t = oracle.ORACLE_TABLEAUX[name]
    A_im = np.array(t["a_im"])
    s = A_im.shape[0]
    R = 1 + z * np.array(t["b_im"]) @ np.linalg.solve(np.eye(s) - z * A_im, np.ones(s))
    out = oracle.imex_rk_step(mv, mp, t, dt, nu, [ev, np.zeros_like(ev)])
    # 1e-7: the eigen-projected mode carries ~1e-8 x-mode impurities (degenerate eigenspace);
    # a wrong tableau entry or sign moves the result by O(|z| 1e-1)
    assert np.abs(out[0] - R * ev).max() <= 1e-7
    assert np.abs(out[1]).max() <= 1e-7


ORDER = {"RK-TR": 2, "RK-CB2": 2, "RK-CB3e": 3, "RK-ARS3": 3}


def imex_order_defects(t, order):
    """Defects of the IMEX Runge-Kutta order conditions up to `order` (coupled conditions of
    the additive/partitioned RK theory): sum b = 1; b.c = 1/2; b.c^2 = 1/3 and b.A.c = 1/6 for
    every pairing of b in {b_im, b_ex} with A in {A_im, A_ex}; and the shared abscissae
    A_im 1 = A_ex 1 = c."""
    Ai, Ae = np.asarray(t["a_im"], float), np.asarray(t["a_ex"], float)
    bi, be = np.asarray(t["b_im"], float), np.asarray(t["b_ex"], float)
    c = Ae.sum(1)
    d = [np.abs(Ai.sum(1) - c).max()]
    for b in (bi, be):
        d += [b.sum() - 1.0, b @ c - 0.5]
        if order >= 3:
            d += [b @ c ** 2 - 1.0 / 3.0] + [b @ A @ c - 1.0 / 6.0 for A in (Ai, Ae)]
    return np.abs(np.array(d))


@pytest.mark.parametrize("name", sorted(ORDER))
def test_oracle_tableaux_order_conditions(name):
    """Every tableau typed from the paper's appendix satisfies the IMEX order
    conditions of its stated order, and every single non-zero explicit or implicit entry is
    pinned: perturbing it by 1e-3 violates at least one condition."""
    t = oracle.ORACLE_TABLEAUX[name]
    k = ORDER[name]
    assert imex_order_defects(t, k).max() < 1e-14
    for key in ("a_ex", "a_im"):
        A = np.asarray(t[key], float)
        for i, j in zip(*np.nonzero(A)):
            tp = {kk: np.array(v, float) for kk, v in t.items()}
            tp[key][i, j] += 1e-3
            assert imex_order_defects(tp, k).max() > 1e-4, (key, i, j)
