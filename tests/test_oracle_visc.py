"""Pins of the oracle's variable-viscosity pieces (Alg. 3 lines 4-15,
P:815-892; F_d2 / F_d3; the VVP test of P:1189-1256):

* the closed-form VVP forcing (workloads.vvp_forcing) equals central differences of its
  definition f = d_t v + div(v v) - div[nu (grad v + grad v^T)] + grad p;
* the central-flux DG derivative is exact on continuous polynomials of degree <= P (elements
  away from the periodic seam) and M D_c is skew (u^T M D_c w = -w^T M D_c u);
* for constant nu, F_d2 + F_d3 = 0 exactly (the D_c commute on tensor-product meshes);
* F_d1 + F_d2 + F_d3 of the exact VVP field converges spectrally to div[nu (grad v + grad v^T)];
* the variable-viscosity step keeps a uniform flow and, with nu1 = 0, multiplies a viscous
  shear mode by the DIRK stability function R(z) (as the constant-nu step).
"""
import math

import numpy as np
import pytest

import oracle
from workloads import node_coords
from workloads.inputs import vvp_exact, vvp_forcing


def test_vvp_forcing_matches_its_definition():
    rng = np.random.default_rng(0)
    X = [rng.uniform(-0.5, 0.5, 25) for _ in range(3)]
    t, nu0, nu1, h = 0.137, 0.01, 0.02, 1e-4
    vmax = 2.0

    def v_at(Y, tt):
        return np.array(vvp_exact(Y, tt)[0])

    def shift(Y, e, s):
        return [y + (s if k == e else 0.0) for k, y in enumerate(Y)]

    def d(fun, Y, e):
        return (fun(shift(Y, e, h)) - fun(shift(Y, e, -h))) / (2 * h)

    def stress(Y, e):  # nu (d_e v_c + d_c v_e), all c
        vv = v_at(Y, t)
        nu = nu0 + nu1 * (vv ** 2).sum(0) / vmax ** 2
        gd = [d(lambda Z: v_at(Z, t), Y, j) for j in range(3)]
        return nu * np.array([gd[e][c] + gd[c][e] for c in range(3)])

    dv_dt = (v_at(X, t + h) - v_at(X, t - h)) / (2 * h)
    conv = sum(d(lambda Y: v_at(Y, t)[e] * v_at(Y, t), X, e) for e in range(3))
    visc = sum(d(lambda Y: stress(Y, e), X, e) for e in range(3))
    gp = np.array([d(lambda Y: vvp_exact(Y, t)[1], X, e) for e in range(3)])
    f = np.array(vvp_forcing(X, t, nu0, nu1, vmax))
    assert np.abs(f - (dv_dt + conv - visc + gp)).max() <= 1e-5 * np.abs(f).max()


@pytest.mark.parametrize("dim,N,P", [(3, (4, 3, 4), 4), (2, (4, 5), 6)])
def test_dg_derivative_exact_and_skew(dim, N, P):
    L = (1.0, 1.1, 0.9)[:dim]
    m = oracle.Mesh(dim, N, L, P)
    X = node_coords(dim, N, L, P)
    if dim == 3:
        u = X[0] ** 2 * X[1] + X[2] ** 3 - X[0] * X[2]
        du = [2 * X[0] * X[1] - X[2], X[0] ** 2, 3 * X[2] ** 2 - X[0]]
    else:
        u = X[0] ** 3 * X[1] ** 2 - X[1]
        du = [3 * X[0] ** 2 * X[1] ** 2, 2 * X[0] ** 3 * X[1] - 1.0]
    d = oracle.dg_derivative(m, u)
    inner = [e for e in range(m.n_el) if all(0 < c < N[k] - 1 for k, c in enumerate(oracle._elem_coords(m, e)))]
    for c in range(dim):
        assert np.abs(d[c][inner] - du[c][inner]).max() <= 1e-12 * max(1.0, np.abs(du[c]).max())
    rng = np.random.default_rng(1)
    a, b = rng.uniform(-1, 1, (2, m.n_el, m.npe))
    M = oracle.mass(m)
    for c in range(dim):
        lhs = (M * a * oracle.dg_derivative(m, b)[c]).sum()
        rhs = -(M * b * oracle.dg_derivative(m, a)[c]).sum()
        assert abs(lhs - rhs) <= 1e-13 * np.abs(M * a).sum() * 10


def test_constant_nu_f_d2_plus_f_d3_vanishes():
    m = oracle.Mesh(3, (3, 2, 3), (1.0, 0.8, 1.2), 4)
    rng = np.random.default_rng(2)
    v = [rng.uniform(-1, 1, (m.n_el, m.npe)) for _ in range(3)]
    Fd3, Fd23 = oracle.viscous_explicit(m, v, np.full((m.n_el, m.npe), 0.37))
    scale = max(np.abs(x).max() for x in Fd3)
    assert scale > 1.0
    assert max(np.abs(x).max() for x in Fd23) <= 1e-13 * scale


def test_viscous_terms_converge_to_closed_form():
    """F_d1 + F_d2 + F_d3 of the exact VVP velocity with nu = nu(v) at the nodes vs the closed form
    div[nu (grad v + grad v^T)] = nu lap v + (grad v + grad v^T) grad nu (div v = 0): spectral
    convergence in P on 4^3 elements of [0, 1]^3."""
    nu0, nu1, vmax, t = 0.01, 0.01, 2.0, 0.1
    k = 2 * math.pi
    errs = []
    for P in (4, 7):
        m = oracle.Mesh(3, (4, 4, 4), (1.0, 1.0, 1.0), P)
        X = node_coords(3, (4, 4, 4), (1.0, 1.0, 1.0), P)
        v, _ = vvp_exact(X, t)
        nu = oracle.visc_model(v, nu0, nu1, vmax)
        M = oracle.mass(m)
        Fd3, Fd23 = oracle.viscous_explicit(m, v, nu)
        Fd1 = [-oracle.sip_apply(m, 0.0, v[c], nu=nu) / M for c in range(3)]
        # closed form from the gradient tensor of the exact field (as in vvp_forcing)
        A, B, C = k * (X[0] + t), k * (X[1] + t), k * (X[2] + t)
        sA, cA, sB, cB, sC, cC = np.sin(A), np.cos(A), np.sin(B), np.cos(B), np.sin(C), np.cos(C)
        G = [[k * cA * sC, -k * sB * sC, k * (sA + cB) * cC],
             [-k * sA * sC, k * cB * sC, k * (cA + sB) * cC],
             [-k * sA * cC, -k * sB * cC, -k * (cA + cB) * sC]]
        gnu = [2 * nu1 / vmax ** 2 * sum(v[c] * G[c][e] for c in range(3)) for e in range(3)]
        exact = [nu * (-2 * k * k * v[c]) + sum(gnu[e] * (G[c][e] + G[e][c]) for e in range(3)) for c in range(3)]
        err = max(np.abs(Fd1[c] + Fd23[c] - exact[c]).max() for c in range(3))
        errs.append(err / max(np.abs(e).max() for e in exact))
    assert errs[1] < 1e-3 and errs[1] < errs[0] / 50, errs


TAB = oracle.ORACLE_TABLEAUX


@pytest.mark.parametrize("name", ["RK-CB3e", "RK-ARS3"])
def test_vv_step_keeps_a_uniform_flow(name):
    dim, N, L, P = 2, (3, 2), (1.0, 1.3), 3
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    v = [np.full((mv.n_el, mv.npe), c) for c in (0.7, -0.2)]
    out = oracle.imex_rk_step_vv(mv, mp, TAB[name], 0.05, (0.02, 0.03, 1.0), v)
    for c in range(dim):
        assert np.abs(out[c] - v[c]).max() < 1e-12


def test_vv_step_shear_mode_with_nu1_zero_is_the_dirk_stability_function():
    dim, N, L, P = 2, (2, 4), (1.0, 1.0), 5
    mv, mp = oracle.Mesh(dim, N, L, P), oracle.Mesh(dim, N, L, P - 1)
    X = node_coords(dim, N, L, P)
    u0 = np.sin(2 * np.pi * X[1])
    nu = 0.02
    A = oracle.sip_dense(mv, 0.0, nu_const=nu)
    m = oracle.mass(mv).reshape(-1)
    w, V = np.linalg.eigh(A / np.sqrt(np.outer(m, m)))
    y = np.sqrt(m) * u0.reshape(-1)
    k = int(np.argmax(np.abs(V.T @ y)))
    sel = np.abs(w - w[k]) <= 1e-9 * w[k]
    ev = V[:, sel] @ (V[:, sel].T @ y) / np.sqrt(m)
    mu = -w[k]
    ev = ev.reshape(mv.n_el, mv.npe) / np.abs(ev).max()
    z = -0.7
    dt = z / mu
    t = TAB["RK-ARS3"]
    A_im = np.array(t["a_im"])
    s = A_im.shape[0]
    R = 1 + z * np.array(t["b_im"]) @ np.linalg.solve(np.eye(s) - z * A_im, np.ones(s))
    out = oracle.imex_rk_step_vv(mv, mp, t, dt, (nu, 0.0, 1.0), [ev, np.zeros_like(ev)])
    assert np.abs(out[0] - R * ev).max() <= 1e-7
    assert np.abs(out[1]).max() <= 1e-7
