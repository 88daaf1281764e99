"""Pins for the oracle's divergence / mass-flux stabilisation (reading A26).

The paper cites the formulation without writing it; what the reading fixes -- and these pins
check -- are properties of its definition:
  * zero coefficients give the identity (v^ = v'');
  * M + a_D K_D + a_C K_C is symmetric, K_D + K_C positive semi-definite (a wrong face sign or a
    one-sided jump makes it indefinite);
  * fields with zero broken divergence and continuous normal components (v_x a function of
    (y, z) only, etc., even discontinuous across tangential faces) are left unchanged;
  * the step contracts in the mass norm, ||v^||_M <= ||v''||_M;
  * as a_D, a_C -> inf the penalised quantities of v^ -- the broken divergence and the normal
    jumps, SURVEY §8(f) NEXT-1's "discrete divergence of v''" -- decrease like 1/a;
  * U is the RMS velocity (a constant field gives |v|).
"""
import numpy as np
import pytest

import oracle
from oracle.stab import div_measures, div_stab_apply, div_stab_coefficients, div_stab_solve


def rand_v(m, seed):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, (m.n_el, m.npe)) for _ in range(m.dim)]


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 3), (3, (2, 2, 2), 2)])
def test_zero_coefficients_identity(dim, N, P):
    m = oracle.Mesh(dim, N, (1.0, 1.2, 0.9)[:dim], P)
    v = rand_v(m, 1)
    out = div_stab_apply(m, v, 0.0, 0.0)
    mm = oracle.mass(m)
    for c in range(dim):
        assert np.abs(out[c] - mm * v[c]).max() < 1e-15
    vh, it, _ = div_stab_solve(m, v, 0.1, coeffs=(0.0, 0.0, 1.0))
    for c in range(dim):
        assert np.abs(vh[c] - v[c]).max() < 1e-14


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 3), (2, (1, 2), 2), (3, (2, 2, 2), 2), (3, (2, 1, 2), 2)])
def test_symmetric_positive(dim, N, P):
    m = oracle.Mesh(dim, N, (1.0, 1.2, 0.9)[:dim], P)
    n = m.ndof
    K = np.zeros((dim * n, dim * n))
    for j in range(dim * n):
        e = np.zeros(dim * n)
        e[j] = 1.0
        v = [e[c * n:(c + 1) * n].reshape(m.n_el, m.npe) for c in range(dim)]
        K[:, j] = np.concatenate([x.reshape(-1) for x in div_stab_apply(m, v, 0.7, 1.3)])
    Mv = np.concatenate([oracle.mass(m).reshape(-1)] * dim)
    assert np.abs(K - K.T).max() < 1e-14 * np.abs(K).max()
    ev = np.linalg.eigvalsh(K - np.diag(Mv))
    assert ev.min() > -1e-12 * ev.max()                 # K_D + K_C PSD
    assert (ev < 1e-10 * ev.max()).sum() > 0            # with a non-trivial null space


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 4), (3, (2, 3, 2), 3)])
def test_solenoidal_normal_continuous_fields_unchanged(dim, N, P):
    """v_d independent of x_d (random in the transverse node positions, discontinuous across
    tangential faces): zero broken divergence, no normal jumps -> A v = M v, v^ = v."""
    m = oracle.Mesh(dim, N, (1.0, 1.2, 0.9)[:dim], P)
    rng = np.random.default_rng(5)
    n = P + 1
    shape = tuple(m.N[:dim][::-1]) + (n,) * dim            # (ez, ey, ex, k, j, i) / (ey, ex, j, i)
    v = []
    for d in range(dim):
        R = rng.uniform(-1, 1, shape)
        el_ax, nd_ax = dim - 1 - d, 2 * dim - 1 - d
        R = np.repeat(np.take(R, [0], axis=el_ax), m.N[d], axis=el_ax)     # same in every element along d
        R = np.repeat(np.take(R, [0], axis=nd_ax), n, axis=nd_ax)           # constant along the d-lines
        v.append(R.reshape(m.n_el, m.npe))
    out = div_stab_apply(m, v, 3.0, 5.0)
    mm = oracle.mass(m)
    for c in range(dim):
        assert np.abs(out[c] - mm * v[c]).max() < 1e-13
    dv, jv = div_measures(m, v)
    assert dv < 1e-12 and jv < 1e-12


@pytest.mark.parametrize("dim,N,P", [(2, (3, 3), 4), (3, (2, 2, 2), 2)])
def test_cg_solve_matches_dense(dim, N, P):
    m = oracle.Mesh(dim, N, (1.0,) * dim, P)
    v = rand_v(m, 8)
    vh, it, _ = div_stab_solve(m, v, 1.0, coeffs=(0.3, 0.5, 1.0), tol=1e-14)
    ref = dense_solve_ab(m, v, 0.3, 0.5)
    for c in range(dim):
        assert np.abs(vh[c] - ref[c]).max() < 1e-11


def dense_solve_ab(m, v, aD, aC):
    n, dim = m.ndof, m.dim
    K = np.zeros((dim * n, dim * n))
    for j in range(dim * n):
        e = np.zeros(dim * n)
        e[j] = 1.0
        w = [e[c * n:(c + 1) * n].reshape(m.n_el, m.npe) for c in range(dim)]
        K[:, j] = np.concatenate([x.reshape(-1) for x in div_stab_apply(m, w, aD, aC)])
    rhs = np.concatenate([(oracle.mass(m) * x).reshape(-1) for x in v])
    x = np.linalg.solve(K, rhs)
    return [x[c * n:(c + 1) * n].reshape(m.n_el, m.npe) for c in range(dim)]


@pytest.mark.parametrize("dim,N,P", [(2, (3, 3), 4), (3, (2, 2, 2), 2)])
def test_contraction_and_large_penalty_limit(dim, N, P):
    m = oracle.Mesh(dim, N, (1.0,) * dim, P)
    v = rand_v(m, 7)
    mm = oracle.mass(m)
    nrm = lambda w: np.sqrt(sum(np.sum(mm * x ** 2) for x in w))
    d0, j0 = div_measures(m, v)
    prev = None
    for a in (1e-2, 1.0, 1e2, 1e4):
        vh = dense_solve_ab(m, v, a, a)
        assert nrm(vh) <= nrm(v) * (1 + 1e-14)
        d, j = div_measures(m, vh)
        if prev is not None:
            assert d + j < prev
        prev = d + j
        if a >= 1e2:
            assert d + j < 30.0 / a * (d0 + j0)
    assert prev < 1e-2 * (d0 + j0)


def test_velocity_scale():
    m = oracle.Mesh(3, (2, 2, 2), (1.0, 2.0, 0.5), 3)
    v = [np.full((m.n_el, m.npe), c) for c in (0.3, -1.2, 0.4)]
    aD, aC, U = div_stab_coefficients(m, v, 0.01, 2.0, 3.0)
    assert abs(U - np.sqrt(0.09 + 1.44 + 0.16)) < 1e-14
    h = (0.5 * 1.0 * 0.25) ** (1 / 3)
    assert abs(aD - 0.01 * 2.0 * U * h / 4) < 1e-15 and abs(aC - 0.01 * 3.0 * U) < 1e-15
