"""Pins of the oracle's IMEX-RK stage pieces (Alg. 3 lines 4-9)."""
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


@pytest.mark.parametrize("dim,N,P", [(2, (3, 2), 3), (3, (2, 2, 3), 3), (3, (2, 1, 2), 4), (2, (2, 2), 6)])
def test_broken_divergence_exact_for_polynomials(dim, N, P):
    """Collocation derivatives are exact for degree <= P and the interpolation to the P-1
    nodes is exact for degree <= P-1: the result equals the analytic divergence there."""
    L = (1.0, 1.3, 0.8)[:dim]
    om = oracle.Mesh(dim, N, L, P)
    v, _ = _poly(dim, node_coords(dim, N, L, P))
    _, dv = _poly(dim, node_coords(dim, N, L, P - 1))
    got = oracle.broken_divergence_p1(om, v)
    assert np.abs(got - dv).max() <= 1e-13 * np.abs(dv).max()


def test_broken_divergence_detects_transposed_direction():
    dim, N, P, L = 2, (2, 2), 3, (1.0, 1.3)
    om = oracle.Mesh(dim, N, L, P)
    X = node_coords(dim, N, L, P)
    v = [X[1] ** 2, 0.0 * X[0]]          # div = 0 exactly; a swapped axis would give 2y
    assert np.abs(oracle.broken_divergence_p1(om, v)).max() < 1e-13


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
