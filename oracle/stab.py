"""Divergence / mass-flux stabilisation of the projection step -- TEST INFRASTRUCTURE ONLY
(same import rule as the rest of ``oracle/``).

PAPER.md:1040 (§3.3): "For pressure robustness a divergence/mass-flux stabilization is added as
proposed in [Joshi 2016, Akbas 2018]" -- the formula is not in the paper.  Reading A26
(DESIGN.md §2): the standard form of those references, a grad-div penalty plus a penalty on
the normal-velocity (mass-flux) jumps, applied as a postprocessing step after the projection:

  find v^ with, for every vector test function w of the velocity DG space,
    (v^, w) + a_D sum_K (div v^, div w)_K + a_C sum_F ([v^ . n], [w . n])_F = (v'', w),
    a_D = dt zeta_D U h / (P + 1),  a_C = dt zeta_C U,
  U = the mass-weighted RMS velocity sqrt(sum m |v''|^2 / sum m), h = (prod_d h_d)^(1/d),

with GLL collocation quadrature (reading A2: W_q = prod w h/2 on the element GLL grid, W^F on
the face grid), the broken (element-local) divergence, and [g] = g^- - g^+ across every face
(n = +e_d from the '-' element to its +d neighbour, so [w . n] = [w_d] on faces normal to d).
The matrix M + a_D K_D + a_C K_C is SPD; v^ is the M-orthogonal-like contraction of v''
(||v^||_M <= ||v''||_M) and tends to the H(div)-conforming, divergence-free part as a -> inf.

Plain numpy: the operator is assembled per element and per face by explicit quadrature sums
with the basis evaluated at the quadrature points by the product formula (oracle.dense_pair's
tables), the solve is a plain CG to 1e-14.
"""
from __future__ import annotations

import numpy as np

from . import Mesh, _elem_coords, _elem_index, mass
from .dense_pair import _Space


def _h(mesh):
    return [mesh.L[d] / mesh.N[d] for d in range(mesh.dim)]


def div_stab_apply(mesh: Mesh, v, aD, aC):
    """Weak vector (M + a_D K_D + a_C K_C) v, per component [N_el, n^d] (v: dim nodal fields)."""
    dim, P = mesh.dim, mesh.P
    S = _Space(dim, P, P, _h(mesh))
    nv, nel = S.nb ** dim, mesh.n_el
    B, G, W = S.vol()
    vs = [np.asarray(x, float).reshape(nel, nv) for x in v[:dim]]
    m = mass(mesh)
    out = [m * vs[c] for c in range(dim)]                               # (v, w): lumped GLL mass
    for e in range(nel):
        # div v at the quadrature points, sum_q W_q div(x_q) d_c phi_I(x_q)
        divq = sum(G[c] @ vs[c][e] for c in range(dim))
        for c in range(dim):
            out[c][e] += aD * (G[c].T @ (W * divq))
    for e in range(nel):
        ec = _elem_coords(mesh, e)
        for dn in range(dim):
            cn = list(ec)
            cn[dn] += 1
            ep = _elem_index(mesh, cn)
            Fm, WF = S.face(dn, 1)
            Fp, _ = S.face(dn, 0)
            jump = Fm @ vs[dn][e] - Fp @ vs[dn][ep]                        # [v . n] at the face points
            out[dn][e] += aC * (Fm.T @ (WF * jump))                        # [w . n] = +phi on the '-' side
            out[dn][ep] -= aC * (Fp.T @ (WF * jump))                       #          -phi on the '+' side
    return out


def div_stab_coefficients(mesh: Mesh, v, dt, zeta_D=1.0, zeta_C=1.0):
    """(a_D, a_C, U) of reading A26 for the velocity v (dim nodal fields)."""
    m = mass(mesh)
    U = np.sqrt(sum(np.sum(m * np.asarray(x, float).reshape(m.shape) ** 2) for x in v[: mesh.dim]) / np.sum(m))
    h = float(np.prod(_h(mesh))) ** (1.0 / mesh.dim)
    return dt * zeta_D * U * h / (mesh.P + 1), dt * zeta_C * U, U


def div_stab_solve(mesh: Mesh, v, dt, zeta_D=1.0, zeta_C=1.0, tol=1e-14, maxit=5000, coeffs=None):
    """v^ of reading A26 (plain CG on the 3-component system, start v'', stop when
    ||M^-1 r|| <= tol ||v''||).  Returns (v^ list, iterations, (a_D, a_C, U))."""
    dim = mesh.dim
    aD, aC, U = coeffs if coeffs is not None else div_stab_coefficients(mesh, v, dt, zeta_D, zeta_C)
    m = mass(mesh).reshape(-1)
    vv = [np.asarray(x, float).reshape(-1) for x in v[:dim]]
    fn = np.sqrt(sum(x @ x for x in vv))
    A = lambda x: [y.reshape(-1) for y in div_stab_apply(mesh, [z.reshape(mesh.n_el, -1) for z in x], aD, aC)]
    x = [z.copy() for z in vv]
    Ax = A(x)
    r = [m * vv[c] - Ax[c] for c in range(dim)]
    p = [z.copy() for z in r]
    rr = sum(z @ z for z in r)
    it = 0
    while np.sqrt(sum(((z / m) ** 2).sum() for z in r)) > tol * fn and it < maxit:
        q = A(p)
        a = rr / sum(p[c] @ q[c] for c in range(dim))
        for c in range(dim):
            x[c] += a * p[c]
            r[c] -= a * q[c]
        rr2 = sum(z @ z for z in r)
        for c in range(dim):
            p[c] = r[c] + (rr2 / rr) * p[c]
        rr = rr2
        it += 1
    return [z.reshape(mesh.n_el, -1) for z in x], it, (aD, aC, U)


def div_measures(mesh: Mesh, v):
    """(||div_h v||_M, ||[v . n]||_F): the broken divergence at the GLL nodes (mass-weighted L2)
    and the normal-velocity jumps over all faces (face-weighted L2) -- the quantities the
    stabilisation penalises (the 'discrete divergence' of the projected velocity)."""
    dim, P = mesh.dim, mesh.P
    S = _Space(dim, P, P, _h(mesh))
    nv, nel = S.nb ** dim, mesh.n_el
    B, G, W = S.vol()
    vs = [np.asarray(x, float).reshape(nel, nv) for x in v[:dim]]
    d2 = 0.0
    j2 = 0.0
    for e in range(nel):
        divq = sum(G[c] @ vs[c][e] for c in range(dim))
        d2 += float(W @ divq ** 2)
        ec = _elem_coords(mesh, e)
        for dn in range(dim):
            cn = list(ec)
            cn[dn] += 1
            ep = _elem_index(mesh, cn)
            Fm, WF = S.face(dn, 1)
            Fp, _ = S.face(dn, 0)
            jump = Fm @ vs[dn][e] - Fp @ vs[dn][ep]
            j2 += float(WF @ jump ** 2)
    return np.sqrt(d2), np.sqrt(j2)
