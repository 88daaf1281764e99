"""Brute-force dense assembly of the DG divergence / gradient pair and of the velocity-level DG
derivative -- TEST INFRASTRUCTURE ONLY (same import rule as the rest of ``oracle/``).

A second, independent statement of the operators that ``oracle.dg_divergence_weak``,
``oracle.dg_gradient_weak`` and ``oracle.dg_derivative`` compute with element-local tensor
contractions: here every matrix entry is the explicit quadrature sum over ALL quadrature
points of the product of the two basis functions involved, with the basis evaluated at each
point by the product formula (``oracle.lagrange``), element by element and face by face, no
tensor-product factorisation and no sparsity logic (like ``oracle.sip_dense`` for the SIP
operator).  Small meshes only (2x2, 2x2x2).

Definitions (Alg. 3 lines 5-6; P:1036 pressure degree P-1; readings in
DESIGN.md §9; central fluxes {g} = (g^- + g^+)/2, [g] = g^- - g^+, n = +e_d from the '-'
element e to its +d neighbour, quadrature: the velocity GLL grid, W^F the face weights):
  div  D[a, (c, J)] = -sum_K sum_q W_q d_c phi^p_a(x_q) phi^v_J(x_q)
                      + sum_F sum_q W^F_q {phi^v_J} n_c [phi^p_a]
  grad G[(c, i), a] = -sum_K sum_q W_q phi^p_a(x_q) d_c phi^v_i(x_q)
                      + sum_F sum_q W^F_q {phi^p_a} n_c [phi^v_i]
  deriv D_c[i, J]   = m_i^-1 ( -sum_K sum_q W_q phi_J(x_q) d_c phi_i(x_q)
                      + sum_F sum_q W^F_q {phi_J} n_c [phi_i] )
"""
from __future__ import annotations

import numpy as np

from . import Mesh, _elem_coords, _elem_index, gll, lagrange, mass


def _tables(Pb, nodes_b, xq):
    """1-D basis of degree Pb (nodes nodes_b) at points xq and at the two ends: values, derivs."""
    L = np.array([lagrange(Pb, nodes_b, x)[0] for x in xq])
    dL = np.array([lagrange(Pb, nodes_b, x)[1] for x in xq])
    Le = np.array([lagrange(Pb, nodes_b, x)[0] for x in (-1.0, 1.0)])
    return L, dL, Le


def _tp(mats):
    """Tensor-product basis values [points, functions] from per-direction 1-D tables
    (direction 0 fastest in both the point and the function index)."""
    out = mats[0]
    for M in mats[1:]:
        out = np.kron(M, out)
    return out


class _Space:
    """Element basis of degree Pb evaluated on the velocity GLL grid of degree Pq."""

    def __init__(self, dim, Pb, Pq, h):
        xq, wq = gll(Pq)
        xb, _ = gll(Pb)
        self.dim, self.nq, self.nb = dim, Pq + 1, Pb + 1
        self.L, self.dL, self.Le = _tables(Pb, xb, xq)
        self.h = h
        self.wq = wq

    def vol(self):
        """B[q, J] (values) and G[c][q, J] (physical d_c) at the volume points, and W[q]."""
        d = self.dim
        B = _tp([self.L] * d)
        G = []
        for c in range(d):
            G.append(_tp([self.dL * (2.0 / self.h[k]) if k == c else self.L for k in range(d)]))
        W = _tp([(self.wq * 0.5 * self.h[k])[:, None] for k in range(d)])[:, 0]
        return B, G, W

    def face(self, dn, end):
        """Values [qf, J] at the face points of the face normal to dn at reference end (0: -1,
        1: +1), and the face weights W^F[qf] (points ordered over the tangential directions)."""
        d = self.dim
        mats, wts = [], []
        for k in range(d):
            if k == dn:
                mats.append(self.Le[end][None, :])
                wts.append(np.ones((1, 1)))
            else:
                mats.append(self.L)
                wts.append((self.wq * 0.5 * self.h[k])[:, None])
        return _tp(mats), _tp(wts)[:, 0]


def _h(mesh):
    return [mesh.L[d] / mesh.N[d] for d in range(mesh.dim)]


def div_dense(mv: Mesh):
    """Dense weak DG divergence [N_el P^d, dim * N_el (P+1)^d]; column block c = component c."""
    dim, P = mv.dim, mv.P
    h = _h(mv)
    Vs, Ps = _Space(dim, P, P, h), _Space(dim, P - 1, P, h)
    nv, npp = Vs.nb ** dim, Ps.nb ** dim
    nel = mv.n_el
    D = np.zeros((nel * npp, dim * nel * nv))
    Bv, _, W = Vs.vol()
    _, Gp, _ = Ps.vol()
    for e in range(nel):
        for c in range(dim):
            blk = -np.einsum("q,qa,qj->aj", W, Gp[c], Bv)
            D[e * npp:(e + 1) * npp, c * nel * nv + e * nv:c * nel * nv + (e + 1) * nv] += blk
    for e in range(nel):
        ec = _elem_coords(mv, e)
        for dn in range(dim):
            cn = list(ec)
            cn[dn] += 1
            ep = _elem_index(mv, cn)                      # '+' element across face x_dn = right end of e
            Fv_m, WF = Vs.face(dn, 1)
            Fv_p, _ = Vs.face(dn, 0)
            Fp_m, _ = Ps.face(dn, 1)
            Fp_p, _ = Ps.face(dn, 0)
            c = dn                                         # n = +e_dn: only component dn
            for (rows, Fp, sgn) in ((e, Fp_m, 1.0), (ep, Fp_p, -1.0)):      # [phi^p] = phi^- - phi^+
                for (cols, Fv) in ((e, Fv_m), (ep, Fv_p)):                   # {v} = (v^- + v^+)/2
                    blk = sgn * 0.5 * np.einsum("q,qa,qj->aj", WF, Fp, Fv)
                    D[rows * npp:(rows + 1) * npp, c * nel * nv + cols * nv:c * nel * nv + (cols + 1) * nv] += blk
    return D


def grad_dense(mp: Mesh):
    """Dense weak DG gradient [dim * N_el (P+1)^d, N_el P^d] for the pressure mesh mp
    (velocity degree P = mp.P + 1); row block c = component c."""
    dim, P = mp.dim, mp.P + 1
    h = _h(mp)
    Vs, Ps = _Space(dim, P, P, h), _Space(dim, P - 1, P, h)
    nv, npp = Vs.nb ** dim, Ps.nb ** dim
    nel = mp.n_el
    G = np.zeros((dim * nel * nv, nel * npp))
    _, Gv, W = Vs.vol()
    Bp, _, _ = Ps.vol()
    for e in range(nel):
        for c in range(dim):
            blk = -np.einsum("q,qi,qa->ia", W, Gv[c], Bp)
            G[c * nel * nv + e * nv:c * nel * nv + (e + 1) * nv, e * npp:(e + 1) * npp] += blk
    for e in range(nel):
        ec = _elem_coords(mp, e)
        for dn in range(dim):
            cn = list(ec)
            cn[dn] += 1
            ep = _elem_index(mp, cn)
            Fv_m, WF = Vs.face(dn, 1)
            Fv_p, _ = Vs.face(dn, 0)
            Fp_m, _ = Ps.face(dn, 1)
            Fp_p, _ = Ps.face(dn, 0)
            c = dn
            for (rows, Fv, sgn) in ((e, Fv_m, 1.0), (ep, Fv_p, -1.0)):      # [phi^v] n_c
                for (cols, Fp) in ((e, Fp_m), (ep, Fp_p)):                   # {psi}
                    blk = sgn * 0.5 * np.einsum("q,qi,qa->ia", WF, Fv, Fp)
                    G[c * nel * nv + rows * nv:c * nel * nv + (rows + 1) * nv, cols * npp:(cols + 1) * npp] += blk
    return G


def deriv_dense(m: Mesh):
    """Dense nodal central-flux DG derivatives [D_0, ..., D_{dim-1}], each [ndof, ndof]."""
    dim, P = m.dim, m.P
    h = _h(m)
    S = _Space(dim, P, P, h)
    nv, nel = S.nb ** dim, m.n_el
    B, Gd, W = S.vol()
    out = [np.zeros((nel * nv, nel * nv)) for _ in range(dim)]
    for e in range(nel):
        for c in range(dim):
            out[c][e * nv:(e + 1) * nv, e * nv:(e + 1) * nv] -= np.einsum("q,qi,qj->ij", W, Gd[c], B)
    for e in range(nel):
        ec = _elem_coords(m, e)
        for dn in range(dim):
            cn = list(ec)
            cn[dn] += 1
            ep = _elem_index(m, cn)
            F_m, WF = S.face(dn, 1)
            F_p, _ = S.face(dn, 0)
            for (rows, Fr, sgn) in ((e, F_m, 1.0), (ep, F_p, -1.0)):
                for (cols, Fc) in ((e, F_m), (ep, F_p)):
                    out[dn][rows * nv:(rows + 1) * nv, cols * nv:(cols + 1) * nv] += \
                        sgn * 0.5 * np.einsum("q,qi,qj->ij", WF, Fr, Fc)
    mi = mass(m).reshape(-1)
    return [o / mi[:, None] for o in out]
