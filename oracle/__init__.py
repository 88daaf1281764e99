"""CPU oracle for the SIP-DG implicit-stage hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2112_04167_b200``) never imports it and shares no code with it.

Thin ctypes wrapper around ``dg_oracle.c`` (plain C, explicit quadrature, fp64,
``-ffp-contract=off``); see ``dg_oracle.h`` for the definitions and PAPER.md citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "dg_oracle.c")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_long)


class _Mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("N", ctypes.c_int * 3), ("L", ctypes.c_double * 3), ("P", ctypes.c_int)]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dg_oracle.h"))
    ):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.oracle_gll.argtypes = [ctypes.c_int, _dp, _dp]
        L.oracle_gauss.argtypes = [ctypes.c_int, _dp, _dp]
        L.oracle_lagrange.argtypes = [ctypes.c_int, _dp, ctypes.c_double, _dp, _dp]
        L.oracle_lagrange.restype = None
        mp = ctypes.POINTER(_Mesh)
        L.oracle_sip_apply.argtypes = [mp, ctypes.c_double, _dp, ctypes.c_double, _dp, _dp, _lp, ctypes.c_long]
        L.oracle_sip_diag.argtypes = [mp, ctypes.c_double, _dp, ctypes.c_double, _dp, _lp, ctypes.c_long]
        L.oracle_sip_dense.argtypes = [mp, ctypes.c_double, _dp, ctypes.c_double, _dp]
        L.oracle_pcg_solve.argtypes = [mp, ctypes.c_double, _dp, ctypes.c_double, _dp, ctypes.c_double,
                                       ctypes.c_int, ctypes.c_int, _dp, ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.oracle_convect.argtypes = [mp, ctypes.POINTER(_dp), ctypes.POINTER(_dp), _lp, ctypes.c_long]
        L.oracle_convect_q.argtypes = [mp, ctypes.c_int, ctypes.POINTER(_dp), ctypes.POINTER(_dp), _lp, ctypes.c_long]
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class Mesh:
    """Periodic Cartesian mesh description (dim, N[], L[], P)."""

    def __init__(self, dim, N, L, P):
        self.dim, self.P = int(dim), int(P)
        N = list(N) + [1] * (3 - len(N))
        L = list(L) + [1.0] * (3 - len(L))
        self.N = tuple(int(x) if i < dim else 1 for i, x in enumerate(N[:3]))
        self.L = tuple(float(x) for x in L[:3])
        self._m = _Mesh(self.dim, (ctypes.c_int * 3)(*self.N), (ctypes.c_double * 3)(*self.L), self.P)

    @property
    def n(self):
        return self.P + 1

    @property
    def npe(self):
        return self.n ** self.dim

    @property
    def n_el(self):
        return int(np.prod(self.N[: self.dim]))

    @property
    def ndof(self):
        return self.n_el * self.npe

    def ref(self):
        return ctypes.byref(self._m)


def gll(P):
    xi = np.zeros(P + 1)
    w = np.zeros(P + 1)
    if lib().oracle_gll(P, _ptr(xi), _ptr(w)):
        raise ValueError("oracle_gll failed")
    return xi, w


def gauss(Q):
    z = np.zeros(Q)
    w = np.zeros(Q)
    if lib().oracle_gauss(Q, _ptr(z), _ptr(w)):
        raise ValueError("oracle_gauss failed")
    return z, w


def lagrange(P, xi, x):
    xi = _f64(xi)
    l = np.zeros(P + 1)
    dl = np.zeros(P + 1)
    lib().oracle_lagrange(P, _ptr(xi), float(x), _ptr(l), _ptr(dl))
    return l, dl


def _elems(elems):
    if elems is None:
        return None, 0, None
    e = np.ascontiguousarray(elems, dtype=np.int64)
    return e, len(e), e.ctypes.data_as(_lp)


def sip_apply(mesh: Mesh, lam, u, nu=None, nu_const=1.0, elems=None):
    """Weak-form SIP-DG Helmholtz action; rows of ``elems`` (compact) or all."""
    u = _f64(u).reshape(-1)
    nu = _f64(nu)
    e, k, ep = _elems(elems)
    cnt = mesh.n_el if e is None else k
    y = np.zeros((cnt, mesh.npe))
    if lib().oracle_sip_apply(mesh.ref(), float(lam), _ptr(nu), float(nu_const), _ptr(u), _ptr(y), ep, k):
        raise ValueError("oracle_sip_apply failed")
    return y


def sip_diag(mesh: Mesh, lam, nu=None, nu_const=1.0, elems=None):
    nu = _f64(nu)
    e, k, ep = _elems(elems)
    cnt = mesh.n_el if e is None else k
    d = np.zeros((cnt, mesh.npe))
    if lib().oracle_sip_diag(mesh.ref(), float(lam), _ptr(nu), float(nu_const), _ptr(d), ep, k):
        raise ValueError("oracle_sip_diag failed")
    return d


def sip_dense(mesh: Mesh, lam, nu=None, nu_const=1.0):
    nu = _f64(nu)
    A = np.zeros((mesh.ndof, mesh.ndof))
    rc = lib().oracle_sip_dense(mesh.ref(), float(lam), _ptr(nu), float(nu_const), _ptr(A))
    if rc:
        raise ValueError("oracle_sip_dense failed (%d)" % rc)
    return A


def pcg_solve(mesh: Mesh, lam, f, nu=None, nu_const=1.0, tol=1e-14, maxit=100000, precond=True, u0=None):
    """Returns (u, iters, relres, removed_mean, status)."""
    f = _f64(f).reshape(-1)
    nu = _f64(nu)
    u = np.zeros(mesh.ndof) if u0 is None else _f64(u0).reshape(-1).copy()
    it = ctypes.c_int(0)
    rr = ctypes.c_double(0.0)
    rm = ctypes.c_double(0.0)
    st = lib().oracle_pcg_solve(mesh.ref(), float(lam), _ptr(nu), float(nu_const), _ptr(f), float(tol),
                                int(maxit), int(bool(precond)), _ptr(u), ctypes.byref(it), ctypes.byref(rr),
                                ctypes.byref(rm))
    if st < 0:
        raise ValueError("oracle_pcg_solve failed (%d)" % st)
    return u.reshape(mesh.n_el, mesh.npe), it.value, rr.value, rm.value, st


def convect(mesh: Mesh, v, elems=None, Q=None):
    """LLF DG convective tendency F_c (nodal), per component; rows of ``elems``.  Q: Gauss
    points per direction (default: reading A13, floor(3P/2)+1)."""
    vs = [_f64(x).reshape(-1) for x in v[: mesh.dim]]
    e, k, ep = _elems(elems)
    cnt = mesh.n_el if e is None else k
    outs = [np.zeros((cnt, mesh.npe)) for _ in range(mesh.dim)]
    vin = (_dp * 3)(*[_ptr(x) for x in vs] + [None] * (3 - mesh.dim))
    vout = (_dp * 3)(*[_ptr(x) for x in outs] + [None] * (3 - mesh.dim))
    rc = (lib().oracle_convect(mesh.ref(), vin, vout, ep, k) if Q is None
          else lib().oracle_convect_q(mesh.ref(), int(Q), vin, vout, ep, k))
    if rc:
        raise ValueError("oracle_convect failed")
    return outs


def mass(mesh: Mesh):
    """GLL-lumped mass m_I = prod_d w_{i_d} h_d/2, [N_el, n^d] (from oracle_gll)."""
    _, w = gll(mesh.P)
    m = np.ones([1] * 0)
    wd = []
    for d in range(mesh.dim):
        wd.append(w * mesh.L[d] / mesh.N[d] * 0.5)
    if mesh.dim == 2:
        m = (wd[1][:, None] * wd[0][None, :]).reshape(-1)
    else:
        m = (wd[2][:, None, None] * wd[1][None, :, None] * wd[0][None, None, :]).reshape(-1)
    return np.broadcast_to(m, (mesh.n_el, mesh.npe)).copy()


# ---------------------------------------------------------------------------
# IMEX-RK stage -- plain numpy composition of the functions above.
# ---------------------------------------------------------------------------
def imex_stage(mv: Mesh, mp: Mesh, dt, a_ex21, a_im21, a_im22, nu, v, tol=1e-14, stab=None):
    """Alg. 3 stage i = 2, constant nu, F_s = 0, under the readings of
    include/dg.h dg_imex_stage: returns (vout[dim], psi, v'').  Exact discrete solves
    (oracle PCG to tol).  stab = (zeta_D, zeta_C): the divergence / mass-flux stabilisation of
    v'' after line 6 (reading A26; oracle.stab)."""
    dim = mv.dim
    m = mass(mv)
    Fc = convect(mv, v)                                                     # F_c(v)
    Fd = [-sip_apply(mv, 0.0, v[c], nu_const=nu) / m for c in range(dim)]  # F_d1(v) = -M^-1 A_0 v
    gd = dg_gradient_weak(mp, dg_divergence_weak(mv, v) / mass(mp))        # grad div v
    Fg = [nu * gd[c] / m for c in range(dim)]                               # = F_d2 = -F_d3
    vp = [np.asarray(v[c]) + dt * a_ex21 * (Fc[c] + Fd[c] - Fg[c]) for c in range(dim)]  # line 4
    fp = -dg_divergence_weak(mv, vp) / mass(mp)                             # line 5 rhs: b = -D v'
    psi, *_ = pcg_solve(mp, 0.0, fp, nu_const=1.0, tol=tol)                 # line 5 (lam = 0)
    gw = dg_gradient_weak(mp, psi)
    vpp = [vp[c] - gw[c] / m for c in range(dim)]                           # line 6
    if stab is not None:                                                    # P:1040 (reading A26)
        from .stab import div_stab_solve
        vpp, _, _ = div_stab_solve(mv, vpp, dt, stab[0], stab[1], tol=tol)
    lam = 1.0 / (dt * a_im22)
    out = []
    for c in range(dim):
        g = vpp[c] + dt * ((a_im21 - a_ex21) * Fd[c] + a_ex21 * Fg[c])      # line 8
        u, *_ = pcg_solve(mv, lam, lam * g, nu_const=nu, tol=tol)           # line 9
        out.append(u)
    return out, psi, vpp


# ---------------------------------------------------------------------------
# DG divergence / gradient pair of the projection step (Alg. 3 lines
# 5-6): velocity degree P, pressure degree P-1, central fluxes,
# integrals on the velocity GLL grid (exact for these integrands: degree <= 2P-1 per
# direction).  Plain numpy; element loops, library tensor contractions as steps.
# ---------------------------------------------------------------------------
def _pv_tables(P):
    """GLL nodes of P and P-1, velocity weights w, pressure basis at velocity nodes E[i, a]
    and its derivative Ed[i, a], velocity derivative matrix Dv[i, j] (product formula)."""
    xv, wv = gll(P)
    xp, _ = gll(P - 1)
    E = np.zeros((P + 1, P))
    Ed = np.zeros((P + 1, P))
    Dv = np.zeros((P + 1, P + 1))
    for i, x in enumerate(xv):
        E[i], Ed[i] = lagrange(P - 1, xp, x)
        _, Dv[i] = lagrange(P, xv, x)
    return xv, wv, E, Ed, Dv


def _elem_coords(mesh, e):
    N = mesh.N
    return [e % N[0], (e // N[0]) % N[1], e // (N[0] * N[1])][: mesh.dim]


def _elem_index(mesh, c):
    N = mesh.N
    c = [c[d] % N[d] for d in range(mesh.dim)]
    return c[0] + N[0] * (c[1] + (N[1] * c[2] if mesh.dim == 3 else 0))


def _apply_1d(M, arr, axis):
    """Contract matrix M[out, in] with array axis `axis`."""
    return np.moveaxis(np.tensordot(M, arr, axes=([1], [axis])), 0, axis)


def dg_divergence_weak(mv: Mesh, v):
    """d_a = -sum_K sum_q W_q v(x_q).grad phi^p_a(x_q) + sum_F sum_q W^F_q ({v}.n)[phi^p_a],
    the weak DG divergence of the nodal velocity v (dim arrays [N_el, (P+1)^d]) tested with
    the degree-(P-1) pressure basis; returns [N_el, P^d] (pressure-mesh layout)."""
    P, dim = mv.P, mv.dim
    n, m = P + 1, P
    _, wv, E, Ed, _ = _pv_tables(P)
    h = [mv.L[d] / mv.N[d] for d in range(dim)]
    vs = [np.asarray(v[c], dtype=np.float64).reshape((mv.n_el,) + (n,) * dim) for c in range(dim)]
    out = np.zeros((mv.n_el,) + (m,) * dim)
    # array axes of an element block: (k, j, i) -> direction d sits at axis dim-1-d
    ax = lambda d: dim - 1 - d
    Wq = np.ones((n,) * dim)
    for d in range(dim):
        shp = [1] * dim
        shp[ax(d)] = n
        Wq = Wq * (wv * 0.5 * h[d]).reshape(shp)
    for e in range(mv.n_el):
        acc = np.zeros((m,) * dim)
        for c in range(dim):  # volume: -(v_c, d_c phi^p)
            t = Wq * vs[c][e]
            for d in range(dim):
                t = _apply_1d((Ed * (2.0 / h[d])).T if d == c else E.T, t, ax(d))
            acc -= t
        ec = _elem_coords(mv, e)
        for d in range(dim):  # faces normal to d; n = +e_d from the - side to the + side
            Wf = np.ones((n,) * (dim - 1))
            tdirs = [dd for dd in range(dim) if dd != d]
            for k, dd in enumerate(tdirs):
                shp = [1] * (dim - 1)
                shp[dim - 2 - k] = n
                Wf = Wf * (wv * 0.5 * h[dd]).reshape(shp)
            for side in (0, 1):
                cn = list(ec)
                cn[d] += 1 if side else -1
                en = _elem_index(mv, cn)
                own = np.take(vs[d][e], P if side else 0, axis=ax(d))     # own face trace v_d
                nbr = np.take(vs[d][en], 0 if side else P, axis=ax(d))    # neighbour's trace
                flux = Wf * 0.5 * (own + nbr)                              # W^F {v}.e_d
                # own test functions on the face: [phi] = +phi (own is '-', side 1) or -phi
                t = flux
                for k, dd in enumerate(tdirs):
                    t = _apply_1d(E.T, t, dim - 2 - k)
                layer = np.zeros(m)
                layer[m - 1 if side else 0] = 1.0
                shp = [1] * dim
                shp[ax(d)] = m
                acc += (1.0 if side else -1.0) * np.expand_dims(t, ax(d)) * layer.reshape(shp)
        out[e] = acc
    return out.reshape(mv.n_el, m ** dim)


def dg_gradient_weak(mp: Mesh, psi):
    """g_{c,i} = -sum_K sum_q W_q psi_h(x_q) d_c phi^v_i(x_q) + sum_F sum_q W^F_q {psi_h} n_c [phi^v_i]
    for the degree-(P-1) pressure psi ([N_el, P^d] on mesh mp, P = mp.P + 1); returns dim
    arrays [N_el, (P+1)^d] (velocity layout).  -g is the adjoint of dg_divergence_weak."""
    P, dim = mp.P + 1, mp.dim
    n, m = P + 1, P
    _, wv, E, _, Dv = _pv_tables(P)
    h = [mp.L[d] / mp.N[d] for d in range(dim)]
    ps = np.asarray(psi, dtype=np.float64).reshape((mp.n_el,) + (m,) * dim)
    ax = lambda d: dim - 1 - d
    Wq = np.ones((n,) * dim)
    for d in range(dim):
        shp = [1] * dim
        shp[ax(d)] = n
        Wq = Wq * (wv * 0.5 * h[d]).reshape(shp)

    def interp(a):  # pressure nodes -> velocity nodes (all directions)
        for d in range(dim):
            a = _apply_1d(E, a, ax(d))
        return a

    outs = [np.zeros((mp.n_el,) + (n,) * dim) for _ in range(dim)]
    for e in range(mp.n_el):
        ph = interp(ps[e])
        ec = _elem_coords(mp, e)
        for c in range(dim):
            # volume: -(psi_h, d_c phi^v_i) = -(2/h_c) sum_q D[q_c][i_c] W_q psi_h(q)
            outs[c][e] -= _apply_1d((Dv * (2.0 / h[c])).T, Wq * ph, ax(c))
            # faces normal to c
            d = c
            tdirs = [dd for dd in range(dim) if dd != d]
            Wf = np.ones((n,) * (dim - 1))
            for k, dd in enumerate(tdirs):
                shp = [1] * (dim - 1)
                shp[dim - 2 - k] = n
                Wf = Wf * (wv * 0.5 * h[dd]).reshape(shp)
            for side in (0, 1):
                cn = list(ec)
                cn[d] += 1 if side else -1
                en = _elem_index(mp, cn)
                own = np.take(ph, P if side else 0, axis=ax(d))
                nbr = np.take(interp(ps[en]), 0 if side else P, axis=ax(d))
                val = (1.0 if side else -1.0) * Wf * 0.5 * (own + nbr)   # W^F {psi} n_c [phi_i]
                idx = [slice(None)] * dim
                idx[ax(d)] = P if side else 0
                outs[c][e][tuple(idx)] += val
    return [o.reshape(mp.n_el, n ** dim) for o in outs]


# ---------------------------------------------------------------------------
# IMEX Runge-Kutta step (Alg. 3) composed from the oracle pieces.
# Tableaux typed from the paper's appendix, independently of the product's.
# ---------------------------------------------------------------------------
ORACLE_TABLEAUX = {
    "RK-TR": dict(
        a_im=[[0, 0, 0], [0, 1, 0], [1 / 2, 0, 1 / 2]],
        a_ex=[[0, 0, 0], [1, 0, 0], [1 / 2, 1 / 2, 0]],
        b_im=[1 / 2, 0, 1 / 2], b_ex=[1 / 2, 1 / 2, 0]),
    "RK-CB2": dict(
        a_im=[[0, 0, 0], [0, 2 / 5, 0], [0, 5 / 6, 1 / 6]],
        a_ex=[[0, 0, 0], [2 / 5, 0, 0], [0, 1, 0]],
        b_im=[0, 5 / 6, 1 / 6], b_ex=[0, 5 / 6, 1 / 6]),
    "RK-CB3e": dict(  # implicit (left), explicit (right)
        a_im=[[0, 0, 0, 0], [0, 1 / 3, 0, 0], [0, 1 / 2, 1 / 2, 0], [0, 3 / 4, -1 / 4, 1 / 2]],
        a_ex=[[0, 0, 0, 0], [1 / 3, 0, 0, 0], [0, 1, 0, 0], [0, 3 / 4, 1 / 4, 0]],
        b_im=[0, 3 / 4, -1 / 4, 1 / 2], b_ex=[0, 3 / 4, -1 / 4, 1 / 2]),
    "RK-ARS3": dict(
        a_im=[[0, 0, 0, 0, 0], [0, 1 / 2, 0, 0, 0], [0, 1 / 6, 1 / 2, 0, 0], [0, -1 / 2, 1 / 2, 1 / 2, 0],
              [0, 3 / 2, -3 / 2, 1 / 2, 1 / 2]],
        a_ex=[[0, 0, 0, 0, 0], [1 / 2, 0, 0, 0, 0], [11 / 18, 1 / 18, 0, 0, 0], [5 / 6, -5 / 6, 1 / 2, 0, 0],
              [1 / 4, 7 / 4, 3 / 4, -7 / 4, 0]],
        b_im=[0, 3 / 2, -3 / 2, 1 / 2, 1 / 2], b_ex=[1 / 4, 7 / 4, 3 / 4, -7 / 4, 0]),
}


def imex_rk_step(mv: Mesh, mp: Mesh, tab, dt, nu, v, tol=1e-14, stab=None):
    """One step of Alg. 3 under the readings of include/dg.h dg_imex_rk_step (constant nu,
    F_s = 0, F_d2 = -F_d3 = nu grad div u with the DG pair, final projection skipped):
    returns v^{n+1} (dim arrays)."""
    dim = mv.dim
    m, mpm = mass(mv), mass(mp)
    A_im, A_ex = np.asarray(tab["a_im"], float), np.asarray(tab["a_ex"], float)
    s = A_im.shape[0]

    def forces(u):
        gd = dg_gradient_weak(mp, dg_divergence_weak(mv, u) / mpm)                   # grad div u
        return (convect(mv, u), [-sip_apply(mv, 0.0, u[c], nu_const=nu) / m for c in range(dim)],
                [nu * gd[c] / m for c in range(dim)])

    Fc, Fd, Fg = [None] * s, [None] * s, [None] * s
    Fc[0], Fd[0], Fg[0] = forces([np.asarray(x, float) for x in v])
    u = None
    for i in range(1, s):
        # line 4 with F_d + F_d3 = F_d1 - nu grad div u (constant nu; rotational form)
        vp = [np.asarray(v[c], float) + dt * sum(A_ex[i, j] * (Fc[j][c] + Fd[j][c] - Fg[j][c]) for j in range(i))
              for c in range(dim)]
        psi, *_ = pcg_solve(mp, 0.0, -dg_divergence_weak(mv, vp) / mpm, nu_const=1.0, tol=tol)  # line 5
        gw = dg_gradient_weak(mp, psi)
        vpp = [vp[c] - gw[c] / m for c in range(dim)]                                   # line 6
        if stab is not None:                                                            # P:1040, A26
            from .stab import div_stab_solve
            vpp, _, _ = div_stab_solve(mv, vpp, dt, stab[0], stab[1], tol=tol)
        u = []
        for c in range(dim):
            g = vpp[c] + dt * sum((A_im[i, j] - A_ex[i, j]) * Fd[j][c] + A_ex[i, j] * Fg[j][c]
                                  for j in range(i))                                    # line 8
            if A_im[i, i] > 0:
                lam = 1.0 / (dt * A_im[i, i])
                x, *_ = pcg_solve(mv, lam, lam * g, nu_const=nu, tol=tol)                # line 9
                u.append(x)
            else:
                u.append(g)
        Fc[i], Fd[i], Fg[i] = forces(u)
    out = []
    for c in range(dim):                                                                # line 11
        out.append(u[c] + dt * sum((tab["b_ex"][j] - A_ex[s - 1, j]) * Fc[j][c]
                                   + (tab["b_im"][j] - A_im[s - 1, j]) * Fd[j][c] for j in range(s)))
    return out


# ---------------------------------------------------------------------------
# Two-level additive Schwarz preconditioner for the SIP system (
# P:1045-1046 "Krylov-accelerated Schwarz/multigrid methods ... for solving the implicit
# pressure and diffusion problems").  The paper gives no formula; DESIGN.md §9 states the
# reading taken (both sides):
#     B r = sum_K R_K^T A_KK^-1 R_K r  +  P_1 A_c^+ P_1^T r,   A_c = P_1^T A P_1,
# with R_K the restriction to the nodes of element K (non-overlapping subdomains = elements,
# A_KK the diagonal block of the assembled SIP matrix) and P_1 the prolongation of the
# continuous vertex-based Q1 space on the same mesh to the DG nodes (trilinear hats
# (1 -/+ xi)/2 evaluated at the GLL nodes, periodic vertex numbering).  A_c^+ is the
# pseudo-inverse (lam = 0: the constant null space, reading A8).  Definitions written out:
# A_KK and A_c by applying the oracle's own operator to unit / hat vectors, dense numpy
# linear algebra (library routines) for the inverses.  Small meshes only.
# ---------------------------------------------------------------------------
def q1_prolongation(mesh: Mesh):
    """Dense P_1 [ndof, NV]: column v = the periodic Q1 hat of vertex v at every DG node.
    Vertex index v = vx + Nx (vy + Ny vz), vertex (vx, vy, vz) at x = vx h (periodic)."""
    dim, N, n = mesh.dim, mesh.N, mesh.n
    xi, _ = gll(mesh.P)
    hat = [(1.0 - xi) / 2.0, (1.0 + xi) / 2.0]  # corner 0 (left), corner 1 (right)
    NV = mesh.n_el
    Pm = np.zeros((mesh.n_el, mesh.npe, NV))
    for e in range(mesh.n_el):
        ec = _elem_coords(mesh, e)
        for corner in range(2 ** dim):
            a = [(corner >> d) & 1 for d in range(dim)]
            v = _elem_index(mesh, [ec[d] + a[d] for d in range(dim)])
            if dim == 2:
                val = np.outer(hat[a[1]], hat[a[0]])
            else:
                val = hat[a[2]][:, None, None] * hat[a[1]][None, :, None] * hat[a[0]][None, None, :]
            Pm[e, :, v] += val.reshape(-1)  # += : with N_d = 1 two corners are one vertex
    return Pm.reshape(mesh.ndof, NV)


def q1_coarse_operator(mesh: Mesh, lam, nu_const=1.0):
    """A_c = P_1^T A P_1 (dense [NV, NV]), the oracle's operator applied to every hat."""
    Pm = q1_prolongation(mesh)
    Ac = np.zeros((Pm.shape[1], Pm.shape[1]))
    for v in range(Pm.shape[1]):
        Ac[:, v] = Pm.T @ sip_apply(mesh, lam, Pm[:, v], nu_const=nu_const).reshape(-1)
    return Ac, Pm


def element_block(mesh: Mesh, lam, e, nu_const=1.0):
    """A_KK [npe, npe]: rows and columns of element e of the assembled SIP matrix."""
    B = np.zeros((mesh.npe, mesh.npe))
    for j in range(mesh.npe):
        u = np.zeros(mesh.ndof)
        u[e * mesh.npe + j] = 1.0
        B[:, j] = sip_apply(mesh, lam, u, nu_const=nu_const, elems=[e]).reshape(-1)
    return B


class Schwarz2:
    """B = sum_K R_K^T A_KK^-1 R_K + P_1 A_c^+ P_1^T (see above); constant nu."""

    def __init__(self, mesh: Mesh, lam, nu_const=1.0, coarse=True):
        self.mesh = mesh
        self.binv = [np.linalg.inv(element_block(mesh, lam, e, nu_const)) for e in range(mesh.n_el)]
        self.coarse = coarse
        if coarse:
            Ac, self.Pm = q1_coarse_operator(mesh, lam, nu_const)
            self.Acp = np.linalg.pinv(Ac, rcond=1e-13) if lam == 0.0 else np.linalg.inv(Ac)

    def __call__(self, r):
        r = np.asarray(r, dtype=np.float64).reshape(self.mesh.n_el, self.mesh.npe)
        z = np.stack([self.binv[e] @ r[e] for e in range(self.mesh.n_el)])
        if self.coarse:
            z = z + (self.Pm @ (self.Acp @ (self.Pm.T @ r.reshape(-1)))).reshape(z.shape)
        return z


def pcg_precond(mesh: Mesh, lam, f, B, nu_const=1.0, tol=1e-12, maxit=10000):
    """Preconditioned CG for A u = M f with preconditioner z = B(r) (plain numpy loop; the
    stopping rule of reading A7, lam = 0 handled as reading A8).  Returns (u, iters)."""
    m = mass(mesh).reshape(-1)
    f = np.asarray(f, dtype=np.float64).reshape(-1)
    if lam == 0.0:
        f = f - (m @ f) / m.sum()
    fn = np.linalg.norm(f)
    A = lambda x: sip_apply(mesh, lam, x, nu_const=nu_const).reshape(-1)
    u = np.zeros_like(f)
    r = m * f
    z = B(r).reshape(-1)
    p = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        q = A(p)
        a = rz / (p @ q)
        u += a * p
        r -= a * q
        if lam == 0.0:
            r -= r.mean()
        if np.linalg.norm(r / m) <= tol * fn:
            break
        z = B(r).reshape(-1)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    if lam == 0.0:
        u -= (m @ u) / m.sum()
    return u.reshape(mesh.n_el, mesh.npe), it


# ---------------------------------------------------------------------------
# Variable viscosity: Alg. 3 line 7 nu_i = nu(v''_i) with the model of
# P:1218-1224, the explicit viscous parts F_d2 = div(nu grad(v)^T) and F_d3 = -grad(nu div v)
# (P:693-703), line 11 and the final projection (lines 12-15).  Readings (DESIGN.md
# §9): the derivatives in F_d2 / F_d3 are the velocity-level central-flux DG derivative
#     (Dc u)_i = m_i^-1 [ -sum_K sum_q W_q u(x_q) d_c phi_i(x_q) + sum_F sum_q W^F_q {u} n_c [phi_i] ]
# (GLL_P quadrature), so F_d2,c = sum_e D_e(nu D_c v_e), F_d3,c = -D_c(nu sum_e D_e v_e); the
# stage forces of stage i use nu_i (the viscosity of its implicit solve).
# ---------------------------------------------------------------------------
def dg_derivative(mesh: Mesh, u):
    """Nodal central-flux DG derivatives [D_0 u, ..., D_{dim-1} u] of the degree-P field u
    ([N_el, (P+1)^d]); each [N_el, (P+1)^d]."""
    P, dim, n = mesh.P, mesh.dim, mesh.n
    xv, wv = gll(P)
    Dv = np.zeros((n, n))
    for i, x in enumerate(xv):
        _, Dv[i] = lagrange(P, xv, x)
    h = [mesh.L[d] / mesh.N[d] for d in range(dim)]
    us = np.asarray(u, dtype=np.float64).reshape((mesh.n_el,) + (n,) * dim)
    ax = lambda d: dim - 1 - d
    Wq = np.ones((n,) * dim)
    for d in range(dim):
        shp = [1] * dim
        shp[ax(d)] = n
        Wq = Wq * (wv * 0.5 * h[d]).reshape(shp)
    outs = [np.zeros((mesh.n_el,) + (n,) * dim) for _ in range(dim)]
    for e in range(mesh.n_el):
        ec = _elem_coords(mesh, e)
        for c in range(dim):
            # volume: -(u, d_c phi_i) = -(2/h_c) sum_q D[q_c][i_c] W_q u(q)
            outs[c][e] -= _apply_1d((Dv * (2.0 / h[c])).T, Wq * us[e], ax(c))
            tdirs = [dd for dd in range(dim) if dd != c]
            Wf = np.ones((n,) * (dim - 1))
            for k, dd in enumerate(tdirs):
                shp = [1] * (dim - 1)
                shp[dim - 2 - k] = n
                Wf = Wf * (wv * 0.5 * h[dd]).reshape(shp)
            for side in (0, 1):
                cn = list(ec)
                cn[c] += 1 if side else -1
                en = _elem_index(mesh, cn)
                own = np.take(us[e], P if side else 0, axis=ax(c))
                nbr = np.take(us[en], 0 if side else P, axis=ax(c))
                idx = [slice(None)] * dim
                idx[ax(c)] = P if side else 0
                outs[c][e][tuple(idx)] += (1.0 if side else -1.0) * Wf * 0.5 * (own + nbr)  # W^F {u} n_c [phi_i]
    m = mass(mesh)
    return [o.reshape(mesh.n_el, mesh.npe) / m for o in outs]


def visc_model(v, nu0, nu1, vmax):
    """nu(v) = nu0 + nu1 (|v| / v_max)^2, pointwise at the nodes."""
    return nu0 + nu1 * sum(np.asarray(x, float) ** 2 for x in v) / vmax ** 2


def viscous_explicit(mv: Mesh, v, nu):
    """(F_d3, F_d2 + F_d3) of the nodal velocity v with the nodal viscosity field nu."""
    dim = mv.dim
    Dv = [dg_derivative(mv, v[e]) for e in range(dim)]            # Dv[e][c] = D_c v_e
    div = sum(Dv[e][e] for e in range(dim))
    Fd3 = [-g for g in dg_derivative(mv, nu * div)]
    Fd2 = [sum(dg_derivative(mv, nu * Dv[e][c])[e] for e in range(dim)) for c in range(dim)]
    return Fd3, [Fd2[c] + Fd3[c] for c in range(dim)]


def imex_rk_step_vv(mv: Mesh, mp: Mesh, tab, dt, visc, v, fs=None, final_projection=True, tol=1e-14):
    """One step of Alg. 3 with the solution-dependent viscosity nu(v) =
    nu0 + nu1 (|v|/v_max)^2 (visc = (nu0, nu1, vmax)) and forcing fs[j][c] (nodal, at
    t + c_j dt; None = 0), under the readings of include/dg.h dg_imex_rk_step_vv."""
    dim = mv.dim
    m, mpm = mass(mv), mass(mp)
    A_im, A_ex = np.asarray(tab["a_im"], float), np.asarray(tab["a_ex"], float)
    s = A_im.shape[0]
    nu0, nu1, vmax = visc
    F = (lambda j, c: 0.0) if fs is None else (lambda j, c: np.asarray(fs[j][c], float))

    def forces(u, nu):
        Fd3, Fd23 = viscous_explicit(mv, u, nu)
        Fd1 = [-sip_apply(mv, 0.0, u[c], nu=nu) / m for c in range(dim)]         # F_d1 = div nu grad u
        return convect(mv, u), Fd1, Fd3, Fd23

    def project(w):  # lines 5-6 / 13-14: solve lap psi = div w, w - grad psi
        psi, *_ = pcg_solve(mp, 0.0, -dg_divergence_weak(mv, w) / mpm, nu_const=1.0, tol=tol)
        gw = dg_gradient_weak(mp, psi)
        return [w[c] - gw[c] / m for c in range(dim)]

    v0 = [np.asarray(x, float) for x in v]
    Fc, Fd1, Fd3, Fd23 = [None] * s, [None] * s, [None] * s, [None] * s
    Fc[0], Fd1[0], Fd3[0], Fd23[0] = forces(v0, visc_model(v0, nu0, nu1, vmax))
    u = v0
    for i in range(1, s):
        vp = [v0[c] + dt * (sum(A_ex[i, j] * (Fc[j][c] + Fd1[j][c] + Fd23[j][c] + Fd3[j][c]) for j in range(i))
                            + sum(A_im[i, j] * F(j, c) for j in range(i + 1)))
              for c in range(dim)]                                                   # line 4
        vpp = project(vp)                                                            # lines 5-6
        nu_i = visc_model(vpp, nu0, nu1, vmax)                                       # line 7
        u = []
        for c in range(dim):
            g = vpp[c] + dt * sum((A_im[i, j] - A_ex[i, j]) * Fd1[j][c] - A_ex[i, j] * Fd3[j][c]
                                  for j in range(i))                                 # line 8
            if A_im[i, i] > 0:
                lam = 1.0 / (dt * A_im[i, i])
                x, *_ = pcg_solve(mv, lam, lam * g, nu=nu_i, tol=tol)                 # line 9
                u.append(x)
            else:
                u.append(g)
        Fc[i], Fd1[i], Fd3[i], Fd23[i] = forces(u, nu_i)
    out = []
    for c in range(dim):                                                             # line 11
        out.append(u[c] + dt * sum((tab["b_ex"][j] - A_ex[s - 1, j]) * (Fc[j][c] + Fd23[j][c])
                                   + (tab["b_im"][j] - A_im[s - 1, j]) * (Fd1[j][c] + F(j, c))
                                   for j in range(s)))
    if final_projection:
        out = project(out)                                                           # lines 12-15
    return out
