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


def convect(mesh: Mesh, v, elems=None):
    """LLF DG convective tendency F_c (nodal), per component; rows of ``elems``."""
    vs = [_f64(x).reshape(-1) for x in v[: mesh.dim]]
    e, k, ep = _elems(elems)
    cnt = mesh.n_el if e is None else k
    outs = [np.zeros((cnt, mesh.npe)) for _ in range(mesh.dim)]
    vin = (_dp * 3)(*[_ptr(x) for x in vs] + [None] * (3 - mesh.dim))
    vout = (_dp * 3)(*[_ptr(x) for x in outs] + [None] * (3 - mesh.dim))
    if lib().oracle_convect(mesh.ref(), vin, vout, ep, k):
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
def _lagrange_matrix(P, xi, pts):
    """B[a, j] = l_j(pts[a]), dB[a, j] = l_j'(pts[a]) on the nodes xi (product formula)."""
    B = np.zeros((len(pts), P + 1))
    dB = np.zeros((len(pts), P + 1))
    for a, x in enumerate(pts):
        B[a], dB[a] = lagrange(P, xi, x)
    return B, dB


def broken_divergence_p1(mesh: Mesh, v):
    """Element-local (broken) collocation divergence of the nodal velocity v at the GLL
    nodes of degree P, interpolated to the GLL nodes of degree P-1, returned as
    [N_el, P^d] (pressure-mesh layout).  The stand-in Poisson rhs of SURVEY §8(a) a8:
    div v (x_q) = sum_d (2/h_d) sum_j l_j'(xi_{q_d}) v_d(.., x_j, ..) at the velocity nodes,
    then the degree-P interpolant evaluated at the degree-(P-1) nodes."""
    P, dim, n = mesh.P, mesh.dim, mesh.P + 1
    xi, _ = gll(P)
    xp, _ = gll(P - 1)
    _, Dm = _lagrange_matrix(P, xi, xi)        # Dm[i, j] = l_j'(xi_i)
    Ip, _ = _lagrange_matrix(P, xi, xp)        # Ip[a, j] = l_j(xp_a)
    shp = (mesh.n_el,) + (n,) * dim            # node axes (k, j, i): x last
    div = np.zeros(shp)
    for d in range(dim):
        vd = np.asarray(v[d], dtype=np.float64).reshape(shp)
        ax = dim - d                            # array axis of direction d
        div += (2.0 * mesh.N[d] / mesh.L[d]) * np.moveaxis(np.tensordot(Dm, vd, axes=([1], [ax])), 0, ax)
    for d in range(dim):
        ax = dim - d
        div = np.moveaxis(np.tensordot(Ip, div, axes=([1], [ax])), 0, ax)
    return div.reshape(mesh.n_el, P ** dim)


def imex_stage(mv: Mesh, mp: Mesh, dt, a_ex21, a_im21, a_im22, nu, v, tol=1e-14):
    """Alg. 3 stage i = 2, constant nu, F_s = 0, under the readings of
    include/dg.h dg_imex_stage: returns (vout[dim], psi, v').  Exact discrete solves
    (oracle PCG to tol)."""
    dim = mv.dim
    m = mass(mv)
    Fc = convect(mv, v)                                                     # F_c(v)
    Fd = [-sip_apply(mv, 0.0, v[c], nu_const=nu) / m for c in range(dim)]  # F_d1(v) = -M^-1 A_0 v
    vp = [np.asarray(v[c]) + dt * a_ex21 * (Fc[c] + Fd[c]) for c in range(dim)]         # line 4
    fp = -broken_divergence_p1(mv, vp)                                       # line 5 rhs: -div v'
    psi, *_ = pcg_solve(mp, 0.0, fp, nu_const=1.0, tol=tol)                 # line 5 (lam = 0)
    lam = 1.0 / (dt * a_im22)
    out = []
    for c in range(dim):
        g = vp[c] + dt * (a_im21 - a_ex21) * Fd[c]                          # line 8 (v'' = v')
        u, *_ = pcg_solve(mv, lam, lam * g, nu_const=nu, tol=tol)           # line 9
        out.append(u)
    return out, psi, vp
