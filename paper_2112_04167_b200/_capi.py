"""ctypes binding for libdgsip.so -- same names as include/dg.h, marshalling only.

Field arguments are torch tensors (CUDA, float64, contiguous) passed by ``data_ptr()``,
or raw integer device pointers.  Host variants take numpy float64 arrays.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("DG_LIBRARY", os.path.join(_HERE, "libdgsip.so"))

DG_OK, DG_EINVAL, DG_ECUDA, DG_ENCCL, DG_ENOMEM, DG_ENOTCONV, DG_EBREAKDOWN, DG_EUNSUPPORTED = range(8)
_NAMES = {0: "DG_OK", 1: "DG_EINVAL", 2: "DG_ECUDA", 3: "DG_ENCCL", 4: "DG_ENOMEM", 5: "DG_ENOTCONV",
          6: "DG_EBREAKDOWN", 7: "DG_EUNSUPPORTED"}

if not os.path.exists(_LIBPATH):
    raise ImportError(
        "libdgsip.so not found at %s -- build it with `python paper_2112_04167_b200/build.py` "
        "(there is no CPU fallback)" % _LIBPATH)

_lib = ctypes.CDLL(_LIBPATH)
_vp = ctypes.c_void_p
_d = ctypes.c_double
_i = ctypes.c_int
_ll = ctypes.c_longlong


class SolveInfo(ctypes.Structure):
    _fields_ = [("iters", _i), ("rel_res", _d), ("removed_mean", _d), ("f_norm", _d), ("kappa_est", _d)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class StageInfo(ctypes.Structure):
    _fields_ = [("pressure", SolveInfo), ("velocity", SolveInfo * 3), ("stab", SolveInfo)]

    def as_dict(self):
        return {"pressure": self.pressure.as_dict(), "velocity": [x.as_dict() for x in self.velocity],
                "stab": self.stab.as_dict()}


RK_MAX = 8


class Tableau(ctypes.Structure):
    _fields_ = [("s", _i), ("c", _d * RK_MAX), ("a_im", (_d * RK_MAX) * RK_MAX), ("a_ex", (_d * RK_MAX) * RK_MAX),
                ("b_im", _d * RK_MAX), ("b_ex", _d * RK_MAX)]

    @classmethod
    def from_dict(cls, t):
        tab = cls()
        s = len(t["c"])
        tab.s = s
        for i in range(s):
            tab.c[i] = float(t["c"][i])
            tab.b_im[i] = float(t["b_im"][i])
            tab.b_ex[i] = float(t["b_ex"][i])
            for j in range(s):
                tab.a_im[i][j] = float(t["a_im"][i][j])
                tab.a_ex[i][j] = float(t["a_ex"][i][j])
        return tab


class StepInfo(ctypes.Structure):
    _fields_ = [("stages", _i), ("pressure_iters", _i), ("velocity_iters", _i), ("stab_iters", _i)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ViscModel(ctypes.Structure):
    """nu(v) = nu0 + nu1 (|v| / vmax)^2."""
    _fields_ = [("nu0", _d), ("nu1", _d), ("vmax", _d)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_c = {
    "dg_nccl_unique_id": _sig("dg_nccl_unique_id", _i, [ctypes.c_char_p]),
    "dg_mesh_create": _sig("dg_mesh_create", _i, [_i, ctypes.POINTER(_i), ctypes.POINTER(_d), _i, _i, _i,
                                                  ctypes.c_char_p, _vp, ctypes.POINTER(_vp)]),
    "dg_mesh_destroy": _sig("dg_mesh_destroy", None, [_vp]),
    "dg_mesh_set_stream": _sig("dg_mesh_set_stream", _i, [_vp, _vp]),
    "dg_mesh_local_ndof": _sig("dg_mesh_local_ndof", _ll, [_vp]),
    "dg_mesh_local_elements": _sig("dg_mesh_local_elements", _ll, [_vp]),
    "dg_mesh_element_offset": _sig("dg_mesh_element_offset", _ll, [_vp]),
    "dg_mesh_launch_count": _sig("dg_mesh_launch_count", _ll, [_vp]),
    "dg_mesh_node_coords": _sig("dg_mesh_node_coords", _i, [_vp, _vp]),
    "dg_mesh_mass": _sig("dg_mesh_mass", _i, [_vp, _vp]),
    "dg_helmholtz_apply": _sig("dg_helmholtz_apply", _i, [_vp, _d, _vp, _d, _vp, _vp]),
    "dg_helmholtz_diag": _sig("dg_helmholtz_diag", _i, [_vp, _d, _vp, _d, _vp]),
    "dg_pcg_solve": _sig("dg_pcg_solve", _i, [_vp, _d, _vp, _d, _vp, _d, _i, _vp, ctypes.POINTER(SolveInfo)]),
    "dg_convect_rhs": _sig("dg_convect_rhs", _i, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "dg_last_apply_kernel": _sig("dg_last_apply_kernel", ctypes.c_char_p, []),
    "dg_derivative": _sig("dg_derivative", _i, [_vp, _vp, ctypes.POINTER(_vp)]),
    "dg_mesh_set_div_stab": _sig("dg_mesh_set_div_stab", _i, [_vp, _d, _d]),
    "dg_div_stab_apply": _sig("dg_div_stab_apply", _i, [_vp, _d, _d, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "dg_div_stab_solve": _sig("dg_div_stab_solve", _i, [_vp, _d, _d, _d, ctypes.POINTER(_vp), _d, _i,
                                                        ctypes.POINTER(_d), ctypes.POINTER(SolveInfo)]),
    "dg_imex_rk_step_vv": _sig("dg_imex_rk_step_vv", _i, [_vp, _vp, ctypes.POINTER(Tableau), _d,
                                                          ctypes.POINTER(ViscModel), ctypes.POINTER(_vp), _i,
                                                          ctypes.POINTER(_vp), _vp, _d, _i, ctypes.POINTER(StepInfo)]),
    "dg_mesh_set_precond": _sig("dg_mesh_set_precond", _i, [_vp, _i]),
    "dg_mesh_get_precond": _sig("dg_mesh_get_precond", _i, [_vp]),
    "dg_schwarz_apply": _sig("dg_schwarz_apply", _i, [_vp, _d, _d, _vp, _vp]),
    "dg_imex_rk_step": _sig("dg_imex_rk_step", _i, [_vp, _vp, ctypes.POINTER(Tableau), _d, _d, ctypes.POINTER(_vp),
                                                    _vp, _d, _i, ctypes.POINTER(StepInfo)]),
    "dg_divergence": _sig("dg_divergence", _i, [_vp, _vp, ctypes.POINTER(_vp), _vp]),
    "dg_gradient": _sig("dg_gradient", _i, [_vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "dg_imex_stage": _sig("dg_imex_stage", _i, [_vp, _vp, _d, _d, _d, _d, _d, ctypes.POINTER(_vp),
                                                ctypes.POINTER(_vp), _vp, _d, _i, ctypes.POINTER(StageInfo)]),
    "dg_helmholtz_apply_host": _sig("dg_helmholtz_apply_host", _i, [_vp, _d, _vp, _d, _vp, _vp]),
    "dg_pcg_solve_host": _sig("dg_pcg_solve_host", _i, [_vp, _d, _vp, _d, _vp, _d, _i, _vp,
                                                        ctypes.POINTER(SolveInfo)]),
    "dg_gll_tables": _sig("dg_gll_tables", _i, [_i, _vp, _vp, _vp]),
    "dg_check_field": _sig("dg_check_field", _i, [_vp, _vp, _i]),
    "dg_last_error": _sig("dg_last_error", ctypes.c_char_p, []),
    "dg_version": _sig("dg_version", ctypes.c_char_p, []),
}

EXPORTED = sorted(_c)


def library_path() -> str:
    return _LIBPATH


class DGError(RuntimeError):
    def __init__(self, status, msg, info=None):
        super().__init__("%s: %s" % (_NAMES.get(status, status), msg))
        self.status = status
        self.info = info


def dg_last_error() -> str:
    return _c["dg_last_error"]().decode()


def dg_version() -> str:
    return _c["dg_version"]().decode()


def _check(st, info=None, allow=()):
    if st != DG_OK and st not in allow:
        raise DGError(st, dg_last_error(), info)
    return st


def _ptr(x):
    """Device pointer of a torch tensor (checked) / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    import torch

    if not isinstance(x, torch.Tensor):
        raise TypeError("expected a torch tensor")
    if not x.is_cuda or x.dtype != torch.float64 or not x.is_contiguous():
        raise TypeError("fields must be contiguous CUDA float64 tensors")
    return x.data_ptr()


def _hptr(a):
    if a is None:
        return None
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise TypeError("host fields must be C-contiguous float64 numpy arrays")
    return a.ctypes.data


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Mesh:
    """Owning handle of a ``dg_mesh*``."""

    def __init__(self, handle, dim, N, L, P, rank, nranks):
        self._h = handle
        self.dim, self.N, self.L, self.P, self.rank, self.nranks = dim, tuple(N), tuple(L), P, rank, nranks

    @property
    def handle(self):
        if not self._h:
            raise DGError(DG_EINVAL, "mesh destroyed")
        return self._h

    @property
    def n(self):
        return self.P + 1

    @property
    def npe(self):
        return self.n ** self.dim

    @property
    def ndof(self):
        return dg_mesh_local_ndof(self)

    @property
    def n_el(self):
        return dg_mesh_local_elements(self)

    @property
    def element_offset(self):
        return dg_mesh_element_offset(self)

    def close(self):
        if self._h:
            dg_mesh_destroy(self)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dg_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_c["dg_nccl_unique_id"](buf))
    return buf.raw


def dg_mesh_create(dim, N, L, P, rank=0, nranks=1, nccl_uid=None, stream=None, halo_mode=False) -> Mesh:
    """halo_mode (one rank): route the slab-boundary faces through the NCCL face-trace exchange
    (a 1-rank communicator, self send/recv) instead of the local periodic wrap (dg.h)."""
    N3 = (list(N) + [1, 1, 1])[:3]
    L3 = (list(L) + [1.0, 1.0, 1.0])[:3]
    h = _vp()
    if halo_mode and nccl_uid is None:
        nccl_uid = dg_nccl_unique_id()
    uid = None if nccl_uid is None else bytes(nccl_uid)
    _check(_c["dg_mesh_create"](int(dim), (_i * 3)(*N3), (_d * 3)(*L3), int(P), int(rank), int(nranks), uid,
                                _stream_ptr(stream), ctypes.byref(h)))
    return Mesh(h.value, dim, N3[:dim], L3[:dim], P, rank, nranks)


def dg_mesh_destroy(m: Mesh):
    if m._h:
        _c["dg_mesh_destroy"](m._h)
        m._h = None


def dg_mesh_set_stream(m: Mesh, stream):
    _check(_c["dg_mesh_set_stream"](m.handle, _stream_ptr(stream)))


def dg_mesh_local_ndof(m: Mesh) -> int:
    return int(_c["dg_mesh_local_ndof"](m.handle))


def dg_mesh_local_elements(m: Mesh) -> int:
    return int(_c["dg_mesh_local_elements"](m.handle))


def dg_mesh_element_offset(m: Mesh) -> int:
    return int(_c["dg_mesh_element_offset"](m.handle))


def dg_mesh_launch_count(m: Mesh) -> int:
    return int(_c["dg_mesh_launch_count"](m.handle))


def dg_mesh_node_coords(m: Mesh, xyz):
    _check(_c["dg_mesh_node_coords"](m.handle, _ptr(xyz)))


def dg_mesh_mass(m: Mesh, mass):
    _check(_c["dg_mesh_mass"](m.handle, _ptr(mass)))


def dg_helmholtz_apply(m: Mesh, lam, nu, nu_const, u, out):
    _check(_c["dg_helmholtz_apply"](m.handle, float(lam), _ptr(nu), float(nu_const), _ptr(u), _ptr(out)))


def dg_helmholtz_diag(m: Mesh, lam, nu, nu_const, diag):
    _check(_c["dg_helmholtz_diag"](m.handle, float(lam), _ptr(nu), float(nu_const), _ptr(diag)))


def dg_pcg_solve(m: Mesh, lam, nu, nu_const, f, tol, maxit, u, raise_on_notconv=True) -> SolveInfo:
    info = SolveInfo()
    st = _c["dg_pcg_solve"](m.handle, float(lam), _ptr(nu), float(nu_const), _ptr(f), float(tol), int(maxit),
                            _ptr(u), ctypes.byref(info))
    _check(st, info, allow=() if raise_on_notconv else (DG_ENOTCONV,))
    return info


DG_PC_JACOBI = 0
DG_PC_SCHWARZ2 = 1


def dg_mesh_set_precond(m: Mesh, precond):
    """Preconditioner of later dg_pcg_solve calls on m: DG_PC_JACOBI or DG_PC_SCHWARZ2 -- include/dg.h."""
    _check(_c["dg_mesh_set_precond"](m.handle, int(precond)))


def dg_mesh_get_precond(m: Mesh) -> int:
    return int(_c["dg_mesh_get_precond"](m.handle))


def dg_schwarz_apply(m: Mesh, lam, nu_const, r, z):
    """z = B r, the two-level additive Schwarz preconditioner -- include/dg.h."""
    _check(_c["dg_schwarz_apply"](m.handle, float(lam), float(nu_const), _ptr(r), _ptr(z)))


def dg_convect_rhs(m: Mesh, v, out):
    vin = (_vp * 3)(*([_ptr(x) for x in v] + [None] * (3 - len(v))))
    vout = (_vp * 3)(*([_ptr(x) for x in out] + [None] * (3 - len(out))))
    _check(_c["dg_convect_rhs"](m.handle, vin, vout))


def dg_imex_rk_step(mv: Mesh, mp: Mesh, tableau, dt, nu, v, psi, tol, maxit) -> StepInfo:
    """One IMEX-RK step (Alg. 3) in place on v -- include/dg.h.  tableau: dict (tableaux.py) or Tableau."""
    tab = tableau if isinstance(tableau, Tableau) else Tableau.from_dict(tableau)
    vv = (_vp * 3)(*([_ptr(x) for x in v] + [None] * (3 - len(v))))
    info = StepInfo()
    _check(_c["dg_imex_rk_step"](mv.handle, mp.handle, ctypes.byref(tab), dt, nu, vv, _ptr(psi), tol, maxit,
                                 ctypes.byref(info)), info)
    return info


def dg_derivative(m: Mesh, u, out):
    """Velocity-level central-flux DG derivatives out[c] = D_c u (None skips c) -- include/dg.h."""
    o = (_vp * 3)(*([_ptr(x) for x in out] + [None] * (3 - len(out))))
    _check(_c["dg_derivative"](m.handle, _ptr(u), o))


def dg_last_apply_kernel() -> str:
    return _c["dg_last_apply_kernel"]().decode()


def dg_mesh_set_div_stab(mv: Mesh, zeta_D=1.0, zeta_C=1.0):
    """Divergence / mass-flux stabilisation of every projection on this velocity mesh -- dg.h."""
    _check(_c["dg_mesh_set_div_stab"](mv.handle, float(zeta_D), float(zeta_C)))


def dg_div_stab_apply(m: Mesh, a_D, a_C, v, out):
    vi = (_vp * 3)(*([_ptr(x) for x in v] + [None] * (3 - len(v))))
    vo = (_vp * 3)(*([_ptr(x) for x in out] + [None] * (3 - len(out))))
    _check(_c["dg_div_stab_apply"](m.handle, float(a_D), float(a_C), vi, vo))


def dg_div_stab_solve(m: Mesh, dt, zeta_D, zeta_C, v, tol=1e-12, maxit=2000):
    """v (in: v'', out: v^) in place; returns (SolveInfo, (a_D, a_C, U)) -- dg.h."""
    vi = (_vp * 3)(*([_ptr(x) for x in v] + [None] * (3 - len(v))))
    coef = (_d * 3)()
    info = SolveInfo()
    _check(_c["dg_div_stab_solve"](m.handle, float(dt), float(zeta_D), float(zeta_C), vi, float(tol), int(maxit),
                                   coef, ctypes.byref(info)), info)
    return info, (coef[0], coef[1], coef[2])


def dg_imex_rk_step_vv(mv: Mesh, mp: Mesh, tableau, dt, visc, v, psi, tol, maxit, fs=None, final_projection=True):
    """One IMEX-RK step (Alg. 3) with nu(v) = nu0 + nu1 (|v|/vmax)^2, forcing fs[j][c] (device
    tensors at t + c_j dt, or None) and the final projection, in place on v -- include/dg.h."""
    tab = tableau if isinstance(tableau, Tableau) else Tableau.from_dict(tableau)
    vm = ViscModel(*[float(x) for x in visc])
    vv = (_vp * 3)(*([_ptr(x) for x in v] + [None] * (3 - len(v))))
    fsp = None
    if fs is not None:
        flat = [_ptr(fs[j][c]) for j in range(len(fs)) for c in range(len(v))]
        fsp = (_vp * len(flat))(*flat)
    info = StepInfo()
    _check(_c["dg_imex_rk_step_vv"](mv.handle, mp.handle, ctypes.byref(tab), float(dt), ctypes.byref(vm), fsp,
                                    int(bool(final_projection)), vv, _ptr(psi), float(tol), int(maxit),
                                    ctypes.byref(info)), info)
    return info


def dg_divergence(mv: Mesh, mp: Mesh, v, div_weak):
    """Weak DG divergence of v (velocity mesh) tested with the pressure basis -- include/dg.h."""
    vin = (_vp * 3)(*([_ptr(x) for x in v] + [None] * (3 - len(v))))
    _check(_c["dg_divergence"](mv.handle, mp.handle, vin, _ptr(div_weak)))


def dg_gradient(mp: Mesh, mv: Mesh, psi, grad_weak):
    """Weak DG gradient of psi (pressure mesh) tested with the velocity basis -- include/dg.h."""
    go = (_vp * 3)(*([_ptr(x) for x in grad_weak] + [None] * (3 - len(grad_weak))))
    _check(_c["dg_gradient"](mp.handle, mv.handle, _ptr(psi), go))


def dg_imex_stage(mv: Mesh, mp: Mesh, dt, a_ex21, a_im21, a_im22, nu, v, vout, psi, tol, maxit) -> StageInfo:
    """One IMEX-RK stage (Alg. 3 lines 4-9) -- see include/dg.h."""
    vin = (_vp * 3)(*([_ptr(x) for x in v] + [None] * (3 - len(v))))
    vo = (_vp * 3)(*([_ptr(x) for x in vout] + [None] * (3 - len(vout))))
    info = StageInfo()
    _check(_c["dg_imex_stage"](mv.handle, mp.handle, dt, a_ex21, a_im21, a_im22, nu, vin, vo, _ptr(psi), tol, maxit,
                               ctypes.byref(info)), info)
    return info


def dg_helmholtz_apply_host(m: Mesh, lam, nu, nu_const, u, out):
    _check(_c["dg_helmholtz_apply_host"](m.handle, float(lam), _hptr(nu), float(nu_const), _hptr(u), _hptr(out)))


def dg_pcg_solve_host(m: Mesh, lam, nu, nu_const, f, tol, maxit, u) -> SolveInfo:
    info = SolveInfo()
    _check(_c["dg_pcg_solve_host"](m.handle, float(lam), _hptr(nu), float(nu_const), _hptr(f), float(tol),
                                   int(maxit), _hptr(u), ctypes.byref(info)), info)
    return info


def dg_gll_tables(P):
    xi = np.zeros(P + 1)
    w = np.zeros(P + 1)
    D = np.zeros((P + 1, P + 1))
    _check(_c["dg_gll_tables"](int(P), xi.ctypes.data, w.ctypes.data, D.ctypes.data))
    return xi, w, D


def dg_check_field(m: Mesh, x, positive=True):
    _check(_c["dg_check_field"](m.handle, _ptr(x), int(bool(positive))))


