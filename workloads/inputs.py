"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json ``configs``).

Nothing here computes any part of the method.  The only numerics are:

* node positions used to SAMPLE analytic fields (x = e*h + (xi+1)*h/2), where the
  GLL abscissae xi come from numpy's Legendre module (roots of P_P'), a library
  primitive independent of both the oracle's and the CUDA path's own tables;
* numpy PCG64 streams seeded with ``[20211208, cfg, field]``.

Layout of every nodal array: canonical global order ``[N_el][n^d]`` with element
index ``e = ex + Nx*(ey + Ny*ez)`` (z slowest) and node index ``i + n*(j + n*k)``
(x fastest) -- SURVEY.md §8(a) row a2.

Paper workloads these stand in for:
  c1  laminar traveling Taylor-Green, 2D, coarse
  c2  variable viscosity, 2D
  c3  transition Taylor-Green DNS at Re 1600, coarse
  c4  one IMEX-RK stage of the TG DNS: 32^3 hexes as in PAPER.md:1474
  c5  variable-viscosity vortex scaled up
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED0 = 20211208
GAMMA_SDIRK3 = 0.4358665  # BASELINE.json configs[1..2]; SURVEY.md §8(c) A11


def rng(cfg: int, field: int) -> np.random.Generator:
    """PCG64 stream for (config, field) -- SURVEY.md §8(d) 'Seeds'."""
    return np.random.default_rng([SEED0, cfg, field])


def gll_points_for_sampling(P: int) -> np.ndarray:
    """GLL abscissae on [-1,1] for sampling analytic input fields only.

    Uses numpy's Legendre class (companion-matrix roots of P_P'), i.e. a library
    routine, so that input generation shares no code with either implementation.
    """
    if P < 1:
        raise ValueError("P must be >= 1")
    inner = np.polynomial.legendre.Legendre.basis(P).deriv().roots() if P > 1 else np.array([])
    return np.concatenate([[-1.0], np.sort(np.real(inner)), [1.0]])


def node_coords(dim: int, N, L, P: int):
    """Physical coordinates of every node, canonical global order.

    Returns a list of ``dim`` float64 arrays of shape ``[N_el, n^dim]``.
    """
    N = list(N)[:dim]
    L = list(L)[:dim]
    n = P + 1
    xi = gll_points_for_sampling(P)
    out = []
    for d in range(dim):
        h = L[d] / N[d]
        # 1-D coordinates of (element index along d, node index along d)
        c1 = (np.arange(N[d])[:, None] * h + (xi[None, :] + 1.0) * 0.5 * h)  # [N_d, n]
        # place into axes [ez, ey, ex, k, j, i] (element axes slow..fast, then node axes)
        shape = [1] * (2 * dim)
        shape[dim - 1 - d] = N[d]
        shape[2 * dim - 1 - d] = n
        full = np.broadcast_to(c1.reshape(shape), tuple(N[::-1]) + (n,) * dim)
        out.append(np.ascontiguousarray(full).reshape(int(np.prod(N)), n ** dim))
    return out


def uniform_field(cfg: int, field: int, shape, lo=-1.0, hi=1.0) -> np.ndarray:
    return rng(cfg, field).uniform(lo, hi, size=shape)


@dataclasses.dataclass(frozen=True)
class Config:
    cid: int
    name: str
    dim: int
    N: tuple
    L: tuple
    P: int
    P_p: int            # pressure degree, P-1
    lam: float          # Helmholtz lambda
    nu0: float          # constant viscosity (or scale of the variable one)
    variable_nu: bool
    tol: float
    shaped_like: str

    @property
    def n(self) -> int:
        return self.P + 1

    @property
    def n_el(self) -> int:
        return int(np.prod(self.N[: self.dim]))

    @property
    def ndof(self) -> int:
        return self.n_el * self.n ** self.dim

    def coords(self, P=None):
        return node_coords(self.dim, self.N, self.L, self.P if P is None else P)

    # ---- fields -------------------------------------------------------------
    def nu(self):
        """Nodal viscosity [N_el, n^d] or None for constant nu (= self.nu0)."""
        if not self.variable_nu:
            return None
        X = self.coords()
        if self.cid == 2:   # nu = 0.01 (1 + 0.5 sin x cos y)      (BASELINE configs[1])
            return self.nu0 * (1.0 + 0.5 * np.sin(X[0]) * np.cos(X[1]))
        if self.cid == 5:   # nu = nu0 (1 + 0.5 tanh(4 sin x sin y sin z))  (configs[4])
            return self.nu0 * (1.0 + 0.5 * np.tanh(4.0 * np.sin(X[0]) * np.sin(X[1]) * np.sin(X[2])))
        raise ValueError("no variable nu for config %d" % self.cid)

    def apply_input(self):
        """Seeded U[-1,1] DOF vector for the apply benchmarks (field 0)."""
        return uniform_field(self.cid, 0, (self.n_el, self.n ** self.dim))

    def rhs(self, comp: int = 0):
        """Nodal right-hand side f for the Helmholtz solve of component ``comp``."""
        if self.cid == 1:   # f from manufactured u = sin x sin y: f = (lam + 2 nu) u
            X = self.coords()
            return (self.lam + 2.0 * self.nu0) * np.sin(X[0]) * np.sin(X[1])
        return uniform_field(self.cid, 10 + comp, (self.n_el, self.n ** self.dim))

    # ---- rank slabs (multi-GPU): the same values as the global arrays' slices ----------
    def _slab_uniform(self, field: int, el_off: int, nel: int, npe: int):
        g = rng(self.cid, field)
        g.bit_generator.advance(int(el_off) * npe)  # PCG64 draws one 64-bit word per double
        return g.uniform(-1.0, 1.0, size=(nel, npe))

    def coords_slab(self, el_off: int, nel: int, P=None):
        """Node coordinates of the global elements [el_off, el_off + nel) (canonical order)."""
        P = self.P if P is None else P
        n = P + 1
        xi = gll_points_for_sampling(P)
        N = list(self.N[: self.dim])
        e = np.arange(el_off, el_off + nel)
        ec = [e % N[0], (e // N[0]) % N[1]] + ([e // (N[0] * N[1])] if self.dim == 3 else [])
        out = []
        for d in range(self.dim):
            h = self.L[d] / N[d]
            shape = [nel] + [1] * self.dim
            shape[self.dim - d] = n            # node axes (k, j, i): x fastest
            loc = ((xi + 1.0) * 0.5 * h).reshape(shape[1:])
            x = ec[d].reshape([nel] + [1] * self.dim) * h + loc[None]
            out.append(np.ascontiguousarray(np.broadcast_to(x, [nel] + [n] * self.dim)).reshape(nel, n ** self.dim))
        return out

    def apply_input_slab(self, el_off: int, nel: int):
        return self._slab_uniform(0, el_off, nel, self.n ** self.dim)

    def rhs_slab(self, comp: int, el_off: int, nel: int):
        if self.cid == 1:
            X = self.coords_slab(el_off, nel)
            return (self.lam + 2.0 * self.nu0) * np.sin(X[0]) * np.sin(X[1])
        return self._slab_uniform(10 + comp, el_off, nel, self.n ** self.dim)

    def nu_slab(self, el_off: int, nel: int):
        if not self.variable_nu:
            return None
        X = self.coords_slab(el_off, nel)
        if self.cid == 2:
            return self.nu0 * (1.0 + 0.5 * np.sin(X[0]) * np.cos(X[1]))
        if self.cid == 5:
            return self.nu0 * (1.0 + 0.5 * np.tanh(4.0 * np.sin(X[0]) * np.sin(X[1]) * np.sin(X[2])))
        raise ValueError("no variable nu for config %d" % self.cid)

    def poisson_rhs_raw(self):
        """Seeded U[-1,1] Poisson rhs on the pressure mesh (mass-mean removed by the solver)."""
        n_p = self.P_p + 1
        return uniform_field(self.cid, 20, (self.n_el, n_p ** self.dim))

    def tg_velocity(self, noise: float = 1e-3):
        """Config 4: u = (sin x cos y cos z, -cos x sin y cos z, 0) + noise*U[-1,1] per component."""
        X = self.coords()
        v0 = np.sin(X[0]) * np.cos(X[1]) * np.cos(X[2])
        v1 = -np.cos(X[0]) * np.sin(X[1]) * np.cos(X[2])
        v2 = np.zeros_like(v0)
        out = []
        for c, v in enumerate((v0, v1, v2)):
            out.append(v + noise * uniform_field(self.cid, c, v.shape))
        return out


TWO_PI = 2.0 * math.pi
LAM_3 = 1.0 / (GAMMA_SDIRK3 * 1e-2)   # 229.43

CONFIGS = {
    1: Config(1, "c1-2d-4x4-P4", 2, (4, 4, 1), (TWO_PI,) * 3, 4, 3, 1.0, 1.0, False, 1e-11,
              "laminar traveling TG 2D (PAPER.md:1089-1125), coarse"),
    2: Config(2, "c2-2d-32x32-P8-varnu", 2, (32, 32, 1), (TWO_PI,) * 3, 8, 7,
              1.0 / (GAMMA_SDIRK3 * 1e-3), 0.01, True, 1e-11,
              "variable viscosity (PAPER.md:1189-1244), 2D"),
    3: Config(3, "c3-3d-16^3-P7", 3, (16, 16, 16), (TWO_PI,) * 3, 7, 6, LAM_3, 1.0 / 1600.0, False, 1e-10,
              "TG transition DNS Re=1600 (PAPER.md:1449-1483), coarse"),
    4: Config(4, "c4-3d-32^3-P7-stage", 3, (32, 32, 32), (TWO_PI,) * 3, 7, 6, LAM_3, 1.0 / 1600.0, False, 1e-10,
              "one IMEX-RK stage of the TG DNS, 32^3 hexes (PAPER.md:1474)"),
    5: Config(5, "c5-3d-64^3-P5-varnu", 3, (64, 64, 64), (TWO_PI,) * 3, 5, 4, LAM_3, 1e-3, True, 1e-10,
              "variable-viscosity vortex (PAPER.md:1189-1244), scaled up"),
}


def config(cid: int) -> Config:
    return CONFIGS[cid]


# ---------------------------------------------------------------------------
# 3-D vortex with solution-dependent viscosity, case VVP: the paper's
# closed-form exact solution, viscosity model and manufactured forcing, sampled at nodes.
# (Input data of the convergence experiment; none of the method's discrete arithmetic.)
# ---------------------------------------------------------------------------
VVP_VMAX = 2.0  # v^ex_max


def vvp_exact(X, t):
    """(v^ex, p^ex) of eq. var-visc-test at coordinates X = (x, y, z)."""
    k = 2.0 * math.pi
    A, B, C = k * (X[0] + t), k * (X[1] + t), k * (X[2] + t)
    v = [(np.sin(A) + np.cos(B)) * np.sin(C),
         (np.cos(A) + np.sin(B)) * np.sin(C),
         (np.cos(A) + np.cos(B)) * np.cos(C)]
    p = np.sin(A) * np.sin(B) * np.sin(C)
    return v, p


def vvp_forcing(X, t, nu0, nu1, vmax=VVP_VMAX):
    """f = d_t v + div(v v) - div[nu(v) (grad v + grad v^T)] + grad p for the exact VVP solution
    (PAPER.md:1229-1239), nu(v) = nu0 + nu1 (|v|/vmax)^2, in closed form:
    with the phases A, B, C = 2 pi (x + t, y + t, z + t): div v = 0, lap v = -2 (2 pi)^2 v,
    d_t = d_x + d_y + d_z, div(v v) = (v . grad) v, div[nu S] = nu lap v + S grad nu."""
    k = 2.0 * math.pi
    A, B, C = k * (X[0] + t), k * (X[1] + t), k * (X[2] + t)
    sA, cA, sB, cB, sC, cC = np.sin(A), np.cos(A), np.sin(B), np.cos(B), np.sin(C), np.cos(C)
    v, _ = vvp_exact(X, t)
    # G[c][e] = d_e v_c
    G = [[k * cA * sC, -k * sB * sC, k * (sA + cB) * cC],
         [-k * sA * sC, k * cB * sC, k * (cA + sB) * cC],
         [-k * sA * cC, -k * sB * cC, -k * (cA + cB) * sC]]
    gp = [k * cA * sB * sC, k * sA * cB * sC, k * sA * sB * cC]
    nu = nu0 + nu1 * (v[0] ** 2 + v[1] ** 2 + v[2] ** 2) / vmax ** 2
    gnu = [2.0 * nu1 / vmax ** 2 * sum(v[c] * G[c][e] for c in range(3)) for e in range(3)]
    f = []
    for c in range(3):
        dt_v = G[c][0] + G[c][1] + G[c][2]
        conv = sum(v[e] * G[c][e] for e in range(3))
        visc = nu * (-2.0 * k * k * v[c]) + sum(gnu[e] * (G[c][e] + G[e][c]) for e in range(3))
        f.append(dt_v + conv - visc + gp[c])
    return f
