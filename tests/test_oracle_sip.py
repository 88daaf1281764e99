"""Pins for the oracle's SIP-DG operator, diagonal and solve.

The operator is the symmetric interior-penalty DG form for lam*u - div(nu grad u)
("interior penalty method for pressure and viscous diffusion";
Alg. 3 lines 5 and 9) on GLL tensor-product elements,
with the readings A1-A8 listed in DESIGN.md.  Every check below is pinned to something
other than the oracle's own apply routine: a brute-force dense assembly that evaluates
the full tensor-product basis at every quadrature point, closed forms (critical penalty,
polynomial reproduction, the Laplacian spectrum k^2, manufactured solutions), invariants
(symmetry, null space), or LAPACK (numpy.linalg).
"""
import itertools
import math

import numpy as np
import pytest

import oracle

TWO_PI = 2 * math.pi


def mesh(dim, N, P, L=TWO_PI):
    return oracle.Mesh(dim, N, [L] * 3 if np.isscalar(L) else L, P)


def coords(m):
    """Node coordinates from the oracle's GLL nodes (test helper)."""
    xi, _ = oracle.gll(m.P)
    n = m.n
    out = []
    for d in range(m.dim):
        h = m.L[d] / m.N[d]
        c1 = np.arange(m.N[d])[:, None] * h + (xi[None, :] + 1) * h / 2
        shape = [1] * (2 * m.dim)
        shape[m.dim - 1 - d] = m.N[d]
        shape[2 * m.dim - 1 - d] = n
        full = np.broadcast_to(c1.reshape(shape), tuple(m.N[: m.dim][::-1]) + (n,) * m.dim)
        out.append(np.ascontiguousarray(full).reshape(m.n_el, m.npe))
    return out


def rand_nu(m, seed=3):
    X = coords(m)
    nu = 1.0 + 0.4 * np.sin(X[0] + 0.3) * np.cos(X[1] - 0.2)
    if m.dim == 3:
        nu = nu * (1.0 + 0.3 * np.sin(X[2]))
    return 0.05 * nu


# ---------------------------------------------------------------------------
# Q11: brute-force dense agreement (explicit all-triples assembly)
# ---------------------------------------------------------------------------
CASES_2X2 = [(2, (2, 2), P) for P in (1, 2, 3, 4, 6, 8)] + [(3, (2, 2, 2), P) for P in (1, 2, 3)]


@pytest.mark.parametrize("dim,N,P", CASES_2X2)
@pytest.mark.parametrize("varnu", [False, True])
def test_apply_matches_dense_bruteforce(dim, N, P, varnu):
    m = mesh(dim, N, P)
    nu = rand_nu(m) if varnu else None
    lam = 2.5
    A = oracle.sip_dense(m, lam, nu=nu, nu_const=0.7)
    rng = np.random.default_rng(7)
    for _ in range(3):
        u = rng.uniform(-1, 1, m.ndof)
        y = oracle.sip_apply(m, lam, u, nu=nu, nu_const=0.7).reshape(-1)
        ref = A @ u
        assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    # diagonal (a different evaluation: quadratic form with full tensor basis)
    d = oracle.sip_diag(m, lam, nu=nu, nu_const=0.7).reshape(-1)
    assert np.abs(d - np.diag(A)).max() <= 1e-13 * np.abs(np.diag(A)).max()


@pytest.mark.parametrize("dim,N,P", [(2, (1, 1), 3), (2, (1, 3), 2), (2, (3, 2), 3), (3, (1, 2, 1), 2),
                                     (3, (3, 1, 2), 1), (2, (2, 1), 5)])
def test_apply_dense_self_and_double_adjacency(dim, N, P):
    """N=1 (element is its own neighbour) and N=2 (two faces, same neighbour)."""
    m = mesh(dim, N, P, L=[1.3, 2.1, 0.9])
    nu = rand_nu(m)
    A = oracle.sip_dense(m, 0.8, nu=nu)
    U = np.eye(m.ndof)
    Y = np.stack([oracle.sip_apply(m, 0.8, U[:, j], nu=nu).reshape(-1) for j in range(m.ndof)], axis=1)
    assert np.abs(Y - A).max() <= 1e-13 * np.abs(A).max()
    d = oracle.sip_diag(m, 0.8, nu=nu).reshape(-1)
    assert np.abs(d - np.diag(A)).max() <= 1e-13 * np.abs(A).max()


# ---------------------------------------------------------------------------
# Q3 / Q4 / Q5: symmetry, null space, coercivity
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dim,N,P", [(2, (2, 2), 3), (2, (3, 2), 4), (2, (1, 1), 2), (3, (2, 2, 2), 2),
                                     (2, (4, 3), 2)])
@pytest.mark.parametrize("varnu", [False, True])
def test_symmetric_psd_nullspace(dim, N, P, varnu):
    m = mesh(dim, N, P)
    nu = rand_nu(m) if varnu else None
    A0 = oracle.sip_dense(m, 0.0, nu=nu)
    assert np.abs(A0 - A0.T).max() <= 1e-15 * np.abs(A0).max() * 10
    # lam = 0: A 1 = 0 and null space exactly span{1}
    one = np.ones(m.ndof)
    assert np.abs(A0 @ one).max() <= 1e-13 * np.abs(A0).max()
    ev = np.linalg.eigvalsh(0.5 * (A0 + A0.T))
    scale = ev[-1]
    assert abs(ev[0]) <= 1e-12 * scale
    assert ev[1] > 1e-8 * scale
    # lam > 0: SPD
    A1 = oracle.sip_dense(m, 1.0, nu=nu)
    assert np.linalg.eigvalsh(0.5 * (A1 + A1.T))[0] > 0


def line_operator(Nx, P, L, nu=1.0):
    """1-D SIP line operator K (N n x N n), extracted from the 2-D oracle with N_y = 1 and
    u = g(x) (x) 1(y):  A(g (x) 1) = m^y_j (K g)  at lam = 0 (transverse weight m^y_j)."""
    m = oracle.Mesh(2, (Nx, 1), (L, 1.0), P)
    n = P + 1
    _, w = oracle.gll(P)
    my = w * 1.0 / 2.0
    K = np.zeros((Nx * n, Nx * n))
    for col in range(Nx * n):
        g = np.zeros(Nx * n)
        g[col] = 1.0
        u = np.zeros((Nx, n, n))  # [ex][j][i]
        u[:] = g.reshape(Nx, 1, n)
        y = oracle.sip_apply(m, 0.0, u.reshape(Nx, n * n), nu_const=nu).reshape(Nx, n, n)
        for j in range(n):  # every transverse node gives the same K g
            np.testing.assert_allclose(y[:, j, :] / my[j], y[:, 0, :] / my[0], rtol=1e-12, atol=1e-12)
        K[:, col] = (y[:, 0, :] / my[0]).reshape(-1)
    return K


def mass_1d(Nx, P, L):
    _, w = oracle.gll(P)
    return np.tile(w * (L / Nx) / 2, Nx)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 6, 7, 8])
def test_critical_penalty_1d(P):
    """Q5: in 1-D the SIP form (GLL collocation) is PSD iff tau >= P(P+1)/(2h)
    (GLL trace inequality w_0 a_0^2 <= sum_k w_k a_k^2 with w_0 = 2/(P(P+1))); the bound is
    attained by the alternating Bloch mode, so N must be even.
    The oracle uses tau = (P+1)^2/h; strip that penalty, then probe +-0.1 % around tau_c."""
    Nx, L = 4, 2.0
    h = L / Nx
    n = P + 1
    K = line_operator(Nx, P, L)
    S = np.zeros_like(K)  # sum_F [phi][phi]^T, built independently from the node layout
    for e in range(Nx):
        jv = np.zeros(Nx * n)
        jv[e * n + P] += 1.0
        jv[((e + 1) % Nx) * n + 0] -= 1.0
        S += np.outer(jv, jv)
    tau = (P + 1) ** 2 / h
    K0 = K - tau * S

    def eigs(t):
        return np.linalg.eigvalsh(K0 + t * S)

    tc = P * (P + 1) / (2 * h)
    above, below = eigs(1.001 * tc), eigs(0.999 * tc)
    scale = above[-1]
    assert abs(above[0]) < 1e-12 * scale and above[1] > 0  # PSD, null space = constants
    assert below[0] < -1e-10 * scale                      # indefinite just below tau_c


def test_line_separability_kronecker():
    """Q7: constant nu: A = lam My(x)Mx + My(x)Kx + Ky(x)Mx (2-D), independent of how the
    apply loops are organised."""
    P, Nx, Ny, Lx, Ly, lam, nu = 3, 3, 2, 2.0, 1.5, 0.7, 1.3
    n = P + 1
    Kx = line_operator(Nx, P, Lx, nu)
    Ky = line_operator(Ny, P, Ly, nu)
    Mx, My = np.diag(mass_1d(Nx, P, Lx)), np.diag(mass_1d(Ny, P, Ly))
    Akron = lam * np.kron(My, Mx) + np.kron(My, Kx) + np.kron(Ky, Mx)
    m = oracle.Mesh(2, (Nx, Ny), (Lx, Ly, 1.0), P)
    A = oracle.sip_dense(m, lam, nu_const=nu)
    # permutation: our index (e = ex + Nx ey) * n^2 + i + n j  <->  (ey n + j) * (Nx n) + ex n + i
    perm = np.zeros(m.ndof, dtype=int)
    for ey, ex, j, i in itertools.product(range(Ny), range(Nx), range(n), range(n)):
        ours = (ex + Nx * ey) * n * n + i + n * j
        perm[ours] = (ey * n + j) * (Nx * n) + ex * n + i
    B = Akron[np.ix_(perm, perm)]
    assert np.abs(A - B).max() <= 1e-13 * np.abs(A).max()


@pytest.mark.parametrize("P,N", [(5, 7), (4, 6), (7, 4)])
def test_laplacian_spectrum_k2(P, N):
    """Q9: low eigenvalues of M^-1 K on [0, 2pi] approximate k^2 = 0,1,1,4,4,9,9."""
    K = line_operator(N, P, TWO_PI)
    m = mass_1d(N, P, TWO_PI)
    Ms = 1.0 / np.sqrt(m)
    ev = np.sort(np.linalg.eigvalsh(Ms[:, None] * K * Ms[None, :]))
    expect = np.array([0, 1, 1, 4, 4, 9, 9], dtype=float)
    assert abs(ev[0]) < 1e-11
    np.testing.assert_allclose(ev[1:7], expect[1:], rtol=2e-3)


def test_bloch_symbol_1d():
    """Q8: block-circulant structure -> eig(M^-1 K) = union over theta of the Bloch blocks."""
    P, N, L = 4, 6, TWO_PI
    n = P + 1
    K = line_operator(N, P, L)
    m = mass_1d(N, P, L)
    K0 = K[n:2 * n, n:2 * n]
    Kp = K[n:2 * n, 2 * n:3 * n]
    Km = K[n:2 * n, 0:n]
    assert np.abs(K[n:2 * n, 3 * n:]).max() == 0.0  # nearest-neighbour coupling only
    ms = m[:n]
    ev_bloch = []
    for jt in range(N):
        th = 2 * math.pi * jt / N
        Kt = K0 + Kp * np.exp(1j * th) + Km * np.exp(-1j * th)
        ev_bloch.extend(np.linalg.eigvalsh((Kt / np.sqrt(ms)[:, None]) / np.sqrt(ms)[None, :]))
    Ms = 1.0 / np.sqrt(m)
    ev = np.linalg.eigvalsh(Ms[:, None] * K * Ms[None, :])
    np.testing.assert_allclose(np.sort(ev), np.sort(np.real(ev_bloch)), atol=1e-10 * ev.max())


# ---------------------------------------------------------------------------
# Q6: polynomial reproduction away from the periodic seam
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dim,P", [(2, 3), (2, 5), (2, 7), (3, 3), (3, 4)])
def test_polynomial_reproduction(dim, P):
    N = [4] * dim
    L = [1.0, 1.4, 0.8][:dim]
    m = oracle.Mesh(dim, N, L + [1.0] * (3 - dim), P)
    X = coords(m)
    rng = np.random.default_rng(11)
    Pol = np.polynomial.Polynomial
    lam = 1.7
    # u = prod_d a_d(x_d), deg a_d = P-1 ; nu = prod_d b_d(x_d), deg b_d = 2  (deg sum = P+1)
    a = [Pol(rng.uniform(-1, 1, P)) for _ in range(dim)]
    b = [Pol([1.0, 0.2 * rng.uniform(-1, 1), 0.1 * rng.uniform(-1, 1)]) for _ in range(dim)]
    cen = [l / 2 for l in L]
    ev = lambda p, d: p(X[d] - cen[d])
    u = np.prod([ev(a[d], d) for d in range(dim)], axis=0)
    nu = np.prod([ev(b[d], d) for d in range(dim)], axis=0)
    div = np.zeros_like(u)
    for d in range(dim):
        term = ev((b[d] * a[d].deriv()).deriv(), d)
        for dd in range(dim):
            if dd != d:
                term = term * ev(b[dd] * a[dd], dd)
        div += term
    strong = lam * u - div
    y = oracle.sip_apply(m, lam, u, nu=nu)
    mass = oracle.mass(m)
    # elements whose closure avoids the seam: 1 <= e_d <= N_d - 2
    ok = []
    for e in range(m.n_el):
        ec = [e % N[0], (e // N[0]) % N[1]] + ([e // (N[0] * N[1])] if dim == 3 else [])
        if all(1 <= c <= N[d] - 2 for d, c in enumerate(ec)):
            ok.append(e)
    ok = np.array(ok)
    ref = mass[ok] * strong[ok]
    err = np.abs(y[ok] - ref).max() / np.abs(ref).max()
    assert err < 1e-11, err
    # and it must FAIL when deg nu + deg u = P + 2 (guards against a vacuous test)
    b2 = [Pol([1.0, 0.2, 0.1, 0.3]) for _ in range(dim)]
    nu2 = np.prod([ev(b2[d], d) for d in range(dim)], axis=0)
    div2 = np.zeros_like(u)
    for d in range(dim):
        term = ev((b2[d] * a[d].deriv()).deriv(), d)
        for dd in range(dim):
            if dd != d:
                term = term * ev(b2[dd] * a[dd], dd)
        div2 += term
    y2 = oracle.sip_apply(m, lam, u, nu=nu2)
    ref2 = mass[ok] * (lam * u - div2)[ok]
    assert np.abs(y2[ok] - ref2).max() / np.abs(ref2).max() > 1e-9


# ---------------------------------------------------------------------------
# Q12 / Q13 / Q14: solves
# ---------------------------------------------------------------------------
def test_pcg_matches_lapack_dense():
    m = mesh(2, (3, 2), 4)
    nu = rand_nu(m)
    lam = 3.0
    f = np.random.default_rng(5).uniform(-1, 1, m.ndof)
    A = oracle.sip_dense(m, lam, nu=nu)
    b = oracle.mass(m).reshape(-1) * f
    ref = np.linalg.solve(A, b)
    for pre in (True, False):
        u, it, rr, _, st = oracle.pcg_solve(m, lam, f, nu=nu, tol=1e-14, precond=pre)
        assert st == 0 or rr < 1e-13
        assert np.linalg.norm(u.reshape(-1) - ref) <= 1e-12 * np.linalg.norm(ref)


def test_pcg_poisson_nullspace():
    """lam = 0 (Alg. 3 line 5, periodic): f projected to zero mass-mean, u zero mass-mean."""
    m = mesh(3, (2, 2, 2), 2)
    f = np.random.default_rng(6).uniform(-1, 1, m.ndof)
    mass = oracle.mass(m).reshape(-1)
    u, it, rr, rm, st = oracle.pcg_solve(m, 0.0, f, tol=1e-13)
    assert abs(rm - (mass @ f) / mass.sum()) < 1e-15
    assert abs(mass @ u.reshape(-1)) < 1e-13 * np.abs(u).max() * mass.sum()
    A = oracle.sip_dense(m, 0.0)
    fp = f - rm
    # pseudo-inverse solution, then zero mass-mean (LAPACK lstsq)
    ref = np.linalg.lstsq(A, mass * fp, rcond=1e-12)[0]
    ref -= (mass @ ref) / mass.sum()
    assert np.linalg.norm(u.reshape(-1) - ref) <= 1e-10 * np.linalg.norm(ref)


def mms_error(dim, N, P, lam=1.0, nu=1.0):
    m = mesh(dim, [N] * dim, P)
    X = coords(m)
    uex = np.prod([np.sin(X[d]) for d in range(dim)], axis=0)
    f = (lam + dim * nu) * uex
    u, it, rr, _, st = oracle.pcg_solve(m, lam, f, nu_const=nu, tol=1e-13)
    return math.sqrt(np.mean((u - uex) ** 2)), m


@pytest.mark.parametrize("dim,P,Ns", [(2, 2, (4, 8, 16)), (2, 3, (4, 8, 16)), (2, 4, (4, 8)), (3, 2, (2, 4, 8))])
def test_mms_convergence_order(dim, P, Ns):
    """Q12: u = sin x sin y (sin z), f = (lam + d nu) u: nodal RMS error EOC >= P+1 - 0.2."""
    errs = [mms_error(dim, N, P)[0] for N in Ns]
    eoc = [math.log(errs[i] / errs[i + 1]) / math.log(Ns[i + 1] / Ns[i]) for i in range(len(Ns) - 1)]
    assert eoc[-1] >= P + 1 - 0.2, (errs, eoc)


def test_single_fourier_mode_closed_form():
    """Q13 (SPEC.md:440 analogue): lam u - nu lap u = sin(k.x) -> sin(k.x)/(lam + nu|k|^2)."""
    P, N = 6, 4
    m = mesh(2, (N, N), P)
    X = coords(m)
    k = (2, 1)
    lam, nu = 0.5, 0.3
    g = np.sin(k[0] * X[0] + k[1] * X[1])
    u, *_ = oracle.pcg_solve(m, lam, g, nu_const=nu, tol=1e-13)
    ref = g / (lam + nu * (k[0] ** 2 + k[1] ** 2))
    assert np.abs(u - ref).max() < 5e-5 * np.abs(ref).max()
