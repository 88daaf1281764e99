"""Pins of the oracle's two-level additive Schwarz preconditioner (
P:1045-1046 "Krylov-accelerated Schwarz/multigrid", formula not in the paper; reading in
DESIGN.md §9):  B = sum_K R_K^T A_KK^-1 R_K + P_1 A_c^+ P_1^T,  A_c = P_1^T A P_1.

What fixes it independently of its own code:
* A_c equals the textbook Q1 finite-element matrices on the periodic vertex grid (1-D
  stiffness circ(2, -1)/h, mass circ(4, 1) h/6, Kronecker-summed) -- every SIP face term
  carries a jump and vanishes on continuous functions; GLL_P quadrature is exact for Q1
  products when P >= 2 and lumps the mass (circ(1, 0) h) when P = 1;
* A_KK equals the diagonal block of the brute-force all-triples dense assembly
  (oracle.sip_dense, a separate code path);
* B is symmetric positive definite (on 1-perp for lam = 0);
* Schwarz-PCG converges to the LAPACK solution, in an h-independent number of iterations
  (the two-level property) while Jacobi-PCG's count grows.
"""
import numpy as np
import pytest

import oracle


def circ(N, c0, c1):
    C = np.zeros((N, N))
    for i in range(N):
        C[i, i] += c0
        C[i, (i + 1) % N] += c1
        C[i, (i - 1) % N] += c1
    return C


def kron_sum(mats_K, mats_M, lam, nu):
    """lam M_z(x)M_y(x)M_x + nu sum_d (M with K in slot d): x fastest, as the vertex index."""
    def kron_list(lst):  # lst[0] = x (fastest) ... lst[-1] = slowest
        out = lst[-1]
        for a in lst[-2::-1]:
            out = np.kron(out, a)
        return out
    A = lam * kron_list(mats_M)
    for k in range(len(mats_K)):
        A = A + nu * kron_list([mats_K[j] if j == k else mats_M[j] for j in range(len(mats_K))])
    return A


@pytest.mark.parametrize("dim,N,L,P,lam,nu", [
    (2, (5, 4), (1.0, 1.3), 3, 0.7, 1.3),
    (2, (2, 3), (2.0, 1.0), 5, 0.0, 1.0),
    (3, (3, 2, 4), (1.0, 0.8, 1.2), 2, 2.0, 0.5),
    (2, (4, 3), (1.0, 1.0), 1, 1.5, 1.0),  # P = 1: GLL lumps the Q1 mass
])
def test_coarse_operator_is_textbook_q1(dim, N, L, P, lam, nu):
    m = oracle.Mesh(dim, N, L, P)
    Ac, Pm = oracle.q1_coarse_operator(m, lam, nu_const=nu)
    Ks, Ms = [], []
    for d in range(dim):
        h = L[d] / N[d]
        Ks.append(circ(N[d], 2.0 / h, -1.0 / h))
        Ms.append(circ(N[d], 4.0 * h / 6.0, h / 6.0) if P >= 2 else circ(N[d], h, 0.0))
    ref = kron_sum(Ks, Ms, lam, nu)
    assert np.abs(Ac - ref).max() <= 1e-13 * np.abs(ref).max()
    # the hats are a partition of unity (P_1 1 = 1)
    assert np.allclose(Pm.sum(axis=1), 1.0, atol=1e-15)


@pytest.mark.parametrize("dim,N,P,lam", [(2, (3, 3), 4, 0.0), (3, (3, 3, 3), 2, 1.7), (2, (2, 3), 3, 0.5)])
def test_element_block_is_dense_diagonal_block(dim, N, P, lam):
    m = oracle.Mesh(dim, N, (1.0, 1.1, 0.9)[:dim], P)
    A = oracle.sip_dense(m, lam, nu_const=0.8)
    for e in (0, m.n_el - 1):
        sl = slice(e * m.npe, (e + 1) * m.npe)
        B = oracle.element_block(m, lam, e, nu_const=0.8)
        assert np.abs(B - A[sl, sl]).max() <= 1e-13 * np.abs(A).max()


@pytest.mark.parametrize("lam", [0.0, 2.0])
def test_schwarz_symmetric_positive(lam):
    m = oracle.Mesh(2, (3, 4), (1.0, 1.2), 3)
    B = oracle.Schwarz2(m, lam)
    Bm = np.stack([B(np.eye(m.ndof)[j]).reshape(-1) for j in range(m.ndof)], axis=1)
    assert np.abs(Bm - Bm.T).max() <= 1e-12 * np.abs(Bm).max()
    ev = np.linalg.eigvalsh(0.5 * (Bm + Bm.T))
    if lam == 0.0:  # on 1-perp (the residuals of the Poisson system)
        Q = np.eye(m.ndof) - 1.0 / m.ndof
        ev = np.linalg.eigvalsh(Q @ Bm @ Q)[1:]
    assert ev.min() > 0.0


@pytest.mark.parametrize("lam", [0.0, 3.0])
def test_schwarz_pcg_matches_lapack(lam):
    m = oracle.Mesh(2, (4, 3), (2.0, 1.5), 4)
    f = np.random.default_rng(11).uniform(-1, 1, (m.n_el, m.npe))
    A = oracle.sip_dense(m, lam)
    ms = oracle.mass(m).reshape(-1)
    fv = f.reshape(-1)
    if lam == 0.0:
        fv = fv - (ms @ fv) / ms.sum()
        ref = np.linalg.lstsq(A, ms * fv, rcond=None)[0]
        ref -= (ms @ ref) / ms.sum()
    else:
        ref = np.linalg.solve(A, ms * fv)
    u, it = oracle.pcg_precond(m, lam, f, oracle.Schwarz2(m, lam), tol=1e-13)
    assert np.linalg.norm(u.reshape(-1) - ref) <= 1e-10 * np.linalg.norm(ref)


def test_two_level_iterations_h_independent():
    its_s, its_j = [], []
    for N in (4, 8, 16):
        m = oracle.Mesh(2, (N, N), (2 * np.pi, 2 * np.pi), 4)
        f = np.random.default_rng(N).uniform(-1, 1, (m.n_el, m.npe))
        _, it = oracle.pcg_precond(m, 0.0, f, oracle.Schwarz2(m, 0.0), tol=1e-10)
        its_s.append(it)
        _, itj, *_ = oracle.pcg_solve(m, 0.0, f, tol=1e-10)
        its_j.append(itj)
    assert its_s[2] <= its_s[0] + 8, its_s
    assert its_j[2] >= 2.5 * its_j[0], its_j
    assert its_s[2] < 0.5 * its_j[2]
