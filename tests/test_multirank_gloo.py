"""Multi-rank host logic on CPU: world-size 2 and 4 ``gloo`` process groups.

What the N > 1 path relies on, checked without GPUs:
* the slab partition (``paper_2112_04167_b200.slabs.slab``) tiles the mesh exactly and each
  rank's seeded inputs (``workloads`` ``*_slab``) equal the global arrays' slices bit for bit;
* the halo pairing of capi.cpp ``exchange`` (last layer -> next, first layer -> prev,
  periodic ring, R = 2 where both neighbours coincide) delivers exactly the neighbour
  layers: the oracle's SIP apply evaluated on (slab + lo/hi halos only, everything else
  NaN) reproduces the global apply on the slab bit for bit (the apply is
  partition-independent);
* the PCG dot products summed with an all-reduce over ranks match the global sums.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2112_04167_b200 import slabs
from workloads import config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "apply":
            _check_apply(rank, world)
        elif case == "traces":
            _check_traces(rank, world)
        else:
            _check_inputs(rank, world)
    finally:
        dist.destroy_process_group()


def _check_apply(rank, world):
    dim, N, L, P = 3, (3, 2, 4), (1.0, 1.3, 0.9), 2
    om = oracle.Mesh(dim, N, L, P)
    g = np.random.default_rng(7)  # identical global arrays on every rank
    u = g.uniform(-1, 1, (om.n_el, om.npe))
    nu = 0.5 + g.uniform(0, 1, (om.n_el, om.npe))
    lam = 2.5
    ref = oracle.sip_apply(om, lam, u, nu=nu)
    off, nel, layer = slabs.slab(dim, N, rank, world)
    us, nus = torch.from_numpy(u[off:off + nel].copy()), torch.from_numpy(nu[off:off + nel].copy())
    lo, hi = slabs.exchange_layers(us, layer, rank, world, dist)
    nlo, nhi = slabs.exchange_layers(nus, layer, rank, world, dist)
    # extended array: own slab + received halos, NaN elsewhere (a missing value poisons the result)
    ext_u = np.full_like(u, np.nan)
    ext_nu = np.full_like(nu, np.nan)
    ext_u[off:off + nel], ext_nu[off:off + nel] = us.numpy(), nus.numpy()
    lo_off = (off - layer) % om.n_el
    hi_off = (off + nel) % om.n_el
    ext_u[lo_off:lo_off + layer], ext_nu[lo_off:lo_off + layer] = lo.numpy(), nlo.numpy()
    ext_u[hi_off:hi_off + layer], ext_nu[hi_off:hi_off + layer] = hi.numpy(), nhi.numpy()
    mine = oracle.sip_apply(om, lam, ext_u, nu=ext_nu, elems=np.arange(off, off + nel))
    assert np.array_equal(mine, ref[off:off + nel]), np.nanmax(np.abs(mine - ref[off:off + nel]))
    # all-reduced dot products (PCG p.q and sum q) against the global ones
    loc = torch.tensor([float(np.dot(us.numpy().ravel(), mine.ravel())), float(mine.sum())], dtype=torch.float64)
    dist.all_reduce(loc)
    glob = np.array([np.dot(u.ravel(), ref.ravel()), ref.sum()])
    assert np.allclose(loc.numpy(), glob, rtol=1e-13, atol=1e-13 * np.abs(ref).sum())


def _face_traces(u, nu, dim, Nl, n, D0, sd, layer_idx, node):
    """(u, nu (2/h) (D u)_node, nu) at the S-face node ``node`` (0 or P) of one element layer,
    written with the oracle's differentiation matrix (test-side arithmetic, not product code)."""
    npe = n ** dim
    lay = int(np.prod(Nl[: dim - 1]))
    NF = n ** (dim - 1)
    F = lay * NF
    out = np.zeros(3 * F)
    for fe in range(lay):
        e = layer_idx * lay + fe
        for inface in range(NF):
            line = u[e, inface + NF * np.arange(n)]
            f = fe * NF + inface
            out[f] = line[node]
            nv = nu[e, inface + NF * node]
            out[F + f] = nv * sd * float(D0[node] @ line)
            out[2 * F + f] = nv
    return out


def _check_traces(rank, world):
    """The face-trace pairing of capi.cpp trace_exchange: every rank receives the top-face
    traces of the layer below its slab (tr_lo) and the bottom-face traces of the layer above
    (tr_hi), periodic; R = 1 (halo mode) receives its own faces (the local wrap)."""
    dim, N, L, P = 3, (3, 2, 8), (1.0, 1.3, 0.9), 3
    n = P + 1
    om = oracle.Mesh(dim, N, L, P)
    g = np.random.default_rng(8)
    u = g.uniform(-1, 1, (om.n_el, om.npe))
    nu = 0.5 + g.uniform(0, 1, (om.n_el, om.npe))
    xi, _ = oracle.gll(P)
    D0 = np.array([oracle.lagrange(P, xi, x)[1] for x in xi])  # D[i][j] = l_j'(xi_i)
    sd = 2.0 / (L[2] / N[2])
    off, nel, layer = slabs.slab(dim, N, rank, world)
    Nl = (N[0], N[1], N[2] // world)
    us, nus = u[off:off + nel], nu[off:off + nel]
    send_lo = torch.from_numpy(_face_traces(us, nus, dim, Nl, n, D0, sd, 0, 0))
    send_hi = torch.from_numpy(_face_traces(us, nus, dim, Nl, n, D0, sd, Nl[2] - 1, P))
    assert send_lo.numel() == 3 * slabs.face_count(dim, Nl, n)
    tr_lo, tr_hi = slabs.exchange_traces(send_lo, send_hi, rank, world, dist)
    # the neighbours' faces from the global arrays
    zl = (rank * Nl[2] - 1) % N[2]
    zh = ((rank + 1) * Nl[2]) % N[2]
    want_lo = _face_traces(u, nu, dim, N, n, D0, sd, zl, P)
    want_hi = _face_traces(u, nu, dim, N, n, D0, sd, zh, 0)
    assert np.array_equal(tr_lo.numpy(), want_lo)
    assert np.array_equal(tr_hi.numpy(), want_hi)
    assert slabs.face_index(dim, Nl, n, 2, 1, 5) == (2 + 3 * 1) * 16 + 5


def _check_inputs(rank, world):
    for cid in (2, 3):
        c = config(cid)
        off, nel, _ = slabs.slab(c.dim, c.N, rank, world)
        parts = [c.apply_input_slab(off, nel), c.rhs_slab(0, off, nel)]
        if c.variable_nu:
            parts.append(c.nu_slab(off, nel))
        loc = torch.from_numpy(np.concatenate([p.ravel() for p in parts]))
        gathered = [torch.empty_like(loc) for _ in range(world)]
        dist.all_gather(gathered, loc)
        if rank == 0:
            full = [c.apply_input(), c.rhs(0)] + ([c.nu()] if c.variable_nu else [])
            for r in range(world):
                o, ne, _ = slabs.slab(c.dim, c.N, r, world)
                want = np.concatenate([f[o:o + ne].ravel() for f in full])
                assert np.array_equal(gathered[r].numpy(), want), (cid, r)


@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_reproduces_global_apply(world):
    mp.spawn(_worker, args=(world, _free_port(), "apply"), nprocs=world, join=True)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_face_trace_exchange_pairing(world):
    mp.spawn(_worker, args=(world, _free_port(), "traces"), nprocs=world, join=True)


@pytest.mark.parametrize("world", [2, 4])
def test_rank_slab_inputs_match_global(world):
    mp.spawn(_worker, args=(world, _free_port(), "inputs"), nprocs=world, join=True)


def test_slab_partition_tiles_the_mesh():
    for dim, N, R in [(3, (4, 3, 8), 4), (3, (2, 2, 2), 2), (2, (5, 6), 3), (3, (1, 1, 8), 8)]:
        offs = [slabs.slab(dim, N, r, R) for r in range(R)]
        assert offs[0][0] == 0
        for (o0, n0, _), (o1, _, _) in zip(offs, offs[1:]):
            assert o1 == o0 + n0
        assert offs[-1][0] + offs[-1][1] == int(np.prod(N[:dim]))
    with pytest.raises(ValueError):
        slabs.slab(3, (2, 2, 3), 0, 2)
    assert slabs.peers(0, 2) == (1, 1) and slabs.peers(3, 4) == (2, 0)
