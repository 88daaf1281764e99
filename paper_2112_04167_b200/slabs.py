"""Host-side slab partition and halo pairing of the multi-GPU path.

The C library (``dg_mesh_create`` / ``exchange`` in csrc/capi.cpp) owns the device-side
exchange over NCCL.  This module states the same contract in Python so that the launcher
(bench.py) generates each rank's inputs consistently and so that the partition and the
halo pairing can be tested on CPU with a ``gloo`` process group:

* the slowest direction (z in 3-D, y in 2-D) is split into ``nranks`` equal slabs; rank r
  owns global elements ``[r E, (r + 1) E)``, ``E = N_el / nranks`` (element index
  ``ex + Nx (ey + Ny ez)``, so a slab is one contiguous range);
* one face exchange per operator application: every rank sends its LAST element layer to
  ``next = (r + 1) % R`` and its FIRST layer to ``prev = (r - 1) % R`` and receives the
  ``lo`` halo (the layer below its first one) from ``prev`` and the ``hi`` halo from
  ``next`` -- periodic in the slowest direction, so with R = 2 both neighbours are the same
  rank and the two messages are told apart by their order (NCCL) or tag (here).

* per operator application of a halo mesh the exchanged data are FACE TRACES, not layers
  (capi.cpp ``trace_exchange``, halo.cu): each rank sends the traces of its TOP face (last
  layer) to ``next`` and of its BOTTOM face (first layer) to ``prev``, receives ``tr_lo`` (the
  top face of the layer below) from ``prev`` and ``tr_hi`` (the bottom face of the layer
  above) from ``next``, posted in that order (send top, send bottom, recv lo, recv hi), so
  R = 2 (prev == next) and R = 1 (the halo mode: both peers are the rank itself) pair
  correctly; a trace array holds 3 F values ``[u | nu d_n u | nu]`` with F face nodes of one
  layer, face node index ``face_index``.

No method arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

TAG_UP = 11    # last layer -> next rank (arrives as its lo halo)
TAG_DOWN = 12  # first layer -> prev rank (arrives as its hi halo)


def slab(dim: int, N, rank: int, nranks: int):
    """(element offset, local element count, layer size in elements) of ``rank``."""
    N = list(N)[:dim]
    S = dim - 1
    if N[S] % nranks:
        raise ValueError("N of the slowest direction (%d) must be divisible by nranks (%d)" % (N[S], nranks))
    layer = int(np.prod(N[:S]))
    nel = layer * (N[S] // nranks)
    return rank * nel, nel, layer


def peers(rank: int, nranks: int):
    """(prev, next) ranks of the periodic slab ring."""
    return (rank - 1) % nranks, (rank + 1) % nranks


def face_count(dim: int, Nl, n: int) -> int:
    """F: face nodes of one slab layer of the slowest direction (the trace array holds 3 F)."""
    return (Nl[0] * Nl[1] * n * n) if dim == 3 else (Nl[0] * n)


def face_index(dim: int, Nl, n: int, c0: int, c1: int, inface: int) -> int:
    """Index in [0, F) of the face node with in-face index ``inface`` (a + n b: a along x, b
    along y in 3-D; a along x in 2-D) of the face element (c0, c1) -- dg_internal.h Halo."""
    return ((c0 + Nl[0] * c1) * n * n + inface) if dim == 3 else (c0 * n + inface)


def exchange_traces(send_lo, send_hi, rank: int, nranks: int, dist):
    """The face-trace swap of capi.cpp ``trace_exchange`` with torch.distributed P2P calls in the
    same posting order (top -> next, bottom -> prev; lo <- prev, hi <- next).  send_lo: traces
    of the rank's bottom face, send_hi: of its top face.  Returns (tr_lo, tr_hi)."""
    import torch

    prev, nxt = peers(rank, nranks)
    if nranks == 1:  # the halo mode's self send/recv (NCCL supports it, gloo P2P does not)
        return send_hi.clone(), send_lo.clone()
    lo = torch.empty_like(send_hi)
    hi = torch.empty_like(send_lo)
    ops = [dist.P2POp(dist.isend, send_hi.contiguous(), nxt, tag=TAG_UP),
           dist.P2POp(dist.isend, send_lo.contiguous(), prev, tag=TAG_DOWN),
           dist.P2POp(dist.irecv, lo, prev, tag=TAG_UP),
           dist.P2POp(dist.irecv, hi, nxt, tag=TAG_DOWN)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return lo, hi


def exchange_layers(field, layer_elems: int, rank: int, nranks: int, dist):
    """Halo exchange of an element-major slab field ``[nel][npe]`` (torch tensor, CPU) with
    ``torch.distributed`` point-to-point calls in the pairing of capi.cpp ``exchange``.
    Returns ``(lo, hi)``: the neighbour layers below the first and above the last layer."""
    import torch

    prev, nxt = peers(rank, nranks)
    first = field[:layer_elems].contiguous()
    last = field[-layer_elems:].contiguous()
    lo = torch.empty_like(first)
    hi = torch.empty_like(first)
    ops = [dist.P2POp(dist.isend, last, nxt, tag=TAG_UP),
           dist.P2POp(dist.isend, first, prev, tag=TAG_DOWN),
           dist.P2POp(dist.irecv, lo, prev, tag=TAG_UP),
           dist.P2POp(dist.irecv, hi, nxt, tag=TAG_DOWN)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return lo, hi
