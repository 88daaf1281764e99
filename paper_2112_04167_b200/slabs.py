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
