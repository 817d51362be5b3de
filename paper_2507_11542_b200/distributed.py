"""Host-side gathers of slab-decomposed fields over torch.distributed.

The device path keeps each rank's slab of the last axis (lsg_slab_partition);
consumers of whole fields — the reference's snapshot files (snapshot.cpp:68-93)
and solve_brt's checkpoint vector (reachability.cpp:160-170) — need the
global column-major array, which is the slabs concatenated in rank order.

`gather_slabs` moves host slabs to rank 0 with point-to-point messages in
1 GiB chunks on any torch.distributed backend (gloo: CPU tensors; NCCL: the
chunks travel through the rank's current CUDA device).  The C ABI has the same
operation over the context's own NCCL communicator (lsg_gather_field,
lsg_solver_write_snapshot), which needs no torch process group.
"""
from __future__ import annotations

import numpy as np

from . import _lib

_CHUNK = 1 << 27  # doubles


def slab_nodes(g, nranks, rank):
    """(first node, node count) of rank's slab of grid g."""
    n_last = g.counts[g.dim - 1]
    plane = _lib.node_count(g) // n_last
    z0, nz = _lib.slab_partition(n_last, nranks, rank)
    return z0 * plane, nz * plane


def take_slab(field, g, nranks, rank):
    """This rank's slab of a global column-major field (a view)."""
    off, n = slab_nodes(g, nranks, rank)
    return np.ascontiguousarray(field, dtype=np.float64)[off:off + n]


def gather_slabs(local, g, group=None):
    """Global field on rank 0 (None elsewhere) from every rank's host slab."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    local = np.ascontiguousarray(local, dtype=np.float64)
    off, n = slab_nodes(g, world, rank)
    if local.size != n:
        raise ValueError(f"gather_slabs: rank {rank} holds {local.size} values, its slab has {n}")
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    if rank != 0:
        for k in range(0, n, _CHUNK):
            dist.send(torch.from_numpy(local[k:k + _CHUNK]).to(dev), dst=0, group=group)
        return None
    out = np.empty(_lib.node_count(g), dtype=np.float64)
    out[off:off + n] = local
    for r in range(1, world):
        ro, rn = slab_nodes(g, world, r)
        for k in range(0, rn, _CHUNK):
            c = min(_CHUNK, rn - k)
            buf = torch.empty(c, dtype=torch.float64, device=dev)
            dist.recv(buf, src=r, group=group)
            out[ro + k:ro + k + c] = buf.cpu().numpy()
    return out


def write_snapshot(g, local, time, path, group=None):
    """snapshot.cpp:68-93 file of the whole grid from per-rank slabs (rank 0 writes)."""
    full = gather_slabs(local, g, group)
    if full is not None:
        _lib.write_snapshot(g, full, time, path)
    return full is not None
