"""CPU multi-process tests (torch.distributed, gloo, world_size 2 and 3) of the
slab decomposition the multi-GPU path uses.

Each rank takes its slab of the last axis with the product's own partition
rule (lsg_slab_partition, host-only), exchanges W ghost planes per stage with
its neighbours in the product's message order (send up, send down, receive
from below, receive from above; a ring when the axis is periodic), reduces the
v range with all_reduce(MIN/MAX), and evaluates each stage with the CPU oracle
on its halo-padded slab.  The gathered result must equal the single-domain
oracle integration bit for bit — the same property the device path is held to
(tests/test_gpu_parity.py::test_slabs_equal_single_device_bitwise).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grid(nz, periodic_z, abi):
    # spacing 1 along the slab axis keeps every sub-grid's spacing and axis bit-exact
    periodic = (2,) if periodic_z else ()
    return abi.make_grid([-1.0, 0.0, 0.0], [1.0, 2.0, float(nz - 1)], [10, 9, nz], periodic)


def _worker(rank, world, port, nz, periodic_z, scheme, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import oracle as O
    from paper_2507_11542_b200 import _lib, abi

    port_ = O.port()
    g = _grid(nz, periodic_z, abi)
    W = {0: 1, 1: 2, 2: 3, 3: 3}[scheme]
    p = abi.make_problem(abi.HAM_LINEAR, scheme, abi.linear_params([0.3, -0.8, 1.1]), abi.GROW, True)
    plane = 10 * 9
    v_full = np.random.default_rng(7).uniform(-1, 1, plane * nz)
    z0, nzl = _lib.slab_partition(nz, world, rank)
    v = v_full[z0 * plane:(z0 + nzl) * plane].copy()
    _, bound = port_.term_lf(g, p, 0.0, v_full)
    dt = 0.32 * bound

    lo = rank - 1 if rank > 0 else (world - 1 if periodic_z else -1)
    hi = rank + 1 if rank < world - 1 else (0 if periodic_z else -1)

    def exchange(u):
        """ghost planes below/above u's slab, in the product's message order."""
        send_up = torch.from_numpy(u[(nzl - W) * plane:].copy())
        send_dn = torch.from_numpy(u[:W * plane].copy())
        recv_lo = torch.empty(W * plane, dtype=torch.float64)
        recv_hi = torch.empty(W * plane, dtype=torch.float64)
        reqs = []
        if hi >= 0:
            reqs.append(dist.isend(send_up, hi))
        if lo >= 0:
            reqs.append(dist.isend(send_dn, lo))
        if lo >= 0:
            reqs.append(dist.irecv(recv_lo, lo))
        if hi >= 0:
            reqs.append(dist.irecv(recv_hi, hi))
        for r in reqs:
            r.wait()
        return (recv_lo.numpy() if lo >= 0 else None), (recv_hi.numpy() if hi >= 0 else None)

    def stage_term(u):
        glo, ghi = exchange(u)
        parts, zlo = [], float(z0)
        if glo is not None:
            parts.append(glo)
            zlo -= W
        parts.append(u)
        if ghi is not None:
            parts.append(ghi)
        padded = np.concatenate(parts)
        nzp = padded.size // plane
        sub = abi.make_grid([-1.0, 0.0, zlo], [1.0, 2.0, zlo + nzp - 1], [10, 9, nzp])
        if glo is None and ghi is None and periodic_z:  # single slab keeps the global rule
            sub = g
        d, _ = port_.term_lf(sub, p, 0.0, padded)
        off = W * plane if glo is not None else 0
        return d[off:off + nzl * plane]

    # one TVD-RK3 step (integrator.cpp:70-85) with the fused stage forms
    d1 = stage_term(v)
    v1 = v + dt * d1
    d2 = stage_term(v1)
    vh = v + 0.25 * ((v1 + dt * d2) - v)
    d3 = stage_term(vh)
    vn = v + (2.0 / 3.0) * ((vh + dt * d3) - v)

    rng = torch.tensor([vn.min(), -vn.max()], dtype=torch.float64)
    dist.all_reduce(rng, op=dist.ReduceOp.MIN)
    sizes = [None] * world
    dist.all_gather_object(sizes, (z0, vn))
    if rank == 0:
        full = np.empty(plane * nz)
        for zz, part in sizes:
            full[zz * plane: zz * plane + part.size] = part
        ref_v, ref_steps, _ = port_.integrate(g, p, abi.CFL3, 0.0, dt, v_full, abi.make_opts(max_step=dt))
        same = bool(np.array_equal(full.view(np.int64), ref_v.view(np.int64)))
        rng_ok = (rng[0].item() == ref_steps[0, 3]) and (-rng[1].item() == ref_steps[0, 4])
        result_q.put((same, rng_ok, len(ref_steps)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nz,periodic_z,scheme", [
    (2, 17, False, 2),   # ENO3, extrapolated ends
    (2, 16, True, 2),    # ENO3, periodic ring of two: both neighbours are the same rank
    (3, 20, True, 3),    # WENO5 ring of three, uneven slabs 7/7/6
    (3, 11, False, 1),   # ENO2, thin slabs 4/4/3
])
def test_slab_decomposition_gloo(world, nz, periodic_z, scheme):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), nz, periodic_z, scheme, q), nprocs=world,
                       join=True, start_method="spawn")
    same, rng_ok, nsteps = q.get(timeout=60)
    assert nsteps == 1
    assert same, "slab-decomposed RK3 step differs from the single-domain oracle"
    assert rng_ok, "all-reduced v range differs from the oracle's step log"


def test_partition_rule():
    from paper_2507_11542_b200 import _lib

    for n, P in [(41, 8), (101, 3), (512, 8), (7, 7)]:
        spans = [_lib.slab_partition(n, P, r) for r in range(P)]
        assert spans[0][0] == 0 and sum(s[1] for s in spans) == n
        for a, b in zip(spans, spans[1:]):
            assert a[0] + a[1] == b[0] and a[1] >= b[1] >= a[1] - 1
    with pytest.raises(ValueError):
        _lib.slab_partition(4, 5, 5)
