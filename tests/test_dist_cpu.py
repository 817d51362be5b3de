"""CPU multi-process tests (torch.distributed, gloo, world_size 2 and 3) of the
slab decomposition the multi-GPU path uses.

Each rank takes its slab of the last axis with the product's own partition
rule (lsg_slab_partition, host-only), exchanges W ghost planes per stage with
its neighbours by the product's own halo plan (lsg_halo_plan: the messages
the NCCL exchange issues, in its order — send up, send down, receive from
below, receive from above; a ring when the axis is periodic), reduces the
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


def _order_key(v):
    """lsg_device.cuh order_key: monotone u64 key, -0.0 sharing +0.0's key."""
    b = v.view(np.uint64).copy()
    b[b == np.uint64(0x8000000000000000)] = np.uint64(0)
    neg = (b >> np.uint64(63)) == np.uint64(1)
    return np.where(neg, ~b, b | np.uint64(0x8000000000000000))


def _key_to_double(k):
    k = np.uint64(k)
    b = (k & np.uint64(0x7FFFFFFFFFFFFFFF)) if (k >> np.uint64(63)) else ~k
    return np.array([b], dtype=np.uint64).view(np.float64)[0]


def _worker(rank, world, port, nz, periodic_z, scheme, zero_speed, result_q):
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
    speed = [0.0, 0.0, 0.0] if zero_speed else [0.3, -0.8, 1.1]
    p = abi.make_problem(abi.HAM_LINEAR, scheme, abi.linear_params(speed), abi.GROW, True)
    plane = 10 * 9
    v_full = np.random.default_rng(7).uniform(-1, 1, plane * nz)
    if zero_speed:  # field >= 0 with +0 and -0 in different slabs: the step log's v_min is a zero
        v_full = 1.0 + np.abs(v_full)
        first, later = (-0.0, 0.0) if zero_speed == 1 else (0.0, -0.0)
        v_full[(nz - 2) * plane + 5] = later  # later in index order (last slab)
        v_full[1 * plane + 3] = first         # first zero in index order (first slab)
    z0, nzl = _lib.slab_partition(nz, world, rank)
    v = v_full[z0 * plane:(z0 + nzl) * plane].copy()
    _, bound = port_.term_lf(g, p, 0.0, v_full)
    dt = 0.32 * bound if np.isfinite(bound) else 0.01

    plan = _lib.halo_plan(nz, world, rank, W, periodic_z)  # the product's own message list (lsg_halo_plan)

    def exchange(u):
        """ghost planes below/above u's slab: the product's halo plan (the
        messages the NCCL exchange issues, in its order) over gloo."""
        ghost = {}
        reqs = []
        for kind, peer, first, count in plan:
            if kind == "send":
                reqs.append(dist.isend(torch.from_numpy(u[first * plane:(first + count) * plane].copy()), peer))
            else:
                buf = torch.empty(count * plane, dtype=torch.float64)
                ghost[first] = buf
                reqs.append(dist.irecv(buf, peer))
        for r in reqs:
            r.wait()
        glo = ghost[-W].numpy() if -W in ghost else None
        ghi = ghost[nzl].numpy() if nzl in ghost else None
        return glo, ghi

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

    # the product's per-step range slot: {~min key, max key, ~first zero code},
    # every word max-reduced across ranks as unsigned 64-bit (lsg_kernels.cuh
    # block_range, lsg_host.cu run_leg), then decoded like the host
    def reduced_range(u):
        keys = _order_key(u)
        zeros = np.flatnonzero(u == 0.0)
        gidx = (z0 * plane + zeros).astype(np.uint64)
        codes = (gidx << np.uint64(1)) | (u[zeros].view(np.uint64) >> np.uint64(63))
        fz = codes.min() if codes.size else np.uint64(0xFFFFFFFFFFFFFFFF)
        gathered = [None] * world
        dist.all_gather_object(gathered, [int(~keys.min()), int(keys.max()), int(~np.uint64(fz))])
        w = [max(gw[i] for gw in gathered) for i in range(3)]
        lo, hi = _key_to_double(~np.uint64(w[0])), _key_to_double(w[1])
        code = int(~np.uint64(w[2]))
        if code != 0xFFFFFFFFFFFFFFFF:
            zero = -0.0 if code & 1 else 0.0
            lo = zero if lo == 0.0 else lo
            hi = zero if hi == 0.0 else hi
        return lo, hi

    vmin, vmax = reduced_range(vn)
    v0min, v0max = reduced_range(v)  # the initial field keeps its signed zeros
    sizes = [None] * world
    dist.all_gather_object(sizes, (z0, vn))
    if rank == 0:
        full = np.empty(plane * nz)
        for zz, part in sizes:
            full[zz * plane: zz * plane + part.size] = part
        ref_v, ref_steps, _ = port_.integrate(g, p, abi.CFL3, 0.0, dt, v_full, abi.make_opts(max_step=dt))
        same = bool(np.array_equal(full.view(np.int64), ref_v.view(np.int64)))
        bits = lambda x: np.array([x], dtype=np.float64).view(np.int64)[0]  # noqa: E731
        rng_ok = bits(vmin) == bits(ref_steps[0, 3]) and bits(vmax) == bits(ref_steps[0, 4])
        # integrator.cpp:87-90 over the initial field: sequential std::min/max
        smin = smax = v_full[0]
        for x in v_full[1:]:
            smin = x if x < smin else smin
            smax = x if smax < x else smax
        rng_ok = rng_ok and bits(v0min) == bits(smin) and bits(v0max) == bits(smax)
        expect = {0: None, 1: -0.0, 2: 0.0}[zero_speed]
        zero_ok = expect is None or bits(v0min) == bits(expect)
        result_q.put((same, rng_ok, len(ref_steps), zero_ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nz,periodic_z,scheme,zero_speed", [
    (2, 17, False, 2, 0),       # ENO3, extrapolated ends
    (2, 16, True, 2, 0),        # ENO3, periodic ring of two: both neighbours are the same rank
    (3, 20, True, 3, 0),        # WENO5 ring of three, uneven slabs 7/7/6
    (3, 11, False, 1, 0),       # ENO2, thin slabs 4/4/3
    (3, 12, True, 2, 1),        # -0 first, +0 in a later slab: the first zero's sign wins across ranks
    (3, 12, True, 2, 2),        # +0 first, -0 later
])
def test_slab_decomposition_gloo(world, nz, periodic_z, scheme, zero_speed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), nz, periodic_z, scheme, zero_speed, q), nprocs=world,
                       join=True, start_method="spawn")
    same, rng_ok, nsteps, zero_ok = q.get(timeout=60)
    assert nsteps == 1
    assert same, "slab-decomposed RK3 step differs from the single-domain oracle"
    assert rng_ok, "reduced v range (product's word scheme) differs from the oracle's step log"
    assert zero_ok, "the first zero's sign did not decide v_min across ranks"


def test_partition_rule():
    from paper_2507_11542_b200 import _lib

    for n, P in [(41, 8), (101, 3), (512, 8), (7, 7)]:
        spans = [_lib.slab_partition(n, P, r) for r in range(P)]
        assert spans[0][0] == 0 and sum(s[1] for s in spans) == n
        for a, b in zip(spans, spans[1:]):
            assert a[0] + a[1] == b[0] and a[1] >= b[1] >= a[1] - 1
    with pytest.raises(ValueError):
        _lib.slab_partition(4, 5, 5)


def _snap_worker(rank, world, port, nz, tmpdir, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2507_11542_b200 import _lib, abi
    from paper_2507_11542_b200 import distributed as D

    g = abi.make_grid([-1.0, 0.0, 0.5], [1.0, 2.0, 3.25], [10, 9, nz], (2,))
    full = np.random.default_rng(11).uniform(-1, 1, 90 * nz)
    full[7] = -0.0
    local = D.take_slab(full, g, world, rank).copy()
    path = os.path.join(tmpdir, "gathered.snap")
    wrote = D.write_snapshot(g, local, 0.125, path)
    gathered = D.gather_slabs(local, g)
    if rank == 0:
        ref = os.path.join(tmpdir, "single.snap")
        _lib.write_snapshot(g, full, 0.125, ref)
        same_file = open(path, "rb").read() == open(ref, "rb").read()
        same_field = bool(np.array_equal(gathered.view(np.int64), full.view(np.int64)))
        result_q.put((wrote, same_file, same_field))
    else:
        assert not wrote and gathered is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nz", [(2, 17), (3, 4), (3, 20)])  # (3, 4): slabs of 2/1/1 planes
def test_snapshot_gather_gloo(world, nz, tmp_path):
    """Per-rank slabs gathered on rank 0 (paper_2507_11542_b200.distributed)
    give a file byte-identical to a single-process write of the whole field
    (snapshot.cpp:68-93), also when slabs hold fewer than 3 planes."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_snap_worker, args=(world, _free_port(), nz, str(tmp_path), q), nprocs=world, join=True,
                       start_method="spawn")
    wrote, same_file, same_field = q.get(timeout=60)
    assert wrote and same_field and same_file


def test_halo_plan():
    """lsg_halo_plan (the message list the distributed exchange issues): ends
    of an open axis talk to one neighbour, a periodic axis is a ring, a
    2-rank ring sends both messages to the same peer in a matching order."""
    from paper_2507_11542_b200 import _lib

    assert _lib.halo_plan(20, 3, 0, 3, False) == [("send", 1, 4, 3), ("recv", 1, 7, 3)]
    assert _lib.halo_plan(20, 3, 2, 3, False) == [("send", 1, 0, 3), ("recv", 1, -3, 3)]
    assert _lib.halo_plan(20, 3, 1, 3, False) == [("send", 2, 4, 3), ("send", 0, 0, 3), ("recv", 0, -3, 3),
                                                  ("recv", 2, 7, 3)]
    assert _lib.halo_plan(16, 2, 0, 2, True) == [("send", 1, 6, 2), ("send", 1, 0, 2), ("recv", 1, -2, 2),
                                                 ("recv", 1, 8, 2)]
    assert _lib.halo_plan(11, 1, 0, 3, True) == [("send", 0, 8, 3), ("send", 0, 0, 3), ("recv", 0, -3, 3),
                                                 ("recv", 0, 11, 3)]
    assert _lib.halo_plan(11, 1, 0, 3, False) == []
    # every send has a matching receive at the peer, in the same relative order
    for n, P, per in [(41, 8, True), (41, 8, False), (512 * 8, 8, True), (7, 7, True)]:
        plans = [_lib.halo_plan(n, P, r, 3, per) for r in range(P)]
        for r in range(P):
            for kind, peer, first, count in plans[r]:
                if kind == "send":
                    assert any(k == "recv" and q == r and c == count for k, q, _, c in plans[peer])
