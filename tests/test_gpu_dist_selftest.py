"""The distributed (NCCL) branch on one GPU: LSG_DIST_SELFTEST=1 with a
one-rank communicator makes solvers take the multi-rank path (halo planes,
NCCL send/recv with the rank as its own neighbour on a periodic slab axis,
overlapped interior/boundary launches, NCCL max-all-reduce of alpha, error
flags and per-step v range).  Results must equal the single-device solver
bit for bit.  No two ranks wait on each other (B200_PROFILING.md), so this
is safe on one GPU; the multi-rank message pattern itself is covered by the
gloo tests in test_dist_cpu.py."""
import os

import pytest

import helpers as H
from conftest import assert_bitwise
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dctx():
    old = os.environ.get("LSG_DIST_SELFTEST")
    os.environ["LSG_DIST_SELFTEST"] = "1"
    try:
        c = _lib.Context(0, 0, 1, _lib.nccl_unique_id())
    finally:
        if old is None:
            del os.environ["LSG_DIST_SELFTEST"]
        else:
            os.environ["LSG_DIST_SELFTEST"] = old
    yield c
    c.close()


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("name", ["cfg2", "cfg1", "cfg3", "cfg4", "cfg5", "rockets"])
def test_dist_branch_equals_single_device(ctx, dctx, port, monkeypatch, name, overlap):
    monkeypatch.setenv("LSG_HALO_OVERLAP", overlap)
    S = P.CONFIGS[name](**H.small(name))
    v0 = H.initial_value(port, S)
    one = _lib.Solver(ctx, S.grid, S.problem, S.method)
    dist = _lib.Solver(dctx, S.grid, S.problem, S.method)
    assert dist.local_nodes == v0.size
    one.set_field(v0)
    dist.set_field(v0)
    s1, t1 = one.integrate(0.0, 0.04, abi.make_opts())
    s2, t2 = dist.integrate(0.0, 0.04, abi.make_opts())
    assert t1 == t2
    assert_bitwise(s1, s2, "step log")
    assert_bitwise(one.get_field(), dist.get_field(), "value function")
    # the per-step API (ring slots, one sync per call) through the same branch
    dt = 0.32 * one.step_bound()
    one.step(t1, dt)
    dist.step(t2, dt)
    assert_bitwise(one.get_field(), dist.get_field(), "after step()")


def test_dist_branch_stateless_calls(ctx, dctx, port):
    S = P.cfg2_air3d(21)
    v0 = H.initial_value(port, S)
    a, ba = ctx.term_lf(S.grid, S.problem, 0.0, v0)
    b, bb = dctx.term_lf(S.grid, S.problem, 0.0, v0)
    assert ba == bb
    assert_bitwise(a, b, "term")
    va, sa, _ = ctx.integrate(S.grid, S.problem, S.method, 0.0, 0.05, v0)
    vb, sb, _ = dctx.integrate(S.grid, S.problem, S.method, 0.0, 0.05, v0)
    assert_bitwise(sa, sb, "steps")
    assert_bitwise(va, vb, "v")


def test_dist_branch_snapshot_and_gather(ctx, dctx, port, tmp_path):
    """The collective snapshot (lsg_solver_write_snapshot on a distributed
    context: NCCL gather to rank 0, which writes) and lsg_gather_field through
    the NCCL branch give the single-device file and field byte for byte."""
    S = P.cfg2_air3d(21)
    v0 = H.initial_value(port, S)
    one = _lib.Solver(ctx, S.grid, S.problem, S.method)
    dist = _lib.Solver(dctx, S.grid, S.problem, S.method)
    one.set_field(v0)
    dist.set_field(v0)
    one.integrate(0.0, 0.03)
    dist.integrate(0.0, 0.03)
    a, b = tmp_path / "one.snap", tmp_path / "dist.snap"
    one.write_snapshot(0.03, a)
    dist.write_snapshot(0.03, b)
    assert a.read_bytes() == b.read_bytes()
    g = dctx.gather_field(S.grid, dist.get_field())
    assert_bitwise(g, one.get_field(), "gathered field")
    ck, times, steps, _ = dctx.solve_brt(S.grid, S.problem, v0, (0.0, 0.05), 3, gather=True)
    ck1, times1, steps1, _ = ctx.solve_brt(S.grid, S.problem, v0, (0.0, 0.05), 3)
    assert_bitwise(ck, ck1, "gathered checkpoints")
    assert_bitwise(steps, steps1, "step log")
