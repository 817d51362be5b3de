"""GPU parity: the sm_100a path (through the C ABI) against the oracle.

Bit-exact for the ENO/First schemes, step bounds, dt sequences and step
counts, and — because the WENO5 kernel keeps the reference's operation order
with IEEE divisions — for WENO5 as well.  The north_star tolerance (1e-10
relative in fp64) is the fallback bar asserted where noted.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import assert_bitwise, rel_inf
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P
import helpers as H

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="module")
def sums():
    with open(os.path.join(GOLDEN, "golden_sums.json")) as f:
        return json.load(f)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_pad_and_shift_vs_golden(ctx, golden):
    g = abi.make_grid([0.0] * 3, [1.0] * 3, [5, 6, 7], [0, 1, 2])
    v = golden["pad/periodic/in"]
    for d in range(3):
        p = ctx.pad_ghost(g, v, d, 2)
        assert_bitwise(p, golden[f"pad/periodic/d{d}"], f"pad periodic d{d}")
        for off in (-2, -1, 0, 1, 2):
            back = ctx.shift_along_dim(g, ctx.pad_ghost(g, ctx.shift_along_dim(g, p, d, 2, off), d, 2), d, 2, -off)
            assert_bitwise(back, v, "shift round trip")
    g = abi.make_grid([0.0] * 3, [1.0] * 3, [5, 6, 7])
    for d in range(3):
        assert_bitwise(ctx.pad_ghost(g, golden["pad/extrap/in"], d, 3), golden[f"pad/extrap/d{d}"], f"pad extrap d{d}")
    with pytest.raises(ValueError):
        ctx.pad_ghost(abi.make_grid([0.0], [1.0], [4]), np.zeros(4), 0, 4)


@pytest.mark.parametrize("key", ["A", "B", "C"])
def test_upwind_vs_golden(ctx, golden, key):
    from golden.make_golden import UPWIND_GRIDS

    g, _ = UPWIND_GRIDS[key]
    v = golden[f"upwind/{key}/in"]
    for s in range(4):
        for d in range(g.dim):
            L, R = ctx.upwind(g, v, d, s)
            assert_bitwise(L, golden[f"upwind/{key}/s{s}/d{d}/L"], f"{key} s{s} d{d} L")
            assert_bitwise(R, golden[f"upwind/{key}/s{s}/d{d}/R"], f"{key} s{s} d{d} R")


@pytest.mark.parametrize("dims", [(7,), (9, 8), (8, 7, 9), (7, 7, 7, 8), (7, 7, 7, 7, 7), (7,) * 6])
def test_upwind_vs_oracle_all_dims(ctx, port, dims):
    D = len(dims)
    for periodic in [(), tuple(range(D))]:
        g = abi.make_grid([-1.0] * D, [1.5] * D, list(dims), periodic)
        v = H.random_field(g, 11 + D)
        for s in range(4):
            for d in range(D):
                a, b = ctx.upwind(g, v, d, s), port.upwind(g, v, d, s)
                assert_bitwise(a[0], b[0], f"D{D} s{s} d{d} L")
                assert_bitwise(a[1], b[1], f"D{D} s{s} d{d} R")


def test_upwind_errors(ctx):
    g = abi.make_grid([0.0], [1.0], [5])
    ctx.upwind(g, np.zeros(5), 0, abi.SCHEME_ENO2)
    for s, dim in [(abi.SCHEME_ENO3, 0), (abi.SCHEME_WENO5, 0), (abi.SCHEME_FIRST, 1)]:
        with pytest.raises(ValueError):
            ctx.upwind(g, np.zeros(5), dim, s)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "rockets", "rotation"])
def test_term_vs_golden(ctx, port, sums, name):
    S = P.CONFIGS[name](**H.small(name))
    v0 = H.initial_value(port, S)
    dvdt, bound = ctx.term_lf(S.grid, S.problem, 0.0, v0)
    e = sums[f"term/{name}"]
    assert bound.hex() == e["bound"], "step bound must be bit-exact"
    if sha(dvdt) != e["dvdt"]:
        ref_dvdt, _ = port.term_lf(S.grid, S.problem, 0.0, v0)
        assert_bitwise(dvdt, ref_dvdt, f"dvdt {name}")


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
@pytest.mark.parametrize("clamp", [False, True])
def test_term_linear_all_schemes(ctx, port, scheme, clamp):
    g = abi.make_grid([0.0, -1.0, 0.0], [1.0, 1.0, 2.0], [12, 9, 10], [2])
    v = H.random_field(g, 99)
    p = abi.make_problem(abi.HAM_LINEAR, scheme, abi.linear_params([0.7, -1.3, 0.2]), abi.SHRINK, clamp)
    a, ba = ctx.term_lf(g, p, 0.0, v)
    b, bb = port.term_lf(g, p, 0.0, v)
    assert_bitwise(a, b, "dvdt")
    assert ba == bb


def test_term_kats(ctx):
    # test_hamiltonian.cpp:54-193 on the device path
    lin = lambda c, bounds=None, offset=0.0, scheme=abi.SCHEME_ENO2: abi.make_problem(  # noqa: E731
        abi.HAM_LINEAR, scheme, abi.linear_params(c, bounds, offset))
    g = abi.make_grid([0.0], [1.0], [11])
    assert ctx.term_lf(g, lin([2.0]), 0.0, np.zeros(11))[1] == pytest.approx(0.05, rel=1e-14)
    assert ctx.term_lf(g, lin([0.0]), 0.0, np.zeros(11))[1] == math.inf
    g = abi.make_grid([0.0], [2.0], [5])
    x = np.linspace(0.0, 2.0, 5)
    assert ctx.term_lf(g, lin([1.0], [0.0], scheme=abi.SCHEME_FIRST), 0.0, x * x)[0][2] == pytest.approx(-2.0)
    g = abi.make_grid([0.0], [1.0], [17])
    d, _ = ctx.term_lf(g, lin([0.25], [0.25], 0.125), 0.0, 1.5 * np.arange(17) / 16.0)
    assert np.all(d == -(0.25 * 1.5 + 0.125))
    g = abi.make_grid([0.0], [1.0], [5])
    with pytest.raises(RuntimeError):
        ctx.term_lf(g, lin([math.nan]), 0.0, np.ones(5))
    with pytest.raises(RuntimeError):
        ctx.term_lf(g, lin([1.0], [-1.0]), 0.0, np.ones(5))
    with pytest.raises(RuntimeError):
        ctx.term_lf(g, lin([1.0], [math.inf]), 0.0, np.ones(5))
    assert list(ctx.restrict_update(np.array([-2.0, 0.0, 3.0]), abi.GROW)) == [-2.0, 0.0, 0.0]
    assert list(ctx.restrict_update(np.array([-2.0, 0.0, 3.0]), abi.SHRINK)) == [0.0, 0.0, 3.0]


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "rotation"])
def test_integrate_vs_oracle(ctx, port, name):
    S = P.CONFIGS[name](**H.small(name))
    v0 = H.initial_value(port, S)
    tf = 0.03
    va, sa, ta = ctx.integrate(S.grid, S.problem, S.method, 0.0, tf, v0, abi.make_opts())
    vb, sb, tb = port.integrate(S.grid, S.problem, S.method, 0.0, tf, v0, abi.make_opts())
    assert ta == tb
    assert_bitwise(sa, sb, "step log (t, dt, bound, v_min, v_max)")
    assert_bitwise(va, vb, "final value function")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5", "rotation"])
def test_integrate_vs_golden(ctx, port, sums, name):
    e = sums[f"integrate/{name}"]
    S = P.CONFIGS[name](**e["kw"])
    v0 = H.initial_value(port, S)
    v, steps, tfin = ctx.integrate(S.grid, S.problem, S.method, 0.0, e["tf"], v0, abi.make_opts())
    assert len(steps) == e["n_steps"]
    assert [[x.hex() for x in row] for row in steps] == e["steps"]
    assert tfin.hex() == e["t_final"]
    assert sha(v) == e["out"]


def test_integrate_methods_and_checkpoints(ctx, port):
    S = P.cfg2_air3d(15)
    v0 = H.initial_value(port, S)
    o = abi.make_opts(checkpoint_times=[0.011, 0.05], max_step=0.02)
    for m in (abi.CFL1, abi.CFL2, abi.CFL3):
        a = ctx.integrate(S.grid, S.problem, m, 0.0, 0.07, v0, o)
        b = port.integrate(S.grid, S.problem, m, 0.0, 0.07, v0, o)
        assert_bitwise(a[1], b[1], f"steps m{m}")
        assert_bitwise(a[0], b[0], f"v m{m}")
        assert 0.011 in a[1][:, 0] and 0.05 in a[1][:, 0]


def test_integrate_errors(ctx, port):
    S = P.cfg1_circle(21)
    v0 = H.initial_value(port, S)
    for bad in [abi.make_opts(cfl_factor=0.0), abi.make_opts(max_step=-1.0),
                abi.make_opts(checkpoint_times=[0.5, 0.2])]:
        with pytest.raises(ValueError):
            ctx.integrate(S.grid, S.problem, abi.CFL1, 0.0, 1.0, v0, bad)
    with pytest.raises(ValueError):
        ctx.integrate(S.grid, S.problem, abi.CFL1, 1.0, 0.0, v0)
    v, steps, t = ctx.integrate(S.grid, S.problem, abi.CFL2, 4.0, 4.0, v0)
    assert t == 4.0 and len(steps) == 0 and np.array_equal(v, v0)
    nan_p = abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_ENO2, abi.linear_params([math.nan, 1.0], [1.0, 1.0]))
    with pytest.raises(RuntimeError):
        ctx.integrate(S.grid, nan_p, abi.CFL3, 0.0, 0.1, v0)
    # a rockets problem on a 2-D grid is rejected like rocket_hamiltonian does
    rk = P.rockets(9).problem
    with pytest.raises(ValueError):
        ctx.integrate(S.grid, rk, abi.CFL3, 0.0, 0.1, v0)


def test_solve_brt_rockets20_vs_golden(ctx, golden):
    S = P.rockets(20)
    v0 = golden["brt/rockets20/in"]
    ck, times, steps, secs = ctx.solve_brt(S.grid, S.problem, v0, (-0.5, 0.0), 3, abi.CFL3, abi.make_opts())
    assert_bitwise(ck, golden["brt/rockets20/ck"], "checkpoints")
    assert_bitwise(times, golden["brt/rockets20/times"], "checkpoint times")
    assert_bitwise(steps, golden["brt/rockets20/steps"], "step log")
    assert secs > 0


def test_solve_brt_rockets50_acceptance(ctx, port, sums):
    """acceptance.cpp:381-419: rockets N=50, (-2.5, 0), 11 checkpoints -> 490 steps,
    full step log and final field bit-identical to the reference."""
    S = P.rockets(50)
    v0 = H.initial_value(port, S)
    ck, times, steps, _ = ctx.solve_brt(S.grid, S.problem, v0, (-2.5, 0.0), 11, abi.CFL3, abi.make_opts())
    e = sums["rockets50"]
    assert len(steps) == 490
    assert [[x.hex() for x in row] for row in steps] == e["steps"]
    assert sha(ck[-1]) == e["out"]
    assert np.all(np.diff(ck, axis=0) <= 0.0), "the Grow clamp makes checkpoints non-increasing"


def test_cfg1_full_size_vs_golden(ctx, port, sums):
    """BASELINE configs[0] end to end: 101^2 ENO2 + odeCFL2 over (0, 0.5)."""
    e = sums["integrate/cfg1"]
    S = P.cfg1_circle(101)
    v0 = H.initial_value(port, S)
    v, steps, t = ctx.integrate(S.grid, S.problem, S.method, 0.0, 0.5, v0, abi.make_opts())
    assert sha(v) == e["out"] and len(steps) == e["n_steps"] == 118


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("name,nslabs", [("cfg2", 2), ("cfg2", 3), ("cfg5", 4), ("cfg3", 2), ("cfg1", 5),
                                         ("cfg4", 2), ("cfg2", 4), ("cfg3", 3), ("rotation", 7)])
def test_slabs_equal_single_device_bitwise(ctx, port, monkeypatch, name, nslabs, overlap):
    """P slabs along the last axis == the single-slab result, bit for bit,
    including the step log, in both halo modes: overlapped (ghost planes move
    on a second stream while the interior planes are computed; thin slabs
    (nz <= 2W) take the boundary-only path) and exchange-then-stage (the
    large-slab mode)."""
    monkeypatch.setenv("LSG_HALO_OVERLAP", overlap)
    S = P.CONFIGS[name](**H.small(name))
    v0 = H.initial_value(port, S)
    one = _lib.Solver(ctx, S.grid, S.problem, S.method)
    many = _lib.Solver(ctx, S.grid, S.problem, S.method, nslabs=nslabs)
    one.set_field(v0)
    many.set_field(v0)
    s1, t1 = one.integrate(0.0, 0.04, abi.make_opts())
    s2, t2 = many.integrate(0.0, 0.04, abi.make_opts())
    assert t1 == t2
    assert_bitwise(s1, s2, "step log")
    assert_bitwise(one.get_field(), many.get_field(), "value function")


def test_device_initial_conditions(ctx, port):
    for name in ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "rockets", "rotation"]:
        S = P.CONFIGS[name](**H.small(name))
        s = _lib.Solver(ctx, S.grid, S.problem, S.method)
        shape, center, radius, ignored = S.ic
        s.init_shape(shape, center, radius, ignored)
        assert_bitwise(s.get_field(), H.initial_value(port, S), f"IC {name}")


def test_cfg2_full_size_two_steps_vs_oracle(ctx, port):
    """The bench workload (Air3D 101^3, ENO3 LF + RK3) against the oracle."""
    S = P.cfg2_air3d(101)
    v0 = H.initial_value(port, S)
    solver = _lib.Solver(ctx, S.grid, S.problem, S.method)
    solver.set_field(v0)
    tf = 2 * 0.32 * solver.step_bound()
    sa, ta = solver.integrate(0.0, tf)
    vb, sb, tb = port.integrate(S.grid, S.problem, S.method, 0.0, tf, v0)
    assert len(sa) == len(sb) >= 2
    assert_bitwise(sa, sb, "step log")
    assert_bitwise(solver.get_field(), vb, "v after 2 steps")


def test_cfg5_full_size_properties(ctx):
    """512^3 periodic WENO5 (1.07 GB per field): translating the initial field by
    one node along each periodic axis translates the result bit for bit
    (test_spatial_derivatives.cpp:171-192 lifted to a whole RK3 step), and the
    4-slab decomposition equals the single-slab run."""
    S = P.cfg5_normal(512)
    n = 512
    base = _lib.Solver(ctx, S.grid, S.problem, S.method)
    base.init_shape(*S.ic[:3], S.ic[3])
    v0 = base.get_field()
    dt = 0.32 * base.step_bound()
    base.step(0.0, dt)
    out0 = base.get_field().reshape(n, n, n)
    moved = _lib.Solver(ctx, S.grid, S.problem, S.method)
    for axis in range(3):
        moved.set_field(np.roll(v0.reshape(n, n, n), 1, axis=axis).ravel())
        moved.step(0.0, dt)
        assert_bitwise(moved.get_field(), np.roll(out0, 1, axis=axis).ravel(), f"translation axis {axis}")
    del moved
    slabs = _lib.Solver(ctx, S.grid, S.problem, S.method, nslabs=4)
    slabs.set_field(v0)
    slabs.step(0.0, dt)
    assert_bitwise(slabs.get_field(), out0.ravel(), "4 slabs vs 1")


@pytest.mark.parametrize("counts,periodic", [
    ((300, 20, 9), ()),            # x-segment tiles with x-halo columns, extrapolated edges
    ((300, 20, 9), (0, 1, 2)),     # wrapped x/y halo slots, periodic z window
    ((257, 13, 11), (1,)),         # ragged last x tile (1 column), periodic y only
    ((7, 300, 8), (0, 2)),         # tiny rows: many rows per tile, full-row periodic wrap
    ((33, 7, 7), ()),              # minimum stencil room along y and z
    ((160, 9, 8), (0,)),           # rows too long for full-row tiles: 32-wide segments
    ((250, 11, 7), (2,)),          # ... ragged last segment
])
def test_march3_tilings_vs_oracle(ctx, port, counts, periodic):
    """The 2.5-D tiled 3-D kernel on awkward shapes, all schemes, bit for bit."""
    g = abi.make_grid([-1.0, 0.0, 2.0], [1.0, 3.0, 5.0], list(counts), periodic)
    v = H.random_field(g, sum(counts))
    for s in range(4):
        p = abi.make_problem(abi.HAM_LINEAR, s, abi.linear_params([0.7, -1.1, 0.4]), abi.GROW, s % 2 == 1)
        a, ba = ctx.term_lf(g, p, 0.0, v)
        b, bb = port.term_lf(g, p, 0.0, v)
        assert ba == bb
        assert_bitwise(a, b, f"term scheme {s}")
        va, sa, _ = ctx.integrate(g, p, abi.CFL3, 0.0, 2.5 * 0.32 * ba, v)
        vb, sb, _ = port.integrate(g, p, abi.CFL3, 0.0, 2.5 * 0.32 * bb, v)
        assert_bitwise(sa, sb, f"steps scheme {s}")
        assert_bitwise(va, vb, f"v scheme {s}")


@pytest.mark.parametrize("counts,periodic", [
    ((300, 20, 9), (0, 1, 2)),     # TMA tiles 32x16, chunks of odd and even length
    ((160, 9, 8), (0,)),           # full rows of 160: R = 3 made even for the y pass
    ((250, 11, 7), (2,)),          # ragged last segment
    ((64, 64, 37), (0, 1, 2)),     # z chunks of 5 planes (below): the z pairs' odd last plane
    ((101, 21, 13), ()),           # odd rows: the cp.async tile kernel
])
def test_march3_tilings_fast_weno5_matches_generic(ctx, monkeypatch, counts, periodic):
    """The fast WENO5 on the tile kernels (y pass, z pairs) against the
    one-node-per-thread kernel: the same per-node arithmetic, so the same bits
    (a few RK3 steps)."""
    g = abi.make_grid([-1.0, 0.0, 2.0], [1.0, 3.0, 5.0], list(counts), periodic)
    v = H.random_field(g, sum(counts) + 1)
    p = abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_WENO5, abi.linear_params([0.7, -1.1, 0.4]), abi.GROW, False,
                         options=abi.OPT_WENO5_FAST)
    out = []
    if counts[2] == 37:
        monkeypatch.setenv("LSG_M3_CHUNK", "5")
    for kernel in (None, "generic"):
        if kernel:
            monkeypatch.setenv("LSG_KERNEL", kernel)
        s = _lib.Solver(ctx, g, p, abi.CFL3)
        s.set_field(v)
        dt = 0.32 * s.step_bound()
        log, _ = s.integrate(0.0, 3 * dt)
        out.append((np.asarray(log), s.get_field()))
        s.close()
    assert len(out[0][0]) >= 2
    assert_bitwise(out[0][0], out[1][0], "step log, tiles vs generic")
    assert_bitwise(out[0][1], out[1][1], "v, tiles vs generic")


def test_generic_kernel_3d_still_exact(ctx, port, monkeypatch):
    """LSG_KERNEL=generic forces the one-thread-per-node kernel on 3-D grids."""
    monkeypatch.setenv("LSG_KERNEL", "generic")
    S = P.cfg2_air3d(17)
    v0 = H.initial_value(port, S)
    va, sa, _ = ctx.integrate(S.grid, S.problem, S.method, 0.0, 0.03, v0)
    vb, sb, _ = port.integrate(S.grid, S.problem, S.method, 0.0, 0.03, v0)
    assert_bitwise(sa, sb, "steps")
    assert_bitwise(va, vb, "v")


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5", "rotation"])
def test_weno5_fast_within_tolerance(ctx, port, name):
    """LSG_OPT_WENO5_FAST (one division per side) stays within the north_star
    tolerance of the exact reference: 1e-10 relative (inf-norm) on the value
    function, identical step log (dt does not depend on v)."""
    S = P.CONFIGS[name](**H.small(name))
    fast = abi.make_problem(S.problem.kind, abi.SCHEME_WENO5, list(S.problem.params), S.problem.direction,
                            bool(S.problem.restrict_update), options=abi.OPT_WENO5_FAST)
    v0 = H.initial_value(port, S)
    va, sa, ta = ctx.integrate(S.grid, fast, S.method, 0.0, 0.05, v0)
    vb, sb, tb = port.integrate(S.grid, S.problem, S.method, 0.0, 0.05, v0)
    assert ta == tb and len(sa) == len(sb)
    assert_bitwise(sa[:, :3], sb[:, :3], "t, dt, bound")
    assert rel_inf(va, vb) <= 1e-10, rel_inf(va, vb)
    assert rel_inf(sa[:, 3:], sb[:, 3:]) <= 1e-10
    # sign / zero-level-set membership away from ties
    tie = 1e-9 * np.max(np.abs(vb))
    away = np.abs(vb) > tie
    assert np.array_equal(np.sign(va[away]), np.sign(vb[away]))


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
@pytest.mark.parametrize("profile", ["sin", "linear"])
def test_convergence_study_matches_reference(ctx, ref, scheme, profile):
    """runner.cpp:298-341 (acceptance criterion 1) on the device kernels: the
    table equals the reference's bit for bit and shows the design orders."""
    import ctypes as C
    from paper_2507_11542_b200.studies import convergence_study

    rows = convergence_study(ctx, scheme, 3, profile)
    buf = (C.c_double * 64)()
    n = C.c_int()
    assert ref.lib.ref_convergence_study(scheme, 3, 1 if profile == "sin" else 0, buf, C.byref(n)) == 0
    ref_rows = [tuple(buf[4 * k:4 * k + 4]) for k in range(n.value)]
    assert len(rows) == len(ref_rows) == 4
    for a, b in zip(rows, ref_rows):
        assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]
        assert (np.isnan(a[3]) and np.isnan(b[3])) or a[3] == b[3]
    if profile == "sin":
        assert rows[-1][3] >= {0: 0.9, 1: 1.8, 2: 2.7, 3: 4.3}[scheme]
    else:
        assert rows[-1][2] <= 1e-12


def test_solver_snapshot_roundtrip(ctx, port, tmp_path):
    S = P.cfg2_air3d(21)
    s = _lib.Solver(ctx, S.grid, S.problem, S.method)
    s.init_shape(*S.ic[:3], S.ic[3])
    s.write_snapshot(0.0, tmp_path / "ck.bin")
    g, v, t = _lib.read_snapshot(tmp_path / "ck.bin")
    assert t == 0.0 and g.counts[2] == 21
    assert_bitwise(v, H.initial_value(port, S), "snapshot payload")


def test_cfg3_full_size_slabs(ctx):
    """BASELINE configs[2] at full size (81^4, 344 MB per field, WENO5 exact):
    three slabs with overlapped halo exchange == one slab, bit for bit, after a step."""
    S = P.cfg3_dblint4(81)
    one = _lib.Solver(ctx, S.grid, S.problem, S.method)
    one.init_shape(*S.ic[:3], S.ic[3])
    v0 = one.get_field()
    dt = 0.32 * one.step_bound()
    one.step(0.0, dt)
    a = one.get_field()
    one.close()
    three = _lib.Solver(ctx, S.grid, S.problem, S.method, nslabs=3)
    three.set_field(v0)
    three.step(0.0, dt)
    assert_bitwise(three.get_field(), a, "3 slabs vs 1 at 81^4")
    assert np.all(np.isfinite(a)) and np.all(a <= v0)  # Grow clamp: values only decrease


def test_step_log_capacity_retry(ctx, port):
    """A leg longer than the caller's step log is reported (LSG_ERANGE with the
    needed size) before anything runs; the bindings retry transparently."""
    S = P.cfg1_circle(41)
    v0 = H.initial_value(port, S)
    a = ctx.integrate(S.grid, S.problem, S.method, 0.0, 0.2, v0, log_cap=3)
    b = port.integrate(S.grid, S.problem, S.method, 0.0, 0.2, v0)
    assert len(a[1]) == len(b[1]) > 3
    assert_bitwise(a[0], b[0], "v")
    assert_bitwise(a[1], b[1], "steps")
    ck, times, steps, _ = ctx.solve_brt(S.grid, S.problem, v0, (0.0, 0.2), 3, S.method, log_cap=2)
    rk, rt, rs = port.solve_brt(S.grid, S.problem, v0, (0.0, 0.2), 3, S.method)
    assert_bitwise(ck, rk, "checkpoints")
    assert_bitwise(steps, rs, "steps")


def _ref_zero_set(ref, g, v):
    import ctypes as C

    cap = 1 << 18
    seg = np.empty((cap, 4))
    n, length = C.c_size_t(), C.c_double()
    assert ref.lib.ref_extract_zero_set_2d(C.byref(g), abi.dptr(np.ascontiguousarray(v)), abi.dptr(seg),
                                           C.c_size_t(cap), C.byref(n), C.byref(length)) == 0
    return seg[: n.value], length.value


@pytest.mark.parametrize("case", ["circle", "random_saddles", "cfg1_after_solve"])
def test_zero_set_matches_reference(ctx, port, ref, case):
    """contour.cpp:27-97 on the device: same segments, same order, same bits."""
    if case == "circle":
        S = P.rotation(101)
        g, v = S.grid, H.initial_value(port, S)
    elif case == "random_saddles":
        g = abi.make_grid([-1.0, 0.0], [1.0, 3.0], [37, 29])
        v = H.random_field(g, 5)  # many saddle cells (codes 5 and 10)
    else:
        S = P.cfg1_circle(101)
        g = S.grid
        v, _, _ = ctx.integrate(g, S.problem, S.method, 0.0, 0.5, H.initial_value(port, S))
    seg = ctx.extract_zero_set_2d(g, v)
    rseg, rlen = _ref_zero_set(ref, g, v)
    assert len(seg) == len(rseg) > 0
    assert_bitwise(seg, rseg, "segments")
    length = float(np.hypot(seg[:, 2] - seg[:, 0], seg[:, 3] - seg[:, 1]).sum())
    assert abs(length - rlen) <= 1e-12 * rlen


@pytest.mark.parametrize("case", ["zero_lines", "sprinkled_signed_zeros", "all_zero"])
def test_zero_set_exact_zero_nodes(ctx, port, ref, case):
    """Marching squares with node values exactly +-0.0 (whole zero rows and
    columns, scattered signed zeros, an all-zero field): same segments, order
    and bits as contour.cpp:27-97."""
    g = abi.make_grid([-1.0, -1.0], [1.0, 1.0], [21, 17])  # x = 0 and y = 0 are grid lines
    x = np.array([port.axis(g, 0)[i] for i in range(21)])
    y = np.array([port.axis(g, 1)[j] for j in range(17)])
    X, Y = np.meshgrid(x, y, indexing="xy")  # column-major: index = i + 21 * j
    if case == "zero_lines":
        v = (X * Y).ravel()
    elif case == "sprinkled_signed_zeros":
        v = H.random_field(g, 11)
        rng = np.random.default_rng(4)
        idx = rng.choice(v.size, 60, replace=False)
        v[idx[:30]] = 0.0
        v[idx[30:]] = -0.0
    else:
        v = np.zeros(g.counts[0] * g.counts[1])
    seg = ctx.extract_zero_set_2d(g, v)
    rseg, rlen = _ref_zero_set(ref, g, v)
    assert len(seg) == len(rseg)
    assert_bitwise(seg, rseg, "segments")


def test_slice_2d_matches_reference(ctx, port, ref):
    import ctypes as C

    S = P.cfg2_air3d(21)
    v = H.initial_value(port, S)
    for fixed, idx in [(2, 7), (0, 3), (1, 20)]:
        out = ctx.slice_2d(S.grid, v, fixed, idx)
        r = np.empty_like(out)
        assert ref.lib.ref_slice_2d(C.byref(S.grid), abi.dptr(v), fixed, idx, abi.dptr(r)) == 0
        assert_bitwise(out, r, f"slice {fixed}={idx}")
    with pytest.raises(ValueError):
        ctx.slice_2d(S.grid, v, 2, 21)


def test_stateless_call_cache_limits(ctx, port, monkeypatch):
    """Stateless calls (term, integrate) give identical results whether their
    solver is cached, too large to cache (released when the call returns), or
    caching is off; a solver built afterwards is unaffected."""
    S = P.cfg2_air3d(21)
    v0 = H.initial_value(port, S)
    want_t, want_b = port.term_lf(S.grid, S.problem, 0.0, v0)
    for env in [{}, {"LSG_CALL_CACHE_MAX_BYTES": "1"}, {"LSG_CALL_CACHE": "0"}]:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        for _ in range(2):
            a, b = ctx.term_lf(S.grid, S.problem, 0.0, v0)
            assert b == want_b
            assert_bitwise(a, want_t, f"term {env}")
            va, sa, _ = ctx.integrate(S.grid, S.problem, S.method, 0.0, 0.05, v0)
            vb, sb, _ = port.integrate(S.grid, S.problem, S.method, 0.0, 0.05, v0)
            assert_bitwise(va, vb, f"integrate {env}")
        for k in env:
            monkeypatch.delenv(k)
    s = _lib.Solver(ctx, S.grid, S.problem, S.method)
    s.set_field(v0)
    s.integrate(0.0, 0.05)
    assert_bitwise(s.get_field(), vb, "solver after stateless calls")


@pytest.mark.parametrize("D", [5, 6])
@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_integrate_5d_6d_all_schemes(ctx, port, D, scheme):
    """5-D and 6-D grids through the generic kernel: every scheme, mixed
    periodic axes, clamp on, RK3 and RK2, bit for bit against the oracle."""
    counts = [7, 8, 7, 9, 7, 8][:D]
    g = abi.make_grid([-1.0] * D, [1.0 + 0.1 * d for d in range(D)], counts, (1, D - 1))
    c = [0.4, -0.7, 0.2, 1.1, -0.3, 0.5][:D]
    p = abi.make_problem(abi.HAM_LINEAR, scheme, abi.linear_params(c, offset=0.05), abi.SHRINK, True)
    v = H.random_field(g, 100 * D + scheme)
    for method in (abi.CFL3, abi.CFL2):
        va, sa, ta = ctx.integrate(g, p, method, 0.0, 0.02, v)
        vb, sb, tb = port.integrate(g, p, method, 0.0, 0.02, v)
        assert ta == tb
        assert_bitwise(sa, sb, f"steps D={D} s={scheme}")
        assert_bitwise(va, vb, f"v D={D} s={scheme}")


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("nslabs", [1, 2, 7])
def test_launches_per_step_matches_counted_launches(ctx, monkeypatch, nslabs, overlap):
    """lsg_solver_launches_per_step equals the kernels a step actually launches
    (one per stage, or boundary bands + interior per slab; thin slabs one)."""
    import ctypes as C
    monkeypatch.setenv("LSG_HALO_OVERLAP", overlap)
    S = P.cfg2_air3d(21)
    s = _lib.Solver(ctx, S.grid, S.problem, S.method, nslabs=nslabs)
    s.init_shape(*S.ic[:3], S.ic[3])
    dt = 0.32 * s.step_bound()
    s.step(0.0, dt)  # the first stage after a device write also exchanges halos
    ctx.synchronize()
    before = ctx.launches()
    s.step(dt, dt)
    ctx.synchronize()
    assert ctx.launches() - before == s.launches_per_step()


@pytest.mark.parametrize("scale", [1e-310, 1e-300, 3e-290, 1e76, 1e100, 1e150])
def test_weno5_exact_on_subnormal_differences(ctx, port, scale):
    """Exact WENO5 where its fast divisions leave their exact domain: divided
    differences subnormal or near it (constant divisions), or so large that a
    smoothness denominator exceeds 1e300 or overflows (weights) -- the IEEE
    path takes over, bit for bit with the reference arithmetic (upwind
    derivatives and a full LF term, or the same non-finite-H refusal)."""
    g = abi.make_grid([0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [11, 9, 8], (1,))
    v = H.random_field(g, 5) * scale
    for d in range(3):
        la, ra = ctx.upwind(g, v, d, abi.SCHEME_WENO5)
        lb, rb = port.upwind(g, v, d, abi.SCHEME_WENO5)
        assert_bitwise(la, lb, f"L dim {d}")
        assert_bitwise(ra, rb, f"R dim {d}")
    p = abi.make_problem(abi.HAM_NORMAL, abi.SCHEME_WENO5, [1.0], abi.GROW, False)
    try:
        b, bb = port.term_lf(g, p, 0.0, v)
    except RuntimeError as e:  # |p|^2 overflow: the reference refuses, so must the device
        with pytest.raises(RuntimeError, match=str(e).split(":")[0]):
            ctx.term_lf(g, p, 0.0, v)
        return
    a, ba = ctx.term_lf(g, p, 0.0, v)
    assert ba == bb
    assert_bitwise(a, b, "term")


@pytest.mark.parametrize("kernel,counts,nslabs", [("march3", (21, 13, 11), 1), ("box3", (21, 13, 11), 1),
                                                  ("march3", (21, 13, 11), 3), ("generic", (33, 29), 1)])
@pytest.mark.parametrize("first_negative", [False, True])
@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_step_log_signed_zero_extremes(ctx, port, monkeypatch, kernel, counts, nslabs, first_negative, sign):
    """When a step's minimum (or maximum) is zero and the field holds both
    +0.0 and -0.0, the step log reports the sign of the first zero in index
    order, as the reference's sequential std::min/max does
    (integrator.cpp:87-90).  Zero speed keeps the zeros through the stage."""
    D = len(counts)
    g = abi.make_grid([-1.0] * D, [1.0] * D, list(counts), (D - 1,))
    p = abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_ENO3, abi.linear_params([0.0] * D), abi.GROW, False)
    v = sign * (1.0 + H.random_field(g, 3, 0.0, 1.0))
    n = v.size
    i, j = n // 3, 2 * n // 3
    v[i], v[j] = (-0.0, 0.0) if first_negative else (0.0, -0.0)
    if kernel != "march3":
        monkeypatch.setenv("LSG_KERNEL", kernel)
    for method in (abi.CFL1, abi.CFL2, abi.CFL3):
        s = _lib.Solver(ctx, g, p, method, nslabs=nslabs)
        s.set_field(v)
        sa, ta = s.integrate(0.0, 0.1, abi.make_opts(max_step=0.05))
        vb, sb, tb = port.integrate(g, p, method, 0.0, 0.1, v, abi.make_opts(max_step=0.05))
        assert ta == tb
        assert_bitwise(sa, sb, f"step log {kernel} m={method}")
        assert_bitwise(s.get_field(), vb, f"field {kernel} m={method}")


@pytest.mark.parametrize("dims,nslabs", [(2, 1), (3, 1), (3, 3), (4, 1), (4, 2)])
def test_device_implicit_surface_compositions(ctx, ref, dims, nslabs):
    """rectangle, ellipsoid and the set operations on the device-resident field
    (lsg_solver_apply_shape / _complement) against the reference's own
    implicit_surfaces.cpp functions, bit for bit; the stateless lsg_set_op
    on host fields likewise."""
    counts = [21, 17, 15, 9][:dims]
    g = abi.make_grid([-1.0] * dims, [1.0 + 0.25 * d for d in range(dims)], counts)
    p = abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_FIRST, abi.linear_params([0.0] * dims), abi.GROW, False)
    s = _lib.Solver(ctx, g, p, abi.CFL1, nslabs=nslabs)
    lo, up = [-0.5 + 0.1 * d for d in range(dims)], [0.3 + 0.05 * d for d in range(dims)]
    c = [0.1 * (d + 1) for d in range(dims)]

    s.apply_shape(0, 3, center=lo, upper=up)
    want = ref.rectangle(g, lo, up)
    assert_bitwise(s.get_field(), want, "rectangle")
    s.apply_shape(1, 0, center=c, radius=0.6)                       # union with a sphere
    want = ref.set_op(g, 1, want, ref.sphere(g, c, 0.6))
    assert_bitwise(s.get_field(), want, "rectangle u sphere")
    if dims in (2, 3):
        s.apply_shape(2, 4, radius=0.8)                             # intersection with an ellipsoid
        want = ref.set_op(g, 2, want, ref.ellipsoid(g, 0.8))
        assert_bitwise(s.get_field(), want, "... n ellipsoid")
    s.complement()
    want = ref.set_op(g, 3, want)
    assert_bitwise(s.get_field(), want, "complement")
    s.apply_shape(2, 1, center=c, radius=0.4, ignored_dims=(0,))    # intersection with a cylinder
    want = ref.set_op(g, 2, want, ref.cylinder(g, [0], c, 0.4))
    assert_bitwise(s.get_field(), want, "... n cylinder")
    # stateless set operations on host fields
    b = ref.sphere(g, c, 0.3)
    for op in (1, 2, 3):
        assert_bitwise(ctx.set_op(op, want, b), ref.set_op(g, op, want, b), f"lsg_set_op {op}")


def test_implicit_surface_argument_errors(ctx):
    g = abi.make_grid([-1.0] * 4, [1.0] * 4, [7, 7, 7, 7])
    p = abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_FIRST, abi.linear_params([0.0] * 4), abi.GROW, False)
    s = _lib.Solver(ctx, g, p, abi.CFL1)
    with pytest.raises(ValueError, match="ellipsoid: only 2-D and 3-D"):
        s.apply_shape(0, 4, radius=1.0)
    with pytest.raises(ValueError, match="rectangle: upper must exceed lower"):
        s.apply_shape(0, 3, center=[0.0] * 4, upper=[1.0, 1.0, -1.0, 1.0])


@pytest.mark.parametrize("theta_periodic", [False, True])
def test_rocket_plugins_match_reference(ctx, ref, theta_periodic):
    """lsg_eval_hamiltonian / lsg_eval_dissipation for the rockets kind ==
    the reference's rocket_hamiltonian / rocket_dissipation
    (reachability.cpp:19-66) on random costate fields, bit for bit."""
    S = P.rockets(13, theta_periodic=theta_periodic)
    rng = np.random.default_rng(8)
    cs = [rng.uniform(-3, 3, 13 ** 3) for _ in range(3)]
    h, bounds = ref.rocket_plugins(S.grid, list(S.problem.params)[:5], cs)
    assert_bitwise(ctx.eval_hamiltonian(S.grid, S.problem, cs), h, "H")
    for d in range(3):
        assert_bitwise(ctx.eval_dissipation(S.grid, S.problem, d), bounds[d], f"bound {d}")


def test_concurrent_contexts_from_threads(port):
    """Reentrancy (SPEC: the library is used from several host threads, one
    context each): four threads run stateless and solver integrations on
    their own contexts concurrently (ctypes releases the GIL); every result
    is bit-identical to the oracle's, and errors stay per thread."""
    import threading
    cases = [P.CONFIGS[n](**H.small(n)) for n in ("cfg1", "cfg2", "cfg5", "rotation")]
    want = []
    for S in cases:
        v0 = H.initial_value(port, S)
        want.append((v0, port.integrate(S.grid, S.problem, S.method, 0.0, 0.03, v0)))
    results, errors = [None] * len(cases), []

    def work(k):
        try:
            c = _lib.Context(0)
            S, (v0, (vb, sb, tb)) = cases[k], want[k]
            for _ in range(3):
                va, sa, ta = c.integrate(S.grid, S.problem, S.method, 0.0, 0.03, v0)
                s = _lib.Solver(c, S.grid, S.problem, S.method)
                s.set_field(v0)
                ss, ts = s.integrate(0.0, 0.03)
                results[k] = (va, sa, ta, s.get_field(), ss, ts)
                s.close()
                try:  # an error on this thread reports this thread's message
                    c.integrate(S.grid, S.problem, S.method, 1.0, 0.0, v0)
                except ValueError as e:
                    assert "tspan must not be decreasing" in str(e)
            c.close()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k, (v0, (vb, sb, tb)) in enumerate(want):
        va, sa, ta, vs, ss, ts = results[k]
        assert ta == tb and ts == tb
        assert_bitwise(sa, sb, f"steps {k}")
        assert_bitwise(va, vb, f"v {k}")
        assert_bitwise(ss, sb, f"solver steps {k}")
        assert_bitwise(vs, vb, f"solver v {k}")


def test_index_division_paths_bitwise(ctx, monkeypatch):
    """The generic kernel decomposes node indices with the 31-bit multiplier
    division (divmod31) where the dividends fit 31 bits, and with the 64-bit
    double-reciprocal division otherwise (slabs of more than 2^31 nodes take
    it for the first axis only).  LSG_DIV31 forces each combination: all three
    give the same fields bit for bit (6-D ENO3 and WENO5, 4-D WENO5, 1 and 3 slabs)."""
    cases = {
        "cfg4_eno3": (P.cfg4_dubins6(13, scheme=abi.SCHEME_ENO3), 1),
        "cfg4_weno5": (P.cfg4_dubins6(11), 3),
        "cfg3": (P.cfg3_dblint4(25), 1),
    }
    out = {}
    for mask in ("0", "2", "3"):
        monkeypatch.setenv("LSG_DIV31", mask)
        for name, (S, nslabs) in cases.items():
            s = _lib.Solver(ctx, S.grid, S.problem, S.method, nslabs=nslabs)
            s.init_shape(*S.ic[:3], S.ic[3])
            dt = 0.32 * s.step_bound()
            s.step(0.0, dt)
            s.step(dt, dt)
            out[mask, name] = s.get_field()
            s.close()
    for name in cases:
        assert_bitwise(out["0", name], out["3", name], f"{name}: 64-bit vs 31-bit division")
        assert_bitwise(out["2", name], out["3", name], f"{name}: mixed vs 31-bit division")


def test_cfg4_full_size_slabs_step_log(ctx):
    """BASELINE configs[3] at full size: 41^6 = 4.75 G nodes (38 GB per field),
    exact WENO5, with RK2 so both decompositions fit in HBM one after the other
    (76 GB for one slab, 109 GB for three with their halo planes).  One slab
    (node indices above 2^31: 64-bit first-axis division) and three slabs
    (31-bit division, NCCL-free device halo copies) give bit-identical step logs
    over two steps: every entry holds the exact min and max of all 4.75 G values
    and the dt, so a single differing node would show."""
    S = P.cfg4_dubins6(41)
    out = []
    for nslabs in (1, 3):
        s = _lib.Solver(ctx, S.grid, S.problem, abi.CFL2, nslabs=nslabs)
        s.init_shape(*S.ic[:3], S.ic[3])
        tf = 2 * 0.32 * s.step_bound()
        log, t = s.integrate(0.0, tf)
        out.append((np.asarray(log, dtype=np.float64), t))
        s.close()
    assert len(out[0][0]) >= 2
    assert_bitwise(out[0][0], out[1][0], "step log at 41^6, 1 vs 3 slabs")
    assert out[0][1] == out[1][1]
    assert np.all(np.isfinite(out[0][0]))


@pytest.mark.parametrize("dims,periodic", [((9, 8, 7, 8), ()), ((9, 8, 7, 10), (1, 3)), ((8, 7, 7, 7, 7, 8), (2, 5)),
                                           ((7, 9, 7, 7, 7, 7), (0, 1, 2, 3, 4, 5))])
@pytest.mark.parametrize("nslabs", [1, 2])
def test_marchn_kernel_vs_oracle(ctx, port, monkeypatch, dims, periodic, nslabs):
    """LSG_KERNEL=marchn: the 4-D/6-D tile-and-march kernel (lsg_marchn.cuh) for
    every scheme, both clamps, slabs, bit for bit against the oracle (linear
    Hamiltonian in 4-D, the cfg4 Dubins Hamiltonian in 6-D)."""
    monkeypatch.setenv("LSG_KERNEL", "marchn")
    D = len(dims)
    g = abi.make_grid([-1.0] * D, [1.0] * D, list(dims), periodic)
    v = H.random_field(g, sum(dims) + nslabs)
    for s in range(4):
        if D == 4:
            p = abi.make_problem(abi.HAM_LINEAR, s, abi.linear_params([0.7, -1.1, 0.4, 0.9]), abi.GROW, s % 2 == 1)
        else:
            p = abi.make_problem(abi.HAM_DUBINS6, s, [], abi.GROW, s % 2 == 1)
        sol = _lib.Solver(ctx, g, p, abi.CFL3, nslabs=nslabs)
        sol.set_field(v)
        tf = 2.5 * 0.32 * sol.step_bound()
        sa, _ = sol.integrate(0.0, tf)
        va = sol.get_field()
        sol.close()
        vb, sb, _ = port.integrate(g, p, abi.CFL3, 0.0, tf, v)
        assert_bitwise(sa, sb, f"steps scheme {s}")
        assert_bitwise(va, vb, f"v scheme {s}")


def test_solve_brt_resume_from_snapshot(ctx, port, tmp_path):
    """A checkpointed solve_brt resumed from its checkpoint-5 snapshot file
    (reference format, snapshot.cpp:68-129) reproduces the uninterrupted run's
    later checkpoints and step log bit for bit (resume: SURVEY §5)."""
    S = P.rockets(20)
    v0 = port.rocket_initial(20) if hasattr(port, "rocket_initial") else None
    if v0 is None:
        s = _lib.Solver(ctx, S.grid, S.problem, S.method)
        s.init_shape(*S.ic[:3], S.ic[3])
        v0 = s.get_field()
        s.close()
    ck, times, steps, _ = ctx.solve_brt(S.grid, S.problem, v0, S.tspan, S.n_checkpoints)
    k = 5
    path = tmp_path / "ck5.snap"
    _lib.write_snapshot(S.grid, ck[k], times[k], path)
    g2, vk, tk = _lib.read_snapshot(path)
    assert tk == times[k]
    rk, rtimes, rsteps, _ = ctx.solve_brt_resume(S.grid, S.problem, vk, k, tk, S.tspan, S.n_checkpoints)
    assert_bitwise(rk, ck[k:], "checkpoints k..n-1")
    assert_bitwise(rtimes, times[k:], "checkpoint times")
    first = int(np.searchsorted(steps[:, 0], tk))
    assert_bitwise(rsteps, steps[first:], "remaining step log")
