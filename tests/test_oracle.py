"""CPU tests: pin the oracle before trusting it.

The C restatement (oracle/levelset_oracle.c) must equal, bit for bit,
(1) the committed golden vectors made from the reference library itself
(tests/golden/make_golden.py), (2) the reference library compiled from its
own sources (oracle/_ref, when present), and (3) the known-answer tests of the
reference's own doctest suite (/root/reference/proj/tests/test_*.cpp).
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import assert_bitwise
from paper_2507_11542_b200 import abi
from paper_2507_11542_b200 import problems as P
import helpers as H

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


# ---- golden vectors (made from the reference) ------------------------------

def test_golden_pad_ghost(port, golden):
    g = abi.make_grid([0.0] * 3, [1.0] * 3, [5, 6, 7], [0, 1, 2])
    for d in range(3):
        assert_bitwise(port.pad_ghost(g, golden["pad/periodic/in"], d, 2), golden[f"pad/periodic/d{d}"], f"periodic d{d}")
    g = abi.make_grid([0.0] * 3, [1.0] * 3, [5, 6, 7])
    for d in range(3):
        assert_bitwise(port.pad_ghost(g, golden["pad/extrap/in"], d, 3), golden[f"pad/extrap/d{d}"], f"extrap d{d}")


@pytest.mark.parametrize("key", ["A", "B", "C"])
def test_golden_upwind(port, golden, key):
    from golden.make_golden import UPWIND_GRIDS

    g, _ = UPWIND_GRIDS[key]
    v = golden[f"upwind/{key}/in"]
    for s in range(4):
        for d in range(g.dim):
            L, R = port.upwind(g, v, d, s)
            assert_bitwise(L, golden[f"upwind/{key}/s{s}/d{d}/L"], f"{key} s{s} d{d} L")
            assert_bitwise(R, golden[f"upwind/{key}/s{s}/d{d}/R"], f"{key} s{s} d{d} R")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "rockets", "rotation"])
def test_golden_term(port, golden, sums, name):
    S = P.CONFIGS[name](**H.small(name))
    v0 = H.initial_value(port, S)
    e = sums[f"term/{name}"]
    assert sha(v0) == e["in"], "initial condition differs from the reference's"
    dvdt, bound = port.term_lf(S.grid, S.problem, 0.0, v0)
    assert sha(dvdt) == e["dvdt"]
    assert bound.hex() == e["bound"]


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5", "rotation"])
def test_golden_integrate(port, sums, name):
    e = sums[f"integrate/{name}"]
    S = P.CONFIGS[name](**e["kw"])
    v0 = H.initial_value(port, S)
    assert sha(v0) == e["in"]
    v, steps, tfin = port.integrate(S.grid, S.problem, S.method, 0.0, e["tf"], v0, abi.make_opts())
    assert len(steps) == e["n_steps"]
    assert [[x.hex() for x in row] for row in steps] == e["steps"]
    assert tfin.hex() == e["t_final"]
    assert sha(v) == e["out"]


def test_golden_brt_rockets20(port, golden):
    S = P.rockets(20)
    v0 = golden["brt/rockets20/in"]
    assert_bitwise(H.initial_value(port, S), v0, "rocket IC")
    ck, times, steps = port.solve_brt(S.grid, S.problem, v0, (-0.5, 0.0), 3, abi.CFL3, abi.make_opts())
    assert_bitwise(ck, golden["brt/rockets20/ck"], "checkpoints")
    assert_bitwise(times, golden["brt/rockets20/times"], "times")
    assert_bitwise(steps, golden["brt/rockets20/steps"], "step log")


# ---- differential against the compiled reference ----------------------------

@pytest.mark.parametrize("periodic", [(), (0,), (1, 2), (0, 1, 2)])
def test_port_vs_reference_upwind(port, ref, periodic):
    g = abi.make_grid([0.0, -1.0, 2.0], [1.0, 1.0, 3.0], [8, 9, 7], periodic)
    v = H.random_field(g, 5)
    for s in range(4):
        for d in range(3):
            a, b = port.upwind(g, v, d, s), ref.upwind(g, v, d, s)
            assert_bitwise(a[0], b[0], f"L s{s} d{d}")
            assert_bitwise(a[1], b[1], f"R s{s} d{d}")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "rotation"])
def test_port_vs_reference_integrate(port, ref, name):
    S = P.CONFIGS[name](**H.small(name))
    v0 = H.initial_value(ref, S)
    tf = 0.02
    a = port.integrate(S.grid, S.problem, S.method, 0.0, tf, v0, abi.make_opts())
    b = ref.integrate(S.grid, S.problem, S.method, 0.0, tf, v0, abi.make_opts())
    assert_bitwise(a[0], b[0], "v")
    assert_bitwise(a[1], b[1], "steps")
    assert a[2] == b[2]


def test_port_vs_reference_checkpoints_and_errors(port, ref):
    S = P.cfg1_circle(21)
    v0 = H.initial_value(ref, S)
    o = abi.make_opts(checkpoint_times=[0.013, 0.05])
    a = port.integrate(S.grid, S.problem, abi.CFL1, 0.0, 0.08, v0, o)
    b = ref.integrate(S.grid, S.problem, abi.CFL1, 0.0, 0.08, v0, o)
    assert_bitwise(a[1], b[1], "steps")
    assert 0.013 in a[1][:, 0] and 0.05 in a[1][:, 0]
    for bad in [abi.make_opts(cfl_factor=0.0), abi.make_opts(max_step=-1.0),
                abi.make_opts(checkpoint_times=[0.5, 0.2])]:
        for chk in (port, ref):
            with pytest.raises(ValueError):
                chk.integrate(S.grid, S.problem, abi.CFL1, 0.0, 1.0, v0, bad)
    for chk in (port, ref):
        with pytest.raises(ValueError):
            chk.integrate(S.grid, S.problem, abi.CFL1, 1.0, 0.0, v0)
        with pytest.raises(ValueError):
            chk.integrate(S.grid, S.problem, abi.CFL1, 0.0, math.inf, v0)


# ---- the reference's own known-answer tests, on both checkers ----------------

@pytest.fixture(params=["port", "ref"])
def checker(request, port):
    if request.param == "port":
        return port
    return request.getfixturevalue("ref")


def test_kat_pad_ghost(checker):
    # test_grid.cpp:96-114
    g = abi.make_grid([0.0], [3.0], [4], [0])
    assert list(checker.pad_ghost(g, np.array([1.0, 2, 3, 4]), 0, 1)) == [4.0, 1, 2, 3, 4, 1]
    g = abi.make_grid([0.0], [3.0], [4])
    assert list(checker.pad_ghost(g, np.array([0.0, 1, 2, 3]), 0, 2)) == [-2.0, -1, 0, 1, 2, 3, 4, 5]
    # test_grid.cpp:165-171
    g = abi.make_grid([0.0], [1.0], [4])
    for dim, width in [(0, 4), (0, 0), (1, 1)]:
        with pytest.raises(ValueError):
            checker.pad_ghost(g, np.zeros(4), dim, width)


def test_kat_shift(checker):
    # test_grid.cpp:173-189
    g = abi.make_grid([0.0], [3.0], [4], [0])
    p = checker.pad_ghost(g, np.array([1.0, 2, 3, 4]), 0, 1)
    assert list(checker.shift_along_dim(g, p, 0, 1, 1)) == [2.0, 3, 4, 1]
    assert list(checker.shift_along_dim(g, p, 0, 1, -1)) == [4.0, 1, 2, 3]
    with pytest.raises(ValueError):
        checker.shift_along_dim(g, p, 0, 1, 2)


def test_kat_derivatives(checker):
    # test_spatial_derivatives.cpp:58-66: x^2 on dx = 0.5 -> 1.5 / 2.5 at x = 1
    g = abi.make_grid([0.0], [2.0], [5])
    x = checker.axis(g, 0)
    L, R = checker.upwind(g, x * x, 0, abi.SCHEME_FIRST)
    assert L[2] == pytest.approx(1.5, rel=1e-14) and R[2] == pytest.approx(2.5, rel=1e-14)
    # :68-83 linear exact, constant zero
    g = abi.make_grid([-1.0], [1.0], [9])
    x = checker.axis(g, 0)
    for s in range(4):
        L, R = checker.upwind(g, 3.0 * x, 0, s)
        assert np.allclose(L, 3.0, rtol=1e-12) and np.allclose(R, 3.0, rtol=1e-12)
        L, R = checker.upwind(g, np.full(9, 4.25), 0, s)
        assert np.allclose(L, 0.0, atol=1e-12) and np.allclose(R, 0.0, atol=1e-12)
    # :114-133 ENO2 step data
    g = abi.make_grid([0.0], [7.0], [8])
    L, R = checker.upwind(g, np.array([0.0, 0, 0, 0, 1, 1, 1, 1]), 0, abi.SCHEME_ENO2)
    assert abs(L[6]) <= 1e-14 and abs(R[5]) <= 1e-14
    # :135-144 ENO3 cubic exact in the interior
    g = abi.make_grid([-1.0], [1.0], [33])
    x = checker.axis(g, 0)
    L, R = checker.upwind(g, x * x * x, 0, abi.SCHEME_ENO3)
    assert np.allclose(L[3:-3], 3 * x[3:-3] ** 2, rtol=1e-10) and np.allclose(R[3:-3], 3 * x[3:-3] ** 2, rtol=1e-10)
    # :230-237 stencil room
    g = abi.make_grid([0.0], [1.0], [5])
    checker.upwind(g, np.zeros(5), 0, abi.SCHEME_ENO2)
    for s, dim in [(abi.SCHEME_ENO3, 0), (abi.SCHEME_WENO5, 0), (abi.SCHEME_FIRST, 1)]:
        with pytest.raises(ValueError):
            checker.upwind(g, np.zeros(5), dim, s)


def test_kat_orders(checker):
    # test_spatial_derivatives.cpp:164-169 on sin(2 pi x), periodic
    want = {abi.SCHEME_FIRST: 0.9, abi.SCHEME_ENO2: 1.8, abi.SCHEME_ENO3: 2.7, abi.SCHEME_WENO5: 4.3}
    for s, order in want.items():
        errs = []
        for n in (64, 128):
            g = abi.make_grid([0.0], [1.0 - 1.0 / n], [n], [0])
            x = checker.axis(g, 0)
            L, R = checker.upwind(g, np.sin(2 * math.pi * x), 0, s)
            truth = 2 * math.pi * np.cos(2 * math.pi * x)
            errs.append(max(np.abs(L - truth).max(), np.abs(R - truth).max()))
        assert math.log2(errs[0] / errs[1]) >= order


def test_kat_bitwise_translation_and_reversal(checker):
    # test_spatial_derivatives.cpp:171-213
    g = abi.make_grid([0.0, 0.0], [1.0, 1.0], [16, 12], [0, 1])
    v = H.random_field(g, 7).reshape(12, 16)
    for dim in range(2):
        axis = 1 - dim  # numpy (row-major reshape of column-major data): dim 0 is the last numpy axis
        moved = np.roll(v, -1, axis=axis)
        for s in range(4):
            bL, bR = checker.upwind(g, v.ravel(), dim, s)
            mL, mR = checker.upwind(g, moved.ravel(), dim, s)
            assert_bitwise(mL, np.roll(bL.reshape(12, 16), -1, axis=axis).ravel(), "translate L")
            assert_bitwise(mR, np.roll(bR.reshape(12, 16), -1, axis=axis).ravel(), "translate R")
    for periodic in ((), (0,)):
        g = abi.make_grid([-1.0], [1.0], [24], periodic)
        v = H.random_field(g, 41)
        for s in range(4):
            vL, vR = checker.upwind(g, v, 0, s)
            wL, wR = checker.upwind(g, v[::-1].copy(), 0, s)
            assert_bitwise(wL, -vR[::-1], "reverse L")
            assert_bitwise(wR, -vL[::-1], "reverse R")


def _linear(c, bounds=None, offset=0.0, scheme=abi.SCHEME_ENO2, clamp=False, direction=abi.GROW):
    return abi.make_problem(abi.HAM_LINEAR, scheme, abi.linear_params(c, bounds, offset), direction, clamp)


def test_kat_term(checker):
    # test_hamiltonian.cpp:54-60: bound 0.05
    g = abi.make_grid([0.0], [1.0], [11])
    _, b = checker.term_lf(g, _linear([2.0]), 0.0, np.zeros(11))
    assert b == pytest.approx(0.05, rel=1e-14)
    # :62-69 multi-dim
    g = abi.make_grid([0.0, 0.0], [1.0, 2.0], [11, 21])
    _, b = checker.term_lf(g, _linear([3.0, 0.5]), 0.0, np.ones(231))
    assert b * (3.0 / 0.1 + 0.5 / 0.1) == pytest.approx(1.0, rel=1e-14)
    # :71-76 zero dissipation -> +inf
    g = abi.make_grid([0.0], [1.0], [11])
    _, b = checker.term_lf(g, _linear([0.0]), 0.0, np.zeros(11))
    assert b == math.inf
    # :78-93 H sees the central costate
    g = abi.make_grid([0.0], [2.0], [5])
    x = checker.axis(g, 0)
    d, _ = checker.term_lf(g, _linear([1.0], bounds=[0.0], scheme=abi.SCHEME_FIRST), 0.0, x * x)
    assert d[2] == pytest.approx(-2.0, rel=1e-14)
    # :135-165 dyadic linear data: zero dissipation, bitwise dvdt == -H
    g = abi.make_grid([0.0], [1.0], [17])
    x = checker.axis(g, 0)
    d, _ = checker.term_lf(g, _linear([0.25], bounds=[0.25], offset=0.125), 0.0, 1.5 * x)
    assert np.all(d == -(0.25 * 1.5 + 0.125))
    # :110-133 clamp: Grow = min(free, 0), bound unchanged
    g = abi.make_grid([0.0], [1.0 - 1.0 / 32], [32], [0])
    v = np.sin(2 * math.pi * checker.axis(g, 0))
    free, bf = checker.term_lf(g, _linear([1.0]), 0.0, v)
    clamped, bc = checker.term_lf(g, _linear([1.0], clamp=True), 0.0, v)
    assert (free > 0).any() and np.all(clamped == np.minimum(free, 0.0)) and bf == bc
    # :95-108 restrict_update goldens
    assert list(checker.restrict_update(np.array([-2.0, 0.0, 3.0]), abi.GROW)) == [-2.0, 0.0, 0.0]
    assert list(checker.restrict_update(np.array([-2.0, 0.0, 3.0]), abi.SHRINK)) == [0.0, 0.0, 3.0]
    # :167-193 non-finite H and invalid bounds abort
    g = abi.make_grid([0.0], [1.0], [5])
    with pytest.raises(RuntimeError):
        checker.term_lf(g, _linear([math.nan]), 0.0, np.ones(5))
    with pytest.raises(RuntimeError):
        checker.term_lf(g, _linear([1.0], bounds=[-1.0]), 0.0, np.ones(5))
    with pytest.raises(RuntimeError):
        checker.term_lf(g, _linear([1.0], bounds=[math.inf]), 0.0, np.ones(5))


def test_kat_integrator(checker):
    # test_integrator.cpp:111-133: dt <= cfl*bound, <= max_step, exact t bookkeeping
    g = abi.make_grid([0.0], [1.0 - 1.0 / 64], [64], [0])
    v0 = np.sin(2 * math.pi * checker.axis(g, 0))
    p = _linear([1.0], scheme=abi.SCHEME_FIRST)
    o = abi.make_opts(cfl_factor=0.5, max_step=0.009)
    v, steps, tf = checker.integrate(g, p, abi.CFL3, 0.0, 0.25, v0, o)
    assert tf == 0.25 and len(steps)
    t = 0.0
    for e in steps:
        assert e[0] == t and 0 < e[1] <= 0.5 * e[2] and e[1] <= 0.009
        t = e[0] + e[1]
    # :184-202 determinism
    a = checker.integrate(g, _linear([-0.6], scheme=abi.SCHEME_FIRST), abi.CFL3, 0.0, 0.5, v0)
    b = checker.integrate(g, _linear([-0.6], scheme=abi.SCHEME_FIRST), abi.CFL3, 0.0, 0.5, v0)
    assert_bitwise(a[0], b[0]) and assert_bitwise(a[1], b[1])
    # :204-214 zero-length span
    v, steps, tf = checker.integrate(g, p, abi.CFL2, 4.0, 4.0, v0)
    assert tf == 4.0 and len(steps) == 0 and np.array_equal(v, v0)
    # :238-244 a vanishing bound (here: alpha -> inf makes the bound 0) aborts
    with pytest.raises(RuntimeError):
        checker.integrate(g, _linear([1.0], bounds=[1e308], scheme=abi.SCHEME_FIRST), abi.CFL1, 0.0, 1.0, v0,
                          abi.make_opts(cfl_factor=1e-300))


def test_kat_tvd(checker):
    # test_integrator.cpp:156-182: TV does not grow for upwinded step advection
    n = 80
    g = abi.make_grid([0.0], [1.0 - 1.0 / n], [n], [0])
    x = checker.axis(g, 0)
    v0 = np.where((x >= 0.25) & (x < 0.65), 1.0, 0.0)
    p = _linear([1.0], scheme=abi.SCHEME_FIRST)
    for m in (abi.CFL2, abi.CFL3):
        v, tv_prev = v0, 2.0
        for _ in range(60):
            dt = 0.32 / (1.0 / (x[1] - x[0]))
            v, steps, _ = checker.integrate(g, p, m, 0.0, dt, v, abi.make_opts(max_step=dt))
            assert len(steps) == 1
            tv = np.abs(np.roll(v, -1) - v).sum()
            assert tv <= tv_prev + 1e-10
            tv_prev = tv


def test_kat_rockets(checker):
    # test_reachability.cpp:166-206 wiring: cylinder radius 1.5 around the theta axis
    S = P.rockets(9)
    v0 = H.initial_value(checker, S)
    center = 4 + 9 * 4
    assert v0[center] == pytest.approx(-1.5, rel=1e-15)
    for k in range(9):
        assert v0[6 + 9 * 4 + 81 * k] == pytest.approx(32.0 - 1.5, rel=1e-15)
    # :232-257 backward span, monotone under the Grow clamp
    ck, times, steps = checker.solve_brt(S.grid, S.problem, v0, (-0.1, 0.0), 3, abi.CFL3, abi.make_opts())
    assert len(ck) == 3 and times[0] == 0.0 and times[2] == pytest.approx(0.1, rel=1e-15) and len(steps)
    assert np.all(ck[1] <= ck[0]) and np.all(ck[2] <= ck[1])
    ck, times, steps = checker.solve_brt(S.grid, S.problem, v0, (0.0, 0.0), 5)
    assert len(ck) == 1 and len(steps) == 0
    with pytest.raises(ValueError):
        checker.solve_brt(S.grid, S.problem, v0, (0.0, 1.0), 0)


@pytest.mark.slow
def test_kat_rockets_acceptance_490_steps(port, sums):
    """acceptance.cpp:381-419 (criterion 5): the reference takes 490 steps; the
    port must reproduce the full step log and final field bit for bit."""
    S = P.rockets(50)
    v0 = H.initial_value(port, S)
    ck, times, steps = port.solve_brt(S.grid, S.problem, v0, (-2.5, 0.0), 11, abi.CFL3, abi.make_opts())
    e = sums["rockets50"]
    assert len(steps) == e["n_steps"] == 490
    assert [[x.hex() for x in row] for row in steps] == e["steps"]
    assert sha(ck[-1]) == e["out"]


@pytest.mark.parametrize("dims", [2, 3, 4])
def test_port_vs_reference_implicit_surfaces(port, ref, dims):
    """rectangle / ellipsoid / set_union / set_intersection / set_complement
    (implicit_surfaces.cpp:73-151): restatement == compiled reference, bit for
    bit, signed zeros and NaN operands of the set operations included."""
    g = abi.make_grid([-1.0] * dims, [1.0 + 0.25 * d for d in range(dims)], [9, 8, 7, 6][:dims])
    lo, up = [-0.5 + 0.1 * d for d in range(dims)], [0.3 + 0.05 * d for d in range(dims)]
    assert_bitwise(port.rectangle(g, lo, up), ref.rectangle(g, lo, up), "rectangle")
    if dims in (2, 3):
        assert_bitwise(port.ellipsoid(g, 0.7), ref.ellipsoid(g, 0.7), "ellipsoid")
    rng = np.random.default_rng(dims)
    n = int(np.prod([9, 8, 7, 6][:dims]))
    a, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    a[:4], b[:4] = [0.0, -0.0, 0.0, np.nan], [-0.0, 0.0, 0.0, 1.0]
    b[4] = np.nan
    for op in (1, 2, 3):
        assert_bitwise(port.set_op(g, op, a, b), ref.set_op(g, op, a, b), f"set op {op}")
