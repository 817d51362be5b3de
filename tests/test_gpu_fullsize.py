"""GPU parity at the BASELINE configs' own sizes (SURVEY §8(c) protocol).

* One RK3 step of cfg3 (81^4, 43 M nodes) and cfg5 (512^3, 134 M nodes) with
  the bit-exact WENO5 against the reference compiled from its own sources
  (oracle/_ref): value function and step log bit for bit.
* cfg4 (6-D Dubins) at 17^6 (24 M nodes, the reduced size SURVEY §8(c)
  prescribes), RK3, several steps against the oracle, bit for bit.
* cfg4 at its full 41^6 (4.75 G nodes, 38 GB per field) with RK3: one slab
  vs three slabs (halo exchange), bit-identical step logs (exact min/max over
  all nodes per step) and final fields (compared by checksum).
* The tolerance path (LSG_OPT_WENO5_FAST) over each config's full tspan at a
  reduced size: <= 1e-10 relative (inf-norm) and identical sign membership
  away from ties after the final step (north_star).

The reference needs ~20 GB of host memory and ~1-2 minutes for the 512^3 step.
"""
import numpy as np
import pytest

from conftest import assert_bitwise, rel_inf
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P
import helpers as H

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _one_step_vs_reference(ctx, ref, S):
    v0 = H.initial_value(ref, S)
    solver = _lib.Solver(ctx, S.grid, S.problem, S.method)
    solver.set_field(v0)
    tf = 0.32 * solver.step_bound()
    sa, ta = solver.integrate(0.0, tf)
    va = solver.get_field()
    solver.close()
    vb, sb, tb = ref.integrate(S.grid, S.problem, S.method, 0.0, tf, v0)
    assert len(sa) == len(sb) == 1 and ta == tb
    assert_bitwise(sa, sb, "step log")
    assert_bitwise(va, vb, "v after one RK3 step")
    return va


def test_cfg3_81_one_rk3_step_vs_reference(ctx, ref):
    """BASELINE configs[2] at full size: 81^4 double integrator, WENO5 LF + RK3, Grow clamp
    (integrator.cpp:70-85, spatial_derivatives.cpp:78-97)."""
    v = _one_step_vs_reference(ctx, ref, P.cfg3_dblint4(81))
    assert np.all(np.isfinite(v))


def test_cfg5_512_one_rk3_step_vs_reference(ctx, ref):
    """BASELINE configs[4] at full size (the bench workload): 512^3 periodic normal
    motion, WENO5 LF + RK3."""
    v = _one_step_vs_reference(ctx, ref, P.cfg5_normal(512))
    assert np.all(np.isfinite(v))


def test_cfg4_17_rk3_steps_vs_oracle(ctx, port):
    """BASELINE configs[3] at the reduced size SURVEY §8(c) names (17^6), exact
    WENO5, RK3, three steps, against the C oracle (pinned to the reference)."""
    S = P.cfg4_dubins6(17)
    v0 = H.initial_value(port, S)
    solver = _lib.Solver(ctx, S.grid, S.problem, S.method)
    solver.set_field(v0)
    tf = 3 * 0.32 * solver.step_bound()
    sa, ta = solver.integrate(0.0, tf)
    va = solver.get_field()
    solver.close()
    vb, sb, tb = port.integrate(S.grid, S.problem, S.method, 0.0, tf, v0)
    assert len(sa) == len(sb) >= 3 and ta == tb
    assert_bitwise(sa, sb, "step log")
    assert_bitwise(va, vb, "v after three RK3 steps")


def test_cfg4_41_full_size_rk3_one_vs_three_slabs(ctx):
    """41^6 (4.75 G nodes), exact WENO5, RK3 (3 x 38 GB for one slab, ~164 GB for
    three slabs with their ghost planes, built one after the other): two steps
    give bit-identical step logs and identical field checksums."""
    S = P.cfg4_dubins6(41)
    out = []
    for nslabs in (1, 3):
        s = _lib.Solver(ctx, S.grid, S.problem, abi.CFL3, nslabs=nslabs)
        s.init_shape(*S.ic[:3], S.ic[3])
        tf = 2 * 0.32 * s.step_bound()
        log, t = s.integrate(0.0, tf)
        fp = _checksum(s.get_field())  # 38 GB to host (the box has the RAM), fingerprinted, dropped
        out.append((np.asarray(log, dtype=np.float64), t, fp))
        s.close()
    assert len(out[0][0]) >= 2
    assert_bitwise(out[0][0], out[1][0], "step log at 41^6, 1 vs 3 slabs")
    assert out[0][1] == out[1][1]
    assert out[0][2] == out[1][2], "final field checksums differ (1 vs 3 slabs)"
    assert np.all(np.isfinite(out[0][0]))


def _checksum(v):
    """(sum of the bit patterns, sum of the bit patterns xor a position hash),
    both mod 2^64, in chunks: a fingerprint of a 4.75 G-value field."""
    bits = v.view(np.uint64)
    chunk = 1 << 26
    s1 = s2 = 0
    for off in range(0, bits.size, chunk):
        b = bits[off:off + chunk]
        pos = np.arange(off, off + b.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C1)
        s1 = (s1 + int(b.sum(dtype=np.uint64))) % (1 << 64)
        s2 = (s2 + int(np.bitwise_xor(b, pos).sum(dtype=np.uint64))) % (1 << 64)
    return s1, s2


@pytest.mark.parametrize("name,kw", [("cfg3", dict(n=11)), ("cfg4", dict(n=9)), ("cfg5", dict(n=32)),
                                     ("rotation", dict(n=41))])
def test_weno5_fast_full_tspan_within_tolerance(ctx, port, name, kw):
    """The tolerance path over the config's whole tspan (north_star: value
    function within 1e-10 relative after the final step; identical sign /
    zero-level-set membership away from ties)."""
    S = P.CONFIGS[name](**kw)
    fast = abi.make_problem(S.problem.kind, abi.SCHEME_WENO5, list(S.problem.params), S.problem.direction,
                            bool(S.problem.restrict_update), options=abi.OPT_WENO5_FAST)
    v0 = H.initial_value(port, S)
    t0, tf = S.tspan
    va, sa, ta = ctx.integrate(S.grid, fast, S.method, 0.0, tf - t0, v0)
    vb, sb, tb = port.integrate(S.grid, S.problem, S.method, 0.0, tf - t0, v0)
    assert ta == tb and len(sa) == len(sb) >= 10
    assert_bitwise(sa[:, :3], sb[:, :3], "t, dt, bound")
    err = rel_inf(va, vb)
    assert err <= 1e-10, err
    assert rel_inf(sa[:, 3:], sb[:, 3:]) <= 1e-10
    tie = 1e-9 * np.max(np.abs(vb))
    away = np.abs(vb) > tie
    assert np.array_equal(np.sign(va[away]), np.sign(vb[away]))


@pytest.mark.parametrize("name,kw", [("cfg2", dict(n=51)), ("cfg3", dict(n=21)), ("cfg4", dict(n=9)),
                                     ("cfg5", dict(n=32)), ("cfg1", dict(n=101))])
def test_full_tspan_bitwise_vs_oracle(ctx, port, name, kw):
    """Every config over its whole tspan (hundreds to thousands of RK steps) at a
    reduced size, with the bit-exact schemes: the final value function and the
    whole step log equal the oracle bit for bit (north_star: 'after the final
    step')."""
    S = P.CONFIGS[name](**kw)
    v0 = H.initial_value(port, S)
    t0, tf = S.tspan
    va, sa, ta = ctx.integrate(S.grid, S.problem, S.method, 0.0, tf - t0, v0)
    vb, sb, tb = port.integrate(S.grid, S.problem, S.method, 0.0, tf - t0, v0)
    assert ta == tb and len(sa) == len(sb) >= 10
    assert_bitwise(sa, sb, "step log")
    assert_bitwise(va, vb, "final value function")
