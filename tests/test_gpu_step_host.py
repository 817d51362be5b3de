"""lsg_solver_step_host: one step from a host field to a host result with the
copies chunked along the slab axis and overlapped with the stage kernels.
Must equal set_field + step + get_field bit for bit, for every integrator,
periodic and clamped slab axes, 2-D..6-D, pinned and pageable buffers, in
place and out of place, repeated calls, and the fallbacks (too few planes to
pipeline, in-process slabs, LSG_PIPE=0)."""
import dataclasses
import os

import numpy as np
import pytest

import helpers as H
from conftest import assert_bitwise
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

pytestmark = pytest.mark.gpu


def cases():
    lin6 = abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_WENO5, abi.linear_params([0.3, -0.2, 0.5, 0.1, -0.4, 0.9]),
                            abi.GROW, True)
    g6 = abi.make_grid([-1.0] * 6, [1.0] * 6, [7, 7, 7, 7, 7, 40], (5,))
    return {
        "cfg2_41": (P.cfg2_air3d(41), None),                       # periodic z, tiled 3-D kernel
        "cfg1_41": (P.CONFIGS["cfg1"](n=41), None),                # 2-D, clamped (extrapolated) slab axis
        "cfg3_29": (P.cfg3_dblint4(29), None),                     # 4-D WENO5
        "cfg5_32": (P.cfg5_normal(32), None),                      # periodic box WENO5
        "cfg5_32x120": (P.cfg5_normal(32, nz=120), None),          # wrap planes first, tapered last chunk
        "rockets_30": (P.rockets(30), None),                       # non-periodic heading
        "lin6_40": (dataclasses.replace(P.cfg1_circle(21), grid=g6, problem=lin6, method=abi.CFL3), "random"),
        "cfg2_21_fallback": (P.cfg2_air3d(21), None),              # 21 planes: too few to pipeline
    }


CASES = cases()


def field(port, S, kind):
    if kind == "random":
        return H.random_field(S.grid, 7)
    return H.initial_value(port, S)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("method", [abi.CFL1, abi.CFL2, abi.CFL3])
def test_step_host_bitwise(ctx, port, name, method):
    S0, kind = CASES[name]
    S = dataclasses.replace(S0, method=method)
    v0 = field(port, S, kind)
    ref = _lib.Solver(ctx, S.grid, S.problem, S.method)
    pipe = _lib.Solver(ctx, S.grid, S.problem, S.method)
    dt = 0.32 * ref.step_bound()
    # reference: three explicit set/step/get round trips
    want = []
    v = v0.copy()
    for k in range(3):
        ref.set_field(v)
        ref.step(k * dt, dt)
        v = ref.get_field()
        want.append(v)
    # pinned, in place
    buf = _lib.PinnedArray(v0.size)
    buf.array[:] = v0
    for k in range(3):
        pipe.step_host(k * dt, dt, buf.array, out=buf.array)
        assert_bitwise(buf.array, want[k], f"pinned in-place step {k}")
    # pageable, out of place
    out = pipe.step_host(0.0, dt, v0)
    assert_bitwise(out, want[0], "pageable")
    buf.free()


def test_step_host_fallbacks(ctx, port, monkeypatch):
    S = P.cfg2_air3d(41)
    v0 = H.initial_value(port, S)
    one = _lib.Solver(ctx, S.grid, S.problem, S.method)
    dt = 0.32 * one.step_bound()
    one.set_field(v0)
    one.step(0.0, dt)
    want = one.get_field()
    slabs = _lib.Solver(ctx, S.grid, S.problem, S.method, nslabs=3)
    assert_bitwise(slabs.step_host(0.0, dt, v0), want, "in-process slabs")
    monkeypatch.setenv("LSG_PIPE", "0")
    plain = _lib.Solver(ctx, S.grid, S.problem, S.method)
    assert_bitwise(plain.step_host(0.0, dt, v0), want, "LSG_PIPE=0")
    # the step log of a following leg sees the field step_host left behind
    monkeypatch.delenv("LSG_PIPE")
    a = _lib.Solver(ctx, S.grid, S.problem, S.method)
    a.step_host(0.0, dt, v0)
    sa, _ = a.integrate(dt, 3 * dt)
    one2 = _lib.Solver(ctx, S.grid, S.problem, S.method)
    one2.set_field(want)
    sb, _ = one2.integrate(dt, 3 * dt)
    assert_bitwise(sa, sb, "leg after step_host")
    assert_bitwise(a.get_field(), one2.get_field(), "field after leg")


def test_step_host_errors(ctx):
    S = P.cfg2_air3d(21)
    s = _lib.Solver(ctx, S.grid, S.problem, S.method)
    with pytest.raises(ValueError):
        s.step_host(0.0, 0.01, np.zeros(5))
