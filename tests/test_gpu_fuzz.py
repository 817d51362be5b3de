"""Property-based parity (hypothesis): random grids (1-4-D, extents at and above
the stencil minimum, any periodic mask), schemes, Hamiltonian kinds, clamp
settings, integrators and spans — the device result must equal the oracle bit
for bit (value function, step log, final time)."""
import math

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from conftest import assert_bitwise
from paper_2507_11542_b200 import abi
import helpers as H

pytestmark = pytest.mark.gpu

MIN_NODES = {0: 3, 1: 5, 2: 7, 3: 7}

# The default run replays a fixed case set (derandomized: the same cases on
# every machine); LSG_FUZZ_RANDOM=1 LSG_FUZZ_EXAMPLES=N explores fresh ones.
import os  # noqa: E402
N_EXAMPLES = int(os.environ.get("LSG_FUZZ_EXAMPLES", "80"))
DERANDOMIZE = os.environ.get("LSG_FUZZ_RANDOM") is None


@st.composite
def cases(draw):
    D = draw(st.integers(1, 4))
    scheme = draw(st.integers(0, 3))
    counts = [draw(st.integers(MIN_NODES[scheme], 13 if D >= 3 else 40)) for _ in range(D)]
    periodic = [d for d in range(D) if draw(st.booleans())]
    mins = [draw(st.sampled_from([-1.0, 0.0, -2.5, 0.3])) for _ in range(D)]
    spans = [draw(st.sampled_from([1.0, 2.0, 0.7, 5.0])) for _ in range(D)]
    kind = draw(st.sampled_from([abi.HAM_LINEAR, abi.HAM_NORMAL]))
    if kind == abi.HAM_LINEAR:
        c = [draw(st.floats(-2.0, 2.0, allow_nan=False, width=32)) for _ in range(D)]
        params = abi.linear_params(c, offset=draw(st.sampled_from([0.0, 0.125, -0.3])))
    else:
        params = [draw(st.sampled_from([1.0, 0.5, 2.0]))]
    clamp = draw(st.booleans())
    direction = draw(st.sampled_from([abi.GROW, abi.SHRINK]))
    method = draw(st.integers(0, 2))
    seed = draw(st.integers(0, 2 ** 31))
    nsteps = draw(st.integers(1, 3))
    scale = draw(st.sampled_from([1.0, 1.0, 1.0, 1e-200, 1e-305, 1e-312, 1e150]))  # incl. subnormal differences
    return D, scheme, counts, periodic, mins, spans, kind, params, clamp, direction, method, seed, nsteps, scale


@settings(max_examples=N_EXAMPLES, deadline=None, derandomize=DERANDOMIZE,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(cases())
def test_fuzz_integrate_bitwise(ctx, port, case):
    D, scheme, counts, periodic, mins, spans, kind, params, clamp, direction, method, seed, nsteps, scale = case
    g = abi.make_grid(mins, [m + s for m, s in zip(mins, spans)], counts, periodic)
    p = abi.make_problem(kind, scheme, params, direction, clamp)
    v0 = H.random_field(g, seed) * scale
    try:
        _, bound = port.term_lf(g, p, 0.0, v0)
    except RuntimeError as e:  # e.g. overflowing |p|^2: the device must refuse the same way
        with pytest.raises(RuntimeError, match=str(e).split(":")[0]):
            ctx.term_lf(g, p, 0.0, v0)
        return
    if not math.isfinite(bound):
        bound = 0.01
    tf = nsteps * 0.32 * bound * 0.999
    try:
        vb, sb, tb = port.integrate(g, p, method, 0.0, tf, v0)
    except RuntimeError as e:
        with pytest.raises(RuntimeError, match=str(e).split(":")[0]):
            ctx.integrate(g, p, method, 0.0, tf, v0)
        return
    va, sa, ta = ctx.integrate(g, p, method, 0.0, tf, v0)
    assert ta == tb
    assert_bitwise(sa, sb, "step log")
    assert_bitwise(va, vb, "value function")


@st.composite
def cases3(draw):
    """3-D cases sized for the tiled kernel's edge cases: full-row tiles,
    rows split in three segments (n0 ~ 96-130), searched segment widths
    (n0 > 256 or rows that do not fit), ragged last tiles, thin z."""
    scheme = draw(st.integers(0, 3))
    lo = MIN_NODES[scheme]
    n0 = draw(st.one_of(st.integers(lo, 40), st.integers(90, 130), st.integers(250, 300)))
    n1 = draw(st.integers(lo, 40 if n0 <= 130 else 12))
    n2 = draw(st.integers(lo, 24))
    periodic = [d for d in range(3) if draw(st.booleans())]
    kind = draw(st.sampled_from([abi.HAM_LINEAR, abi.HAM_NORMAL, abi.HAM_AIR3D]))
    if kind == abi.HAM_LINEAR:
        params = abi.linear_params([draw(st.sampled_from([0.7, -1.3, 0.0, 2.0])) for _ in range(3)])
    elif kind == abi.HAM_NORMAL:
        params = [draw(st.sampled_from([1.0, 0.5]))]
    else:
        params = [5.0, 5.0, 1.0, 1.0]
    return (scheme, (n0, n1, n2), periodic, kind, params, draw(st.booleans()),
            draw(st.sampled_from([abi.GROW, abi.SHRINK])), draw(st.integers(0, 2)),
            draw(st.integers(0, 2 ** 31)), draw(st.sampled_from(["march3", "box3", "generic"])),
            draw(st.integers(1, 4)), draw(st.sampled_from([1.0, 1.0, 1e-305, 1e-312])))


@settings(max_examples=(3 * N_EXAMPLES) // 4, deadline=None, derandomize=DERANDOMIZE,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(cases3())
def test_fuzz_3d_kernels_and_slabs_bitwise(ctx, port, case):
    """Each 3-D kernel variant and a random slab count against the oracle."""
    import os
    from paper_2507_11542_b200 import _lib
    scheme, counts, periodic, kind, params, clamp, direction, method, seed, kernel, nslabs, scale = case
    g = abi.make_grid([-6.0, -10.0, 0.0], [20.0, 10.0, 6.0], list(counts), periodic)
    p = abi.make_problem(kind, scheme, params, direction, clamp)
    v0 = H.random_field(g, seed, -3.0, 3.0) * scale
    _, bound = port.term_lf(g, p, 0.0, v0)
    tf = 2 * 0.32 * bound * 0.999 if math.isfinite(bound) else 0.01
    vb, sb, tb = port.integrate(g, p, method, 0.0, tf, v0)
    old = os.environ.get("LSG_KERNEL")
    os.environ["LSG_KERNEL"] = kernel
    try:
        s = _lib.Solver(ctx, g, p, method, nslabs=max(1, min(nslabs, counts[2] // (1, 2, 3, 3)[scheme])))
    finally:
        if old is None:
            del os.environ["LSG_KERNEL"]
        else:
            os.environ["LSG_KERNEL"] = old
    s.set_field(v0)
    sa, ta = s.integrate(0.0, tf)
    assert ta == tb
    assert_bitwise(sa, sb, "step log")
    assert_bitwise(s.get_field(), vb, f"value function ({kernel}, {nslabs} slabs)")
