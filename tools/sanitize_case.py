"""Small cases over every kernel family, for compute-sanitizer memcheck:
march3 (all modes, full-row and segment tiles), in-process slabs (gapped
boundary-band launches on the side stream, halo copies), box3, the generic
kernel in 1-6 D, upwind / pad / shift / restrict, initial shapes, the zero
set and slices."""
import os

import numpy as np

from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

ctx = _lib.Context(0)
rng = np.random.default_rng(3)


def run(g, p, method=abi.CFL3, nslabs=1, steps=2):
    s = _lib.Solver(ctx, g, p, method, nslabs=nslabs)
    v = rng.uniform(-1, 1, _lib.node_count(g))
    s.set_field(v)
    dt = 0.32 * s.step_bound()
    s.integrate(0.0, steps * dt * 0.999)
    s.step(0.0, dt)
    s.step_timed(0.0, dt)
    out = s.get_field()
    s.close()
    return out


lin3 = abi.linear_params([0.7, -1.1, 0.4])
for counts, per in [((21, 13, 11), (2,)), ((300, 9, 8), (0, 1)), ((7, 9, 12), ())]:
    g = abi.make_grid([-1, -1, -1], [1, 1, 1], list(counts), per)
    for sch in range(4):
        p = abi.make_problem(abi.HAM_LINEAR, sch, lin3, abi.GROW, True)
        run(g, p)
        run(g, p, nslabs=2)
        ctx.term_lf(g, p, 0.0, rng.uniform(-1, 1, _lib.node_count(g)))
# TMA-fed tiles (even x extents): interior and border tiles, periodic and
# extrapolated x/y/z (extrapolated ghost planes at a non-periodic z edge), slabs
for counts, per in [((32, 20, 9), ()), ((64, 18, 10), (0, 1, 2)), ((40, 33, 8), (2,)), ((300, 9, 8), (1,))]:
    g = abi.make_grid([-1, -1, -1], [1, 1, 1], list(counts), per)
    for sch in range(4):
        p = abi.make_problem(abi.HAM_LINEAR, sch, lin3, abi.GROW, True)
        run(g, p)
        run(g, p, nslabs=2)
os.environ["LSG_KERNEL"] = "box3"
g = abi.make_grid([-1, -1, -1], [1, 1, 1], [19, 11, 9], (2,))
run(g, abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_ENO3, lin3, abi.GROW, True))
os.environ["LSG_KERNEL"] = "generic"
for D in range(1, 7):
    n = [9] * D
    g = abi.make_grid([-1] * D, [1] * D, n, (D - 1,))
    p = abi.make_problem(abi.HAM_NORMAL, abi.SCHEME_WENO5, [1.0], abi.GROW, False)
    run(g, p, method=abi.CFL2)
    run(g, p, nslabs=2, method=abi.CFL1)
del os.environ["LSG_KERNEL"]
for name in ["cfg1", "cfg2", "cfg3", "cfg4", "rockets", "rotation"]:
    S = P.CONFIGS[name](n={"cfg1": 21, "cfg2": 13, "cfg3": 9, "cfg4": 7, "rockets": 12, "rotation": 21}[name])
    s = _lib.Solver(ctx, S.grid, S.problem, S.method)
    s.init_shape(*S.ic[:3], S.ic[3])
    s.integrate(0.0, 0.01)
    s.close()
g = abi.make_grid([-1, -1], [1, 1], [33, 29], ())
f = rng.uniform(-1, 1, 33 * 29)
for d in range(2):
    for sch in range(4):
        ctx.upwind(g, f, d, sch)
    ctx.shift_along_dim(g, ctx.pad_ghost(g, f, d, 3), d, 3, -2)
ctx.restrict_update(f, abi.GROW)
ctx.extract_zero_set_2d(g, f)
g3 = abi.make_grid([-1, -1, -1], [1, 1, 1], [9, 8, 7], ())
f3 = rng.uniform(-1, 1, 9 * 8 * 7)
for d in range(3):
    ctx.slice_2d(g3, f3, d, 2)
ctx.synchronize()
print("sanitize case done")
