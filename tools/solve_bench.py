"""End-to-end reference-facing solves on the B200 vs the reference CPU library:
acceptance criterion 5 (rockets N=50, (-2.5, 0), 11 checkpoints, 490 steps) and
the cfg1 run (101^2, ENO2 + odeCFL2, (0, 0.5)).  Wall time of the whole call
(host buffers in, checkpoints out)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P
from oracle import oracle as O

ctx = _lib.Context(0)
out = {}
S = P.rockets(50)
ref = O.reference() if O.have_reference() else None
v0 = (ref or O.port()).rocket_initial(50) if ref else None
if v0 is None:
    s = _lib.Solver(ctx, S.grid, S.problem, S.method)
    s.init_shape(*S.ic[:3], S.ic[3])
    v0 = s.get_field()
ctx.solve_brt(S.grid, S.problem, v0, (-2.5, 0.0), 11)  # warm-up
t0 = time.perf_counter()
ck, times, steps, secs = ctx.solve_brt(S.grid, S.problem, v0, (-2.5, 0.0), 11)
wall = time.perf_counter() - t0
out["rockets50_b200"] = {"steps": len(steps), "wall_s": wall, "integration_seconds": secs}
if ref:
    t0 = time.perf_counter()
    rck, rt, rsteps = ref.solve_brt(S.grid, S.problem, v0, (-2.5, 0.0), 11)
    rwall = time.perf_counter() - t0
    out["rockets50_reference_cpu_1thread"] = {"steps": len(rsteps), "wall_s": rwall}
    out["rockets50_bitwise_equal"] = bool(np.array_equal(ck.view(np.int64), rck.view(np.int64)))
S = P.cfg1_circle(101)
g = S.grid
v0 = ref.sphere(g, [-0.25, 0.0], 0.5) if ref else None
ctx.integrate(g, S.problem, S.method, 0.0, 0.5, v0)
t0 = time.perf_counter()
v, steps, t = ctx.integrate(g, S.problem, S.method, 0.0, 0.5, v0)
out["cfg1_b200"] = {"steps": len(steps), "wall_s": time.perf_counter() - t0}
if ref:
    t0 = time.perf_counter()
    rv, rsteps, rt = ref.integrate(g, S.problem, S.method, 0.0, 0.5, v0)
    out["cfg1_reference_cpu_1thread"] = {"steps": len(rsteps), "wall_s": time.perf_counter() - t0}
    out["cfg1_bitwise_equal"] = bool(np.array_equal(v.view(np.int64), rv.view(np.int64)))
print(json.dumps(out, indent=1))
