"""Per-call cost of the stateless reference-facing entry points vs the
stateful solver, host buffers both ways (cfg2 Air3D 101^3 and cfg1 201^2)."""
import ctypes as C
import json
import time

import numpy as np

from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P


def med(f, n=20):
    f()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts)) * 1e3


ctx = _lib.Context(0)
out = {}
for name, S in [("cfg2", P.cfg2_air3d(101)), ("cfg1", P.CONFIGS["cfg1"]())]:
    s = _lib.Solver(ctx, S.grid, S.problem, S.method)
    s.init_shape(*S.ic[:3], S.ic[3])
    v0 = s.get_field()
    dt = 0.32 * s.step_bound()
    tf = dt * 0.999
    out[name] = {
        "term_lf_ms": med(lambda: ctx.term_lf(S.grid, S.problem, 0.0, v0)),
        "integrate_1step_ms": med(lambda: ctx.integrate(S.grid, S.problem, S.method, 0.0, tf, v0)),
        "solver_set_step_get_ms": med(lambda: (s.set_field(v0), s.step(0.0, dt), s.get_field())),
        "solver_create_ms": med(lambda: _lib.Solver(ctx, S.grid, S.problem, S.method).close()),
    }
    N = v0.size
    pin_in, pin_out = _lib.PinnedArray(N), _lib.PinnedArray(N)
    pin_in.array[:] = v0
    b = C.c_double()
    out[name]["term_lf_pinned_ms"] = med(lambda: _lib.call(
        "lsg_term_lf", ctx.h, C.byref(S.grid), C.byref(S.problem), C.c_double(0.0), pin_in.ptr, pin_out.ptr,
        C.byref(b)))
    out[name]["pad_ghost_ms"] = med(lambda: ctx.pad_ghost(S.grid, v0, 0, 1))
    pin_in.free()
    pin_out.free()
print(json.dumps(out, indent=1))
