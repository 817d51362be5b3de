"""Per-stage cost of the slab machinery on one GPU (cfg2 Air3D 101^3):
single slab, in-process slabs (D2D halo copies), and the multi-rank branch on
a one-rank NCCL communicator (LSG_DIST_SELFTEST).  Reports step_timed stage
times and a whole enqueued leg (host enqueue included)."""
import json
import os
import time

import numpy as np

from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P


def measure(ctx, nslabs=1, periodic_z=True):
    S = P.cfg2_air3d(101)
    g = S.grid
    if not periodic_z:
        g = abi.make_grid([g.mins[d] for d in range(3)], [g.maxs[d] for d in range(3)], [101] * 3, ())
    s = _lib.Solver(ctx, g, S.problem, S.method, nslabs=nslabs)
    s.init_shape(*S.ic[:3], S.ic[3])
    dt = 0.32 * s.step_bound()
    t = 0.0
    for _ in range(5):
        s.step(t, dt)
        t += dt
    st = np.array([s.step_timed(t + k * dt, dt)[0] for k in range(30)])
    v = s.get_field()
    s.set_field(v)
    ctx.synchronize()
    t0 = time.perf_counter()
    steps, _ = s.integrate(0.0, 100 * dt * 0.9999, abi.make_opts(max_step=dt))
    leg = (time.perf_counter() - t0) / len(steps)
    return {"stage_ms": [round(x, 4) for x in st.mean(axis=0)], "leg_ms_per_step": round(leg * 1e3, 4),
            "steps": len(steps)}


out = {}
c = _lib.Context(0)
out["single"] = measure(c)
out["slabs2_inprocess"] = measure(c, 2)
os.environ["LSG_DIST_SELFTEST"] = "1"
d = _lib.Context(0, 0, 1, _lib.nccl_unique_id())
out["dist_selftest"] = measure(d)
out["dist_selftest_nonperiodic_z"] = measure(d, periodic_z=False)
out["single_nonperiodic_z"] = measure(c, periodic_z=False)
import ctypes as C
lib = _lib.load()
S = P.cfg2_air3d(101)
s = _lib.Solver(d, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
s.step(0.0, dt)
d.synchronize()
t0 = time.perf_counter()
for k in range(50):
    lib.lsg_solver_step(s.h, C.c_double(0.0), C.c_double(dt))
t1 = time.perf_counter()
d.synchronize()
t2 = time.perf_counter()
out["dist_host_enqueue_ms_per_step"] = (t1 - t0) / 50 * 1e3
out["dist_total_ms_per_step"] = (t2 - t0) / 50 * 1e3
os.environ["LSG_PDL"] = "0"
out["single_nopdl"] = measure(c)
print(json.dumps(out, indent=1))
s.close()
d.close()
c.close()
