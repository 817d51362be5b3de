"""End-to-end step cost with the field crossing PCIe every step (cfg2 Air3D
101^3, pinned buffers): set_field + step + get_field vs lsg_solver_step_host
(copies chunked and overlapped with the stage kernels)."""
import json
import time

from paper_2507_11542_b200 import _lib
from paper_2507_11542_b200 import problems as P

ctx = _lib.Context(0)
S = P.cfg2_air3d(101)
s = _lib.Solver(ctx, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
buf = _lib.PinnedArray(s.local_nodes)
s.get_field(out=buf.array)
N, n = s.local_nodes, 200
out = {}


def timed(f):
    for _ in range(5):
        f()
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    ctx.synchronize()
    return (time.perf_counter() - t0) / n


def plain():
    s.set_field(buf.array)
    s.step(0.0, dt)
    s.get_field(out=buf.array)


out["plain_ms"] = timed(plain) * 1e3
out["step_host_ms"] = timed(lambda: s.step_host(0.0, dt, buf.array, out=buf.array)) * 1e3
for k in ("plain", "step_host"):
    out[k + "_G_node_stages"] = N * 3 / (out[k + "_ms"] * 1e-3) / 1e9
print(json.dumps(out, indent=1))
buf.free()
