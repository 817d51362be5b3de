"""lsg_solver_step_host on a BASELINE grid: wall time per step over a few
steps (pinned buffers), then one traced step when LSG_PIPE_TRACE=1 is set.
Usage: python tools/pipe_trace.py [cfg2|cfg5] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11542_b200 import _lib  # noqa: E402
from paper_2507_11542_b200 import problems as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
trace = os.environ.pop("LSG_PIPE_TRACE", None)
ctx = _lib.Context(0)
S = P.cfg2_air3d(101) if name == "cfg2" else P.cfg5_normal(512)
s = _lib.Solver(ctx, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
buf = _lib.PinnedArray(s.local_nodes)
s.get_field(out=buf.array)
for _ in range(3):
    s.step_host(0.0, dt, buf.array, out=buf.array)
ctx.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    s.step_host(0.0, dt, buf.array, out=buf.array)
ctx.synchronize()
ms = (time.perf_counter() - t0) / n * 1e3
N = s.local_nodes
print(f"{name} step_host: {ms:.3f} ms per step, {N * (S.method + 1) / (ms * 1e-3) / 1e9:.2f} G node-stages/s "
      f"(K={os.environ.get('LSG_PIPE_K', 'default')})", flush=True)
if trace:
    os.environ["LSG_PIPE_TRACE"] = trace
    s.step_host(0.0, dt, buf.array, out=buf.array)
    ctx.synchronize()
