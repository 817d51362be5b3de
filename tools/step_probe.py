"""Back-to-back RK3 step time (no per-stage events) of the bench workload."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_11542_b200 import _lib
from paper_2507_11542_b200 import problems as P
ctx = _lib.Context(0)
S = P.cfg2_air3d(101)
s = _lib.Solver(ctx, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
for _ in range(10):
    s.step(0.0, dt)
ext = torch.cuda.ExternalStream(s.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx.synchronize()
e0.record(ext)
for _ in range(300):
    s.step(0.0, dt)
e1.record(ext)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 300 * 1e3
st = [s.step_timed(0.0, dt)[1] for _ in range(50)]
print(f"PDL={os.environ.get('LSG_PDL','1')} back-to-back step {us:.1f} us ({1030301*3/us/1e3:.1f} G pt-stage/s); step_timed {1e3*sum(st)/len(st):.1f} us")
