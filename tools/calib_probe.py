"""Calibrate: device time of plain memory-bound kernels at the bench's size
(1,030,301 doubles per field) vs one fused stage, all on one stream."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

N = 101 ** 3
a = torch.rand(N, dtype=torch.float64, device="cuda")
b = torch.rand(N, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
def t(fn, reps=200):
    for _ in range(10):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
print(f"copy 8MB->8MB        {t(lambda: c.copy_(a)):.2f} us")
print(f"add  2x8MB->8MB      {t(lambda: torch.add(a, b, out=c)):.2f} us")
print(f"empty-ish (fill 8B)  {t(lambda: c[:1].fill_(0)):.2f} us")
big = torch.rand(64 * N, dtype=torch.float64, device="cuda")
bigc = torch.empty_like(big)
tb = t(lambda: bigc.copy_(big), 20)
print(f"copy 528MB           {tb:.2f} us  -> {2*big.numel()*8/(tb*1e-6)/1e9:.0f} GB/s")
ctx = _lib.Context(0)
S = P.cfg2_air3d(101)
for scheme in [0, 2]:
    prob = abi.make_problem(abi.HAM_LINEAR, scheme, abi.linear_params([1.0, 0.5, 0.25]))
    s = _lib.Solver(ctx, S.grid, prob, abi.CFL1)
    s.init_shape(*S.ic[:3], S.ic[3])
    dt = 0.32 * s.step_bound()
    for _ in range(5):
        s.step(0.0, dt)
    st = np.mean([s.step_timed(0.0, dt)[0][0] for _ in range(50)]) * 1e3
    ctx.synchronize()
    ext = torch.cuda.ExternalStream(s.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(200):
        s.step(0.0, dt)
    e1.record(ext)
    torch.cuda.synchronize()
    print(f"fused RK1 stage scheme {scheme}: timed {st:.2f} us, back-to-back {e0.elapsed_time(e1)/200*1e3:.2f} us")
