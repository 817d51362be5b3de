"""Per-step cost of the e2e path: H2D set_field + step + D2H get_field, with
torch-pinned vs library-pinned host buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2507_11542_b200 import _lib
from paper_2507_11542_b200 import problems as P
ctx = _lib.Context(0)
S = P.cfg2_air3d(101)
s = _lib.Solver(ctx, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
N = s.local_nodes
keep = _lib.PinnedArray(N)
bufs = {"numpy": np.empty(N), "torch_pinned": torch.empty(N, dtype=torch.float64, pin_memory=True).numpy(),
        "lib_pinned": keep.array}
for name, b in bufs.items():
    s.get_field(out=b)
    for rep in range(2):
        t0 = time.perf_counter()
        for _ in range(50):
            s.set_field(b)
        t1 = time.perf_counter()
        for _ in range(50):
            s.step(0.0, dt)
        ctx.synchronize()
        t2 = time.perf_counter()
        for _ in range(50):
            s.get_field(out=b)
        t3 = time.perf_counter()
    print(f"{name:13s} set_field {1e3*(t1-t0)/50:.3f} ms  step {1e3*(t2-t1)/50:.3f} ms  get_field {1e3*(t3-t2)/50:.3f} ms", flush=True)
