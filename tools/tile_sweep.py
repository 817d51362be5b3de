"""Sweep tile height (LSG_M3_R) and z-chunk (LSG_M3_CHUNK) of the 3-D kernel on cfg2 101^3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P
ctx = _lib.Context(0)
S = P.cfg2_air3d(101)
best = None
for R in [2, 3, 4, 5]:
    for chunk in [None, 3, 4, 5, 6, 8, 10, 13]:
        os.environ["LSG_M3_R"] = str(R)
        if chunk is None:
            os.environ.pop("LSG_M3_CHUNK", None)
        else:
            os.environ["LSG_M3_CHUNK"] = str(chunk)
        sol = _lib.Solver(ctx, S.grid, S.problem, S.method)
        sol.init_shape(*S.ic[:3], S.ic[3])
        dt = 0.32 * sol.step_bound()
        for _ in range(3):
            sol.step(0.0, dt)
        st = np.array([sol.step_timed(0.0, dt)[1] for _ in range(30)]).mean()
        print(f"R={R} chunk={chunk} step_us={st*1e3:.1f}", flush=True)
        if best is None or st < best[0]:
            best = (st, R, chunk)
        sol.close()
print("best", best)
