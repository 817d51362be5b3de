"""Per-stage time of the 3-D kernel vs z-chunk length (LSG_M3_CHUNK)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P
os.environ["LSG_M3_VERBOSE"] = "1"
ctx = _lib.Context(0)
n = 101
base = P.cfg2_air3d(n)
for scheme in [0, 2]:
    for chunk in [None, 1, 2, 4, 8, 16, 34, 101]:
        if chunk is None:
            os.environ.pop("LSG_M3_CHUNK", None)
        else:
            os.environ["LSG_M3_CHUNK"] = str(chunk)
        prob = abi.make_problem(abi.HAM_AIR3D, scheme, [5.0, 5.0, 1.0, 1.0], abi.GROW, True)
        sol = _lib.Solver(ctx, base.grid, prob, abi.CFL3)
        sol.init_shape(*base.ic[:3], base.ic[3])
        dt = 0.32 * sol.step_bound()
        for _ in range(3):
            sol.step(0.0, dt)
        st = np.array([sol.step_timed(0.0, dt)[0] for _ in range(20)]).mean(axis=0)
        print(f"scheme={scheme} chunk={chunk} stage_us={[round(x*1e3,1) for x in st]}", flush=True)
        sol.close()
