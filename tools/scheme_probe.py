"""Per-stage device time of the fused 3-D kernel at 101^3 by scheme and Hamiltonian."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

ctx = _lib.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 101
base = P.cfg2_air3d(n)
for kind in ["linear", "air3d"]:
    for s in range(4):
        if kind == "linear":
            prob = abi.make_problem(abi.HAM_LINEAR, s, abi.linear_params([1.0, 0.5, 0.25]))
        else:
            prob = abi.make_problem(abi.HAM_AIR3D, s, [5.0, 5.0, 1.0, 1.0], abi.GROW, True)
        sol = _lib.Solver(ctx, base.grid, prob, abi.CFL3)
        sol.init_shape(*base.ic[:3], base.ic[3])
        dt = 0.32 * sol.step_bound()
        for _ in range(3):
            sol.step(0.0, dt)
        st = np.array([sol.step_timed(0.0, dt)[0] for _ in range(20)]).mean(axis=0)
        print(f"{kind:7s} scheme={['FIRST','ENO2','ENO3','WENO5'][s]:6s} stage_us={[round(x*1e3,1) for x in st]}  "
              f"G pt-stage/s={n**3/st.mean()/1e6:.1f}", flush=True)
        sol.close()
