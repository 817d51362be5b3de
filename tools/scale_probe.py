"""Per-stage device time vs grid size for the fused stage kernels (Air3D ENO3 RK3)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_11542_b200 import _lib
from paper_2507_11542_b200 import problems as P

ctx = _lib.Context(0)
for kern in ["march3", "generic"]:
    if kern == "generic":
        os.environ["LSG_KERNEL"] = "generic"
    for n in [int(a) for a in os.environ.get("SIZES", "48,64,101,128,160,200,256").split(",")]:
        S = P.cfg2_air3d(n)
        s = _lib.Solver(ctx, S.grid, S.problem, S.method)
        s.init_shape(*S.ic[:3], S.ic[3])
        dt = 0.32 * s.step_bound()
        for _ in range(3):
            s.step(0.0, dt)
        st = np.array([s.step_timed(0.0, dt)[0] for _ in range(20)])
        ms = st.mean(axis=0)
        N = n ** 3
        print(f"{kern:8s} n={n:4d} N={N:9d} stage_us={[round(x*1e3,1) for x in ms]}  ns/pt/stage={ms.mean()*1e6/N:.4f}  Gpt/s={N/ms.mean()/1e6:.1f}", flush=True)
        s.close()
