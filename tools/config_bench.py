"""Device-resident throughput of every BASELINE config at full size (one GPU):
per-stage device time of lsg_solver_step_timed after warm-up, no L2 flush.
Usage: python tools/config_bench.py [cfg ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

RUNS = {
    "cfg1": (P.cfg1_circle, {}, [None]),
    "cfg2": (P.cfg2_air3d, {}, [None]),
    "cfg3": (P.cfg3_dblint4, {}, [None, abi.OPT_WENO5_FAST]),
    "cfg5": (P.cfg5_normal, {}, [None, abi.OPT_WENO5_FAST]),
    "cfg5eno3": (P.cfg5_normal, {"scheme": abi.SCHEME_ENO3}, [None]),
    "cfg4": (P.cfg4_dubins6, {}, [abi.OPT_WENO5_FAST, None]),
    "cfg4eno3": (P.cfg4_dubins6, {"scheme": abi.SCHEME_ENO3}, [None]),
    "cfg1eno2": (P.cfg1_circle, {}, [None]),
    # low-arithmetic schemes on the cfg5 grid: how close the tiled kernel's data
    # movement gets to the HBM roofline when FP64 is not the limit
    "cfg5first": (P.cfg5_normal, {"scheme": abi.SCHEME_FIRST}, [None]),
    "cfg5eno2": (P.cfg5_normal, {"scheme": abi.SCHEME_ENO2}, [None]),
}
try:
    HBM_PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    HBM_PEAK = 6546.2
ctx = _lib.Context(0)
names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5", "cfg5eno3"]
out = []
for name in names:
    fn, kw, opts = RUNS[name]
    S = fn(**kw)
    for opt in opts:
        prob = S.problem
        if opt is not None:
            prob = abi.make_problem(prob.kind, prob.scheme, list(prob.params), prob.direction,
                                    bool(prob.restrict_update), options=opt)
        t0 = time.time()
        sol = _lib.Solver(ctx, S.grid, prob, S.method)
        sol.init_shape(*S.ic[:3], S.ic[3])
        dt = 0.32 * sol.step_bound()
        N = _lib.node_count(S.grid)
        reps = 3 if N > 1e9 else 10
        for _ in range(2):
            sol.step(0.0, dt)
        st = np.array([sol.step_timed(0.0, dt)[0] for _ in range(reps)])
        ms = st.mean(axis=0)
        rate = N * len(ms) / (ms.sum() * 1e-3)
        rec = {"config": S.name, "grid": [S.grid.counts[d] for d in range(S.grid.dim)], "nodes": N,
               "scheme": ["FIRST", "ENO2", "ENO3", "WENO5"][prob.scheme] + ("-fast" if opt else ""),
               "stages": len(ms), "stage_ms": [round(float(x), 4) for x in ms],
               "G_node_stage_per_s": round(rate / 1e9, 2),
               "hbm_frac_of_6546": round(rate * (64 / 3 if len(ms) == 3 else 20.0) / 6546.2e9, 4),
               "hbm_gbs": round(rate * (64 / 3 if len(ms) == 3 else 20.0) / 1e9, 1),
               "hbm_frac_measured_peak": round(rate * (64 / 3 if len(ms) == 3 else 20.0) / (HBM_PEAK * 1e9), 4),
               "wall_s": round(time.time() - t0, 1)}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        sol.close()
