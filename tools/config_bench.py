"""Device-resident throughput of every BASELINE config at full size (one GPU),
timed like bench.py: W warm-up steps, then one CUDA event pair around K whole
RK steps on the solver's stream (no per-stage events, so consecutive stages
keep their programmatic-dependent-launch overlap), SM clocks sampled during
the timed region.  Small grids (fields that fit L2) get an L2 flush before
every step and a per-step event pair instead.
Usage: python tools/config_bench.py [cfg ...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_11542_b200 import _lib, abi  # noqa: E402
from paper_2507_11542_b200 import problems as P  # noqa: E402

RUNS = {
    "cfg1": (P.cfg1_circle, {}, [None]),
    "cfg2": (P.cfg2_air3d, {}, [None]),
    "cfg3": (P.cfg3_dblint4, {}, [None, abi.OPT_WENO5_FAST]),
    "cfg5": (P.cfg5_normal, {}, [None, abi.OPT_WENO5_FAST]),
    "cfg5eno3": (P.cfg5_normal, {"scheme": abi.SCHEME_ENO3}, [None]),
    "cfg4": (P.cfg4_dubins6, {}, [abi.OPT_WENO5_FAST, None]),
    "cfg4eno3": (P.cfg4_dubins6, {"scheme": abi.SCHEME_ENO3}, [None]),
    # low-arithmetic schemes on the cfg5 grid: how close the tiled kernel's data
    # movement gets to the HBM roofline when FP64 is not the limit
    "cfg5first": (P.cfg5_normal, {"scheme": abi.SCHEME_FIRST}, [None]),
    "cfg5eno2": (P.cfg5_normal, {"scheme": abi.SCHEME_ENO2}, [None]),
}
HBM_PEAK, _ = bench.peaks()
ctx = _lib.Context(0)
torch.cuda.set_device(0)
fp64_peak = ctx.fp64_rate()
names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5", "cfg5eno3", "cfg4", "cfg4eno3"]
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
        stages = S.method + 1
        stream = torch.cuda.ExternalStream(sol.stream())
        flush = None
        if 8 * N <= 4 * bench.L2_BYTES:
            flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        T = bench.Timed(torch, ctx, sol, dt, stream, flush)
        T.warm(3)
        K = 3 if N > 1e9 else (20 if N > 1e7 else 200)
        sampler = bench.ClockSampler(0)
        with sampler:
            ms, _ = T.run(K, torch.cuda.synchronize)
        rate = N * stages * K / (ms * 1e-3)
        bps = bench.BYTES_PER_PT_STAGE[S.method]
        rec = {"config": S.name, "grid": [S.grid.counts[d] for d in range(S.grid.dim)], "nodes": N,
               "scheme": ["FIRST", "ENO2", "ENO3", "WENO5"][prob.scheme] + ("-fast" if opt else ""),
               "stages": stages, "steps": K, "ms_per_step": round(ms / K, 4),
               "G_node_stage_per_s": round(rate / 1e9, 2),
               "hbm_gbs": round(rate * bps / 1e9, 1),
               "hbm_frac_measured_peak": round(rate * bps / (HBM_PEAK * 1e9), 4),
               "fp64_peak_instr_per_s": fp64_peak,
               "l2": "flushed per step" if flush is not None else "fields >> L2",
               "clocks": sampler.summary(), "wall_s": round(time.time() - t0, 1)}
        print(json.dumps(rec), flush=True)
        sol.close()
