"""Tile-kernel throughput of the cfg5 problem on other cube sizes (bench-style
timing: W warm-up steps, one event pair around K steps, L2 flush per step for
small grids), with the tile the host picks or a forced LSG_M3_TX.
Usage: python tools/grid_probe.py n [n ...]   (env LSG_M3_TX / LSG_M3_VERBOSE apply)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_11542_b200 import _lib, abi  # noqa: E402
from paper_2507_11542_b200 import problems as P  # noqa: E402

ctx = _lib.Context(0)
torch.cuda.set_device(0)
for n in [int(a) for a in sys.argv[1:]]:
    for name, scheme, opt in (("weno5", abi.SCHEME_WENO5, 0), ("eno3", abi.SCHEME_ENO3, 0),
                              ("weno5-fast", abi.SCHEME_WENO5, abi.OPT_WENO5_FAST)):
        S = P.cfg5_normal(n, scheme=scheme)
        prob = abi.make_problem(S.problem.kind, S.problem.scheme, list(S.problem.params), S.problem.direction,
                                bool(S.problem.restrict_update), options=opt)
        sol = _lib.Solver(ctx, S.grid, prob, S.method)
        sol.init_shape(*S.ic[:3], S.ic[3])
        dt = 0.32 * sol.step_bound()
        N = _lib.node_count(S.grid)
        stream = torch.cuda.ExternalStream(sol.stream())
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda") if 8 * N <= 4 * bench.L2_BYTES else None
        T = bench.Timed(torch, ctx, sol, dt, stream, flush)
        T.warm(3)
        K = 20 if N > 1e7 else 100
        ms, _ = T.run(K, torch.cuda.synchronize)
        print(f"n={n} {name} TX={os.environ.get('LSG_M3_TX', 'auto')}: {N * 3 * K / (ms * 1e-3) / 1e9:.2f} G", flush=True)
        sol.close()
