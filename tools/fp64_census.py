"""One RK3 step of each config at a reduced size, in one process: the command
profiled by ONE `ncu --set full` capture of every config's COMBINE-stage
kernel (FP64 and total instructions per node do not depend on the size).
Writes the launch order and node counts to gpurun_out/census_order.json.

    ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
        -k 'regex:stage_kernel<.*\\(int\\)2>|march3_kernel<.*\\(int\\)2, \\(bool\\)1>' \
        -o gpurun_out/census python tools/fp64_census.py
    python tools/fp64_census_summary.py gpurun_out/census.ncu-rep gpurun_out/census_order.json out.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

RUNS = [  # label, builder, size, fast
    ("cfg2_101_exact", P.cfg2_air3d, 101, False),
    ("cfg3_41_exact", P.cfg3_dblint4, 41, False),
    ("cfg3_41_fast", P.cfg3_dblint4, 41, True),
    ("cfg4_17_exact", P.cfg4_dubins6, 17, False),
    ("cfg4_17_fast", P.cfg4_dubins6, 17, True),
    ("cfg4eno3_17_exact", lambda n: P.cfg4_dubins6(n, scheme=abi.SCHEME_ENO3), 17, False),
    ("cfg5_128_exact", P.cfg5_normal, 128, False),
    ("cfg5_128_fast", P.cfg5_normal, 128, True),
    ("cfg5eno3_128_exact", lambda n: P.cfg5_normal(n, scheme=abi.SCHEME_ENO3), 128, False),
]
ctx = _lib.Context(0)
order = []
for label, build, n, fast in RUNS:
    S = build(n)
    prob = S.problem
    if fast:
        prob = abi.make_problem(prob.kind, prob.scheme, list(prob.params), prob.direction,
                                bool(prob.restrict_update), options=abi.OPT_WENO5_FAST)
    s = _lib.Solver(ctx, S.grid, prob, S.method)
    s.init_shape(*S.ic[:3], S.ic[3])
    dt = 0.32 * s.step_bound()
    s.step(0.0, dt)
    ctx.synchronize()
    nodes = _lib.node_count(S.grid)
    # the generic kernel matches twice per RK3 step (stages 2 and 3), the 3-D one once
    order += [{"label": label, "nodes": nodes}] * (1 if S.grid.dim == 3 else 2)
    s.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(order, open("gpurun_out/census_order.json", "w"))
print("ok", len(order), "matching launches")
