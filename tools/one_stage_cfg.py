"""Two RK steps of one BASELINE config on the device, the short command
profiled under ncu for per-config instruction counts (FP64 instructions per
node do not depend on the grid size, so large configs run smaller):

    python tools/one_stage_cfg.py cfg3 [n] [fast]
"""
import sys

from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
fast = len(sys.argv) > 3 and sys.argv[3] == "fast"
build = {"cfg1": P.cfg1_circle, "cfg2": P.cfg2_air3d, "cfg3": P.cfg3_dblint4, "cfg4": P.cfg4_dubins6,
         "cfg5": P.cfg5_normal, "cfg5eno3": lambda n: P.cfg5_normal(n, scheme=abi.SCHEME_ENO3),
         "cfg5first": lambda n: P.cfg5_normal(n, scheme=abi.SCHEME_FIRST),
         "cfg5eno2": lambda n: P.cfg5_normal(n, scheme=abi.SCHEME_ENO2)}[name]
S = build(n) if n else (build() if name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5") else build(512))
prob = S.problem
if fast:
    prob = abi.make_problem(prob.kind, prob.scheme, list(prob.params), prob.direction, bool(prob.restrict_update),
                            options=abi.OPT_WENO5_FAST)
ctx = _lib.Context(0)
s = _lib.Solver(ctx, S.grid, prob, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
for k in range(2):
    s.step(k * dt, dt)
ctx.synchronize()
print("ok", name, _lib.node_count(S.grid))
