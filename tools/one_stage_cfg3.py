"""Two RK3 steps of cfg3 (4-D double integrator 81^4, WENO5 exact): the short
command profiled under ncu for the generic N-D kernel."""
from paper_2507_11542_b200 import _lib
from paper_2507_11542_b200 import problems as P

ctx = _lib.Context(0)
S = P.cfg3_dblint4(81)
s = _lib.Solver(ctx, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
for k in range(2):
    s.step(k * dt, dt)
ctx.synchronize()
print("ok")
