"""A few cfg2 (Air3D 101^3 ENO3 RK3) steps on the device: the short command
profiled under ncu (one capture per change)."""
from paper_2507_11542_b200 import _lib
from paper_2507_11542_b200 import problems as P

ctx = _lib.Context(0)
S = P.cfg2_air3d(101)
s = _lib.Solver(ctx, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
for k in range(3):
    s.step(k * dt, dt)
ctx.synchronize()
print("ok", s.get_field()[:2])
