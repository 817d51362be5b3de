"""One traced lsg_solver_step_host sequence on cfg2 (run with LSG_PIPE_TRACE=1)."""
from paper_2507_11542_b200 import _lib
from paper_2507_11542_b200 import problems as P
ctx = _lib.Context(0)
S = P.cfg2_air3d(101)
s = _lib.Solver(ctx, S.grid, S.problem, S.method)
s.init_shape(*S.ic[:3], S.ic[3])
dt = 0.32 * s.step_bound()
buf = _lib.PinnedArray(s.local_nodes)
s.get_field(out=buf.array)
for k in range(4):
    s.step_host(0.0, dt, buf.array, out=buf.array)
