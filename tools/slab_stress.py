"""Long-run equality of the slab machinery (side stream, comm stream, halo
validity tracking) with the single-slab solver: cfg2 101^3 over 300 RK3 steps
on 3 and 7 in-process slabs, cfg5 512^3 ENO3 over 10 steps on 4 slabs; field
and step log compared bit for bit."""
import numpy as np

from paper_2507_11542_b200 import _lib, abi
from paper_2507_11542_b200 import problems as P

ctx = _lib.Context(0)


def run(S, nslabs, nsteps):
    s = _lib.Solver(ctx, S.grid, S.problem, S.method, nslabs=nslabs)
    s.init_shape(*S.ic[:3], S.ic[3])
    dt = 0.32 * s.step_bound()
    steps, t = s.integrate(0.0, nsteps * dt * 0.9999, abi.make_opts(max_step=dt))
    return s.get_field(), steps


for S, slabs, n in [(P.cfg2_air3d(101), [3, 7], 300), (P.cfg5_normal(512, scheme=abi.SCHEME_ENO3), [4], 10)]:
    v1, s1 = run(S, 1, n)
    for k in slabs:
        vk, sk = run(S, k, n)
        same = np.array_equal(v1.view(np.int64), vk.view(np.int64)) and np.array_equal(
            s1.view(np.int64), sk.view(np.int64))
        print(f"{S.name} {k} slabs x {len(sk)} steps: {'bit-identical' if same else 'DIFFERENT'}")
        assert same
