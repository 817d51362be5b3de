"""Generate the golden fixtures in tests/golden/ from the REFERENCE library.

The reference (/root/reference/proj/core) is compiled from its own sources by
oracle/Makefile into oracle/_ref/libref_levelset.so; this script calls it
through oracle/ref_driver.cpp and records inputs and outputs:

  golden.npz         small inputs/outputs, stored verbatim (float64)
  golden_sums.json   sha256 of larger outputs + their step logs / scalars

Run here (the reference tree is not on the GPU box):
    python tests/golden/make_golden.py
"""
import hashlib
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
from paper_2507_11542_b200 import abi  # noqa: E402
from paper_2507_11542_b200 import problems as P  # noqa: E402
import helpers as H  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

UPWIND_GRIDS = {
    # test_spatial_derivatives.cpp:171-192 uses 16x12 periodic, seed 7
    "A": (abi.make_grid([0.0, 0.0], [1.0, 1.0], [16, 12], [0, 1]), 7),
    "B": (abi.make_grid([0.0, -1.0, 0.5], [1.0, 2.0, 3.0], [9, 10, 11], [1]), 3),
    "C": (abi.make_grid([-1.0], [1.0], [24]), 41),
}

TERM_CASES = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "rockets", "rotation"]

INTEGRATE_CASES = {
    # name: (config kwargs, tf) — cfg1 is BASELINE configs[0] at full size
    "cfg1": (dict(n=101), 0.5),
    "cfg2": (dict(n=21), 0.3),
    "cfg3": (dict(n=11), 0.05),
    "cfg4": (dict(n=7), 0.06),
    "cfg5": (dict(n=24), 0.05),
    "rotation": (dict(n=41), math.pi / 2),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    O.build()
    ref = O.reference()
    arrays = {}
    sums = {}

    # ghost fill (grid.cpp:108-165)
    g = abi.make_grid([0.0] * 3, [1.0] * 3, [5, 6, 7], [0, 1, 2])
    v = H.random_field(g, 17)
    arrays["pad/periodic/in"] = v
    for d in range(3):
        arrays[f"pad/periodic/d{d}"] = ref.pad_ghost(g, v, d, 2)
    g = abi.make_grid([0.0] * 3, [1.0] * 3, [5, 6, 7])
    arrays["pad/extrap/in"] = v
    for d in range(3):
        arrays[f"pad/extrap/d{d}"] = ref.pad_ghost(g, v, d, 3)

    # upwind derivatives (spatial_derivatives.cpp:37-224)
    for key, (g, seed) in UPWIND_GRIDS.items():
        v = H.random_field(g, seed)
        arrays[f"upwind/{key}/in"] = v
        for s in range(4):
            for d in range(g.dim):
                L, R = ref.upwind(g, v, d, s)
                arrays[f"upwind/{key}/s{s}/d{d}/L"] = L
                arrays[f"upwind/{key}/s{s}/d{d}/R"] = R

    # Lax-Friedrichs term (hamiltonian.cpp:11-76)
    for name in TERM_CASES:
        S = P.CONFIGS[name](**H.small(name))
        v0 = H.initial_value(ref, S)
        dvdt, bound = ref.term_lf(S.grid, S.problem, 0.0, v0)
        if v0.size <= 20000:
            arrays[f"term/{name}/in"] = v0
            arrays[f"term/{name}/dvdt"] = dvdt
        sums[f"term/{name}"] = {"in": sha(v0), "dvdt": sha(dvdt), "bound": bound.hex()}

    # integrate (integrator.cpp:22-125)
    for name, (kw, tf) in INTEGRATE_CASES.items():
        S = P.CONFIGS[name](**kw)
        v0 = H.initial_value(ref, S)
        v, steps, tfin = ref.integrate(S.grid, S.problem, S.method, 0.0, tf, v0, abi.make_opts())
        entry = {"kw": kw, "tf": tf, "in": sha(v0), "out": sha(v), "t_final": tfin.hex(), "n_steps": len(steps),
                 "steps": [[x.hex() for x in row] for row in steps]}
        if v.size <= 20000:
            arrays[f"integrate/{name}/out"] = v
        sums[f"integrate/{name}"] = entry

    # the reference's own rockets BRT (acceptance.cpp:381-419): N=50, 490 steps
    v, steps = ref.solve_rockets(50, (-2.5, 0.0), 11)
    sums["rockets50"] = {"out": sha(v), "n_steps": len(steps), "steps": [[x.hex() for x in row] for row in steps],
                         "v_min": float(v.min()), "v_max": float(v.max())}
    # a short rockets solve_brt with checkpoints, small enough to keep verbatim
    S = P.rockets(20)
    v0 = ref.rocket_initial(20)
    ck, times, steps = ref.solve_brt(S.grid, S.problem, v0, (-0.5, 0.0), 3, abi.CFL3, abi.make_opts())
    arrays["brt/rockets20/in"] = v0
    arrays["brt/rockets20/ck"] = ck
    arrays["brt/rockets20/times"] = times
    arrays["brt/rockets20/steps"] = steps

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden_sums.json"), "w") as f:
        json.dump(sums, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(sums)} checksum entries")


if __name__ == "__main__":
    main()
