"""The reference CPU library (oracle/_ref, compiled from the reference's own
sources, 1 thread: the reference is single-threaded) timed on every BASELINE
config beside the B200 numbers.  Configs the host cannot hold
or finish in seconds run on a stated smaller sample of the same problem (the
per-node-stage rate of the CPU path is close to size-independent): cfg4 at
17^6 as SURVEY §8(d) prescribes, cfg3 at 41^4, cfg5 at 128^3.
Prints one JSON object; the B200 column comes from profiles/r1_configs.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import helpers_path  # noqa: F401  (tests/ on sys.path for the initial conditions)
import helpers as H
from oracle import oracle as O
from paper_2507_11542_b200 import abi
from paper_2507_11542_b200 import problems as P

ref = O.reference()
SAMPLES = [
    ("cfg1_circle_2d", "ENO2", P.cfg1_circle(101), "full 101^2"),
    ("cfg2_air3d", "ENO3", P.cfg2_air3d(101), "full 101^3"),
    ("cfg3_dblint4", "WENO5", P.cfg3_dblint4(41), "41^4 sample of 81^4"),
    ("cfg4_dubins6", "WENO5", P.cfg4_dubins6(17), "17^6 sample of 41^6 (SURVEY §8(d))"),
    ("cfg5_normal", "WENO5", P.cfg5_normal(128), "128^3 sample of 512^3"),
    ("cfg5_normal", "ENO3", P.cfg5_normal(128, scheme=abi.SCHEME_ENO3), "128^3 sample of 512^3"),
]
target = float(os.environ.get("CPU_SECONDS", "8"))
out = []
for name, scheme, S, sample in SAMPLES:
    v0 = H.initial_value(ref, S)
    _, bound = ref.term_lf(S.grid, S.problem, 0.0, v0)
    dt = 0.32 * bound
    opts = abi.make_opts(max_step=dt)
    secs1, steps1 = ref.bench(S.grid, S.problem, S.method, v0, dt, opts, 1)
    k = max(1, min(400, int(target / max(secs1, 1e-9))))
    secs, steps = (secs1, steps1) if k == 1 else ref.bench(S.grid, S.problem, S.method, v0, k * dt, opts, 1)
    stages = S.method + 1
    out.append({"config": name, "scheme": scheme, "sample": sample, "nodes": int(v0.size), "steps": int(steps),
                "seconds": round(secs, 3), "ref_1thread_node_stages_per_s": v0.size * stages * steps / secs})
print(json.dumps(out, indent=1))
