"""CPU tests of bench.py's command line: `--gpus N` outside torchrun launches N
ranks itself (torch.distributed.run on 127.0.0.1), and the two arms print the
same config for the same workload."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_spawns_n_ranks(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launch-check"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == list(range(n))
    assert {x["world_size"] for x in lines} == {n}
    assert {x["master_addr"] for x in lines} == {"127.0.0.1"}
    assert {x["nccl_debug"] for x in lines} == {"INFO"}  # communicator init logged (to stderr)


def test_arms_share_config():
    sys.path.insert(0, ROOT)
    import bench

    for cfg in ("cfg5", "cfg4", "cfg3", "cfg2"):
        for ws in (1, 2, 8):
            scheme = bench.DEFAULT_SCHEME[cfg]
            _, c1, s1 = bench.workload(cfg, scheme, ws)
            _, c2, s2 = bench.workload(cfg, scheme, ws)
            assert c1 == c2 and s1 == s2
    _, c, scaling = bench.workload("cfg5", "weno5", 8)
    assert c["grid"] == [512, 512, 4096] and scaling == "weak"
    _, c, scaling = bench.workload("cfg4", "weno5", 8)
    assert c["grid"] == [41] * 6 and scaling == "strong"
