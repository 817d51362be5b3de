"""profiles/ncu_bench_captures.json (read by bench.py) from the captures of
tools/ncu_bench.sh: per-launch time and DRAM bytes of the dominant kernel,
FP64 and total instructions per node from the SASS opcode counts, pipe/issue
utilisation, registers, and the launch-list share of each kernel.

    python tools/ncu_bench_summary.py <tag> [nodes]
"""
import csv
import io
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_ncu_summary import FP64_OPS, num, opcodes, raw  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def summary(rep, nodes):
    d = raw(rep)
    ops = opcodes(rep)
    total = sum(ops.values())
    fp64 = sum(v for k, v in ops.items() if k in FP64_OPS)
    return {
        "kernel_symbol": d["Kernel Name"],
        "capture": f"ncu --set full --clock-control none --import-source on of bench.py (tools/ncu_bench.sh); {os.path.basename(rep)}",
        "gpu_time_us": num(d, "gpu__time_duration.sum"),
        "dram_bytes_per_launch": num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum"),
        "dram_read_bytes": num(d, "dram__bytes_read.sum"),
        "dram_write_bytes": num(d, "dram__bytes_write.sum"),
        "algorithmic_bytes_per_launch": 24 * nodes,
        "fp64_instr_per_node": round(fp64 * 32 / nodes, 1),
        "instr_per_node": round(total * 32 / nodes, 1),
        "per_node_by_opcode": {k: round(v * 32 / nodes, 1) for k, v in ops.most_common(14)},
        "fp64_pipe_active_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "sm_active_fraction": round(num(d, "sm__cycles_active.avg") / num(d, "gpc__cycles_elapsed.max"), 3),
        "registers": num(d, "launch__registers_per_thread"),
        "grid": num(d, "launch__grid_size"),
    }


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)  # skip ==PROF== lines
    rows = rows[start:]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    t = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1.0)
        t[r[ik]][0] += 1
        t[r[ik]][1] += float(r[iv].replace(",", "")) * scale
    tot = sum(v[1] for v in t.values())
    return {k: {"launches": v[0], "total_us": round(v[1], 1), "mean_us": round(v[1] / v[0], 1),
                "share": round(v[1] / tot, 4)} for k, v in sorted(t.items(), key=lambda kv: -kv[1][1])}


def main():
    tag = sys.argv[1]
    nodes = int(sys.argv[2]) if len(sys.argv) > 2 else 512 ** 3
    out_dir = os.path.join(ROOT, "gpurun_out")
    res = {"how": "tools/ncu_bench.sh + tools/ncu_bench_summary.py: `ncu --set full --clock-control none` of one "
                  "COMBINE-stage launch of `python bench.py --scheme S --steps 3 --warmup 3` (cfg5 512^3); cold L2 per replay"}
    for scheme in ("weno5", "eno3", "weno5-fast"):
        rep = os.path.join(out_dir, f"{tag}_cfg5_{scheme}.ncu-rep")
        if os.path.exists(rep):
            res[f"cfg5/{scheme}"] = summary(rep, nodes)
    lp = os.path.join(out_dir, f"{tag}_launches_cfg5.csv")
    if os.path.exists(lp):
        res["launch_list_cfg5_weno5"] = launches(lp)
    path = os.path.join(ROOT, "profiles", "ncu_bench_captures.json")
    json.dump(res, open(path, "w"), indent=1)
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    main()
