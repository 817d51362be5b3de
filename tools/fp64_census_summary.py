"""Per-config FP64 / total instructions per node from one multi-kernel
`ncu --set full` report (tools/fp64_census.py): one row per captured launch,
the last launch of each config kept.

    python tools/fp64_census_summary.py census.ncu-rep census_order.json out.json
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import Counter

FP64_OPS = {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX"}
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def ncu(rep, page, i, extra=()):
    cmd = ["ncu", "-i", rep, "--page", page, "--csv", "--launch-skip", str(i), "--launch-count", "1", *extra]
    return list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))


def main():
    rep, order, out = sys.argv[1], json.load(open(sys.argv[2])), sys.argv[3]
    rows = {}
    for i, o in enumerate(order):
        raw = ncu(rep, "raw", i)
        if len(raw) < 3:
            break
        d = dict(zip(raw[0], raw[2]))
        u = dict(zip(raw[0], raw[1]))
        src = ncu(rep, "source", i, ("--print-source", "sass"))
        h = src[1]
        ia, isrc = h.index("Instructions Executed"), h.index("Source")
        cnt = Counter()
        for r in src[2:]:
            if r and r[0] == "Kernel Name":  # a filtered import can repeat the section: read the first only
                break
            if len(r) > ia and r[ia].isdigit():
                m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc].strip())
                if m:
                    cnt[m.group(2)] += int(r[ia])
        n = o["nodes"]
        f = lambda k: float(d[k].replace(",", ""))
        rows[o["label"]] = {
            "kernel_symbol": d["Kernel Name"],
            "gpu_time_us": round(f("gpu__time_duration.sum") * SCALE.get(u["gpu__time_duration.sum"], 1.0), 2),
            "fp64_instr_per_node": round(sum(v for k, v in cnt.items() if k in FP64_OPS) * 32 / n, 1),
            "instr_per_node": round(sum(cnt.values()) * 32 / n, 1),
            "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "registers": f("launch__registers_per_thread"),
            # cross-check of the source-page total against the raw counter
            "raw_instr_per_node": round(f("smsp__inst_executed.sum") * 32 / n, 1),
            "threads": f("launch__grid_size") * f("launch__block_size"),
            "source_sections": sum(1 for r in src if r and r[0] == "Kernel Name"),
        }
        print(o["label"], rows[o["label"]], flush=True)
    json.dump({"how": "ncu --set full of every config's COMBINE-stage kernel in one process "
                      "(tools/fp64_census.py; reduced sizes, instructions per node are size-independent)",
               "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
