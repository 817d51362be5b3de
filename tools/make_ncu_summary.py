"""Build profiles/ncu_summary.json (read by bench.py) from one `ncu --set full`
capture of the dominant kernel: per-launch time and DRAM bytes, FP64
instructions per node from the SASS opcode counts, pipe/issue utilisation and
the SM-active fraction.

    python tools/make_ncu_summary.py <report.ncu-rep> <nodes> <label> [out.json]
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import Counter

FP64_OPS = {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX"}


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "ns": 1e-3, "us": 1.0, "ms": 1e3}


def raw(rep):
    """metric -> value in base units (bytes, microseconds)."""
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    out = {}
    for k, u, v in zip(rows[0], rows[1], rows[2]):
        try:
            out[k] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
        except ValueError:
            out[k] = v
    return out


def opcodes(rep):
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    h = rows[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    cnt = Counter()
    for r in rows[2:]:
        if len(r) <= ia or not r[ia].isdigit():
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc].strip())
        if m:
            cnt[m.group(2)] += int(r[ia])
    return cnt


def num(d, k):
    return float(d[k])


def main():
    rep, nodes, label = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    d = raw(rep)
    ops = opcodes(rep)
    total = sum(ops.values())
    fp64 = sum(v for k, v in ops.items() if k in FP64_OPS)
    out = {
        "kernel": label,
        "kernel_symbol": d["Kernel Name"],
        "capture": f"ncu --set full --clock-control none --import-source on (cold L2 per replay); {rep}",
        "gpu_time_us": num(d, "gpu__time_duration.sum"),
        "dram_bytes_per_launch": num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum"),
        "dram_read_bytes": num(d, "dram__bytes_read.sum"),
        "dram_write_bytes": num(d, "dram__bytes_write.sum"),
        "fp64_warp_instructions_per_launch": fp64,
        "fp64_instr_per_node": round(fp64 * 32 / nodes, 1),
        "instr_per_node": round(total * 32 / nodes, 1),
        "per_node_by_opcode": {k: round(v * 32 / nodes, 1) for k, v in ops.most_common(12)},
        "fp64_pipe_active_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "sm_active_fraction": round(num(d, "sm__cycles_active.avg") / num(d, "gpc__cycles_elapsed.max"), 3),
        "registers": num(d, "launch__registers_per_thread"),
        "grid": num(d, "launch__grid_size"),
    }
    s = json.dumps(out, indent=1)
    print(s)
    if len(sys.argv) > 4:
        open(sys.argv[4], "w").write(s + "\n")


if __name__ == "__main__":
    main()
