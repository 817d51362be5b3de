"""Summarise ncu captures for profiles/: launch lists (shares per kernel) and
full-set reports (time, DRAM bytes, pipe utilisation, stalls)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__warps_active.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for w in WANT:
            if w in hdr:
                d[w] = f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip()
        out.append(d)
    return out


def launches(path):
    text = open(path).read()
    lines = [l for l in text.splitlines() if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1000.0 if unit in ("nsecond", "ns") else v
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_us": round(v, 2), "avg_us": round(v / cnt[k], 2),
             "share": round(v / s, 4)} for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(full(path) if kind == "full" else launches(path), indent=1))
