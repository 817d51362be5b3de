"""Join the two arms of benchmarks/bench_kernels.cpp (JSON lines) into one
table: per case the reference and drop-in times, the speed-up and whether
the output checksums agree bit for bit.

    python tools/bench_kernels_compare.py b200.jsonl ref.jsonl [out.json]
"""
import json
import sys


def load(path):
    out = {}
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            r = json.loads(line)
            out[r["name"]] = r
    return out


def main():
    b, r = load(sys.argv[1]), load(sys.argv[2])
    rows = []
    for name, x in b.items():
        y = r.get(name)
        row = {"name": name, "b200_us": round(x["ns_per_iter"] / 1e3, 2),
               "b200_items_per_s": x["items_per_s"]}
        if y:
            row.update(ref_us=round(y["ns_per_iter"] / 1e3, 2), ref_items_per_s=y["items_per_s"],
                       speedup=round(y["ns_per_iter"] / x["ns_per_iter"], 2),
                       checksum_equal=x["checksum"] == y["checksum"])
        rows.append(row)
    print(f"{'case':34s} {'ref us':>12s} {'b200 us':>10s} {'x':>8s}  bits")
    for row in rows:
        print(f"{row['name']:34s} {row.get('ref_us', float('nan')):12.1f} {row['b200_us']:10.1f} "
              f"{row.get('speedup', float('nan')):8.2f}  {row.get('checksum_equal')}")
    if len(sys.argv) > 3:
        json.dump(rows, open(sys.argv[3], "w"), indent=1)


if __name__ == "__main__":
    main()
