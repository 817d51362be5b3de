# The FP64 census of profiles/r1_fp64_census.json (run under gpurun, one ncu capture):
#   gpurun -- bash tools/census_run.sh
set -e
python tools/fp64_census.py
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:stage_kernel<.*\(int\)2>|march3_kernel<.*\(int\)2, \(bool\)1>' \
  -o gpurun_out/census -f python tools/fp64_census.py > gpurun_out/census_ncu.log 2>&1
python tools/fp64_census_summary.py gpurun_out/census.ncu-rep gpurun_out/census_order.json gpurun_out/census.json
python - <<'PY'
import subprocess, csv, io, re, json
from collections import Counter
order = json.load(open("gpurun_out/census_order.json"))
for i, o in enumerate(order):
    if o["label"] not in ("cfg4eno3_17_exact", "cfg3_41_exact") or (i + 1 < len(order) and order[i + 1]["label"] == o["label"]):
        continue
    t = subprocess.run(["ncu", "-i", "gpurun_out/census.ncu-rep", "--page", "source", "--csv", "--print-source", "sass",
                        "--launch-skip", str(i), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(t)))
    h = rows[1]; ia, isrc = h.index("Instructions Executed"), h.index("Source")
    cnt = Counter()
    for r in rows[2:]:
        if r and r[0] == "Kernel Name": break
        if len(r) > ia and r[ia].isdigit():
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc].strip())
            if m: cnt[m.group(2)] += int(r[ia])
    print(o["label"], {k: round(v * 32 / o["nodes"], 1) for k, v in cnt.most_common(20)})
PY
rm -f gpurun_out/census.ncu-rep
