# opcode histograms (executed SASS per node) of the COMBINE kernel, TMA vs cp.async, for one scheme
SCH=${SCH:-eno3}; S=${SID:-2}
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:march3_tma_kernelILi${S}ELi7ELi2ELb0E" --launch-skip 1 -c 1 -o gpurun_out/op_tma -f python bench.py --scheme $SCH --steps 3 --no-cpu-baseline --no-e2e --no-extras > /dev/null 2>&1
LSG_TMA=0 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:march3_kernelILi${S}ELi7ELi2ELb0E" --launch-skip 1 -c 1 -o gpurun_out/op_cpa -f python bench.py --scheme $SCH --steps 3 --no-cpu-baseline --no-e2e --no-extras > /dev/null 2>&1
python - <<'PY'
import sys, json
sys.path.insert(0, "tools")
from make_ncu_summary import opcodes, raw
n = 512**3
out = {}
for f in ("op_tma", "op_cpa"):
    ops = opcodes(f"gpurun_out/{f}.ncu-rep")
    out[f] = {k: round(v * 32 / n, 2) for k, v in ops.most_common(40)}
    d = raw(f"gpurun_out/{f}.ncu-rep")
    out[f]["_time"] = d["gpu__time_duration.sum"]
print(json.dumps(out))
json.dump(out, open("gpurun_out/opcodes.json", "w"), indent=1)
PY
ncu -i gpurun_out/op_tma.ncu-rep --page source --csv --print-source sass > gpurun_out/op_tma_sass.csv 2>/dev/null
for f in op_tma op_cpa; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv; done; rm -f gpurun_out/op_*.ncu-rep
