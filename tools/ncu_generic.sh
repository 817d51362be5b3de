# opcode census of the one-node-per-thread kernel on a 6-D config (cfg4 17^6, exact WENO5)
export PYTHONPATH=$PWD
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:stage_kernelILi6ELi3E" -c 1 -o gpurun_out/g6 -f python tools/one_stage_cfg.py cfg4 17 > gpurun_out/g6.log 2>&1
python - <<PY
import sys
sys.path.insert(0, "tools")
from make_ncu_summary import opcodes, raw
ops = opcodes("gpurun_out/g6.ncu-rep"); d = raw("gpurun_out/g6.ncu-rep")
n = 17**6
print({k: round(v*32/n,1) for k,v in ops.most_common(25)})
print("total", sum(ops.values())*32/n, "fp64", sum(v for k,v in ops.items() if k in ("DADD","DMUL","DFMA","DSETP"))*32/n)
for k in d:
    if ("stalled" in k and k.endswith("per_issue_active.ratio") and float(d[k])>0.08) or k in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active","smsp__issue_active.avg.pct_of_peak_sustained_active","launch__registers_per_thread","sm__warps_active.avg.pct_of_peak_sustained_active"): print(k, d[k])
PY
rm -f gpurun_out/g6.ncu-rep
