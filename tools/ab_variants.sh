#!/bin/bash
# A/B the 3-D kernel's launch bounds (rebuilds in place on the GPU box).
F=paper_2507_11542_b200/csrc/lsg_march3.cuh
cp $F /tmp/orig.cuh
run() {
  cp /tmp/orig.cuh $F
  sed -i "s/__launch_bounds__(256, 2) march3_kernel/__launch_bounds__(256, $1) march3_kernel/" $F
  make -C paper_2507_11542_b200/csrc -j32 > /dev/null 2>&1 || { echo build failed; return; }
  python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/v.json')); print('minBlocks=$1:', round(d['value']/1e9,2), 'G pt-stage/s', [round(x*1e3,1) for x in d['config']['stage_ms_mean']], 'frac', round(d['roofline']['frac'],3))"
}
run 2; run 1; run 3
cp /tmp/orig.cuh $F
