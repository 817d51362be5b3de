#!/bin/bash
# Same-box A/B of two builds of liblsg_b200.so: tools/ab_so.sh BASE.so [rounds]
# (the in-tree build is the variant).  Interleaves bench.py runs and the
# per-config probe; prints one line per run.
P=paper_2507_11542_b200
BASE=$1; R=${2:-3}
cp $P/liblsg_b200.so /tmp/ab_var.so; cp $BASE /tmp/ab_base.so
for r in $(seq $R); do
  for v in base var; do
    cp /tmp/ab_$v.so $P/liblsg_b200.so
    python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['value']/1e9,2), 'G', [round(x*1e3,2) for x in d['config']['stage_ms_mean']], 'e2e', round(d['e2e']['value']/1e9,2))"
  done
done
for v in base var; do
  cp /tmp/ab_$v.so $P/liblsg_b200.so
  echo "== $v configs"; python tools/config_bench.py cfg2 cfg3 cfg5 cfg5eno3 2>/dev/null | grep -v "^\s*$" | tail -8
done
cp /tmp/ab_var.so $P/liblsg_b200.so
