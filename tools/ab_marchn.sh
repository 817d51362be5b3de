# correctness of the 4-D..6-D tile-and-march kernel, then A/B against the generic kernel
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_dist_selftest.py -q -x -k "cfg3 or cfg4 or 5d_6d or all_dims or dims or fuzz or slabs or dist" 2>&1 | tail -3
LSG_M3_VERBOSE=1 python tools/config_bench.py cfg3 cfg4eno3 2>&1 | grep -v "^{" | sort | uniq -c | head
for k in marchn generic; do
  if [ $k = generic ]; then export LSG_KERNEL=generic; else unset LSG_KERNEL; fi
  python tools/config_bench.py cfg3 cfg4 cfg4eno3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$k', d['config'], d['scheme'], d['G_node_stage_per_s'], d['ms_per_step'])"
done
