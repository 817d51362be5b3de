for k in marchn generic; do
  export LSG_KERNEL=$k
  python tools/config_bench.py cfg3 cfg4 cfg4eno3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$k', d['config'], d['scheme'], d['G_node_stage_per_s'], d['ms_per_step'])"
done
