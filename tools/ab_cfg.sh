# A/B of the current library against another in-tree build on BASELINE configs
# at full size (tools/config_bench.py), same box, interleaved:
#   gpurun -- bash tools/ab_cfg.sh prev cfg3 cfg4 cfg4eno3
OTHER=$1; shift
for rep in 1 2; do
  for lib in "" $OTHER; do
    LSG_LIB=$lib python tools/config_bench.py "$@" 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('rep $rep lib=${lib:-cur}', d['config'], d['scheme'], d['G_node_stage_per_s'], d['ms_per_step'])"
  done
done
