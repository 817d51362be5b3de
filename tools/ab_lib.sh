# A/B of the current library against another in-tree build (LSG_LIB=<name> ->
# liblsg_b200_<name>.so) on the cfg5 grid, same box, interleaved:
#   gpurun -- bash tools/ab_lib.sh prev "eno3 weno5-fast weno5"
OTHER=${1:-prev}
for rep in 1 2; do
for sch in ${2:-eno3 weno5-fast weno5}; do
  for lib in "" $OTHER; do
    v=$(LSG_LIB=$lib python bench.py --scheme $sch --steps 20 --no-cpu-baseline --no-e2e --no-extras ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']/1e9,2), round(d['ms_per_step'],3))")
    echo "rep $rep $sch lib=${lib:-cur} ${BENCH_ARGS}: $v"
  done
done
done
