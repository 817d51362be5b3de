# A/B of the TMA-fed and cp.async-fed 3-D tile kernels on the cfg5 grid (same box, interleaved)
for rep in 1 2; do
for sch in ${SCHEMES:-eno3 weno5-fast weno5}; do
  for tma in 1 0; do
    v=$(LSG_TMA=$tma python bench.py --scheme $sch --steps 20 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']/1e9,2), round(d['ms_per_step'],3))")
    echo "rep $rep $sch tma=$tma: $v"
  done
done
done
