# 3-D tile width sweep at 512^3 for the TMA kernel (LSG_M3_TX forces TX, R = 256 / (TX/2))
for tx in 32 64 128 16; do
  for sch in weno5 eno3 weno5-fast; do
    v=$(LSG_M3_TX=$tx python bench.py --scheme $sch --steps 20 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']/1e9,2))")
    echo "TX=$tx $sch: $v"
  done
done
