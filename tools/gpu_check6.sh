python -m pytest tests/test_gpu_dist_selftest.py -q 2>&1 | tail -3
python bench.py --scheme eno3 --steps 20 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cfg5 eno3', round(d['value']/1e9,2))"
