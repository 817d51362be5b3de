./tests/cpp/weno5_check; echo "weno5_check rc=$?"
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_b.json 2> gpurun_out/r2_bench_b.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r2_bench_b.json')); print('value', d['value']/1e9, d['ms_per_step']); print({k:(v['value']/1e9, v['ms_per_step']) for k,v in d['extras'].items()})"
