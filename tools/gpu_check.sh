# quick device check: exact-WENO5 blocks, the GPU suite (minus the slow full-size file), a short bench
./tests/cpp/weno5_check; echo "weno5_check rc=$?"
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15
LSG_M3_VERBOSE=1 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo "bench rc=$?"
grep march3 gpurun_out/bench_check.err | sort | uniq -c | head
python -c "
import json; d=json.load(open('gpurun_out/bench_check.json')); print('value', d['value']/1e9, d['ms_per_step']); print({k:(v['value']/1e9, v['ms_per_step']) for k,v in d['extras'].items()})"
