set -e
python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bA.json 2>gpurun_out/bA.err
python -c "import json; d=json.load(open('gpurun_out/bA.json')); print('A (256,2):', round(d['value']/1e9,2), [round(x*1e3,1) for x in d['config']['stage_ms_mean']], round(d['roofline']['frac'],3))"
sed -i 's/__launch_bounds__(256, 2) march3_kernel/__launch_bounds__(256, 1) march3_kernel/' paper_2507_11542_b200/csrc/lsg_march3.cuh
make -C paper_2507_11542_b200/csrc -j16 > /dev/null 2>&1
python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bB.json 2>gpurun_out/bB.err
python -c "import json; d=json.load(open('gpurun_out/bB.json')); print('B (256,1):', round(d['value']/1e9,2), [round(x*1e3,1) for x in d['config']['stage_ms_mean']], round(d['roofline']['frac'],3))"
