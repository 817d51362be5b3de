set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/r2_gputest.log
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
cat gpurun_out/r2_bench.json
python bench.py --impl reference --ref-seconds 40 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"
cat gpurun_out/r2_ref.json
for sk in "weno5 3" "eno3 2" "weno5-fast 4"; do set -- $sk
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:march3_kernel<$2, 7, 2, 0>" --launch-skip 1 -c 1 -o gpurun_out/r2_cfg5_$1 -f python bench.py --scheme $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/r2_ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg5.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/r2_launch.log 2>&1; echo "launches rc=$?"
