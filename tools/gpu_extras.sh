# reference-facing solves and the reference's microbenchmark suite on this build
python tools/solve_bench.py > gpurun_out/r2_solves.json 2> gpurun_out/r2_solves.err; echo "solves rc=$?"
./benchmarks/bench_kernels_b200 --large > gpurun_out/bk_b200.jsonl 2>&1; echo "bk b200 rc=$?"
./oracle/_ref/bench_kernels_ref --large > gpurun_out/bk_ref.jsonl 2>&1; echo "bk ref rc=$?"
python tools/bench_kernels_compare.py gpurun_out/bk_b200.jsonl gpurun_out/bk_ref.jsonl gpurun_out/r2_bench_kernels.json > /dev/null; echo "compare rc=$?"
cat gpurun_out/r2_solves.json
