# full device evidence for the current build: GPU suite, smoke, ncu captures,
# then the bench (both arms; bench.py reads traffic and FP64 counts from the
# captures just written to profiles/ncu_bench_captures.json), one-rank NCCL selftest
set -x
TAG=${1:-r2}
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/${TAG}_gputest.log; cat gpurun_out/${TAG}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/ncu_bench.sh ${TAG}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --dist-selftest --steps 20 --no-cpu-baseline > gpurun_out/${TAG}_selftest.json 2> gpurun_out/${TAG}_selftest.err; echo "selftest rc=$?"
python tools/config_bench.py > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err; echo "configs rc=$?"
