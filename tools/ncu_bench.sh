# ncu evidence for bench.py (run under gpurun, one GPU, after the plain bench exited 0):
#  * one `ncu --set full` capture of the dominant kernel (the COMBINE stage,
#    march3_kernel<S, NORMAL, COMBINE, no-range>) of `bench.py --scheme S` for
#    the bit-exact WENO5, the fast WENO5 and ENO3 on the cfg5 512^3 grid;
#  * the launch list (gpu__time_duration of every launch) of the default command.
# Summarise with: python tools/ncu_bench_summary.py <tag>
TAG=${1:-r2}
for sk in "weno5 3" "eno3 2" "weno5-fast 4"; do set -- $sk
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k "regex:march3_tma_kernelILi$2ELi7ELi2ELb0E" --launch-skip 1 -c 1 -o gpurun_out/${TAG}_cfg5_$1 -f \
      python bench.py --scheme $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras \
      > gpurun_out/${TAG}_ncu_$1.log 2>&1
  echo "ncu $1 rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg5.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_launch.log 2>&1
echo "launches rc=$?"
# summarise on the box (the reports are too large to bring back whole)
python tools/ncu_bench_summary.py ${TAG} && cp profiles/ncu_bench_captures.json gpurun_out/${TAG}_ncu_bench_captures.json
for s in weno5 eno3 weno5-fast; do
  ncu -i gpurun_out/${TAG}_cfg5_$s.ncu-rep --page details --csv > gpurun_out/${TAG}_cfg5_${s}_details.csv 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep; rm -f gpurun_out/${TAG}_cfg5_eno3.ncu-rep gpurun_out/${TAG}_cfg5_weno5-fast.ncu-rep
ls -la gpurun_out/${TAG}_cfg5_weno5.ncu-rep
