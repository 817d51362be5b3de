# Per-instruction (SASS) execution counts and stall samples of the COMBINE
# stage of `bench.py --scheme S` (cfg5 512^3), for reading the hot loop here:
#   gpurun -- bash tools/ncu_source.sh TAG "eno3 2" "weno5-fast 4"
# Writes gpurun_out/TAG_src_S.csv.gz (ncu --page source --print-source sass).
TAG=$1; shift
for sk in "$@"; do set -- $sk
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k "regex:march3_tma_kernelILi$2ELi7ELi2ELb0E" --launch-skip 1 -c 1 -o /tmp/${TAG}_$1 -f \
      python bench.py --scheme $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras \
      > gpurun_out/${TAG}_ncusrc_$1.log 2>&1
  echo "ncu $1 rc=$?"
  ncu -i /tmp/${TAG}_$1.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/${TAG}_src_$1.csv.gz
done
