# compute-sanitizer over tools/sanitize_case.py (every kernel family on small grids)
export PYTHONPATH=$PWD
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.log
done
