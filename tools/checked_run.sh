# Bounds-checked device build (liblsg_b200_checked.so, LSG_CHECKED: every computed
# shared/global index of the stage kernels checked, trap on failure) over the
# small-case suite and the GPU parity tests.  Stand-in for compute-sanitizer,
# which is closed on this GPU pool.
export LSG_LIB=checked PYTHONPATH=$PWD
python tools/sanitize_case.py > gpurun_out/checked_cases.log 2>&1; echo "cases rc=$?"; tail -3 gpurun_out/checked_cases.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_dist_selftest.py tests/test_gpu_step_host.py -q -x -p no:cacheprovider 2>&1 | tail -4
