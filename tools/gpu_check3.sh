python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_selftest.py tests/test_gpu_fuzz.py -q -x -k "march3 or slabs or dist or integrate_vs or cfg5 or signed_zero or fuzz or tiling" 2>&1 | tail -4
bash tools/ab_tma.sh
