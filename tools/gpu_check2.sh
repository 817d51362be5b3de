python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_selftest.py -q -k "march3 or slabs or dist or integrate_vs or cfg5 or signed_zero" 2>&1 | tail -8
