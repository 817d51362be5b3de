python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "fast" 2>&1 | tail -3
SCHEMES="weno5-fast" bash tools/ab_tma.sh
