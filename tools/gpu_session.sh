for k in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -6; done
