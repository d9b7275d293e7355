mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 60 python tools/trace_bench.py medium
timeout 60 python tools/trace_bench.py small
