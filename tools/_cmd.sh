mkdir -p gpurun_out
bash tools/gpu_r2.sh k2q notest default head default head
timeout 900 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_dist.py tests/test_summaries.py -m gpu -x -q > gpurun_out/pytest_k2q.log 2>&1; echo "rc $?" >> gpurun_out/pytest_k2q.log
