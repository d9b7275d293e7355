mkdir -p gpurun_out
bash tools/gpu_r2.sh k2p notest default head mb5
timeout 900 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/pytest_k2p.log 2>&1; echo "rc $?" >> gpurun_out/pytest_k2p.log
