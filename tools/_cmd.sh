mkdir -p gpurun_out
bash tools/gpu_r2.sh pk1 notest default prev default prev
timeout 1200 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_launch_shapes.py tests/test_gpu_dist.py -m gpu -q > gpurun_out/pytest_pk1.log 2>&1; echo "rc $?" >> gpurun_out/pytest_pk1.log
