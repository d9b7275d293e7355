timeout 900 python -m pytest tests/test_gpu_bench_dist.py -m gpu -q > gpurun_out/p7.pytest.log 2>&1; echo "rc $?" >> gpurun_out/p7.pytest.log
bash tools/variant_run.sh p7 r1 dg4 dg16
