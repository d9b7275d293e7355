mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_dist.py -m gpu -q > gpurun_out/pytest_gr1.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gr1.log
for w in tiny small medium; do
  timeout 600 python bench.py --workload $w --steps 200 --no-cpu-baseline > gpurun_out/gr1.$w.log 2>&1
  timeout 600 python bench.py --workload $w --steps 200 --no-cpu-baseline --graph off > gpurun_out/gr1.$w.off.log 2>&1
done
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/gr1.default.log 2>&1
timeout 600 python bench.py --steps 5 --no-cpu-baseline --graph off > gpurun_out/gr1.default.off.log 2>&1
timeout 600 python bench.py --workload ray_sharded --steps 50 --no-cpu-baseline > gpurun_out/gr1.ray.log 2>&1
