# ray-lanes order change: parity + configs[4] bench lines (exact and voxel)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ev2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/ev2_pytest.log
timeout 600 python bench.py --workload ray_sharded --steps 50 > gpurun_out/ev2_bench_ray.log 2>&1
timeout 600 python bench.py --model voxel --workload ray_sharded --steps 50 > gpurun_out/ev2_bench_vxray.log 2>&1
timeout 300 python tools/trace_bench.py ray_sharded --reps 50 > gpurun_out/ev2_tb.log 2>&1
