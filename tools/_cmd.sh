timeout 600 python tools/tune_eps.py ray_sharded --chains 1 > gpurun_out/tune_ray.log 2>&1
cp data/tuned_eps.json gpurun_out/tuned_eps.json
timeout 600 python bench.py --workload ray_sharded > gpurun_out/bench_ray.log 2>&1
