#!/bin/bash
# Ray-sharded (configs[4]) evidence under gpurun: bench line, ncu launch list and
# one --set full capture of the ray-lanes trace + deferred-pair kernels.
# (GPU parity: tools/gpu_iter.sh or pytest -m gpu separately.)
mkdir -p gpurun_out
timeout 600 python bench.py --workload ray_sharded --steps 50 > gpurun_out/ev_bench_ray.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_ray.csv \
  python bench.py --workload ray_sharded --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_rl|k_trace_defer" -s 8 -c 2 \
  -o gpurun_out/k2_ray_r1g -f python tools/trace_bench.py ray_sharded --reps 3 > gpurun_out/ev_ncu2.log 2>&1
