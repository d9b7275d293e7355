#!/bin/bash
# Round-2 ncu evidence under gpurun (one GPU): launch lists of the default and
# ray-sharded bench commands, --set full captures of the trace kernels (8,192
# near-posterior chains, 8,192 prior-draw chains, the one-chain configs[4]) and
# of K3.  Each bench command runs once without ncu first (must exit 0).
# usage: bash tools/evidence_r2.sh TAG
tag=${1:-r2}
mkdir -p gpurun_out
o=gpurun_out/ev_$tag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o.smi.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $o.bench.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o.ncu1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches_ray.csv \
  python bench.py --workload ray_sharded --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o.ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_c2|k_trace_defer" -s 8 -c 2 \
  -o $o.k2_8192 -f python tools/trace_bench.py chain_sharded --reps 3 > $o.ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_rl|k_trace_defer" -s 8 -c 2 \
  -o $o.k2_ray -f python tools/trace_bench.py ray_sharded --reps 3 > $o.ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_finish" -s 4 -c 1 \
  -o $o.k3_8192 -f python tools/trace_bench.py chain_sharded --reps 3 > $o.ncu5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_c2" -s 4 -c 1 \
  -o $o.k2_prior -f python tools/trace_bench.py chain_sharded --prior --reps 3 > $o.ncu6.log 2>&1
echo done > $o.done
