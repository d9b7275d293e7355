#!/bin/bash
# Round-2 final evidence under gpurun: every bench line (tools/bench_all.sh), the
# ncu launch lists of the default and ray-sharded bench commands, a --set full
# capture of the fused-leapfrog K3 (k_finish_g<STEP>) inside the bench step.
mkdir -p gpurun_out
bash tools/bench_all.sh
o=gpurun_out/fin
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o.ncu1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches_ray.csv \
  python bench.py --workload ray_sharded --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o.ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_finish_g" -s 40 -c 2 -o $o.k3_step -f \
  python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e > $o.ncu3.log 2>&1
echo done > $o.done
