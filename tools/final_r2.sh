#!/bin/bash
# Round-2 final evidence under gpurun: the GPU test suite and smoke, every bench
# line (tools/bench_all.sh), the ncu launch lists of the default and ray-sharded
# bench commands (eager launches, so each kernel is listed), --set full captures
# of the trace kernel (8,192 chains) and of the fused-leapfrog K3 in the bench step.
mkdir -p gpurun_out
o=gpurun_out/fin
timeout 2400 python -m pytest tests -m gpu -q > $o.pytest.log 2>&1; echo "rc $?" >> $o.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o.smoke.log 2>&1; echo "rc $?" >> $o.smoke.log
bash tools/bench_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graph off > $o.ncu1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches_ray.csv \
  python bench.py --workload ray_sharded --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --graph off > $o.ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_c2|k_trace_defer" -s 4 -c 2 \
  -o $o.k2_8192 -f python tools/trace_bench.py chain_sharded --reps 3 > $o.ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_finish_g" -s 40 -c 2 -o $o.k3_step -f \
  python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e --graph off > $o.ncu3.log 2>&1
echo done > $o.done
