#!/bin/bash
# Evidence after the in-lane K, M change (chain and ray lanes): GPU suite + smoke,
# the chain-lanes bench lines, launch list, --set full of the trace kernels.
mkdir -p gpurun_out
o=gpurun_out/fin3
timeout 2400 python -m pytest tests -m gpu -q > $o.pytest.log 2>&1; echo "rc $?" >> $o.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o.smoke.log 2>&1; echo "rc $?" >> $o.smoke.log
B=gpurun_out/benchall3
timeout 600 python bench.py > $B.default.log 2>&1
timeout 600 python bench.py --workload medium --steps 20 > $B.medium.log 2>&1
timeout 600 python bench.py --workload small --steps 1000 > $B.small.log 2>&1
timeout 900 python bench.py --states prior > $B.prior.log 2>&1
timeout 600 python bench.py --noncentred > $B.ncp.log 2>&1
timeout 600 python bench.py --sample-r > $B.sampler.log 2>&1
timeout 900 python bench.py --sampler nuts --chains-total 1024 --steps 3 > $B.nuts.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o.ncu1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o.launches_ray.csv \
  python bench.py --workload ray_sharded --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o.ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_c2|k_trace_defer" -s 8 -c 2 \
  -o $o.k2_8192 -f python tools/trace_bench.py chain_sharded --reps 3 > $o.ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_rl|k_trace_defer" -s 8 -c 2 \
  -o $o.k2_ray -f python tools/trace_bench.py ray_sharded --reps 3 > $o.ncu4.log 2>&1
echo done > $o.done
