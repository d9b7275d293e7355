#!/bin/bash
# Prior-draw (worst-case band) evidence under gpurun: bench line and one --set full
# capture of the chain-lanes trace kernel on prior-draw states (DRAM traffic).
mkdir -p gpurun_out
timeout 900 python bench.py --states prior > gpurun_out/ev_bench_prior.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_cl" -s 3 -c 1 \
  -o gpurun_out/k2_prior_r1 -f python tools/trace_bench.py chain_sharded --prior --reps 1 > gpurun_out/ev_ncu_prior.log 2>&1
