#!/bin/bash
# Evidence at HEAD after the per-lane log-likelihood-sum change: chain-lanes bench lines
# whose trace kernel changed, and --set full of k_trace_c2 + k_trace_defer at 8,192 chains.
mkdir -p gpurun_out
o=gpurun_out/fin4
B=gpurun_out/benchall4
timeout 600 python bench.py --workload medium --steps 20 > $B.medium.log 2>&1
timeout 600 python bench.py --workload small --steps 1000 > $B.small.log 2>&1
timeout 900 python bench.py --states prior > $B.prior.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_c2|k_trace_defer" -s 8 -c 2 \
  -o $o.k2_8192 -f python tools/trace_bench.py chain_sharded --reps 3 > $o.ncu3.log 2>&1
echo done > $o.done
