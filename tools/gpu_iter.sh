#!/bin/bash
# One GPU iteration: GPU parity tests, then trace timings (tools/trace_bench.py).
# usage (under gpurun): bash tools/gpu_iter.sh TAG [configs...]
tag=$1; shift
cfgs=${@:-medium small}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$tag.log 2>&1; echo "rc $?" >> gpurun_out/pytest_$tag.log
for c in $cfgs; do timeout 300 python tools/trace_bench.py $c >> gpurun_out/tb_$tag.log 2>&1; done
