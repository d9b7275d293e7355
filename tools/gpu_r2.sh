#!/bin/bash
# Round-2 GPU iteration: parity tests (optional), then trace timings per variant.
# usage (under gpurun): bash tools/gpu_r2.sh TAG [test|notest] [variant ...]
# a variant is "default", a library name (paper_2603_28907_b200/libmt_<name>.so) or ENV=VALUE
tag=$1; shift
mode=$1; shift
cfgs=${CFGS:-medium chain_sharded}
[ -n "$CFG_LIST" ] && cfgs=$CFG_LIST
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$tag.txt 2>&1
if [ "$mode" = "test" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$tag.log 2>&1; echo "rc $?" >> gpurun_out/pytest_$tag.log
fi
for v in "$@"; do
  for c in $cfgs; do
    echo "== $v $c" >> gpurun_out/tb_$tag.log
    if [ "$v" = default ]; then
      timeout 300 python tools/trace_bench.py $c >> gpurun_out/tb_$tag.log 2>&1
    elif [[ "$v" == *=* ]]; then
      env $v timeout 300 python tools/trace_bench.py $c >> gpurun_out/tb_$tag.log 2>&1
    else
      MT_LIB=$PWD/paper_2603_28907_b200/libmt_$v.so timeout 300 python tools/trace_bench.py $c >> gpurun_out/tb_$tag.log 2>&1
    fi
  done
done
