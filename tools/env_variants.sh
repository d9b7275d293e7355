#!/bin/bash
# Time environment-knob variants of the in-tree libmt.so with tools/trace_bench.py,
# interleaved over two passes.  usage: env_variants.sh TAG "ENV=..." ...  ("-" = none)
tag=$1; shift
mkdir -p gpurun_out
o=gpurun_out/var_$tag.log
for pass in 1 2; do
  for v in "$@"; do
    for c in chain_sharded medium; do
      echo "pass $pass variant $v" >> $o
      if [ "$v" = "-" ]; then timeout 300 python tools/trace_bench.py $c --reps 10 >> $o 2>&1
      else env $v timeout 300 python tools/trace_bench.py $c --reps 10 >> $o 2>&1; fi
    done
  done
done
echo done >> $o
