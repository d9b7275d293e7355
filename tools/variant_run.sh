#!/bin/bash
# Time libmt variants (variants/libmt_<name>.so, tools/build_variants.sh) with
# tools/trace_bench.py, interleaved over two passes.  usage: variant_run.sh TAG name...
tag=$1; shift
mkdir -p gpurun_out
o=gpurun_out/var_$tag.log
for pass in 1 2; do
  for v in "$@"; do
    for c in chain_sharded medium; do
      echo "pass $pass variant $v" >> $o
      MT_LIB=variants/libmt_$v.so timeout 300 python tools/trace_bench.py $c --reps 10 >> $o 2>&1
    done
  done
done
for v in "$@"; do
  MT_LIB=variants/libmt_$v.so timeout 600 ncu --metrics launch__shared_mem_config_size,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,smsp__inst_executed.sum -k regex:k_trace_c2 -c 1 \
    python tools/trace_bench.py chain_sharded --reps 1 > gpurun_out/var_${tag}_ncu_$v.txt 2>&1
done
echo done >> $o
