o=gpurun_out/var_p8.log
for pass in 1 2; do for v in "$@"; do
  echo "pass $pass variant $v" >> $o
  MT_LIB=variants/libmt_$v.so timeout 300 python tools/trace_bench.py ray_sharded --reps 20 >> $o 2>&1
done; done
for v in "$@"; do
  MT_LIB=variants/libmt_$v.so timeout 600 ncu --metrics launch__shared_mem_config_size,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,smsp__inst_executed.sum -k regex:k_trace_rl -c 1 \
    python tools/trace_bench.py ray_sharded --reps 1 > gpurun_out/var_p8_ncu_$v.txt 2>&1
done
echo done >> $o
