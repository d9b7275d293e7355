o=gpurun_out/var_p10.log
for pass in 1 2; do for v in - MT_ORDER_DET=1 "MT_ORDER_DET=1 MT_ORDER_Z=0.5" "MT_ORDER_DET=1 MT_ORDER_Z=0.1" "MT_ORDER_Z=0.3"; do
  echo "pass $pass variant $v" >> $o
  if [ "$v" = "-" ]; then timeout 300 python tools/trace_bench.py ray_sharded --reps 20 >> $o 2>&1
  else env $v timeout 300 python tools/trace_bench.py ray_sharded --reps 20 >> $o 2>&1; fi
done; done
echo done >> $o
