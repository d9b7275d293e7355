o=gpurun_out/var_p16.log
for pass in 1 2; do for v in - MT_CHUNK=32 MT_CHUNK=40 MT_CHUNK=64; do
  echo "pass $pass variant $v" >> $o
  if [ "$v" = "-" ]; then timeout 300 python tools/trace_bench.py small --reps 200 >> $o 2>&1
  else env $v timeout 300 python tools/trace_bench.py small --reps 200 >> $o 2>&1; fi
done; done
echo done >> $o
