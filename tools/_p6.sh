o=gpurun_out/var_p6.log
for pass in 1 2; do for v in r1 rc2; do
  echo "pass $pass variant $v" >> $o
  MT_LIB=variants/libmt_$v.so timeout 600 python tools/trace_bench.py chain_sharded --prior --reps 3 >> $o 2>&1
  echo "pass $pass variant $v" >> $o
  MT_LIB=variants/libmt_$v.so timeout 300 python tools/trace_bench.py small --reps 20 >> $o 2>&1
done; done
echo done >> $o
