o=gpurun_out/var_p18.log
for pass in 1 2; do for v in r1 dg16 dg32; do
  echo "pass $pass variant $v" >> $o
  MT_LIB=variants/libmt_$v.so timeout 300 python tools/trace_bench.py small --reps 200 >> $o 2>&1
done; done
echo done >> $o
