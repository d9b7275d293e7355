for v in default g05 g03 g05z; do
  if [ $v = default ]; then unset MT_LIB; else export MT_LIB=$PWD/variants/libmt_$v.so; fi
  timeout 300 python tools/trace_bench.py medium >> gpurun_out/tb_v4.log 2>&1
  timeout 600 python tools/parity_margin.py tiny small medium >> gpurun_out/pm_v4.log 2>&1
done
