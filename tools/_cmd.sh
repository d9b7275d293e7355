for v in default mb5 mb6; do
  if [ $v = default ]; then unset MT_LIB; else export MT_LIB=$PWD/variants/libmt_$v.so; fi
  timeout 300 python tools/trace_bench.py medium >> gpurun_out/tb_v18.log 2>&1
done
