# chain-lanes deferred-pair group size A/B at configs[3] (8,192 chains)
for v in default d4 d16; do
  if [ $v = default ]; then L=""; else L=variants/libmt_$v.so; fi
  MT_LIB=$L python tools/trace_bench.py chain_sharded --reps 10
  MT_LIB=$L python tools/trace_bench.py chain_sharded --reps 10 --prior
done
