# tuning sweep for the ray-lanes path (configs[4]); variants built by tools/build_variants.sh
for v in r8 r16 r32; do MT_LIB=variants/libmt_$v.so python tools/trace_bench.py ray_sharded --reps 50; done
for v in r8 r32; do MT_LIB=variants/libmt_$v.so python tools/trace_bench.py small --chains 4 --reps 50; done
