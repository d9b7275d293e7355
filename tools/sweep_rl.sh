# ray-lanes A/B: 128-thread blocks (8/SM) vs 256 (4/SM)
for r in 1 2; do
python tools/trace_bench.py ray_sharded --reps 50
MT_LIB=variants/libmt_t128.so python tools/trace_bench.py ray_sharded --reps 50
done
for s in 2368 9472; do MT_TRACE_S=$s MT_LIB=variants/libmt_t128.so python tools/trace_bench.py ray_sharded --reps 50; done
MT_LIB=variants/libmt_t128.so python tools/trace_bench.py small --chains 4 --reps 50
python tools/trace_bench.py small --chains 4 --reps 50
