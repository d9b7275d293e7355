# ray-lanes A/B: next-task prefetch (default L1), none, L2
for r in 1 2; do
python tools/trace_bench.py ray_sharded --reps 50
MT_LIB=variants/libmt_p0.so python tools/trace_bench.py ray_sharded --reps 50
MT_LIB=variants/libmt_p2.so python tools/trace_bench.py ray_sharded --reps 50
done
python tools/trace_bench.py small --chains 4 --reps 50
MT_LIB=variants/libmt_p0.so python tools/trace_bench.py small --chains 4 --reps 50
