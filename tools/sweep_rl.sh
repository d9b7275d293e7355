# tuning sweep for the ray-lanes path (configs[4]); variants built by tools/build_variants.sh
python tools/trace_bench.py ray_sharded --reps 50
MT_LIB=variants/libmt_p0.so python tools/trace_bench.py ray_sharded --reps 50
for s in 296 444 888 1184; do MT_TRACE_S=$s python tools/trace_bench.py ray_sharded --reps 50; done
python tools/trace_bench.py small --chains 4 --reps 50
MT_LIB=variants/libmt_p0.so python tools/trace_bench.py small --chains 4 --reps 50
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
