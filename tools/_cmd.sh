mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/k3u.bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k3u.launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --graph off > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_finish_g" -s 1 -c 1 -o gpurun_out/k3u_plain -f python tools/trace_bench.py chain_sharded --reps 2 > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_k3_tiles.py tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q > gpurun_out/pytest_k3u.log 2>&1; echo "rc $?" >> gpurun_out/pytest_k3u.log
