mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_k3c.log 2>&1
bash tools/gpu_r2.sh k3c notest default nogb t128m9 t128m8
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exhaustive.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/pytest_k3c.log 2>&1; echo "rc $?" >> gpurun_out/pytest_k3c.log
timeout 600 ncu --set full --clock-control none -k regex:"k_finish_g" -s 2 -c 1 -o gpurun_out/k3i -f python tools/trace_bench.py chain_sharded --reps 3 > gpurun_out/ncu_k3i.log 2>&1
