timeout 300 python tools/trace_bench.py ray_sharded > gpurun_out/tb_v30.log 2>&1
timeout 300 python tools/trace_bench.py small >> gpurun_out/tb_v30.log 2>&1
timeout 600 python tools/parity_margin.py ray_sharded > gpurun_out/pm_v30.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v30.log 2>&1
