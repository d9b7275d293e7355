timeout 300 python tools/trace_bench.py ray_sharded > gpurun_out/tb_v24.log 2>&1
timeout 300 python tools/trace_bench.py medium >> gpurun_out/tb_v24.log 2>&1
timeout 900 python tools/parity_margin.py ray_sharded medium > gpurun_out/pm_v24.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v24.log 2>&1
