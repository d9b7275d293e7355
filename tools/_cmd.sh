timeout 600 python tools/e2e_diag.py ray_sharded 0 > gpurun_out/e2e2.log 2>&1
timeout 900 python tools/parity_margin.py ray_sharded medium > gpurun_out/pm_v12.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v12.log 2>&1
timeout 300 python tools/trace_bench.py medium > gpurun_out/tb_v12.log 2>&1
