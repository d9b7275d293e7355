timeout 300 python tools/trace_bench.py medium > gpurun_out/tb_v27.log 2>&1
timeout 300 python tools/trace_bench.py medium --chains 8192 --reps 5 >> gpurun_out/tb_v27.log 2>&1
timeout 900 python tools/parity_margin.py medium small > gpurun_out/pm_v27.log 2>&1
