timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/p17.pytest.log 2>&1; echo "rc $?" >> gpurun_out/p17.pytest.log
timeout 600 python bench.py --workload small --steps 1000 > gpurun_out/p17.small.log 2>&1
timeout 600 python bench.py > gpurun_out/p17.default.log 2>&1
for c in small medium; do timeout 300 python tools/trace_bench.py $c --reps 100 >> gpurun_out/p17.tb.log 2>&1; done
