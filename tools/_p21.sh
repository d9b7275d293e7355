timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/p21.pytest.log 2>&1; echo "rc $?" >> gpurun_out/p21.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p21.smoke.log 2>&1; echo "rc $?" >> gpurun_out/p21.smoke.log
timeout 600 python bench.py > gpurun_out/p21.default.log 2>&1
timeout 600 python bench.py --workload medium --steps 20 > gpurun_out/p21.medium.log 2>&1
timeout 600 python bench.py --workload small --steps 1000 > gpurun_out/p21.small.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p21.launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p21.ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_c2|k_trace_defer" -s 8 -c 2 \
  -o gpurun_out/p21.k2_8192 -f python tools/trace_bench.py chain_sharded --reps 3 > gpurun_out/p21.ncu3.log 2>&1
