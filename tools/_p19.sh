timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/p19.pytest.log 2>&1; echo "rc $?" >> gpurun_out/p19.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p19.smoke.log 2>&1; echo "rc $?" >> gpurun_out/p19.smoke.log
timeout 600 python bench.py --workload small --steps 1000 > gpurun_out/p19.small.log 2>&1
timeout 600 python bench.py --workload tiny --steps 2000 > gpurun_out/p19.tiny.log 2>&1
timeout 600 python bench.py > gpurun_out/p19.default.log 2>&1
