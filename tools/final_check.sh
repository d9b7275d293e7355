#!/bin/bash
# End-of-round check under gpurun: build artefacts as committed, GPU parity, smoke, headline bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "rc $?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_bench.log 2>&1
