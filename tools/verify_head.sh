#!/bin/bash
# HEAD verification under gpurun: GPU suite, smoke, default bench, trace timings.
mkdir -p gpurun_out
o=gpurun_out/v
timeout 2400 python -m pytest tests -m gpu -q > $o.pytest.log 2>&1; echo "rc $?" >> $o.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o.smoke.log 2>&1; echo "rc $?" >> $o.smoke.log
timeout 600 python bench.py > $o.bench.log 2>&1; echo "rc $?" >> $o.bench.log
for c in medium chain_sharded; do timeout 300 python tools/trace_bench.py $c >> $o.tb.log 2>&1; done
