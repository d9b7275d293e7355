#!/bin/bash
# Round-2 (late) evidence on the final kernels: GPU suite + smoke, every bench
# line (tools/bench_all.sh), ncu launch lists and --set full captures (tools/evidence_r2.sh).
mkdir -p gpurun_out
o=gpurun_out/fin2
timeout 2400 python -m pytest tests -m gpu -q > $o.pytest.log 2>&1; echo "rc $?" >> $o.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o.smoke.log 2>&1; echo "rc $?" >> $o.smoke.log
bash tools/bench_all.sh
bash tools/evidence_r2.sh r2b
echo done > $o.done
