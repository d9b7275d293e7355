#!/bin/bash
# The remaining bench lines at HEAD (outputs in gpurun_out/benchall5.*.log).
mkdir -p gpurun_out
B=gpurun_out/benchall5
timeout 600 python bench.py --workload tiny --steps 2000 > $B.tiny.log 2>&1
timeout 600 python bench.py --noncentred > $B.ncp.log 2>&1
timeout 600 python bench.py --sample-r > $B.sampler.log 2>&1
timeout 900 python bench.py --sampler nuts --chains-total 1024 --steps 3 > $B.nuts.log 2>&1
timeout 600 python bench.py --workload ray_sharded --steps 50 > $B.ray.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $B.reference.log 2>&1
echo done > $B.done
