#!/bin/bash
# Every bench line committed under profiles/ (run under gpurun; outputs in gpurun_out/benchall.*.log).
mkdir -p gpurun_out
B=gpurun_out/benchall
rm -f $B.*.log
timeout 600 python bench.py > $B.default.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $B.reference.log 2>&1
timeout 600 python bench.py --workload tiny --steps 2000 > $B.tiny.log 2>&1
timeout 600 python bench.py --workload small --steps 1000 > $B.small.log 2>&1
timeout 600 python bench.py --workload medium --steps 20 > $B.medium.log 2>&1
timeout 900 python bench.py --states prior > $B.prior.log 2>&1
timeout 600 python bench.py --workload ray_sharded --steps 50 > $B.ray.log 2>&1
timeout 600 python bench.py --model voxel > $B.voxel.log 2>&1
timeout 600 python bench.py --model voxel --workload ray_sharded --steps 50 > $B.voxelray.log 2>&1
timeout 600 python bench.py --noncentred > $B.ncp.log 2>&1
timeout 600 python bench.py --sample-r > $B.sampler.log 2>&1
timeout 900 python bench.py --sampler nuts --chains-total 1024 --steps 3 > $B.nuts.log 2>&1
