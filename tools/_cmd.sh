mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_full2.log 2>&1; echo "rc $?" >> gpurun_out/pytest_full2.log
CFG_LIST="ray_sharded" bash tools/gpu_r2.sh rlsm notest default rlsm default rlsm
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "rc $?" >> gpurun_out/smoke2.log
