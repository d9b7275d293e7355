mkdir -p gpurun_out
CFG_LIST="ray_sharded" bash tools/gpu_r2.sh rl2a notest default MT_RL_V=2 default MT_RL_V=2
MT_RL_V=2 timeout 1200 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_parity.py tests/test_gpu_launch_shapes.py -m gpu -q > gpurun_out/pytest_rl2a.log 2>&1; echo "rc $?" >> gpurun_out/pytest_rl2a.log
