bash tools/env_variants.sh p4 - MT_ORDER_DET=1 MT_ORDER_Z=0.55
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/p4.pytest.log 2>&1; echo "rc $?" >> gpurun_out/p4.pytest.log
