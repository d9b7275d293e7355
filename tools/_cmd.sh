mkdir -p gpurun_out
bash tools/gpu_r2.sh unp1 notest default unp default unp
CFG_LIST="ray_sharded" bash tools/gpu_r2.sh ra1 notest default ra32 default ra32
