mkdir -p gpurun_out
bash tools/gpu_r2.sh pp1 notest default pp default pp
