mkdir -p gpurun_out
bash tools/gpu_r2.sh pf1 notest default pf default pf
