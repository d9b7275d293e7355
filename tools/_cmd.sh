mkdir -p gpurun_out
bash tools/gpu_r2.sh qe1 notest default qf ex default qf ex
