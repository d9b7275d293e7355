mkdir -p gpurun_out
bash tools/gpu_r2.sh df1 notest default df3 df4 dg4 dg16
