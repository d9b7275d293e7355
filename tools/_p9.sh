bash tools/variant_run.sh p9 "$@"
o=gpurun_out/var_p9_prior.log
for v in "$@"; do echo "pass 1 variant $v" >> $o; MT_LIB=variants/libmt_$v.so timeout 300 python tools/trace_bench.py chain_sharded --prior --reps 2 >> $o 2>&1; done
