mkdir -p gpurun_out
timeout 400 python tools/tune_eps.py medium > gpurun_out/tune.log 2>&1; echo tune rc=$?; tail -2 gpurun_out/tune.log
timeout 120 python tools/tune_eps.py small >> gpurun_out/tune.log 2>&1; tail -1 gpurun_out/tune.log
cp data/tuned_eps.json gpurun_out/tuned_eps.json
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
