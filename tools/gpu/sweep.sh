mkdir -p gpurun_out/sweep
timeout 2400 python tools/config_sweep.py > gpurun_out/sweep/configs.jsonl 2> gpurun_out/sweep/configs.err; echo "sweep rc=$?"
timeout 900 python bench.py > gpurun_out/sweep/bench.json 2> gpurun_out/sweep/bench.err; echo "bench rc=$?"
