# Round-end evidence (second pass): tests, bench, reference arm, launch list,
# ncu --set full of the headline kernel, configuration sweep, fuzz parity.
mkdir -p gpurun_out/final4
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/final4/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final4/gputest.log
timeout 900 python bench.py > gpurun_out/final4/bench.json 2> gpurun_out/final4/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/final4/bench_reference.json 2> gpurun_out/final4/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final4/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final4/launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dbp_block_kernel --launch-skip 3 --launch-count 1 \
  -o gpurun_out/final4/headline python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final4/ncu.log 2>&1; echo "ncu rc=$?"
timeout 2400 python tools/config_sweep.py > gpurun_out/final4/configs.jsonl 2> gpurun_out/final4/configs.err; echo "sweep rc=$?"
timeout 900 python tools/fuzz_parity.py --out gpurun_out/final4/fuzz_parity.json > gpurun_out/final4/fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/final4/fuzz.log
