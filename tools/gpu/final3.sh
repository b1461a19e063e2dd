# Round-end evidence (second pass): tests, bench, reference arm, launch list,
# ncu --set full of the headline kernel, configuration sweep, fuzz parity.
mkdir -p gpurun_out/final3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/final3/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final3/gputest.log
timeout 900 python bench.py > gpurun_out/final3/bench.json 2> gpurun_out/final3/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/final3/bench_reference.json 2> gpurun_out/final3/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final3/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final3/launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dbp_block_kernel --launch-skip 3 --launch-count 1 \
  -o gpurun_out/final3/headline python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final3/ncu.log 2>&1; echo "ncu rc=$?"
timeout 2400 python tools/config_sweep.py > gpurun_out/final3/configs.jsonl 2> gpurun_out/final3/configs.err; echo "sweep rc=$?"
timeout 900 python tools/fuzz_parity.py --out gpurun_out/final3/fuzz_parity.json > gpurun_out/final3/fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/final3/fuzz.log
# driver-contract checks: smoke(), default bench wall time, 2-rank bench (gloo, one GPU), reference arm under torchrun
mkdir -p gpurun_out/contract
( time timeout 600 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/contract/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/contract/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/contract/bench_default.json 2> gpurun_out/contract/bench_default.err; echo "bench rc=$?"; tail -4 gpurun_out/contract/bench_default.err
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/contract/bench_2rank.json 2> gpurun_out/contract/bench_2rank.err; echo "2rank rc=$?"; cat gpurun_out/contract/bench_2rank.json | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/contract/ref_2rank.json 2> gpurun_out/contract/ref_2rank.err; echo "ref2 rc=$?"; cut -c1-200 gpurun_out/contract/ref_2rank.json
