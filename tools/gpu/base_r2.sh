set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest0.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest0.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err; echo "bench rc=$?"
cat gpurun_out/r2_bench0.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dbp_block_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2_base_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu0.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out
