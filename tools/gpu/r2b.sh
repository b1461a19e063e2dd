mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b/gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b/gputest.log
A="--block-len 8192 --overlap 1024 --algorithm ssfm --num-steps 20 --arrangement linear-first --nc 0"
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $A > gpurun_out/r2b/bench_ssfm20_8192.json 2>&1; echo "bench rc=$?"; cut -c1-200 gpurun_out/r2b/bench_ssfm20_8192.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dbp_r2_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2b/r2_ssfm20 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $A > gpurun_out/r2b/ncu.log 2>&1; echo "ncu rc=$?"
B="--block-len 8192 --overlap 1400"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dbp_r2_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2b/r2_essfm python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $B > gpurun_out/r2b/ncu2.log 2>&1; echo "ncu2 rc=$?"
