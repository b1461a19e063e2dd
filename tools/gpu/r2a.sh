mkdir -p gpurun_out
DBP_R2=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "8192 or golden or random or nofir or ffe_kernel_large" > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/r2a_tests.log
for args in "--block-len 8192 --overlap 1400" "--block-len 8192 --overlap 1024 --algorithm ssfm --num-steps 20 --arrangement linear-first --nc 0" "--algorithm ffe --block-len 8192 --overlap 1024" "--block-len 8192 --overlap 1400 --num-steps 4 --nc 33" "--block-len 8192 --overlap 1400 --num-steps 2 --nc 9"; do
  for r2 in 0 1; do
    x=$(DBP_R2=$r2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
    echo "r2=$r2 [$args] $x"
  done
done 2>&1 | tee gpurun_out/ab_r2a.txt
