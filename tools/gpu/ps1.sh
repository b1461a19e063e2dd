# polarisation-split pairs at N = 8192: parity with DBP_POLSPLIT=1, then A/B
mkdir -p gpurun_out
DBP_POLSPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "8192 or golden or random or deterministic or nofir or ffe_kernel_large" > gpurun_out/ps1_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/ps1_tests.log
for args in "--block-len 8192 --overlap 1400" "--block-len 8192 --overlap 1024 --algorithm ssfm --num-steps 20 --arrangement linear-first --nc 0" "--algorithm ffe --block-len 8192 --overlap 1024" "--block-len 8192 --overlap 1400 --num-steps 1 --nc 33"; do
  for ps in 0 1; do
    x=$(DBP_POLSPLIT=$ps timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
    echo "ps=$ps [$args] $x"
  done
done 2>&1 | tee gpurun_out/ab_ps1.txt
