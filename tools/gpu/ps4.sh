mkdir -p gpurun_out
for ml in 11 10; do DBP_POLSPLIT_FFE_MIN_LOGN=$ml timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "golden or ffe or deterministic or polsplit" > gpurun_out/ps4_tests_$ml.log 2>&1; echo "tests ml=$ml rc=$?"; tail -2 gpurun_out/ps4_tests_$ml.log; done
for args in "--algorithm ffe --block-len 1024 --overlap 700" "--algorithm ffe --block-len 1024 --overlap 256"; do
  for r in 1 2; do for ml in 11 10; do
    x=$(DBP_POLSPLIT_FFE_MIN_LOGN=$ml timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
    echo "minlogn=$ml [$args] $x"
  done; done
done 2>&1 | tee gpurun_out/ab_ps4.txt
