mkdir -p gpurun_out
DBP_POLSPLIT_FFE_MIN_LOGN=11 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "golden or ffe or deterministic" > gpurun_out/ps3_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/ps3_tests.log
for args in "--algorithm ffe" "--algorithm ffe --block-len 4096 --overlap 700" "--algorithm ffe --block-len 4096 --overlap 1400"; do
  for r in 1 2; do for ml in 13 11; do
    x=$(DBP_POLSPLIT_FFE_MIN_LOGN=$ml timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
    echo "minlogn=$ml [$args] $x"
  done; done
done 2>&1 | tee gpurun_out/ab_ps3.txt
