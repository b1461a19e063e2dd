mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "golden or ffe or polsplit or warp_ffe" > gpurun_out/ps2_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/ps2_tests.log
for args in "--algorithm ffe --block-len 8192 --overlap 1024" "--algorithm ffe --block-len 8192 --overlap 1400" "--algorithm ffe --block-len 8192 --overlap 700"; do
  for r in 1 2; do for ps in 0 def; do
    if [ $ps = def ]; then x=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
    else x=$(DBP_POLSPLIT=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))"); fi
    echo "ps=$ps [$args] $x"
  done; done
done 2>&1 | tee gpurun_out/ab_ps2.txt
