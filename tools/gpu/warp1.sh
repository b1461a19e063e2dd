# warp-resident FFE kernel: parity first, then A/B against the block kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/warp1_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/warp1_tests.log
for args in "--algorithm ffe" "--algorithm ffe --block-len 1024 --overlap 700" "--algorithm ffe --block-len 4096 --overlap 700"; do
  for r in 1 2; do
    for cfg in "base 0" "base 1" "wcta2 1"; do
      set -- $cfg
      lib=paper_1507_00921_b200/libdbp_b200.so; [ "$1" != base ] && lib=build/variants/$1.so
      x=$(DBP_LIB=$lib DBP_WARP_FFE=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3), d['roofline']['bound'])")
      echo "$1 warp=$2 [$args] $x"
    done
  done
done 2>&1 | tee gpurun_out/ab_warp1.txt
