mkdir -p gpurun_out
for w in 1 0; do
DBP_WARP_FFE=$w timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "golden or ffe or deterministic or random" > gpurun_out/warp2_tests_$w.log 2>&1; echo "warp=$w tests rc=$?"; tail -3 gpurun_out/warp2_tests_$w.log
done
for args in "--algorithm ffe" "--algorithm ffe --block-len 4096 --overlap 700"; do
    for cfg in "base 0" "base 1" "wcta2 1"; do
      set -- $cfg
      lib=paper_1507_00921_b200/libdbp_b200.so; [ "$1" != base ] && lib=build/variants/$1.so
      x=$(DBP_LIB=$lib DBP_WARP_FFE=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3), d['roofline']['bound'])")
      echo "$1 warp=$2 [$args] $x"
    done
done 2>&1 | tee gpurun_out/ab_warp2.txt
DBP_LIB=build/variants/wcta2.so DBP_WARP_FFE=1 timeout 600 ncu --set full --clock-control none -k regex:warp_ffe -c 1 -o gpurun_out/warp_ffe python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --algorithm ffe > gpurun_out/warp_ncu.log 2>&1; echo "ncu rc=$?"
