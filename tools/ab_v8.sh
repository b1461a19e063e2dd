#!/bin/bash
# v8 (direct-form FIR, 64-register fixed-tap kernel at 1024 threads/SM, kProgGenericFir) vs v7d (build/variants/base.so)
for args in "" "--block-len 1024 --overlap 768 --nc 17" "--block-len 512 --overlap 300 --nc 9" "--block-len 128 --overlap 32 --nc 9" "--block-len 256 --overlap 64 --nc 17" "--nc 5" "--block-len 8192 --overlap 1400 --nc 17" "--algorithm ssfm --num-steps 20 --arrangement symmetric"; do
  for r in 1 2; do
    for lib in build/variants/base.so paper_1507_00921_b200/libdbp_b200.so; do
      x=$(DBP_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
      echo "$(basename $lib .so) [$args] $x"
    done
  done
done
