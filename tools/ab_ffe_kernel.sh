#!/bin/bash
# FFE-only kernel instantiation vs the generic operator-program kernel (build/variants/base.so)
for args in "--algorithm ffe --block-len 1024" "--algorithm ffe" "--algorithm ffe --block-len 4096" "--algorithm ffe --block-len 8192 --overlap 1024" "" "--algorithm ssfm --num-steps 20 --arrangement linear-first"; do
  for r in 1 2; do
    for lib in build/variants/base.so paper_1507_00921_b200/libdbp_b200.so; do
      x=$(DBP_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
      echo "$(basename $lib .so) [$args] $x"
    done
  done
done
