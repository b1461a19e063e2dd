#!/bin/bash
# FFE-only kernel occupancy variants (DBP_FFE_THREADS_PER_SM) at N = 1024 / 2048 / 4096
for args in "--algorithm ffe --block-len 1024" "--algorithm ffe" "--algorithm ffe --block-len 4096"; do
  for r in 1 2; do
    for v in base ffe10 ffe10_768 ffe10_1024 ffe10_512; do
      x=$(DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
      echo "$v [$args] $x"
    done
  done
done
