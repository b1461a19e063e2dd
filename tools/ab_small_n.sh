#!/bin/bash
# small-N occupancy / CTA-size A/B: variants x (N, M, algorithm)
for v in "$@"; do
  for args in "--block-len 1024 --overlap 768 --nc 17" "--block-len 1024 --overlap 700 --algorithm ffe" "--block-len 512 --overlap 300 --nc 9" "--block-len 256 --overlap 100 --algorithm ssfm" "--block-len 128 --overlap 32 --nc 9"; do
    r=$(DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
    echo "$v [$args] $r"
  done
done
