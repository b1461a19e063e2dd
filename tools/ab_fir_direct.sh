#!/bin/bash
# direct-form streamed FIR (DBP_FIR_DIRECT) and 64-register ESSFM at 1024 threads per SM
for args in "" "--nc 9" "--nc 33 --block-len 2048 --overlap 1400" "--num-steps 2" "--block-len 1024 --overlap 768" "--block-len 4096 --overlap 1400"; do
  for r in 1 2; do
    for v in base direct direct_1024_nogen; do
      x=$(DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
      echo "$v [$args] $x"
    done
  done
done
