#!/bin/bash
# split write-after-read barriers: more block lengths / programs
for args in "--block-len 512 --overlap 300 --nc 9" "--block-len 256 --overlap 100 --nc 9" "--block-len 4096 --overlap 700 --algorithm ffe" "--block-len 4096 --overlap 1400 --nc 1 --num-steps 4" "--block-len 2048 --overlap 1400 --nc 17 --num-steps 2"; do
 for v in nosplit split nosplit split; do
  x=$(DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))"); echo "$v [$args] $x"
 done
done
