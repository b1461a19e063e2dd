#!/bin/bash
# persistent group loop for N = 1024 / 2048 (DBP_PERSIST_MIN_LOGN=10 build, DBP_PERSISTENT=k) vs the full grid
for args in "" "--algorithm ffe" "--block-len 1024 --overlap 768 --nc 17"; do
  for c in "base -" "persist11 1" "persist11 2" "base -"; do
    set -- $c
    p=$2; [ "$p" = "-" ] && p=""
    x=$(DBP_PERSISTENT=$p DBP_LIB=build/variants/$1.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
    echo "$1 persistent=$2 [$args] $x"
  done
done
