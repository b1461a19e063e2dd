#!/bin/bash
# single vs double-buffered exchange regions under forced shared-memory carve-outs
for args in "" "--algorithm ffe"; do
  for c in "single -" "single 100" "single 50" "double -"; do
    set -- $c
    cv=$2; [ "$cv" = "-" ] && cv=""
    x=$(DBP_CARVEOUT=$cv DBP_LIB=build/variants/$1.so timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
    echo "$1 carve=$2 [$args] $x"
  done
done
