#!/bin/bash
# A/B of library variants on an explicit config list (one config per line in $CFGS)
#   CFGS=$'--algorithm ffe\n--block-len 4096 --overlap 1400' tools/ab_cfg.sh <rounds> <variant>...
rounds=$1; shift
while IFS= read -r args; do
  for r in $(seq "$rounds"); do
    for v in "$@"; do
      x=$(DBP_LIB=build/variants/$v.so timeout 60 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
      echo "$v [$args] $x"
    done
  done
done <<< "$CFGS"
