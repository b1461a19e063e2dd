#!/bin/bash
# A/B of environment settings on an explicit config list (one config per line in $CFGS)
#   CFGS=$'--block-len 8192 --overlap 1400' tools/ab_env.sh <rounds> "DBP_R2T=0" "DBP_R2T=1" ...
rounds=$1; shift
while IFS= read -r args; do
  for r in $(seq "$rounds"); do
    for v in "$@"; do
      x=$(env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])")
      echo "$v [$args] $x"
    done
  done
done <<< "$CFGS"
