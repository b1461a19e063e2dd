#!/bin/bash
# variants x forced carve-out (percent of the 228 KB maximum; "-" = driver default)
#   tools/ab_carve2.sh "<carveouts>" <variant>...
carves=$1; shift
for args in "" "--algorithm ffe"; do
  for cv in $carves; do
    for v in "$@"; do
      c=$cv; [ "$c" = "-" ] && c=""
      x=$(DBP_CARVEOUT=$c DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
      echo "$v carve=$cv [$args] $x"
    done
  done
done
