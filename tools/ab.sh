#!/bin/bash
# A/B of library variants (build/variants/<name>.so, tools/build_variants.py)
# over the headline and neighbouring configs, variants interleaved per config.
#   tools/ab.sh <rounds> <variant>...
rounds=$1; shift
CONFIGS=(
  ""
  "--algorithm ffe"
  "--block-len 1024 --overlap 768 --nc 17"
  "--block-len 512 --overlap 300 --nc 9"
  "--block-len 128 --overlap 32 --nc 9"
  "--algorithm ssfm --num-steps 20 --arrangement symmetric"
)
# AB_CONFIGS=k limits the run to the first k configs
CONFIGS=("${CONFIGS[@]:0:${AB_CONFIGS:-${#CONFIGS[@]}}}")
for args in "${CONFIGS[@]}"; do
  for r in $(seq "$rounds"); do
    for v in "$@"; do
      x=$(DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
      echo "$v [$args] $x"
    done
  done
done
