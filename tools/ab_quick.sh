#!/bin/bash
# headline + FFE throughput and golden-case accuracy for each variant
for v in "$@"; do
  DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v sym', round(d['value'],3))"
  DBP_LIB=build/variants/$v.so timeout 300 python bench.py --algorithm ffe --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v ffe', round(d['value'],3))"
  DBP_LIB=build/variants/$v.so timeout 300 python tools/diag_cases.py 2>/dev/null | head -22 | awk -v v=$v '{printf "%s %s\n", $1, $NF}' | sort -t= -k2 -g | tail -3 | sed "s/^/$v worst: /"
done
