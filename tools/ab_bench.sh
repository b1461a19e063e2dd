#!/bin/bash
# A/B the library variants in build/variants on the GPU box (device-resident value only)
for v in "$@"; do
  DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],3), 'GS/s', round(d['roofline']['frac'],3), d['clocks'])"
done
