#!/bin/bash
# persistent-grid A/B: DBP_PERSISTENT = 0 (one CTA per block group), 1, 2 (x resident CTAs)
for P in 0 1 2; do
  for NM in "2048 700" "4096 1400" "8192 1400"; do
    set -- $NM
    v=$(DBP_PERSISTENT=$P timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline \
        --block-len $1 --overlap $2 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
    echo "P=$P N=$1 essfm $v"
  done
  v=$(DBP_PERSISTENT=$P timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --algorithm ffe \
      | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
  echo "P=$P N=2048 ffe $v"
done
DBP_PERSISTENT=1 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
