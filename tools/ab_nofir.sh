#!/bin/bash
# no-FIR split-step kernel (SSFM / ESSFM N_c = 0) vs the generic kernel, occupancy variants
for args in "--algorithm ssfm --num-steps 20 --arrangement linear-first" "--algorithm ssfm --num-steps 20 --arrangement symmetric" "--algorithm ssfm --num-steps 20 --arrangement linear-first --block-len 8192 --overlap 1024" "--algorithm ssfm --num-steps 20 --arrangement linear-first --block-len 4096 --overlap 1400" "--algorithm ssfm --num-steps 4 --block-len 1024 --overlap 768" "--algorithm essfm --nc 0 --num-steps 1"; do
  for r in 1 2; do
    for v in base nofir nofir_1024; do
      x=$(DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))")
      echo "$v [$args] $x"
    done
  done
done
