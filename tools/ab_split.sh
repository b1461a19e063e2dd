#!/bin/bash
# split (mbarrier) write-after-read barriers vs __syncthreads across block lengths
for args in "" "--algorithm ffe" "--block-len 1024 --overlap 768 --nc 17" "--block-len 4096 --overlap 1400 --nc 17" "--block-len 8192 --overlap 1400 --nc 17" "--block-len 8192 --overlap 1024 --algorithm ssfm --num-steps 20 --arrangement linear-first" "--block-len 256 --overlap 100 --algorithm ssfm"; do
 for v in nosplit split nosplit split; do
  x=$(DBP_LIB=build/variants/$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],3))"); echo "$v [$args] $x"
 done
done
