#!/bin/bash
# quick sweep of each library variant in build/variants (per block length tuning)
for v in "$@"; do
  DBP_LIB=build/variants/$v.so timeout 600 python tools/sweep.py --quick --waveforms 96 --reps 10 2>/dev/null \
    | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], d['algorithm'], d['block_len'], d['overlap'], d['num_steps'], d['arrangement'][:6], round(d['gsamples_per_s'],2))"
done
