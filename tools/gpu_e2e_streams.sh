#!/bin/bash
# e2e H2D copy streams A/B (ST_E2E_STREAMS), two repetitions, same box
for r in 1 2; do for n in 1 2 3 4 6; do
  ST_E2E_STREAMS=$n timeout 300 python bench.py --no-cpu-baseline --no-strong 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']
print('streams $n', round(e['value']/1e6,3), 'M tok/s', round(e['ms_per_step']*1e3,1), 'us/step', 'h2d implied', round(e['h2d_gbs_implied'],1), 'alone', round(e['h2d_gbs_copies_alone'],1))"
done; done
