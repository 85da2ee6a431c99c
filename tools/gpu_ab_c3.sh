#!/bin/bash
# C3 step A/B of library variants (same box)
for r in 1 2; do for v in "$@"; do
  ST_LIB_VARIANT=build/ab/$v.so timeout 600 python bench.py --config c3 --steps 5 --warmup 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), 'ms', d['clocks'])"
done; done
