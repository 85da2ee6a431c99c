#!/bin/bash
# A/B: the step plan's argmax streaming during K1's tail (ST_K3_EARLY), same box
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q 2>&1 | tail -1
for r in 1 2 3; do for v in 0 1; do
  ST_K3_EARLY=$v timeout 300 python bench.py --no-cpu-baseline --no-strong 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('early=$v', round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step']*1e3,2), 'us/step K1', round(d['roofline']['us_per_launch'],2), 'us frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  ST_K3_EARLY=$v timeout 300 python tools/step_modes.py 2>/dev/null | tail -1 | sed "s/^/early=$v /"
done; done
