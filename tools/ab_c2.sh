#!/bin/bash
# Same-box A/B of library builds in build/ab/<name>.so on the C2 bench (step
# time, K1 per launch). Usage: bash tools/ab_c2.sh v1 v2 ...
for rep in 1 2; do
for v in "$@"; do
  ST_LIB_VARIANT=build/ab/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-strong > /tmp/ab.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("/tmp/ab.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(f"== {sys.argv[1]:8s} step {d['ms_per_step']*1e3:6.1f} us  K1 {r['us_per_launch']:6.2f} us (frac {r['frac']:.3f})  "
      f"graph/step {d.get('graph_ms_per_step', 0)*1e3:6.1f} us  sm {d['clocks']['sm_mhz']}  parity {d['parity']['greedy_vs_oracle']}")
PY
done
done
