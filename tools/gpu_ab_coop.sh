#!/bin/bash
# A/B: K1 launched cooperatively (default) vs not (ST_K1_COOP=0), C2 bench.
OUT=gpurun_out; TAG=${1:-coop}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "step or small or suite or k3_tie" > $OUT/$TAG.pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/$TAG.pytest.txt; tail -2 $OUT/$TAG.pytest.txt
for i in 1 2; do
  for c in 1 0; do
    ST_K1_COOP=$c timeout 300 python bench.py --no-cpu-baseline --no-strong > $OUT/$TAG.c$c.$i.json 2>/dev/null
    python -c "import json;d=json.load(open('$OUT/$TAG.c$c.$i.json'));r=d['roofline'];print('coop=$c', round(d['ms_per_step']*1e3,1), 'us/step K1', round(r['us_per_launch'],1), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"
  done
done
