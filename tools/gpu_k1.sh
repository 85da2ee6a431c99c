#!/bin/bash
# K1 change check: tcgen05 parity tests, C2 bench, C5 at T=128 and T=256.
TAG=${1:-k1}; OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "tc or step or k1" > $OUT/$TAG.pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/$TAG.pytest.txt; tail -3 $OUT/$TAG.pytest.txt
for cfg in "" "--config c5 --tree 128" "--config c5 --tree 256" "--config c5 --kv 4096 --tree 256"; do
  timeout 300 python bench.py --no-cpu-baseline --no-strong $cfg > $OUT/$TAG.b.json 2>$OUT/$TAG.b.err
  python -c "import json;d=json.load(open('$OUT/$TAG.b.json'));r=d['roofline'];print('$cfg', round(d['ms_per_step']*1e3,1), 'us/step K1', round(r['us_per_launch'],1), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'], d['parity']['greedy_vs_oracle'])" || tail -5 $OUT/$TAG.b.err
done
