#!/bin/bash
# Schedule A/B: whole-pair (aligned) vs stream-K at C2 / C4 / C5, with traces.
TAG=${1:-s}
OUT=gpurun_out
mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_tc.py -q -x --timeout 120 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo rc=$? >> $OUT/$TAG.pytest.txt
for SL in 6 -1; do
  ST_K1_SLACK=$SL timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.sl$SL.bench.json 2> $OUT/$TAG.sl$SL.bench.err
  ST_K1_SLACK=$SL timeout 120 python tools/k1_trace.py $OUT/$TAG.sl$SL.k1trace.raw > $OUT/$TAG.sl$SL.trace.txt 2>&1
  ST_K1_SLACK=$SL timeout 120 python tools/c4_slice.py --out $OUT/$TAG.sl$SL.c4.json > $OUT/$TAG.sl$SL.c4.txt 2>&1
done
timeout 600 python tools/sweep_c5.py --out $OUT/$TAG.c5_sweep.json > $OUT/$TAG.c5_sweep.txt 2>&1
