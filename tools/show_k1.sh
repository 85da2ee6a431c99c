#!/bin/bash
# Summarise a gpu_k1q/gpu_k1b run: bench K1 numbers, trace epilogue stamps, C4 slice.
T=$1; cd gpurun_out
tail -2 $T.pytest.txt
for f in $T.bench.json $T.sk.bench.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d['roofline'];print('$f step %.1f k1 %.1f bracket %.1f frac %.3f share %.3f'%(d['ms_per_step']*1e3,r['us_per_launch'],r['us_in_step_bracket'],r['frac'],r['share_of_step']))"; done
for f in $T.trace.txt $T.sk.trace.txt; do echo "== $f"; grep -A9 "SM clock" $f | tail -9; grep "per-CTA" $f; done
grep '"k1_us"\|fused_allgather_k1_us' $T.c4.txt
grep -A10 "SM clock" $T.c4trace.txt | tail -9
