#!/bin/bash
# Same-box A/B of library variants on the C4 slice and the GQA sweep.
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for i in 1 2; do for v in "$@"; do
ST_LIB_VARIANT=build/variants/$v.so timeout 120 python tools/c4_slice.py --out $OUT/$TAG.$v.$i.c4.json > /dev/null 2>&1
ST_LIB_VARIANT=build/variants/$v.so timeout 300 python tools/sweep_gqa.py --out $OUT/$TAG.$v.$i.gqa.json > /dev/null 2>&1
done; done
for f in $OUT/$TAG.*.c4.json; do python -c "
import json; d=json.load(open('$f')); g=json.load(open('$f'.replace('.c4.json','.gqa.json')))
print('$f'.split('/')[-1], 'c4 k1 %.1f us (%.3f) fused %.1f' % (d['k1_us'], d['k1_frac'], d['fused_allgather_k1_us']), '| gqa', ' '.join('%d/%dK %.3f' % (r['T'], r['L']//1024, r['frac']) for r in g['rows']))"; done
