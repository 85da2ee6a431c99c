#!/bin/bash
# Same-box A/B of library variants on the M=128 configurations (C5 T=128, GQA G*T=128).
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for i in 1 2; do for v in "$@"; do
ST_LIB_VARIANT=build/variants/$v.so timeout 300 python tools/sweep_c5.py --Ls 4096,16384 --Ts 128 --out $OUT/$TAG.$v.$i.c5.json > /dev/null 2>&1
ST_LIB_VARIANT=build/variants/$v.so timeout 300 python tools/sweep_gqa.py --out $OUT/$TAG.$v.$i.gqa.json > /dev/null 2>&1
done; done
for f in $OUT/$TAG.*.c5.json; do python -c "
import json; c=json.load(open('$f'))['rows']; g=json.load(open('$f'.replace('.c5.json','.gqa.json')))['rows']
print('$f'.split('/')[-1], 'c5', ' '.join('%d/%dK %.3f' % (r['T'], r['L']//1024, r['frac']) for r in c), '| gqa', ' '.join('%d/%dK %.3f' % (r['T'], r['L']//1024, r['frac']) for r in g))"; done
