#!/bin/bash
# Same-box A/B of library variants (build/variants/<name>.so): C2 bench + C5 (T=64/128) + GQA
# Usage: tools/gpu_abv.sh <tag> <variant>...
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for i in 1 2; do for v in "$@"; do
ST_LIB_VARIANT=build/variants/$v.so timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.$v.$i.bench.json 2>/dev/null
ST_LIB_VARIANT=build/variants/$v.so timeout 300 python tools/sweep_c5.py --Ls 4096,16384 --Ts 64,128 --out $OUT/$TAG.$v.$i.c5.json > $OUT/$TAG.$v.$i.c5.txt 2>&1
done; done
