#!/bin/bash
# Same-box A/B of library builds in build/ab/<name>.so: C2 bench, C4 slice,
# a C5 subset and the GQA sweep. Usage: bash tools/ab_k1.sh v1 v2 ...
bash tools/ab_c2.sh "$@"
bash tools/ab_c4.sh "$@" 2>&1 | grep '^=='
for v in "$@"; do
  echo "-- C5 $v"; ST_LIB_VARIANT=build/ab/$v.so timeout 300 python tools/sweep_c5.py --Ls 4096,16384 --Ts 16,64,128,256 --out /tmp/c5.json | grep -v '^$'
  echo "-- GQA $v"; ST_LIB_VARIANT=build/ab/$v.so timeout 300 python tools/sweep_gqa.py --out /tmp/gqa.json 2>&1 | tail -8
done
