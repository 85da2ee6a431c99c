#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 120 python tools/k1_trace.py $OUT/c4a.raw --B 8 --T 61 --H 8 --L 2048 > $OUT/c4a.trace.txt 2>&1
ST_K1_SLACK=100 timeout 120 python tools/k1_trace.py $OUT/c4b.raw --B 8 --T 61 --H 8 --L 2048 > $OUT/c4b.trace.txt 2>&1
timeout 120 python tools/c4_slice.py --out $OUT/c4a.json > /dev/null 2>&1
ST_K1_SLACK=100 timeout 120 python tools/c4_slice.py --out $OUT/c4b.json > /dev/null 2>&1
