#!/bin/bash
# GQA / C4 K1 fixed-cost traces and schedule A/B (diagnostic). Usage (under gpurun): bash tools/gpu_gqa_trace.sh
OUT=gpurun_out; mkdir -p $OUT
timeout 120 python tools/k1_trace.py $OUT/gq8.raw --B 16 --T 8 --H 64 --Hkv 8 --L 4096 --chain > $OUT/gq8.txt 2>&1; echo "gq8 rc=$?"
timeout 120 python tools/k1_trace.py $OUT/gq16.raw --B 16 --T 16 --H 64 --Hkv 8 --L 4096 --chain > $OUT/gq16.txt 2>&1; echo "gq16 rc=$?"
ST_K1_SLACK=-1 timeout 120 python tools/k1_trace.py $OUT/gq16s.raw --B 16 --T 16 --H 64 --Hkv 8 --L 4096 --chain > $OUT/gq16s.txt 2>&1; echo "gq16s rc=$?"
for s in default -1; do echo "== ST_K1_SLACK=$s"; if [ $s = default ]; then timeout 300 python tools/k1_sched_ab.py; else ST_K1_SLACK=$s timeout 300 python tools/k1_sched_ab.py; fi; done > $OUT/schedab.txt 2>&1
