#!/bin/bash
# K1 fixed-cost traces (ST_K1_TRACE) on the shapes furthest below roofline,
# plus the K3 load-variant microbenchmark. Usage (under gpurun): bash tools/gpu_trace.sh <tag>
TAG=${1:-tr}; OUT=gpurun_out; mkdir -p $OUT
make -C paper_2305_09781_b200/csrc -j8 > /dev/null 2>&1
timeout 120 python tools/k1_trace.py $OUT/$TAG.c2.raw > $OUT/$TAG.c2.txt 2>&1; echo "c2 rc=$?"
timeout 120 python tools/k1_trace.py $OUT/$TAG.c4.raw --B 8 --T 61 --H 8 --L 2048 > $OUT/$TAG.c4.txt 2>&1; echo "c4 rc=$?"
timeout 120 python tools/k1_trace.py $OUT/$TAG.gqa.raw --B 16 --T 16 --H 64 --Hkv 8 --L 4096 --chain > $OUT/$TAG.gqa.txt 2>&1; echo "gqa rc=$?"
timeout 120 python tools/k1_trace.py $OUT/$TAG.t128.raw --B 16 --T 128 --H 32 --L 4096 > $OUT/$TAG.t128.txt 2>&1; echo "t128 rc=$?"
timeout 120 python tools/k1_trace.py $OUT/$TAG.t256.raw --B 16 --T 256 --H 32 --L 4096 > $OUT/$TAG.t256.txt 2>&1; echo "t256 rc=$?"
timeout 120 ./tools/argmax_bench > $OUT/$TAG.argmax.txt 2>&1; echo "argmax rc=$?"
