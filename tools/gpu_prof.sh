#!/bin/bash
# ncu evidence for the C2 step: launch list (device time per launch) and one
# --set full capture each of K1 and the K3 argmax kernel.
# Usage (under gpurun): bash tools/gpu_prof.sh <tag>
TAG=${1:-prof}; OUT=gpurun_out; mkdir -p $OUT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 40 --csv \
    --log-file $OUT/$TAG.launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-strong \
    > /dev/null 2> $OUT/$TAG.ncu1.err; echo "launches rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:greedy_argmax -s 5 -c 1 \
    -o $OUT/$TAG.k3 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong \
    > /dev/null 2> $OUT/$TAG.ncu2.err; echo "k3 rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 5 -c 1 \
    -o $OUT/$TAG.k1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong \
    > /dev/null 2> $OUT/$TAG.ncu3.err; echo "k1 rc=$?"
ls -la $OUT | grep $TAG
