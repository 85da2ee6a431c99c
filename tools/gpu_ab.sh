#!/bin/bash
# Same-box A/B of the C2 step: tree rows from their own tensors vs appended to the cache.
TAG=${1:-ab}
OUT=gpurun_out; mkdir -p $OUT
for i in 1 2; do for m in own cache; do
timeout 300 python bench.py --no-cpu-baseline --tree-rows $m > $OUT/$TAG.$m.$i.json 2>/dev/null
done; done
