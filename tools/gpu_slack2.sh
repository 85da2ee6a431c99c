#!/bin/bash
TAG=${1:-sl}
OUT=gpurun_out; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_tc.py tests/test_gpu_peer.py -q -x --timeout 120 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo rc=$? >> $OUT/$TAG.pytest.txt
for i in 1 2; do for s in 6 3; do
ST_K1_SLACK=$s timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.b$s.$i.json 2>/dev/null
done; done
timeout 120 python tools/k1_trace.py $OUT/$TAG.t128.raw --B 16 --T 128 --L 4096 > $OUT/$TAG.t128.txt 2>&1
timeout 600 python tools/sweep_c5.py --out $OUT/$TAG.c5_sweep.json > $OUT/$TAG.c5_sweep.txt 2>&1
