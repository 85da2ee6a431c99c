#!/bin/bash
# Quick K1 check: tc parity, C2 bench aligned + stream-K, traces, C4 slice.
TAG=${1:-k}
OUT=gpurun_out
mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_tc.py tests/test_gpu_peer.py -q -x --timeout 120 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo rc=$? >> $OUT/$TAG.pytest.txt
timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err
timeout 120 python tools/k1_trace.py $OUT/$TAG.k1trace.raw > $OUT/$TAG.trace.txt 2>&1
ST_K1_SLACK=-1 timeout 120 python tools/k1_trace.py $OUT/$TAG.sk.k1trace.raw > $OUT/$TAG.sk.trace.txt 2>&1
ST_K1_SLACK=-1 timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.sk.bench.json 2> $OUT/$TAG.sk.bench.err
timeout 120 python tools/c4_slice.py --out $OUT/$TAG.c4.json > $OUT/$TAG.c4.txt 2>&1
timeout 120 python tools/k1_trace.py $OUT/$TAG.c4.raw --B 8 --T 61 --H 8 --L 2048 > $OUT/$TAG.c4trace.txt 2>&1
