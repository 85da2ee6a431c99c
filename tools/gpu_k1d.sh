#!/bin/bash
# K1 check: tc/peer parity, C2 bench, T=128 trace, C5 sweep, C4 slice, GQA sweep.
TAG=${1:-k}
OUT=gpurun_out
mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_tc.py tests/test_gpu_peer.py tests/test_gpu_model.py -q -x --timeout 120 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo rc=$? >> $OUT/$TAG.pytest.txt
timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err
timeout 120 python tools/k1_trace.py $OUT/$TAG.t128.raw --B 16 --T 128 --L 4096 > $OUT/$TAG.t128.txt 2>&1
timeout 600 python tools/sweep_c5.py --out $OUT/$TAG.c5_sweep.json > $OUT/$TAG.c5_sweep.txt 2>&1
timeout 120 python tools/c4_slice.py --out $OUT/$TAG.c4.json > $OUT/$TAG.c4.txt 2>&1
timeout 600 python tools/sweep_gqa.py --out $OUT/$TAG.gqa.json > $OUT/$TAG.gqa.txt 2>&1
