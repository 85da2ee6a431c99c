#!/bin/bash
# K1 iteration: all GPU parity tests, C2 bench, CTA trace, C5 sweep, C4 slice, K1 ncu.
TAG=${1:-k}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo rc=$? >> $OUT/$TAG.pytest.txt
timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err
timeout 120 python tools/k1_trace.py $OUT/$TAG.k1trace.raw > $OUT/$TAG.trace.txt 2>&1
ST_K1_SLACK=-1 timeout 120 python tools/k1_trace.py $OUT/$TAG.sk.k1trace.raw > $OUT/$TAG.sk.trace.txt 2>&1
ST_K1_SLACK=-1 timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.sk.bench.json 2> $OUT/$TAG.sk.bench.err
timeout 600 python tools/sweep_c5.py --out $OUT/$TAG.c5_sweep.json > $OUT/$TAG.c5_sweep.txt 2>&1
timeout 120 python tools/c4_slice.py --out $OUT/$TAG.c4.json > $OUT/$TAG.c4.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:tree_attn_tc -s 3 -c 2 --csv \
    --log-file $OUT/$TAG.k1dram.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
