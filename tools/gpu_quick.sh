#!/bin/bash
# Quick GPU iteration: K1/K2/K3 parity, CTA-0 trace, bench, launch list.
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_tc.py tests/test_gpu_kernels.py -q -x --timeout 120 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo rc=$? >> $OUT/$TAG.pytest.txt
timeout 120 python tools/k1_trace.py $OUT/$TAG.k1trace.raw > $OUT/$TAG.trace.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv \
    --log-file $OUT/$TAG.launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:greedy_verify -s 3 -c 1 \
    -o $OUT/$TAG.k3 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
