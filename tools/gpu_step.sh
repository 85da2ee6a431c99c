#!/bin/bash
# Step iteration: kernel parity tests, C2 bench, launch list.
TAG=${1:-st}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tc.py -q -x --timeout 200 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo rc=$? >> $OUT/$TAG.pytest.txt
timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 30 --csv \
    --log-file $OUT/$TAG.launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
