#!/bin/bash
# Step iteration: full GPU parity suite, C2 bench, ncu launch list of the step's kernels.
TAG=${1:-st}
OUT=gpurun_out
mkdir -p $OUT
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/$TAG.pytest.txt
timeout 300 python bench.py --no-cpu-baseline > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 35 --csv \
    --log-file $OUT/$TAG.launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/$TAG.ncu1.err
timeout 120 python tools/k1_trace.py $OUT/$TAG.k1trace.raw > $OUT/$TAG.trace.txt 2>&1
