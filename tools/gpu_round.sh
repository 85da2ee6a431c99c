#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full K1 capture.
# Usage (from repo root, under gpurun): bash tools/gpu_round.sh <tag>
TAG=${1:-r}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/$TAG.gpu.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 240 --timeout-method=thread > $OUT/$TAG.pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/$TAG.pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/$TAG.smoke.txt 2>&1
timeout 300 python bench.py > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv \
    --log-file $OUT/$TAG.launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline \
    > /dev/null 2> $OUT/$TAG.ncu1.err
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 3 -c 1 \
    -o $OUT/$TAG.k1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > /dev/null 2> $OUT/$TAG.ncu2.err
ls -la $OUT
timeout 600 python tools/sweep_c5.py --out gpurun_out/$TAG.c5_sweep.json > gpurun_out/$TAG.c5_sweep.txt 2>&1
timeout 900 python bench.py --config c3 --steps 5 --warmup 2 > $OUT/$TAG.c3.json 2> $OUT/$TAG.c3.err
timeout 120 python tools/c4_slice.py --out $OUT/$TAG.c4.json > $OUT/$TAG.c4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/$TAG.c3launches.csv \
    python bench.py --config c3 --steps 1 --warmup 1 > /dev/null 2> $OUT/$TAG.c3ncu.err
timeout 120 python tools/k1_trace.py $OUT/$TAG.k1trace.raw > $OUT/$TAG.trace.txt 2>&1
timeout 600 python tools/sweep_gqa.py --out $OUT/$TAG.gqa_sweep.json > $OUT/$TAG.gqa_sweep.txt 2>&1
timeout 300 python tools/step_breakdown.py > $OUT/$TAG.step_breakdown.txt 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/$TAG.ref.json 2> $OUT/$TAG.ref.err
