#!/bin/bash
# Quick GPU session: parity tests, smoke, default bench, the N>1 code path on
# one GPU (BENCH_SHARED_GPU_TEST: gloo, numbers meaningless), c4 and c5 modes.
# Usage (from repo root, under gpurun): bash tools/gpu_check.sh <tag> [pytest -k expr]
TAG=${1:-r}
K=${2:-}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/$TAG.gpu.txt
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "$K" > $OUT/$TAG.pytest.txt 2>&1
else
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $OUT/$TAG.pytest.txt 2>&1
fi
echo "pytest rc=$?" >> $OUT/$TAG.pytest.txt
tail -3 $OUT/$TAG.pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/$TAG.smoke.txt 2>&1; tail -1 $OUT/$TAG.smoke.txt
timeout 300 python bench.py > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err; echo "bench rc=$?"
BENCH_SHARED_GPU_TEST=1 timeout 300 python bench.py --gpus 2 --steps 5 --warmup 3 --no-strong > $OUT/$TAG.bench2.json 2> $OUT/$TAG.bench2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config c4 > $OUT/$TAG.c4.json 2> $OUT/$TAG.c4.err; echo "c4 rc=$?"
timeout 300 python bench.py --config c5 > $OUT/$TAG.c5.json 2> $OUT/$TAG.c5.err; echo "c5 rc=$?"
