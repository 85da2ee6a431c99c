#!/bin/bash
# Round-2 GPU evidence session: parity tests, smoke, default bench, ncu launch
# list + --set full captures of K1 and K3, C5 sweep (T up to 256), GQA sweep,
# C4 (1 GPU), reference arm. Usage (under gpurun): bash tools/gpu_round2.sh <tag>
TAG=${1:-r02}; OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/$TAG.gpu.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > $OUT/$TAG.pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/$TAG.pytest.txt; tail -3 $OUT/$TAG.pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/$TAG.smoke.txt 2>&1; tail -1 $OUT/$TAG.smoke.txt
timeout 400 python bench.py > $OUT/$TAG.bench.json 2> $OUT/$TAG.bench.err; echo "bench rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 40 --csv \
    --log-file $OUT/$TAG.launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-strong \
    > /dev/null 2> $OUT/$TAG.ncu1.err; echo "launches rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 5 -c 1 \
    -o $OUT/$TAG.k1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong \
    > /dev/null 2> $OUT/$TAG.ncu2.err; echo "k1 rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:greedy_argmax -s 5 -c 1 \
    -o $OUT/$TAG.k3 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong \
    > /dev/null 2> $OUT/$TAG.ncu3.err; echo "k3 rc=$?"
timeout 1200 python tools/sweep_c5.py --cool 2 --out $OUT/$TAG.c5_sweep.json > $OUT/$TAG.c5_sweep.txt 2>&1; echo "c5 rc=$?"
timeout 600 python tools/sweep_gqa.py --out $OUT/$TAG.gqa_sweep.json > $OUT/$TAG.gqa_sweep.txt 2>&1; echo "gqa rc=$?"
timeout 300 python bench.py --config c4 > $OUT/$TAG.c4.json 2> $OUT/$TAG.c4.err; echo "c4 rc=$?"
timeout 120 python tools/c4_slice.py --out $OUT/$TAG.c4_slice.json > $OUT/$TAG.c4_slice.txt 2>&1; echo "c4 slice rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/$TAG.ref.json 2> $OUT/$TAG.ref.err; echo "ref rc=$?"
timeout 300 python tools/gemm_bench.py > $OUT/$TAG.gemm.txt 2>&1; echo "gemm rc=$?"
timeout 600 python bench.py --config c3 --steps 5 --warmup 2 > $OUT/$TAG.c3.json 2> $OUT/$TAG.c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config c3e > $OUT/$TAG.c3e.json 2> $OUT/$TAG.c3e.err; echo "c3e rc=$?"
timeout 300 python tools/step_modes.py > $OUT/$TAG.step_modes.txt 2>&1; echo "modes rc=$?"
timeout 120 python tools/mss_bench.py > $OUT/$TAG.k4.txt 2>&1; echo "k4 rc=$?"
