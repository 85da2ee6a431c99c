#!/bin/bash
# T=256 sweep, N>1 code paths on one GPU (gloo, numbers meaningless), GEMM ncu capture.
OUT=gpurun_out; TAG=${1:-misc}; mkdir -p $OUT
timeout 600 python tools/sweep_c5.py --Ts 256,128 --out $OUT/$TAG.c5.json > $OUT/$TAG.c5.txt 2>&1; cat $OUT/$TAG.c5.txt | grep "T="
for n in 4 8; do
  BENCH_SHARED_GPU_TEST=1 timeout 600 python bench.py --gpus $n --steps 3 --warmup 3 --no-strong > $OUT/$TAG.n$n.json 2> $OUT/$TAG.n$n.err; echo "n=$n rc=$?"
  python -c "import json;d=json.load(open('$OUT/$TAG.n$n.json'));print('n_gpus',d['n_gpus'],d['parity'])"
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm2_kernel -s 2 -c 1 \
    -o $OUT/$TAG.gemm -f python tools/gemm_bench.py > /dev/null 2> $OUT/$TAG.ncu.err; echo "ncu rc=$?"
