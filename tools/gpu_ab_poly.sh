#!/bin/bash
# M=128 softmax: exp2 pairs on the FMA pipe (poly<N>: one pair in N) vs head; parity first
ST_LIB_VARIANT=build/ab/poly4.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_step.py -x -q 2>&1 | tail -1
bash tools/gpu_ab_lib.sh head poly4 poly3 poly8
for v in head poly4 poly3; do echo "== $v"; ST_LIB_VARIANT=build/ab/$v.so timeout 300 python tools/sweep_c5.py --Ls 4096,16384 --Ts 128,256 --cool 2 --out /tmp/c5.json | grep "T="; done
