#!/bin/bash
# A/B: M=128 register reallocation (setmaxnreg) vs base; parity first
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_step.py -x -q 2>&1 | tail -1
bash tools/gpu_ab_lib.sh base reg
for v in base reg; do echo "== $v"; ST_LIB_VARIANT=build/ab/$v.so timeout 300 python tools/sweep_c5.py --Ls 4096,16384 --Ts 128,256 --cool 2 --out /tmp/c5.json | grep "T="; done
