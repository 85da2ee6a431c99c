#!/bin/bash
# TMA-store epilogue: bit-identity vs per-thread stores, parity tests, same-box A/B
ST_K1_OTMA=0 python tools/otma_check.py dump && python tools/otma_check.py compare
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_step.py -x -q 2>&1 | tail -2
for r in 1 2; do
  ST_K1_OTMA=0 timeout 300 python tools/k1_sched_ab.py | sed "s/^/stores /"
  timeout 300 python tools/k1_sched_ab.py | sed "s/^/tma    /"
done
