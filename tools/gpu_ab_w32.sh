#!/bin/bash
# TMA-store epilogue variants, same box: reg (previous build), w32 per-warp stores (ST_K1_OTMA=2), w32 CTA-wide store (=1)
for r in 1 2 3; do
  ST_LIB_VARIANT=build/ab/reg.so timeout 300 python tools/k1_sched_ab.py | sed "s/^/reg /"
  ST_LIB_VARIANT=build/ab/w32.so ST_K1_OTMA=2 timeout 300 python tools/k1_sched_ab.py | sed "s/^/warp /"
  ST_LIB_VARIANT=build/ab/w32.so ST_K1_OTMA=1 timeout 300 python tools/k1_sched_ab.py | sed "s/^/cta /"
done
