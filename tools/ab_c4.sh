#!/bin/bash
# Same-box A/B of library builds in build/ab/<name>.so on the C4 slice (K1,
# fused all-gather K1) and the K1 DSMEM-merge trace. Usage: bash tools/ab_c4.sh v1 v2 ...
for rep in 1 2; do
for v in "$@"; do
  echo "== $v $(ST_LIB_VARIANT=build/ab/$v.so timeout 120 python tools/c4_slice.py --out /tmp/x.json | grep -E '"k1_us"|fused_allgather_k1_us' | tr -d '\n ')"
done
done
for v in "$@"; do
echo "-- $v"
ST_LIB_VARIANT=build/ab/$v.so python tools/k1_trace.py gpurun_out/t0.txt --B 8 --H 8 --T 61 2>&1 | grep -E "DSMEM|whole"
ST_LIB_VARIANT=build/ab/$v.so ST_K1_TRACE_CTA=1 python tools/k1_trace.py gpurun_out/t1.txt --B 8 --H 8 --T 61 2>&1 | grep -E "DSMEM"
done
