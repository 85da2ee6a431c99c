#!/bin/bash
# same-box A/B of library variants build/ab/<name>.so over tools/k1_sched_ab.py (3 reps)
for r in 1 2 3; do for v in "$@"; do ST_LIB_VARIANT=build/ab/$v.so timeout 300 python tools/k1_sched_ab.py | sed "s/^/$v /"; done; done
