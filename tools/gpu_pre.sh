#!/bin/bash
# A/B: tiles per ring issued by the producers' fast start (ST_K1_PRE)
for r in 1 2 3; do for v in 0 2; do ST_K1_PRE=$v timeout 300 python tools/k1_sched_ab.py | sed "s/^/pre$v /"; done; done
