#!/bin/bash
# A/B of K1 library variants on the C5 T=128 points (build/variants/*.so via ST_LIB_VARIANT).
for v in build/variants/9c3db8d.so build/variants/e4388dc.so HEAD HEAD_nocoop; do
  case $v in
    HEAD) ST_LIB_VARIANT= python tools/sweep_c5.py --Ts 128,64 --Ls 4096,32768 --out /tmp/x.json | sed "s|^|HEAD |";;
    HEAD_nocoop) ST_K1_COOP=0 python tools/sweep_c5.py --Ts 128,64 --Ls 4096,32768 --out /tmp/x.json | sed "s|^|nocoop |";;
    *) ST_LIB_VARIANT=$v python tools/sweep_c5.py --Ts 128,64 --Ls 4096,32768 --out /tmp/x.json | sed "s|^|$(basename $v) |";;
  esac
done
