for r in 1 2; do for v in 0 2; do echo "== pre$v"; ST_K1_PRE=$v timeout 300 python tools/sweep_c5.py --Ls 4096,8192 --Ts 128,256 --cool 2 --out /tmp/c5.json | grep "T="; done; done
