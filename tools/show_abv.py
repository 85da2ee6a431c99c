"""Summarise tools/gpu_abv.sh output: python tools/show_abv.py <tag>"""
import glob
import json
import sys

tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{tag}.*.bench.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        c5 = json.load(open(f.replace(".bench.json", ".c5.json")))["rows"]
        print(f"{f.split('/')[-1]:34s} step {d['ms_per_step'] * 1e3:6.1f} k1 {r['us_per_launch']:5.1f} "
              f"frac {r['frac']:.3f} | c5 " + " ".join(f"{x['T']}/{x['L'] // 1024}K {x['frac']:.3f}" for x in c5))
    except Exception as e:  # noqa: BLE001
        print(f, "error", e)
