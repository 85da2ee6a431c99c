"""Diagnostic: where a C3-shape device-engine step (bench.py --config c3e)
spends its time — torch.profiler (CUPTI) kernel totals over the steps of a
short run after the prefill, live clocks (not serialised like ncu).
  python tools/c3e_profile.py [--new 8]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--new", type=int, default=8)
args = ap.parse_args()
NL, d, Hh, Vv, B, PROMPT = 32, 4096, 32, 32000, 32, 128
llm = _capi.DeviceModel(NL, Hh, d, Vv, PROMPT + 64 + 64, 4, seed=42, dtype=torch.float16)
ssm = _capi.DeviceModel(2, Hh, d, Vv, PROMPT + 64 + 64, 4, seed=7, dtype=torch.float16)
eng = _capi.Engine(llm, ssm, B, PROMPT, expansion=(1, 1, 3, 1, 1, 1, 1, 1))
rng = np.random.default_rng(11)
prompts = [rng.integers(0, Vv, PROMPT).tolist() for _ in range(B)]
eng.run(prompts, [4] * B)
torch.cuda.synchronize()
# a run of 1 new token = prefill + 1 step; the difference to --new tokens is the steps
from torch.profiler import ProfilerActivity, profile  # noqa: E402

def totals(n_new):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        seqs, steps = eng.run(prompts, [n_new] * B)
        torch.cuda.synchronize()
    out = {}
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        k = ev.name
        t, c = out.get(k, (0.0, 0))
        out[k] = (t + ev.device_time_total if hasattr(ev, "device_time_total") else t + ev.cuda_time_total, c + 1)
    return out, steps

one, s1 = totals(1)
many, sn = totals(args.new)
nsteps = sn - s1
print(f"steps {s1} -> {sn}: per-step kernel totals (difference of the two runs / {nsteps} steps)")
rows = []
for k, (t, c) in many.items():
    t1, c1 = one.get(k, (0.0, 0))
    rows.append(((t - t1) / nsteps, (c - c1) / nsteps, k))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"kernel time per step: {tot / 1e3:.2f} ms")
for us, cnt, k in rows[:25]:
    print(f"{us:9.1f} us  {cnt:6.1f}x  {k[:110]}")
