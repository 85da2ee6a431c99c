"""Diagnostic: run K1 (default: the C2 shape; --B/--T/--H/--L to change) with
ST_K1_TRACE set and print CTA 0's per-tile pipeline timeline (cycles relative
to the first K load) and per-CTA globaltimer summaries."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse

ap = argparse.ArgumentParser()
ap.add_argument("out", nargs="?", default="gpurun_out/k1_trace.txt")
ap.add_argument("--B", type=int, default=8)
ap.add_argument("--T", type=int, default=64)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--L", type=int, default=2048)
ap.add_argument("--Hkv", type=int, default=0)
ap.add_argument("--chain", action="store_true")
args = ap.parse_args()
out = args.out
os.environ["ST_K1_TRACE"] = out
if os.path.exists(out):
    os.remove(out)
from paper_2305_09781_b200 import _capi  # noqa: E402

B, T, H, D, L = args.B, args.T, args.H, 128, args.L
HKV = args.Hkv or H
dev = "cuda"
q = torch.randn(B, T, H, D, device=dev).half()
kc = torch.randn(B, HKV, L + T, D, device=dev).half()
vc = torch.randn(B, HKV, L + T, D, device=dev).half()
par0 = [-1] + (list(range(T - 1)) if args.chain else [0] * (T - 1))
par = torch.tensor([par0] * B, dtype=torch.int32, device=dev)
n = torch.full((B,), T, dtype=torch.int32, device=dev)
P = torch.full((B,), L, dtype=torch.int32, device=dev)
mask = _capi.build_masks(par, n)
ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, n)
for _ in range(3):
    _capi.tree_attention(q, kc, vc, mask, P, n, workspace=ws)
torch.cuda.synchronize()
lines = [list(map(int, l.split())) for l in open(out)]
rows = lines[-17:-1]
cta = np.array(lines[-1], dtype=np.int64).reshape(-1, 12)
t = np.array(rows, dtype=np.int64)
t0 = t[0][t[0] > 0].min() if (t[0] > 0).any() else 0
names = ["K issue", "V issue", "S issue", "PV issue", "S ready", "P done", "K full(mma)", "V full(mma)", "S loaded", "masked+max", "pv wait done", "rescaled"]
print("tile " + " ".join(f"{x:>12s}" for x in names))
for i in range(64 if t0 else 0):
    print(f"{i:4d} " + " ".join(f"{(t[r][i] - t0) if t[r][i] else -1:12d}" for r in range(12)))
print("segment epilogues (cycles rel. to first K load): PV done | (m,l) merged | O stored | end")
for i in range(64):
    if t[12][i]:
        print(f"{i:4d} " + " ".join(f"{(t[r][i] - t0) if t[r][i] else -1:12d}" for r in range(12, 16)))

su = t[15][56:64]
if su[0]:
    print("traced CTA startup (cycles after entry): tmem+barriers %d | lengths table %d | schedule %d | "
          "K producer fast start: begin %d, scheduled %d, Q + first ring issued %d" % tuple(int(x - su[0]) if x else -1 for x in su[1:7]))


fi = t[13][48:54]
if fi[0]:
    print("fast-start issue (cycles after scheduled): policy %d | Q %d | stage0 %d | stage1 %d | stage2 %d"
          % tuple(int(x - su[5]) if x else -1 for x in fi[:5]))
w = t[13][56:60]
if w[0]:
    print("warp_first_seg (cycles after fast-start begin): loads %d | scan %d | sched %d | ranges %d" % tuple(int(x - su[4]) for x in w))

x = t[14][40:48]
if x[0] or x[4]:
    pv = t[12][0]
    f = lambda v: int(v - pv) if v else -1  # noqa: E731
    print("DSMEM exchange (cycles after the traced CTA's last PV done): receiver: O read %d, peer half landed %d, "
          "merged %d, stored %d | sender: O read %d, peer ring free %d, staged %d, copies issued %d"
          % (f(x[0]), f(x[1]), f(x[3]), f(x[2]), f(x[4]), f(x[5]), f(x[6]), f(x[7])))
e = t[13][40:46]
if e[0] and t[12][0]:
    print("head epilogue (cycles after its PV done): merged pieces landed %d | (m,l) merged %d | chunk0 merged %d, stored %d | chunk1 merged %d, stored %d"
          % tuple(int(x - t[12][0]) if x else -1 for x in e))

st, en, nt = cta[:, 0], cta[:, 1], cta[:, 2]
t0g = st.min()
print("\nper-CTA (us): start min/median/max %.2f %.2f %.2f | end min/median/max %.2f %.2f %.2f" % (
    (st.min() - t0g) / 1e3, (np.median(st) - t0g) / 1e3, (st.max() - t0g) / 1e3,
    (en.min() - t0g) / 1e3, (np.median(en) - t0g) / 1e3, (en.max() - t0g) / 1e3))
dur = (en - st) / 1e3
order = np.argsort(dur)
print("slowest CTAs:", [(int(i), round(float(dur[i]), 1), int(nt[i])) for i in order[-8:]])
print("fastest CTAs:", [(int(i), round(float(dur[i]), 1), int(nt[i])) for i in order[:5]])
hist = np.histogram(dur, bins=8)
print("duration histogram:", hist[0].tolist(), [round(float(x), 1) for x in hist[1]])

rel = lambda k: (cta[:, k] - cta[:, 0]) / 1e3  # noqa: E731
mhz = (cta[:, 7] - cta[:, 6]) / (cta[:, 1] - cta[:, 0]) * 1e3
print("SM clock from clock64/globaltimer (MHz): median %.0f min %.0f max %.0f" % (np.median(mhz), mhz.min(), mhz.max()))
for k, name in [(8, "kernel entry"), (9, "setup done"), (5, "first K issue"), (3, "last PV done"),
                (11, "pieces staging"), (10, "pieces landed"), (4, "O read+written"), (1, "CTA end")]:
    v = rel(k)
    ok = cta[:, k] > 0
    if k == 8:
        v = -v
    print(f"{name:16s} (us after CTA start; entry: before): median {np.median(v[ok]) if ok.any() else -1:7.2f}  max {v[ok].max() if ok.any() else -1:7.2f}  n={ok.sum()}")
ent = cta[:, 8]
e0 = ent.min()
print("kernel entry spread (us): %.2f ; whole kernel entry->last end (us): %.2f" % ((ent.max() - e0) / 1e3, (cta[:, 1].max() - e0) / 1e3))
per_tile = (cta[:, 3] - cta[:, 5]) / np.maximum(nt - 1, 1) / 1e3
print("per-tile (us, first K issue -> last PV done): median %.3f min %.3f max %.3f" % (np.median(per_tile), per_tile.min(), per_tile.max()))
