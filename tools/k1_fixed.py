"""Diagnostic: K1's fixed cost — device time per launch (CUDA events over a
graph of 200 back-to-back launches) of shapes whose streaming work is one or a few tiles
per CTA, so the number is dominated by launch, prologue, first-load latency
and epilogue. Also the C4 per-rank slice for reference.

  python tools/k1_fixed.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402


def run(B, H, T, L, Hkv=None, n=200, early=False):
    Hkv = Hkv or H
    dev = "cuda"
    q = torch.randn(B, T, H, 128, device=dev).half()
    kc = torch.randn(B, Hkv, L + T, 128, device=dev).half()
    vc = torch.randn(B, Hkv, L + T, 128, device=dev).half()
    par = torch.tensor([[-1] + [0] * (T - 1)] * B, dtype=torch.int32, device=dev)
    nn = torch.full((B,), T, dtype=torch.int32, device=dev)
    P = torch.full((B,), L, dtype=torch.int32, device=dev)
    mask = _capi.build_masks(par, nn)
    out = torch.empty_like(q)
    ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, nn)
    for _ in range(10):
        _capi.tree_attention(q, kc, vc, mask, P, nn, out=out, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # device time: the host's per-call cost is off the clock
    with torch.cuda.graph(g):
        for _ in range(n):
            _capi.tree_attention(q, kc, vc, mask, P, nn, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


for name, args in [("1 pair x 1 tile", (1, 1, 1, 1)), ("148 pairs x 1 tile", (4, 37, 16, 64)),
                   ("64 pairs x 2 tiles", (8, 8, 61, 150)), ("C4 slice (64 pairs x 17 tiles)", (8, 8, 61, 2048)),
                   ("C2", (8, 32, 64, 2048))]:
    print(f"{name:34s} {run(*args):8.2f} us")
