"""Diagnostic: K1 device time (graph of 50 launches, two KV copies alternated
so every launch streams from HBM) for a set of shapes, to A/B schedule knobs
set through the environment (ST_K1_SLACK, ST_K1_HEADX, ST_K1_CLUSTER).

  ST_K1_SLACK=20 python tools/k1_sched_ab.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402

SHAPES = [("C2 B8 H32 T64 L2048", 8, 32, 32, 64, 2048), ("C4 slice B8 H8 T61 L2048", 8, 8, 8, 61, 2048),
          ("GQA B16 H64/8 T8 L4096", 16, 64, 8, 8, 4096), ("GQA B16 H64/8 T16 L4096", 16, 64, 8, 16, 4096),
          ("GQA B16 H64/8 T16 L8192", 16, 64, 8, 16, 8192), ("C5 B16 H32 T64 L4096", 16, 32, 32, 64, 4096),
          ("C5 B16 H32 T128 L4096", 16, 32, 32, 128, 4096), ("B4 H32 T64 L8192", 4, 32, 32, 64, 8192)]


def run(B, H, Hkv, T, L, n=50):
    dev = "cuda"
    q = torch.randn(B, T, H, 128, device=dev).half()
    kvs = [(torch.randn(B, Hkv, L + T, 128, device=dev).half(), torch.randn(B, Hkv, L + T, 128, device=dev).half())
           for _ in range(2)]
    par = torch.tensor([[-1] + [0] * (T - 1)] * B, dtype=torch.int32, device=dev)
    nn = torch.full((B,), T, dtype=torch.int32, device=dev)
    P = torch.full((B,), L, dtype=torch.int32, device=dev)
    mask = _capi.build_masks(par, nn)
    out = torch.empty_like(q)
    ws = _capi.tree_attention_workspace(q, kvs[0][0], kvs[0][1], mask, P, nn)
    for i in range(4):
        _capi.tree_attention(q, kvs[i % 2][0], kvs[i % 2][1], mask, P, nn, out=out, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            _capi.tree_attention(q, kvs[i % 2][0], kvs[i % 2][1], mask, P, nn, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    byts = 2 * B * Hkv * (L + T) * 128 * 2 + 2 * B * T * H * 128 * 2
    return us, byts / us / 1e3


knobs = " ".join(f"{k}={os.environ[k]}" for k in ("ST_K1_SLACK", "ST_K1_HEADX", "ST_K1_CLUSTER") if k in os.environ)
for name, *shape in SHAPES:
    us, gbs = run(*shape)
    print(f"[{knobs or 'default'}] {name:28s} {us:8.2f} us {gbs:7.0f} GB/s {gbs / 6553.6:.3f}")
