"""Diagnostic: C2 step time with parts of the step removed (CUDA graphs of 10
steps, CUDA events, inputs > L2). Shows what each kernel adds on the PDL
chain: masks | K1 | argmax(+walk) | walk+commit.

  python tools/step_breakdown.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Restatement  # noqa: E402
from paper_2305_09781_b200 import _capi  # noqa: E402
from tests.treegen import pack, width_depth_seqs  # noqa: E402

R = Restatement()
rng = np.random.default_rng(0)
B, T, H, D, L, V = 8, 64, 32, 128, 2048, 32000
trees = []
while len(trees) < B:
    t = R.merge(width_depth_seqs(rng, 1, 32000, 8, 8), 4096)
    if len(t[0]) <= T:
        trees.append(t)
tok, par, dep, n = pack(trees, T)
dev = "cuda"
tk, pr, nd = (torch.tensor(x, device=dev) for x in (tok, par, n))
P = torch.full((B,), L, dtype=torch.int32, device=dev)
kc = torch.randn(B, H, L + T, D, device=dev).half()
vc = torch.randn(B, H, L + T, D, device=dev).half()
q = torch.randn(B, T, H, D, device=dev).half()
kn = torch.randn(B, T, H, D, device=dev).half()
vn = torch.randn(B, T, H, D, device=dev).half()
logits = torch.randn(B, T, V, device=dev)
mask = torch.zeros(B, T, 1, dtype=torch.int64, device=dev)
out = torch.empty_like(q)
ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, nd)
wv = _capi.verify_workspace(B, T, dev)
vout = (torch.zeros((B, T + 1), dtype=torch.int32, device=dev),
        torch.zeros((B, T + 1), dtype=torch.int32, device=dev), torch.zeros(B, dtype=torch.int32, device=dev))


def masks():
    _capi.build_masks(pr, nd, out=mask)


def k1():
    _capi.tree_attention(q, kc, vc, mask, P, nd, out=out, workspace=ws, k_tree=kn, v_tree=vn)


def verify():
    _capi.verify_greedy(logits, tk, pr, nd, workspace=wv, want_argmax=False, out=vout)


def commit():
    _capi.verify_greedy_compact(logits, tk, pr, nd, P, kc, vc, workspace=wv, want_argmax=False,
                                out=vout, k_tree=kn, v_tree=vn)


variants = {
    "masks": [masks],
    "K1": [k1],
    "argmax+walk": [verify],
    "argmax+walk+commit": [commit],
    "masks K1": [masks, k1],
    "K1 argmax+walk": [k1, verify],
    "masks K1 argmax+walk": [masks, k1, verify],
    "full step (masks K1 argmax walk+commit)": [masks, k1, commit],
}
for name, fns in variants.items():
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            for f in fns:
                f()
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:42s} {e0.elapsed_time(e1) * 1e3 / 50:7.1f} us per step")
