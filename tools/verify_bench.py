"""Diagnostic: st_verify_greedy (K3) alone at the C2 shape (B=8, T=64,
V=32000), cycling 3 logits buffers (196 MB > L2); CUDA events over 50 calls."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402
from tests.treegen import pack, width_depth_seqs  # noqa: E402
from oracle.oracle import Restatement  # noqa: E402

R = Restatement()
rng = np.random.default_rng(0)
B, T, V = 8, 64, 32000
trees = [R.merge(width_depth_seqs(rng, 1, 32000, 8, 7), 4096) for _ in range(B)]
tok, par, dep, n = pack(trees, T)
dev = "cuda"
tk, pr, nd = (torch.tensor(x, device=dev) for x in (tok, par, n))
lg = [torch.randn(B, T, V, device=dev) for _ in range(3)]
ws = _capi.verify_workspace(B, T, dev)
out = (torch.zeros((B, T + 1), dtype=torch.int32, device=dev),
       torch.zeros((B, T + 1), dtype=torch.int32, device=dev), torch.zeros(B, dtype=torch.int32, device=dev))
for i in range(6):
    _capi.verify_greedy(lg[i % 3], tk, pr, nd, workspace=ws, want_argmax=False, out=out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(30):
        _capi.verify_greedy(lg[i % 3], tk, pr, nd, workspace=ws, want_argmax=False, out=out)
for _ in range(2):
    g.replay()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"st_verify_greedy: {e0.elapsed_time(e1) * 1e3 / 150:.2f} us per call")
