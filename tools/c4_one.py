"""One C4 per-rank slice K1 configuration (8 of 64 heads, B=8, merged 3-SSM
trees of 61 nodes, KV 2048, fp16) for an ncu capture: 5 eager launches
through the C-ABI (tools/c4_slice.py times it inside CUDA graphs, which ncu
cannot replay)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402
from paper_2305_09781_b200.tree import TreeBatch  # noqa: E402
from tools.c4_slice import B, D, L, c4_tree  # noqa: E402

rng = np.random.default_rng(65)
tb = TreeBatch([c4_tree(rng, int(rng.integers(0, 32000))) for _ in range(B)])
T, Hl, dev = tb.T, 8, "cuda"
q = torch.empty(B, T, Hl, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
kc = torch.empty(B, Hl, L + T, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
vc = torch.empty(B, Hl, L + T, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
par = torch.tensor(tb.parents, device=dev)
n = torch.tensor(tb.n_nodes, device=dev)
P = torch.full((B,), L, dtype=torch.int32, device=dev)
mask = _capi.build_masks(par, n)
out = torch.empty_like(q)
ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, n)
for _ in range(5):
    _capi.tree_attention(q, kc, vc, mask, P, n, out=out, workspace=ws)
torch.cuda.synchronize()
print("ok", T)
