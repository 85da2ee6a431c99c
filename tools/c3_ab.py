"""Diagnostic: the C3 step (32-layer LLaMA-7B-shape stack, 32 requests x
64-node trees, KV 2048, MSS verify, in-place compaction) through the
round-1 API (st_model_tree_forward + st_verify_mss + st_kv_compact) — runs
against any library build (ST_LIB_VARIANT), e.g. the round-1 cuBLAS one, for a
same-box A/B of the around-path GEMMs.

  ST_LIB_VARIANT=build/variants/r1_cublas.so python tools/c3_ab.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2305_09781_b200 import _capi  # noqa: E402
from paper_2305_09781_b200.tree import TokenTree, TreeBatch  # noqa: E402

NL, d, H, V, B, T, L = 32, 4096, 32, 32000, 32, 64, 2048
dev = "cuda"
model = _capi.DeviceModel(NL, H, d, V, L + T + 64, 4, seed=42, dtype=torch.float16)
kc, vc = model.new_cache(B, L + T)
kc.uniform_(-1, 1)
vc.uniform_(-1, 1)
trees = bench.c2_trees(lambda s: TokenTree.merge_sequences(s, 1 << 20), 3000, V, n_req=B)
batch = TreeBatch([t for t, _ in trees], T)
tok = torch.tensor(batch.tokens, device=dev)
par = torch.tensor(batch.parents, device=dev)
nn = torch.tensor(batch.n_nodes, device=dev)
P = torch.full((B,), L, dtype=torch.int32, device=dev)
pos = (P[:, None] + torch.tensor(batch.depths, device=dev)).to(torch.int32)
mask = _capi.build_masks(par, nn)
g = torch.Generator(device=dev).manual_seed(7)
qd = torch.softmax(torch.randn(B, T, V, device=dev, generator=g) * 3, dim=-1)
U = torch.rand(B, T + 1, device=dev, generator=g)
logits = torch.empty(B, T, V, dtype=torch.float32, device=dev)


def step():
    model.tree_forward(tok, pos, mask, P, nn, kc, vc, logits=logits)
    ver, ids, ln = _capi.verify_mss(logits, qd, tok, par, nn, 1.0, U)
    _capi.kv_compact(ids, ln, P, kc, vc)


for _ in range(3):
    step()
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        step()
    e1.record()
    torch.cuda.synchronize()
    print(f"{os.environ.get('ST_LIB_VARIANT') or 'HEAD'}: C3 step {e0.elapsed_time(e1) / 5:.2f} ms")
