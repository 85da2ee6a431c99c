"""Diagnostic: K1 at the C3 layer shape (B=32, T=64, KV 2048, H=32, k_tree)
with the grid limited to ST_K1_GRID CTAs — how much HBM bandwidth K1 keeps on
a subset of the SMs (the premise of overlapping attention with GEMMs).
  for g in 0 112 96 80 64; do ST_K1_GRID=$g python tools/k1_grid.py; done
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2305_09781_b200 import _capi
B, H, D, L, T = 32, 32, 128, 2048, 64
dev = "cuda"
q = torch.empty(B, T, H, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
kc = torch.empty(B, H, L + T, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
vc = torch.empty_like(kc).uniform_(-1, 1)
kt = torch.empty(B, T, H, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
vt = torch.empty_like(kt).uniform_(-1, 1)
par = torch.tensor([[-1] + [0] * (T - 1)] * B, dtype=torch.int32, device=dev)
n = torch.full((B,), T, dtype=torch.int32, device=dev)
P = torch.full((B,), L, dtype=torch.int32, device=dev)
mask = _capi.build_masks(par, n)
ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, n)
out = torch.empty_like(q)
for _ in range(3):
    _capi.tree_attention(q, kc, vc, mask, P, n, out=out, workspace=ws, k_tree=kt, v_tree=vt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    _capi.tree_attention(q, kc, vc, mask, P, n, out=out, workspace=ws, k_tree=kt, v_tree=vt)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 20
byts = 2 * (2 * B * L * H * D + 4 * B * T * H * D)
print(f"grid {os.environ.get('ST_K1_GRID', 'all')}: {us:.1f} us  {byts / us / 1e3:.0f} GB/s")
