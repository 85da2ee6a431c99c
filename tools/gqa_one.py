"""One GQA K1 configuration (LLaMA-3-70B attention shape: H=64, Hkv=8, D=128,
B=16, T=16, KV 8192, fp16) for an ncu capture: 5 launches through the C-ABI
(--path 2 tcgen05, 1 CUDA-core)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--path", type=int, default=2)
args = ap.parse_args()
B, H, HKV, D, T, L = 16, 64, 8, 128, 16, 8192
dev = "cuda"
kc = torch.empty(B, HKV, L + T, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
vc = torch.empty_like(kc).uniform_(-1, 1)
q = torch.empty(B, T, H, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
par = torch.tensor([[-1] + list(range(T - 1))] * B, dtype=torch.int32, device=dev)  # a chain
n = torch.full((B,), T, dtype=torch.int32, device=dev)
P = torch.full((B,), L, dtype=torch.int32, device=dev)
mask = _capi.build_masks(par, n)
out = torch.empty_like(q)
ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, n, force_path=args.path)
for _ in range(5):
    _capi.tree_attention(q, kc, vc, mask, P, n, out=out, workspace=ws, force_path=args.path)
torch.cuda.synchronize()
