"""Diagnostic (ST_GEMM_PAIR=0: single-CTA tiles only): the tcgen05 GEMM (st_gemm) vs cuBLAS (torch.matmul) at the C3
projection shapes (M = B*T = 2048 rows, d = 4096, FFN 16384, V = 32000), f16,
CUDA events, mean of N launches after warm-up.

  python tools/gemm_bench.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402

M = int(os.environ.get("GEMM_M", "2048"))
SHAPES = [("qkv", 4096, 4096, 3, "store"), ("wo", 4096, 4096, 1, "add_to"),
          ("ffn1", 16384, 4096, 1, "gelu"), ("ffn2", 4096, 16384, 1, "add_to"),
          ("lm_head", 32000, 4096, 1, "store_f32")]


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for name, N, K, Z, epi in SHAPES:
    a = torch.randn(M, K, device="cuda").half()
    w = torch.randn(Z, K, N, device="cuda").half() * K ** -0.5
    out = torch.empty(Z, M, N, device="cuda", dtype=torch.float32 if epi == "store_f32" else torch.half)
    ours = timed(lambda: _capi.gemm(a, w[0] if Z == 1 else w, out=out[0] if Z == 1 else out,
                                    epilogue=epi))
    if Z == 1:
        theirs = timed(lambda: torch.matmul(a, w[0], out=None))
    else:
        theirs = timed(lambda: torch.matmul(a.unsqueeze(0), w))
    fl = 2 * M * N * K * Z
    print(f"{name:8s} M={M} N={N} K={K} Z={Z}: ours {ours:8.1f} us {fl / ours / 1e6:7.1f} TF/s | "
          f"cuBLAS {theirs:8.1f} us {fl / theirs / 1e6:7.1f} TF/s | ratio {theirs / ours:.2f}")
