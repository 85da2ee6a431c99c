"""Diagnostic: K1 outputs with the TMA-store epilogue (default) are bit-identical
to the per-thread stores (ST_K1_OTMA=0 in a second process), on GQA / C2 / C5
shapes with ragged and full trees. Usage: python tools/otma_check.py [dump|compare]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402

SHAPES = [(16, 64, 8, 16, 4096, True), (16, 64, 8, 8, 4096, True), (8, 32, 32, 64, 2048, True),
          (4, 32, 32, 128, 1024, True), (4, 32, 32, 100, 1024, False), (3, 16, 4, 7, 700, False)]


def run():
    outs = []
    for i, (B, H, Hkv, T, L, full) in enumerate(SHAPES):
        g = torch.Generator(device="cuda").manual_seed(i)
        q = torch.randn(B, T, H, 128, device="cuda", generator=g).half()
        kc = torch.randn(B, Hkv, L + T, 128, device="cuda", generator=g).half()
        vc = torch.randn(B, Hkv, L + T, 128, device="cuda", generator=g).half()
        par = torch.tensor([[-1] + [max(0, (j - 1) // 2) for j in range(1, T)]] * B, dtype=torch.int32,
                           device="cuda")
        n = torch.full((B,), T, dtype=torch.int32, device="cuda")
        if not full:
            n[0] = T // 3
            n[-1] = 1
        P = torch.tensor([L - 17 * b for b in range(B)], dtype=torch.int32, device="cuda")
        mask = _capi.build_masks(par, n)
        out = torch.full_like(q, 7.0)
        lse = torch.zeros(B, H, T, device="cuda")
        _capi.tree_attention(q, kc, vc, mask, P, n, out=out, lse=lse)
        torch.cuda.synchronize()
        outs.append((out.cpu(), lse.cpu()))
    return outs


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "dump"
    path = "/tmp/otma_ref.pt"
    if mode == "dump":
        torch.save(run(), path)
    else:
        ref = torch.load(path)
        got = run()
        for s, (a, b) in zip(SHAPES, zip(ref, got)):
            print(s, "out identical" if torch.equal(a[0], b[0]) else "OUT DIFFERS",
                  "lse identical" if torch.equal(a[1], b[1]) else "LSE DIFFERS")
