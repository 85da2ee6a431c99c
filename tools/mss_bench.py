"""Diagnostic: K4 (st_verify_mss) at the C3 verification shape (B=32, T=64,
V=32000, tau=1), CUDA events over 20 calls; also reports the visited depth."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Restatement  # noqa: E402
from paper_2305_09781_b200 import _capi  # noqa: E402
from tests.test_mss import make_case  # noqa: E402

R = Restatement()
rng = np.random.default_rng(1)
B, V = 32, 32000
tok, par, n, logits, q = make_case(R, rng, V, width=8, depth=8, n_req=B)
T = tok.shape[1]
dev = "cuda"
U = torch.tensor(rng.uniform(0, 1, (B, T + 1)).astype(np.float32), device=dev)
args = [torch.tensor(x, device=dev) for x in (logits, q, tok, par, n)]
for _ in range(3):
    ver, ids, ln = _capi.verify_mss(*args, 1.0, U)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ver, ids, ln = _capi.verify_mss(*args, 1.0, U)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 20
L = ln.cpu().numpy()
print(f"K4 B={B} T={T} V={V}: {us:.1f} us per call; accepted lengths mean {L.mean():.2f} max {L.max()}")
