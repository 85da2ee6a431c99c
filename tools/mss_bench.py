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
if os.environ.get("ST_K4_TRACE") and ":" not in os.environ["ST_K4_TRACE"]:
    # trace the request with the longest accepted path (the kernel's critical path)
    Un = U.cpu().numpy()
    lens = [len(R.mss_verify(logits[b, :n[b]], q[b, :n[b]], tok[b, :n[b]], par[b, :n[b]], 1.0, Un[b])[0])
            for b in range(B)]
    os.environ["ST_K4_TRACE"] += ":%d" % int(np.argmax(lens))
    print("tracing request", int(np.argmax(lens)), "accepted", max(lens))
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

print("accepted lengths per request:", L.tolist())
if os.environ.get("ST_K4_TRACE"):
    names = {0: "entry", 1: "node start", 2: "kids found", 3: "z slice loaded", 4: "cluster max",
             5: "exp pass", 7: "owner sums + combine", 8: "scalars waited", 9: "child test",
             10: "slice wait + prefetch", 11: "residual pass", 12: "residual sums + combine",
             13: "final owner sums", 14: "barrier", 15: "leader prefix + search", 16: "chunk scan", 17: "exit barrier"}
    ev = [tuple(map(int, l.split())) for l in open(os.environ["ST_K4_TRACE"].split(":")[0])]
    tot = {}
    for (c0, t0), (c1, t1) in zip(ev, ev[1:]):
        tot[c1] = tot.get(c1, 0) + (t1 - t0)
    span = ev[-1][1] - ev[0][1]
    print(f"request 0 trace: {len(ev)} events, {span} cycles")
    for c in sorted(tot, key=lambda c: -tot[c]):
        print(f"  {names.get(c, c):28s} {tot[c]:8d} cycles  {100 * tot[c] / span:5.1f} %")
