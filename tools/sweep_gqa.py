"""GQA sweep: K1 tree attention with G query heads per KV head (LLaMA-3-70B
attention shape: H=64, Hkv=8, D=128, fp16), batch 16, KV 4K-16K x tree
width 8-16, on one B200 — tcgen05 path (the G*T query rows of a (request, KV
head) pair share one tile) vs the CUDA-core path on the same inputs.

Algorithmic bytes: s*[2*B*L*Hkv*D + B*T*H*D + 2*B*T*Hkv*D + B*T*H*D] + 8*B*T*W.

  python tools/sweep_gqa.py [--out profiles/gqa_sweep.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_09781_b200 import _capi  # noqa: E402
from paper_2305_09781_b200.tree import TokenTree, TreeBatch  # noqa: E402

B, H, HKV, D = 16, 64, 8, 128


def trees_of(T, seed):
    rng = np.random.default_rng(seed)
    w = 2 if T < 16 else 3
    out = []
    for _ in range(B):
        root = int(rng.integers(0, 32000))
        seqs = [[root] + rng.integers(0, 32000, (T - 1) // w).tolist() for _ in range(w)]
        out.append(TokenTree.merge_sequences(seqs, 1 << 20))
    return TreeBatch(out, T)


def time_k1(args_, iters, path):
    """Device time per launch. tcgen05: `iters` launches captured in one CUDA
    graph, alternating two KV copies (each launch streams from HBM: 268 MB+
    per copy > L2) — eager launches through the Python wrapper are host-bound
    at 4K (~50 us of host work per call, more than the kernel). CUDA-core
    (milliseconds per launch): eager."""
    q, kvs, mask, P, n, out, ws = args_

    def launch(i):
        kc, vc = kvs[i % len(kvs)]
        _capi.tree_attention(q, kc, vc, mask, P, n, out=out, workspace=ws, force_path=path)
    for i in range(4):
        launch(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if path == 2:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(iters):
                launch(i)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
    else:
        e0.record()
        for i in range(iters):
            launch(i)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "gqa_sweep.json"))
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    dev = "cuda"
    Ls, Ts = [4096, 8192, 16384], [8, 16]
    Lmax = max(Ls) + max(Ts)
    kvs = [(torch.empty(B, HKV, Lmax, D, dtype=torch.float16, device=dev).uniform_(-1, 1),
            torch.empty(B, HKV, Lmax, D, dtype=torch.float16, device=dev).uniform_(-1, 1)) for _ in range(2)]
    kc, vc = kvs[0]
    rows = []
    for T in Ts:
        tb = trees_of(T, T)
        par = torch.tensor(tb.parents, device=dev)
        n = torch.tensor(tb.n_nodes, device=dev)
        mask = _capi.build_masks(par, n)
        q = torch.empty(B, T, H, D, dtype=torch.float16, device=dev).uniform_(-1, 1)
        out = torch.empty_like(q)
        for L in Ls:
            P = torch.full((B,), L, dtype=torch.int32, device=dev)
            ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, n)
            us_tc = time_k1((q, kvs, mask, P, n, out, ws), 2 * args.iters, 2)
            _capi.tree_attention(q, kc, vc, mask, P, n, out=out, workspace=ws, force_path=2)
            ref = out.clone()
            us_cc = time_k1((q, [(kc, vc)], mask, P, n, out, ws), max(2, args.iters // 5), 1)
            err = (out.float() - ref.float()).abs().max().item()
            W = (T + 63) // 64
            byts = 2 * (2 * B * L * HKV * D + B * T * H * D + 2 * B * T * HKV * D + B * T * H * D) \
                + 8 * B * T * W
            gbs = byts / (us_tc * 1e-6) / 1e9
            rows.append(dict(L=L, T=T, G=H // HKV, B=B, us_tc=us_tc, us_cuda_core=us_cc, bytes=byts,
                             gbs=gbs, frac=gbs / peak, tc_vs_cc_maxabs=err))
            print(f"L={L:6d} T={T:3d} G={H // HKV}: tcgen05 {us_tc:7.1f} us {gbs:6.0f} GB/s "
                  f"{gbs / peak:5.3f} of peak | cuda-core {us_cc:7.1f} us | max|diff| {err:.1e}")
    json.dump({"config": f"GQA: B={B}, H={H}, Hkv={HKV}, D={D}, fp16", "peak_gbs": peak,
               "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
