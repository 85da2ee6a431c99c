"""C5 sweep (BASELINE.json configs[4]): K1 tree attention at LLaMA-7B shape
(H=32, D=128, fp16), batch 16, KV 4K-32K x tree width 16-128, on one B200.

For each point: K1 device time (CUDA events, mean of N launches; the KV
working set exceeds L2 at every point), algorithmic bytes
(s*[2BLHD + BTHD + 2BTHD + BTHD] + 8BT*ceil(T/64)) and the
fraction of the measured HBM copy peak. Trees: W root-to-leaf paths of depth
ceil((T-1)/W), W = 4/8/8/16 for T = 16/32/64/128, trimmed to exactly T nodes.

  python tools/sweep_c5.py [--out profiles/c5_sweep.json]
"""
import argparse
import time
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_09781_b200 import _capi  # noqa: E402
from paper_2305_09781_b200.tree import TokenTree, TreeBatch  # noqa: E402

B, H, D = 16, 32, 128
WIDTH = {4: 2, 8: 2, 16: 4, 32: 8, 64: 8, 128: 16, 256: 16}


def trees_of(T, seed):
    rng = np.random.default_rng(seed)
    out = []
    W = WIDTH[T]
    depth = -(-(T - 1) // W)
    for _ in range(B):
        root = int(rng.integers(0, 32000))
        seqs = [[root] + rng.integers(0, 32000, depth).tolist() for _ in range(W)]
        t = TokenTree.merge_sequences(seqs, 1 << 20)
        i = len(seqs) - 1
        while t.size > T:
            if len(seqs[i]) > 1:
                seqs[i] = seqs[i][:-1]
            else:
                i -= 1
            t = TokenTree.merge_sequences(seqs, 1 << 20)
        out.append(t)
    return TreeBatch(out, T)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "c5_sweep.json"))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--Ls", default="4096,8192,16384,32768")
    ap.add_argument("--Ts", default="16,32,64,128,256")
    ap.add_argument("--cool", type=float, default=0.0,
                    help="seconds idle before each point (0: back to back, clocks as they fall)")
    args = ap.parse_args()
    try:   # SM clock / power sampled DURING each point's timed loop (the sweep runs power-capped)
        import threading

        import pynvml
        pynvml.nvmlInit()
        nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:  # noqa: BLE001
        nvh = None

    def sampled(fn):
        """Run fn() while a thread samples the SM clock and board power (median)."""
        if nvh is None:
            fn()
            return None, None
        got, stop = [], threading.Event()

        def poll():
            while not stop.is_set():
                got.append((pynvml.nvmlDeviceGetClockInfo(nvh, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(nvh) / 1e3))
                time.sleep(0.002)
        th = threading.Thread(target=poll)
        th.start()
        fn()
        stop.set()
        th.join()
        if not got:
            return None, None
        got.sort()
        return got[len(got) // 2][0], round(sorted(g[1] for g in got)[len(got) // 2])
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    dev = "cuda"
    Ls = [int(x) for x in args.Ls.split(",")]
    Ts = [int(x) for x in args.Ts.split(",")]
    Lmax = max(Ls) + max(Ts)
    # two KV copies alternated launch by launch: every launch streams from HBM
    kvs = [(torch.empty(B, H, Lmax, D, dtype=torch.float16, device=dev).uniform_(-1, 1),
            torch.empty(B, H, Lmax, D, dtype=torch.float16, device=dev).uniform_(-1, 1)) for _ in range(2)]
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
            if args.cool > 0:
                time.sleep(args.cool)
            def launch(i):
                _capi.tree_attention(q, kvs[i % 2][0], kvs[i % 2][1], mask, P, n, out=out, workspace=ws)
            for i in range(4):
                launch(i)
            torch.cuda.synchronize()
            # device time: the timed launches are one CUDA graph (eager launches
            # through the Python wrapper are host-bound on the short points)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(args.iters):
                    launch(i)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

            def timed():
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
            mhz, pw = sampled(timed)
            us = e0.elapsed_time(e1) * 1e3 / args.iters
            W = (T + 63) // 64
            byts = 2 * (2 * B * L * H * D + B * T * H * D + 2 * B * T * H * D + B * T * H * D) + 8 * B * T * W
            gbs = byts / (us * 1e-6) / 1e9
            row = dict(L=L, T=T, B=B, us=us, bytes=byts, gbs=gbs, frac=gbs / peak, sm_mhz=mhz, power_w=pw,
                       path=_capi.tree_attention_path(q, kc, vc, mask, P, n))
            rows.append(row)
            print(f"L={L:6d} T={T:4d}: {us:8.1f} us  {gbs:7.0f} GB/s  {gbs / peak:5.3f} of measured peak"
                  f"  (SM {mhz} MHz, {pw} W)")
    json.dump({"config": "C5: B=16, H=32, D=128, fp16", "peak_gbs": peak, "rows": rows},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
