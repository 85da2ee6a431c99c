"""Diagnostic: the C2 step (bench.VerifyStep) timed three ways, CUDA events,
inputs > L2:
  graph/step : one CUDA-graph replay per step (what bench.py times)
  graph/10   : ten steps captured in one graph (programmatic launch chains
               across step boundaries; no per-replay gap)
  eager      : the four launches issued from Python every step (PDL chains
               across steps, but host launch cost per step)
The gap between graph/step and graph/10 is the per-replay boundary cost.

  python tools/step_modes.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
st = bench.VerifyStep(dev, 0)
for _ in range(3):
    st.run()
torch.cuda.synchronize()
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1):
    st.run()
g10 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g10):
    for _ in range(10):
        st.run()


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


# variant: no masks kernel in the chain (masks precomputed once), K1 right after
# the previous step's commit (early_kv off: that commit writes committed rows)
st.capi.build_masks(st.par, st.nn, W=st.W, out=st.mask)


def run_nomask():
    a = st.resident
    st.capi.tree_attention(st.q, st.kc, st.vc, st.mask, st.P, st.nn, out=st.out,
                           workspace=st.ws_attn, k_tree=st.knew, v_tree=st.vnew, early_kv=False)
    st.post(a)


gn = torch.cuda.CUDAGraph()
run_nomask()
torch.cuda.synchronize()
with torch.cuda.graph(gn):
    for _ in range(10):
        run_nomask()

for rnd in range(2):
    a = timed(g1.replay, 100)
    b = timed(g10.replay, 10) / 10
    c = timed(st.run, 100)
    extra = ""
    if hasattr(st, "run_native"):
        extra = f"  native {timed(st.run_native, 100):6.1f}"
    d = timed(gn.replay, 10) / 10
    print(f"graph/step {a:6.1f} us  graph/10 {b:6.1f} us  eager {c:6.1f} us  "
          f"graph/10 without masks kernel {d:6.1f} us{extra}")
