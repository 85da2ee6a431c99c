import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2305_09781_b200 import _capi
from paper_2305_09781_b200.tree import TokenTree, TreeBatch
import bench
NL, d, Hh, Vv, B, T, L = 32, 4096, 32, 32000, 32, 64, 2048
dev = "cuda"
model = _capi.DeviceModel(NL, Hh, d, Vv, L + T + 64, 4, seed=42, dtype=torch.float16)
kc, vc = model.new_cache(B, L + T)
trees = bench.c2_trees(lambda s_: TokenTree.merge_sequences(s_, 1 << 20), 3000, Vv, n_req=B)
batch = TreeBatch([t for t, _ in trees], T)
tok = torch.tensor(batch.tokens, device=dev); par = torch.tensor(batch.parents, device=dev)
nn = torch.tensor(batch.n_nodes, device=dev); P = torch.full((B,), L, dtype=torch.int32, device=dev)
pos = (P[:, None] + torch.tensor(batch.depths, device=dev)).to(torch.int32)
mask = _capi.build_masks(par, nn)
logits = torch.empty(B, T, Vv, dtype=torch.float32, device=dev)
tq = model.new_tree_qkv(B, T)
for _ in range(2):
    model.tree_forward(tok, pos, mask, P, nn, kc, vc, logits=logits, tree_qkv=tq)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    model.tree_forward(tok, pos, mask, P, nn, kc, vc, logits=logits, tree_qkv=tq)
    torch.cuda.synchronize()
tot = {}
for ev in prof.events():
    if ev.device_type.name != "CUDA": continue
    t, c = tot.get(ev.name, (0.0, 0)); tot[ev.name] = (t + ev.device_time_total, c + 1)
for k, (t, c) in sorted(tot.items(), key=lambda x: -x[1][0])[:10]:
    print(f"{t/1e3:8.2f} ms {c:4d}x {t/c:8.1f} us  {k[:90]}")
