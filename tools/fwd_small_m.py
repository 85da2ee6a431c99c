import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2305_09781_b200 import _capi
from paper_2305_09781_b200.tree import TokenTree, TreeBatch
import bench
NL, d, Hh, Vv, B, T, L = 32, 4096, 32, 32000, 32, 21, 160
dev = "cuda"
model = _capi.DeviceModel(NL, Hh, d, Vv, L + T + 64, 4, seed=42, dtype=torch.float16)
kc, vc = model.new_cache(B, L + T)
trees = bench.c2_trees(lambda s_: TokenTree.merge_sequences(s_, 1 << 20), 3000, Vv, n_req=B, nodes=T)
batch = TreeBatch([t for t, _ in trees], T)
tok = torch.tensor(batch.tokens, device=dev); par = torch.tensor(batch.parents, device=dev)
nn = torch.tensor(batch.n_nodes, device=dev); P = torch.full((B,), L, dtype=torch.int32, device=dev)
pos = (P[:, None] + torch.tensor(batch.depths, device=dev)).to(torch.int32)
mask = _capi.build_masks(par, nn)
logits = torch.empty(B, T, Vv, dtype=torch.float32, device=dev)
for _ in range(3):
    model.tree_forward(tok, pos, mask, P, nn, kc, vc, logits=logits)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    model.tree_forward(tok, pos, mask, P, nn, kc, vc, logits=logits)
e1.record(); torch.cuda.synchronize()
print(f"splitk={os.environ.get('ST_GEMM_SPLITK','1')}: 32-layer forward at M={B*T}: {e0.elapsed_time(e1)/10:.2f} ms")
