"""Parity of the tcgen05 tree-attention kernel (K1, f16/bf16, D=128).

Checked against the f64 CPU restatement on the same (rounded) inputs with the
north-star tolerance: max-abs 2e-3. Shapes exercise the stream-K split
(pairs cut across CTAs and merged), tiles straddling the prefix/tree border,
ragged node counts, and the 128-node maximum.
"""
import numpy as np
import pytest
import torch

from tests.test_gpu_kernels import TOL, check_k1, make_batch, run_k1
from tests.treegen import expansion_seqs, pack, width_depth_seqs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    return _capi


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("B,H,P_range", [(3, 2, (1, 60)), (4, 8, (100, 700)), (2, 3, (1000, 1300)),
                                         (9, 16, (0, 300)),
                                         # long pairs over ~2 tiles per CTA: one pair
                                         # leaves ~70 pieces, past the staged ones
                                         (1, 2, (19000, 20000))])
def test_tc_matches_oracle(capi, restatement, dtype, B, H, P_range):
    rng = np.random.default_rng(B * 100 + H)
    bt = make_batch(restatement, rng, B, H, H, 128, dtype=dtype, P_range=P_range)
    out, lse = run_k1(capi, bt, dtype, force_path=2, lse=True)
    check_k1(restatement, bt, out, dtype, lse)


@pytest.mark.parametrize("B,empty", [(40, (0, 7, 39)), (136, (5,))])
def test_tc_batch_table_and_empty_requests(capi, restatement, B, empty):
    """B <= 128 uses the shared-memory tile table (binary search over the
    cumulative tile counts), B = 136 the global-memory walk; requests with no
    tree nodes own no tiles and must be skipped by both."""
    rng = np.random.default_rng(B)
    bt = make_batch(restatement, rng, B, 2, 2, 128, dtype=torch.float16, P_range=(0, 300))
    for b in empty:
        bt["n"][b] = 0
    out, _ = run_k1(capi, bt, torch.float16, force_path=2)
    keep = [b for b in range(B) if b not in empty]
    sub = {k: (v[keep] if isinstance(v, np.ndarray) and v.shape[:1] == (B,) else v)
           for k, v in bt.items()}
    check_k1(restatement, sub, out[keep], torch.float16)


def _dummy(bt, dtype):
    dev = "cuda"
    q = torch.zeros(bt["q"].shape, dtype=dtype, device=dev)
    kc = torch.zeros(bt["kc"].shape, dtype=dtype, device=dev)
    mask = torch.zeros(bt["mask"].shape, dtype=torch.int64, device=dev)
    P = torch.tensor(bt["P"], device=dev)
    n = torch.tensor(bt["n"], device=dev)
    return q, kc, kc, mask, P, n


@pytest.mark.parametrize("T,width,depth", [(16, 4, 3), (64, 9, 7), (128, 16, 7), (61, 0, 0)])
def test_tc_tree_widths(capi, restatement, T, width, depth):
    rng = np.random.default_rng(T)
    trees = []
    for _ in range(3):
        if width == 0:   # C4: merged tree of 3 SSMs, expansion <1,1,3,1,1,1,1,1>
            seqs = expansion_seqs(rng, 5, 32000, 3, [1, 1, 3, 1, 1, 1, 1, 1])
        else:
            seqs = width_depth_seqs(rng, 5, 32000, width, depth)
        t = restatement.merge(seqs, 4096)
        assert len(t[0]) <= T
        trees.append(t)
    bt = make_batch(restatement, rng, 3, 4, 4, 128, trees=trees, T=T, P_range=(50, 400),
                    dtype=torch.float16)
    out, lse = run_k1(capi, bt, torch.float16, force_path=2, lse=True)
    check_k1(restatement, bt, out, torch.float16, lse)


def test_tc_bitwise_deterministic_and_non_ancestor_invariant(capi, restatement):
    rng = np.random.default_rng(4)
    trees = [restatement.merge([[9, 3, 5, 6], [9, 3, 7, 8]])] * 2
    bt = make_batch(restatement, rng, 2, 32, 32, 128, trees=trees, P_range=(900, 900),
                    dtype=torch.float16)
    a, _ = run_k1(capi, bt, torch.float16, force_path=2)
    b, _ = run_k1(capi, bt, torch.float16, force_path=2)
    assert torch.equal(a, b)
    P = int(bt["P"][0])
    bt["kc"][:, :, P + 4:P + 6] += 3.0
    bt["vc"][:, :, P + 4:P + 6] -= 2.0
    c, _ = run_k1(capi, bt, torch.float16, force_path=2)
    assert torch.equal(a[:, :4], c[:, :4])


def test_tc_c2_shape_sampled_heads(capi, restatement):
    """C2 (B=8, T=64, L=2048, H=32, D=128, f16): full launch, checked on a
    sample of (b, h) pairs with a vectorised f64 reference."""
    rng = np.random.default_rng(2)
    B, T, H, D, L = 8, 64, 32, 128, 2048
    trees = []
    while len(trees) < B:
        t = restatement.merge(width_depth_seqs(rng, 1, 32000, 8, 8), 4096)
        if len(t[0]) <= T:
            trees.append(t)
    tok, par, dep, n = pack(trees, T)
    dev = "cuda"
    Lmax = L + T
    P = np.full(B, L, np.int32)
    q = torch.rand(B, T, H, D, device=dev, dtype=torch.float16) * 2 - 1
    kc = torch.rand(B, H, Lmax, D, device=dev, dtype=torch.float16) * 2 - 1
    vc = torch.rand(B, H, Lmax, D, device=dev, dtype=torch.float16) * 2 - 1
    from tests.treegen import masks
    m = masks(restatement, par, n, 1)
    mask = torch.tensor(m.view(np.int64), device=dev)
    out = capi.tree_attention(q, kc, vc, mask, torch.tensor(P, device=dev),
                              torch.tensor(n, device=dev), force_path=2)
    torch.cuda.synchronize()
    worst = 0.0
    for (b, h) in [(0, 0), (3, 17), (7, 31), (5, 8)]:
        qq = q[b, :, h].double().cpu().numpy()
        kk = kc[b, h].double().cpu().numpy()
        vv = vc[b, h].double().cpu().numpy()
        s = qq @ kk[: L + n[b]].T / np.sqrt(D)
        vis = np.ones_like(s, dtype=bool)
        for u in range(T):
            for v in range(n[b]):
                vis[u, L + v] = bool((int(m[b, u, 0]) >> v) & 1) if u < n[b] else False
        s = np.where(vis, s, -np.inf)
        s -= s.max(axis=1, keepdims=True)
        pr = np.exp(s)
        pr /= pr.sum(axis=1, keepdims=True)
        ref = pr @ vv[: L + n[b]]
        got = out[b, : n[b], h].double().cpu().numpy()
        worst = max(worst, np.abs(got - ref[: n[b]]).max())
    assert worst <= 2e-3, worst


@pytest.mark.parametrize("G,T,dtype", [(2, 32, torch.float16), (4, 16, torch.bfloat16),
                                       (8, 16, torch.float16), (4, 32, torch.bfloat16),
                                       (2, 64, torch.float16), (16, 8, torch.float16)])
def test_tc_gqa_head_groups(capi, restatement, G, T, dtype):
    """GQA: G query heads share each KV head; the tcgen05 kernel stacks the
    group's G*T query rows into one M=64/128 tile per (request, KV head), so
    every KV tile read serves G heads. Checked against the f64 restatement
    (same rounded inputs), with LSE, ragged trees and split pairs."""
    rng = np.random.default_rng(G * 100 + T)
    w = 2 if T < 16 else 3
    trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 50)), 50, w, (T - 1) // w),
                               4096) for _ in range(5)]   # <= 1 + w*depth <= T nodes
    Hkv = 3
    bt = make_batch(restatement, rng, 5, G * Hkv, Hkv, 128, trees=trees, T=T, P_range=(0, 900),
                    dtype=dtype)
    assert capi is not None
    out, lse = run_k1(capi, bt, dtype, force_path=2, lse=True)
    check_k1(restatement, bt, out, dtype, lse)


@pytest.mark.parametrize("path,G,dtype,early", [(2, 1, torch.float16, False), (2, 4, torch.bfloat16, False),
                                                (2, 1, torch.float16, True), (2, 4, torch.float16, True),
                                                (1, 1, torch.float16, False), (1, 2, torch.float32, False)])
def test_k1_tree_rows_from_k_tree(capi, restatement, path, G, dtype, early):
    """st_attn_args.k_tree/v_tree: the tree rows come from the tree's own
    [B][T][Hkv][D] tensors (no append); cache rows [P, P+n) hold junk (finite,
    large) that must not leak into any output."""
    rng = np.random.default_rng(40 + path * 10 + G)
    Hkv, T = 2, 32
    trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 50)), 50, 3, 10), 4096)
             for _ in range(6)]
    bt = make_batch(restatement, rng, 6, G * Hkv, Hkv, 128, trees=trees, T=T, P_range=(0, 500),
                    dtype=dtype)
    bt["P"][0] = 0          # no committed prefix at all
    bt["P"][1] = 256        # prefix ends on a tile boundary
    dev = "cuda"
    q = torch.tensor(bt["q"], device=dev).to(dtype)
    kc = torch.tensor(bt["kc"], device=dev).to(dtype)
    vc = torch.tensor(bt["vc"], device=dev).to(dtype)
    B = q.shape[0]
    kt = torch.zeros(B, T, Hkv, 128, dtype=dtype, device=dev)
    vt = torch.zeros_like(kt)
    for b in range(B):
        P, n = int(bt["P"][b]), int(bt["n"][b])
        kt[b, :n] = kc[b, :, P:P + n].transpose(0, 1)
        vt[b, :n] = vc[b, :, P:P + n].transpose(0, 1)
        kc[b, :, P:P + n] = 300.0   # junk where the appended rows would be
        vc[b, :, P:P + n] = -500.0
    mask = torch.tensor(bt["mask"].view(np.int64), device=dev)
    out = torch.zeros_like(q)
    lse = torch.zeros((B, G * Hkv, T), dtype=torch.float32, device=dev)
    Pd, nd = torch.tensor(bt["P"], device=dev), torch.tensor(bt["n"], device=dev)
    q_src = q.clone()
    q.zero_()
    q.copy_(q_src)   # the kernel right before K1 writes Q (allowed with early_kv)
    capi.tree_attention(q, kc, vc, mask, Pd, nd, out=out, lse=lse, force_path=path,
                        k_tree=kt, v_tree=vt, early_kv=early)
    torch.cuda.synchronize()
    check_k1(restatement, bt, out, dtype, lse)


def test_verify_compact_from_k_tree(capi, restatement):
    """st_verify_greedy_compact with k_tree/v_tree: the accepted rows are copied
    from the tree's own K/V into cache rows [P, P+len) — the same cache as
    append + in-place compaction."""
    rng = np.random.default_rng(8)
    V, Hkv, D, Lmax, layers = 500, 6, 128, 300, 2
    trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 8)), 8, 2, 12), 1024)
             for _ in range(4)]
    tok, par, dep, n = pack(trees)
    B, T = tok.shape
    logits = rng.standard_normal((B, T, V)).astype(np.float32)
    for b in range(B):
        for u in range(n[b]):
            kids = [v for v in range(n[b]) if par[b, v] == u]
            if kids and rng.random() < 0.9:
                logits[b, u, tok[b, kids[0]]] = 10.0
    dev = "cuda"
    lg, tk, pr, nd = (torch.tensor(x, device=dev) for x in (logits, tok, par, n))
    P = torch.tensor(rng.integers(0, 100, B), dtype=torch.int32, device=dev)
    kc = torch.randn(layers, B, Hkv, Lmax, D, device=dev).half()
    vc = torch.randn(layers, B, Hkv, Lmax, D, device=dev).half()
    kt = torch.randn(layers, B, T, Hkv, D, device=dev).half()
    vt = torch.randn(layers, B, T, Hkv, D, device=dev).half()
    # reference flow: append each layer's tree rows, then in-place compaction
    k1, v1 = kc.clone(), vc.clone()
    for l in range(layers):
        capi.kv_append(kt[l], vt[l], P, nd, k1[l], v1[l])
    a1, ver1, ids1, ln1 = capi.verify_greedy(lg, tk, pr, nd)
    capi.kv_compact(ids1, ln1, P, k1, v1)
    k2, v2 = kc.clone(), vc.clone()
    a2, ver2, ids2, ln2 = capi.verify_greedy_compact(lg, tk, pr, nd, P, k2, v2, k_tree=kt,
                                                     v_tree=vt)
    torch.cuda.synchronize()
    assert torch.equal(ln1, ln2) and torch.equal(ver1, ver2) and torch.equal(ids1, ids2)
    assert int(ln1.max()) > 3
    for b in range(B):
        p, L = int(P[b]), int(ln1[b])
        assert torch.equal(k1[:, b, :, : p + L], k2[:, b, :, : p + L])
        assert torch.equal(v1[:, b, :, : p + L], v2[:, b, :, : p + L])


@pytest.mark.parametrize("B,H,P,T", [(2, 4, 3000, 32), (8, 8, 2048, 61), (8, 8, 1500, 100),
                                     (1, 3, 700, 128)])
def test_tc_split_schedule(capi, restatement, B, H, P, T):
    """Uniform pairs with Np <= G/2 take the split schedule: every pair cut into
    S = G/Np single-segment pieces, the head piece min(kHeadExtra, nt - S)
    tiles longer (S = 18 for 8 pairs: the head owner merges 17 pieces, 2 staged
    in shared memory and the rest from L2; the last case has nt == S, so no
    extra tile). 64 pairs (C4's per-rank slice, M=64, and an M=128 tree) give
    S = 2 on 2-CTA clusters: two equal pieces that exchange (m, l) and one d
    half of O over DSMEM, each CTA writing the other half."""
    rng = np.random.default_rng(B * 7 + H)
    w = 3 if T >= 16 else 2
    trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 50)), 50, w, (T - 1) // w),
                               4096) for _ in range(B)]
    bt = make_batch(restatement, rng, B, H, H, 128, trees=trees, T=T, P_range=(P, P),
                    dtype=torch.float16)
    bt["n"][:] = bt["n"].max()   # uniform tile counts (pad the node counts)
    out, lse = run_k1(capi, bt, torch.float16, force_path=2, lse=True)
    check_k1(restatement, bt, out, torch.float16, lse)


def test_tc_fuzz(capi, restatement):
    """Random configurations through the tcgen05 kernel vs the f64 restatement:
    GQA group, tree width/depth, ragged prefixes (incl. 0 and tile
    boundaries), dtype, tree rows in the cache or in their own tensors,
    early_kv. Every schedule (whole pairs, equal pieces, stream-K) occurs."""
    rng = np.random.default_rng(2024)
    dev = "cuda"
    for case in range(24):
        G = int(rng.choice([1, 1, 2, 4, 8]))
        T = int(rng.choice([8, 16, 32, 61, 64, 100, 128]))
        while G * T > 128:
            T //= 2
        Hkv = int(rng.integers(1, 5))
        B = int(rng.integers(1, 7))
        dtype = torch.float16 if rng.random() < 0.6 else torch.bfloat16
        w = int(rng.integers(1, 5))
        trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 40)), 40, w,
                                                    max(1, (T - 1) // w)), 4096) for _ in range(B)]
        uniform = rng.random() < 0.3
        lo = int(rng.choice([0, 1, 127, 128, 300]))
        P_range = (lo, lo) if uniform else (lo, lo + int(rng.integers(0, 700)))
        bt = make_batch(restatement, rng, B, G * Hkv, Hkv, 128, trees=trees, T=T, P_range=P_range,
                        dtype=dtype)
        if uniform:
            bt["n"][:] = bt["n"].max()
        own, early = bool(rng.random() < 0.5), bool(rng.random() < 0.5)
        q = torch.tensor(bt["q"], device=dev).to(dtype)
        kc = torch.tensor(bt["kc"], device=dev).to(dtype)
        vc = torch.tensor(bt["vc"], device=dev).to(dtype)
        kt = vt = None
        if own:
            kt = torch.zeros(B, T, Hkv, 128, dtype=dtype, device=dev)
            vt = torch.zeros_like(kt)
            for b in range(B):
                P, n = int(bt["P"][b]), int(bt["n"][b])
                kt[b, :n] = kc[b, :, P:P + n].transpose(0, 1)
                vt[b, :n] = vc[b, :, P:P + n].transpose(0, 1)
                kc[b, :, P:P + n] = 7.0
                vc[b, :, P:P + n] = -9.0
        out = torch.zeros_like(q)
        lse = torch.zeros((B, G * Hkv, T), dtype=torch.float32, device=dev)
        capi.tree_attention(q, kc, vc, torch.tensor(bt["mask"].view(np.int64), device=dev),
                            torch.tensor(bt["P"], device=dev), torch.tensor(bt["n"], device=dev),
                            out=out, lse=lse, force_path=2, k_tree=kt, v_tree=vt, early_kv=early)
        torch.cuda.synchronize()
        check_k1(restatement, bt, out, dtype, lse)


def test_tc_fuzz_cluster_paths(capi, restatement):
    """Random configurations aimed at the 2-CTA cluster paths vs the f64
    restatement: uniform batches of 50-74 pairs (the split schedule with two
    pieces per pair — M=64: the piece's bulk copy into the head's first freed
    K stage; M=128: the symmetric half exchange) and trees past 128 rows (two
    row blocks per pair, K/V tiles multicast into both CTAs of a slot), with
    dtype, k_tree and early_kv drawn at random."""
    rng = np.random.default_rng(4096)
    dev = "cuda"
    for case in range(16):
        two_blocks = case % 3 == 2
        dtype = torch.float16 if rng.random() < 0.6 else torch.bfloat16
        if two_blocks:   # 128 < G*T <= 256, ragged everything
            G = int(rng.choice([1, 2]))
            T = int(rng.integers(129, 257)) // G
            Hkv = int(rng.integers(1, 4))
            B = int(rng.integers(1, 5))
            uniform = False
        else:            # 50..74 uniform pairs -> two pieces per pair
            G = int(rng.choice([1, 1, 2, 4]))
            T = int(rng.choice([16, 40, 61, 64, 100, 128])) // G
            np_target = int(rng.integers(50, 75))
            Hkv = int(rng.choice([d for d in range(1, 9) if np_target // d >= 1]))
            B = max(1, np_target // Hkv)
            uniform = True
        w = int(rng.integers(1, 5))
        trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 40)), 40, w,
                                                    max(1, (T - 1) // w)), 4096) for _ in range(B)]
        lo = int(rng.choice([0, 127, 128, 700, 1500]))
        P_range = (lo, lo) if uniform else (lo, lo + int(rng.integers(0, 900)))
        bt = make_batch(restatement, rng, B, G * Hkv, Hkv, 128, trees=trees, T=T, P_range=P_range,
                        dtype=dtype)
        if uniform:
            bt["n"][:] = bt["n"].max()
        own, early = bool(rng.random() < 0.5), bool(rng.random() < 0.5)
        q = torch.tensor(bt["q"], device=dev).to(dtype)
        kc = torch.tensor(bt["kc"], device=dev).to(dtype)
        vc = torch.tensor(bt["vc"], device=dev).to(dtype)
        kt = vt = None
        if own:   # the tree rows from their own tensors; the cache's copy poisoned
            kt = torch.zeros(B, T, Hkv, 128, dtype=dtype, device=dev)
            vt = torch.zeros_like(kt)
            for b in range(B):
                P, n = int(bt["P"][b]), int(bt["n"][b])
                kt[b, :n] = kc[b, :, P:P + n].transpose(0, 1)
                vt[b, :n] = vc[b, :, P:P + n].transpose(0, 1)
                kc[b, :, P:P + n] = 7.0
                vc[b, :, P:P + n] = -9.0
        out = torch.zeros_like(q)
        lse = torch.zeros((B, G * Hkv, T), dtype=torch.float32, device=dev)
        capi.tree_attention(q, kc, vc, torch.tensor(bt["mask"].view(np.int64), device=dev),
                            torch.tensor(bt["P"], device=dev), torch.tensor(bt["n"], device=dev),
                            out=out, lse=lse, force_path=2, k_tree=kt, v_tree=vt, early_kv=early)
        torch.cuda.synchronize()
        check_k1(restatement, bt, out, dtype, lse)


@pytest.mark.parametrize("T,G,dtype", [(1, 1, torch.float16), (2, 1, torch.bfloat16),
                                       (4, 1, torch.float16), (8, 1, torch.float16),
                                       (4, 2, torch.bfloat16), (15, 1, torch.float16)])
def test_tc_small_trees_auto_path(capi, restatement, T, G, dtype):
    """G*T < 16 (a few live query rows per tile): the auto dispatch now takes
    the tcgen05 kernel (one pass over the KV for all rows), checked against the
    f64 restatement with ragged prefixes, split pairs and LSE."""
    rng = np.random.default_rng(300 + T * 10 + G)
    Hkv = 4
    trees = []
    for _ in range(6):
        w = 1 if T <= 2 else 2
        t = restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 50)), 50, w,
                                               max(0, (T - 1) // w)), 4096)
        trees.append(tuple(a[:T] for a in t))
    bt = make_batch(restatement, rng, 6, G * Hkv, Hkv, 128, trees=trees, T=T,
                    P_range=(0, 3000), dtype=dtype)
    dev = "cuda"
    q = torch.tensor(bt["q"], device=dev).to(dtype)
    kc = torch.tensor(bt["kc"], device=dev).to(dtype)
    mask = torch.tensor(bt["mask"].view(np.int64), device=dev)
    Pd, nd = torch.tensor(bt["P"], device=dev), torch.tensor(bt["n"], device=dev)
    assert capi.tree_attention_path(q, kc, kc, mask, Pd, nd) == 2
    out, lse = run_k1(capi, bt, dtype, force_path=0, lse=True)
    check_k1(restatement, bt, out, dtype, lse)


@pytest.mark.parametrize("T,G,width,own,dtype,P_range", [
    (256, 1, 16, False, torch.float16, (50, 3000)),
    (256, 1, 32, True, torch.float16, (0, 700)),
    (200, 1, 20, True, torch.bfloat16, (1000, 1300)),
    (129, 1, 16, False, torch.float16, (127, 129)),
    (100, 2, 11, True, torch.float16, (300, 2500)),   # G*T = 200: two row blocks
    (64, 4, 8, False, torch.bfloat16, (0, 900)),      # G*T = 256
])
def test_tc_large_trees_two_row_blocks(capi, restatement, T, G, width, own, dtype, P_range):
    """G*T in (128, 256] (the reference bench's --max-tree-nodes 256,
    proj/tests/cli_roundtrip.cmake:69-71): each pair's rows are split into two
    128-row blocks run by a CTA pair over the same KV tiles; up to 4 mask
    words; k_tree mode with two tree tiles. Checked against the f64
    restatement with LSE, ragged prefixes and split pairs."""
    rng = np.random.default_rng(T * 3 + G + int(own))
    Hkv, B = 3, 5
    depth = -(-(T - 1) // width)
    trees = []
    for _ in range(B):
        t = restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 500)), 500, width, depth),
                              1 << 20)
        trees.append(tuple(a[:T] for a in t))
    bt = make_batch(restatement, rng, B, G * Hkv, Hkv, 128, trees=trees, T=T, P_range=P_range,
                    dtype=dtype)
    assert bt["W"] == (T + 63) // 64
    dev = "cuda"
    q = torch.tensor(bt["q"], device=dev).to(dtype)
    kc = torch.tensor(bt["kc"], device=dev).to(dtype)
    vc = torch.tensor(bt["vc"], device=dev).to(dtype)
    mask = torch.tensor(bt["mask"].view(np.int64), device=dev)
    Pd, nd = torch.tensor(bt["P"], device=dev), torch.tensor(bt["n"], device=dev)
    assert capi.tree_attention_path(q, kc, vc, mask, Pd, nd) == 2
    kt = vt = None
    if own:
        kt = torch.zeros(B, T, Hkv, 128, dtype=dtype, device=dev)
        vt = torch.zeros_like(kt)
        for b in range(B):
            P, n = int(bt["P"][b]), int(bt["n"][b])
            kt[b, :n] = kc[b, :, P:P + n].transpose(0, 1)
            vt[b, :n] = vc[b, :, P:P + n].transpose(0, 1)
            kc[b, :, P:P + n] = 5.0
            vc[b, :, P:P + n] = -3.0
    out = torch.zeros_like(q)
    lse = torch.zeros((B, G * Hkv, T), dtype=torch.float32, device=dev)
    capi.tree_attention(q, kc, vc, mask, Pd, nd, out=out, lse=lse, k_tree=kt, v_tree=vt)
    torch.cuda.synchronize()
    check_k1(restatement, bt, out, dtype, lse)


@pytest.mark.parametrize("G,T,slices,dtype", [(1, 61, [(0, 1), (1, 2), (2, 12), (12, 61)], torch.float16),
                                              (4, 21, [(0, 1), (5, 21)], torch.bfloat16),
                                              (1, 200, [(3, 170), (100, 200)], torch.float16)])
@pytest.mark.parametrize("path,tree", [(2, True), (1, True), (1, False)])
def test_tc_q_node_slices(capi, restatement, G, T, slices, dtype, path, tree):
    """st_attn_args.q_rows / q_node0 (ABI 5): Q, o and lse hold only the nodes
    [u0, u0 + rows) — one level of a draft tree grown level by level — while
    the masks and the tree rows (k_tree) span all T nodes. Every slice vs the
    f64 restatement of the whole tree's rows; ragged n (rows past n[b] are
    not written). Both kernels: the CUDA-core path also slices with the tree
    rows in the cache (no k_tree)."""
    rng = np.random.default_rng(T + G)
    B, Hkv = 3, 2
    w = 3
    trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, 40)), 40, w, max(1, (T - 1) // w)),
                               4096) for _ in range(B)]
    bt = make_batch(restatement, rng, B, G * Hkv, Hkv, 128, trees=trees, T=T, P_range=(0, 400),
                    dtype=dtype)
    D = 128
    dev = "cuda"
    ref, ref_lse = restatement.tree_attention(bt["q"], bt["kc"], bt["vc"], bt["mask"], bt["P"], bt["n"],
                                              1.0 / np.sqrt(D), want_lse=True)
    q = torch.tensor(bt["q"], device=dev).to(dtype)
    kc = torch.tensor(bt["kc"], device=dev).to(dtype)
    vc = torch.tensor(bt["vc"], device=dev).to(dtype)
    Tt = q.shape[1]
    kt = torch.zeros(B, Tt, Hkv, D, dtype=dtype, device=dev)
    vt = torch.zeros_like(kt)
    for b in range(B):
        P, n = int(bt["P"][b]), int(bt["n"][b])
        kt[b, :n] = kc[b, :, P:P + n].transpose(0, 1)
        vt[b, :n] = vc[b, :, P:P + n].transpose(0, 1)
    mask = torch.tensor(bt["mask"].view(np.int64), device=dev)
    P_t, n_t = torch.tensor(bt["P"], device=dev), torch.tensor(bt["n"], device=dev)
    for u0, u1 in slices:
        u1 = min(u1, Tt)
        qs = q[:, u0:u1].contiguous()
        out = torch.full_like(qs, 7.0)
        lse = torch.zeros((B, G * Hkv, u1 - u0), dtype=torch.float32, device=dev)
        capi.tree_attention(qs, kc, vc, mask, P_t, n_t, out=out, lse=lse, force_path=path,
                            k_tree=kt if tree else None, v_tree=vt if tree else None, q_node0=u0)
        torch.cuda.synchronize()
        got, L = out.double().cpu().numpy(), lse.double().cpu().numpy()
        for b in range(B):
            k = int(bt["n"][b])
            hi = min(u1, k)
            if hi > u0:
                assert np.abs(got[b, : hi - u0] - ref[b, u0:hi]).max() <= TOL[dtype]
                np.testing.assert_allclose(L[b, :, : hi - u0], ref_lse[b, :, u0:hi], atol=1e-4, rtol=0)
            if u1 > max(k, u0):   # rows past n[b] untouched
                assert torch.all(out[b, max(k, u0) - u0:] == 7.0)
