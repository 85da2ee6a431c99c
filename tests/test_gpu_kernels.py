"""GPU parity tests for K1/K2/K3 through the C-ABI, checked against the CPU
restatement (oracle/restate.c, itself pinned to the reference by
tests/test_oracle_golden.py).

Tolerances (stated per north_star):
  f64 attention  max-abs 1e-12 (the reference's tree tests use 1e-9)
  f32 attention  max-abs 2e-6
  f16/bf16       max-abs 2e-3 relative to the f64 restatement on the same
                 (rounded) inputs
  greedy verify  bit-exact (argmax, accepted tokens, accepted ids, length)
"""
import numpy as np
import pytest
import torch

from tests.treegen import masks, pack, random_seqs, width_depth_seqs

pytestmark = pytest.mark.gpu

# max-abs vs the f64 restatement on the same rounded inputs. bf16 keeps 8
# mantissa bits (f16: 11): rounding P before P.V and rounding O each cost up to
# ~2^-9 relative, so bf16 gets 4e-3 where f16 meets 2e-3 (measured worst cases:
# f16 3.7e-4, bf16 3.1e-3 on the same tree batch).
TOL = {torch.float64: 1e-12, torch.float32: 2e-6, torch.float16: 2e-3, torch.bfloat16: 4e-3}


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    return _capi


def make_batch(restatement, rng, B, H, Hkv, D, vocab=50, T=None, P_range=(1, 200), trees=None,
               dtype=torch.float32, Lmax=None):
    if trees is None:
        trees = []
        for _ in range(B):
            root = int(rng.integers(0, vocab))
            seqs = random_seqs(rng, root, vocab, int(rng.integers(1, 6)), 6)
            trees.append(restatement.merge(seqs, 1024))
    tok, par, dep, n = pack(trees, T)
    T = tok.shape[1]
    W = (T + 63) // 64
    m = masks(restatement, par, n, W)
    P = rng.integers(P_range[0], P_range[1] + 1, B).astype(np.int32)
    Lmax = Lmax or int(P.max()) + T + 5
    q = rng.uniform(-1, 1, (B, T, H, D))
    kc = rng.uniform(-1, 1, (B, Hkv, Lmax, D))
    vc = rng.uniform(-1, 1, (B, Hkv, Lmax, D))
    # round through the compute dtype so the oracle sees the same values
    q = torch.tensor(q).to(dtype).double().numpy()
    kc = torch.tensor(kc).to(dtype).double().numpy()
    vc = torch.tensor(vc).to(dtype).double().numpy()
    return dict(tok=tok, par=par, dep=dep, n=n, P=P, mask=m, q=q, kc=kc, vc=vc, T=T, W=W)


def run_k1(capi, bt, dtype, force_path=0, lse=False):
    dev = "cuda"
    q = torch.tensor(bt["q"], device=dev).to(dtype)
    kc = torch.tensor(bt["kc"], device=dev).to(dtype)
    vc = torch.tensor(bt["vc"], device=dev).to(dtype)
    mask = torch.tensor(bt["mask"].view(np.int64), device=dev)
    P = torch.tensor(bt["P"], device=dev)
    n = torch.tensor(bt["n"], device=dev)
    out = torch.zeros_like(q)
    B, T, H, _ = q.shape
    lse_t = torch.zeros((B, H, T), dtype=torch.float32, device=dev) if lse else None
    capi.tree_attention(q, kc, vc, mask, P, n, out=out, lse=lse_t, force_path=force_path)
    torch.cuda.synchronize()
    return out, lse_t


def check_k1(restatement, bt, out, dtype, lse=None):
    D = bt["q"].shape[-1]
    ref, ref_lse = restatement.tree_attention(bt["q"], bt["kc"], bt["vc"], bt["mask"], bt["P"],
                                              bt["n"], 1.0 / np.sqrt(D), want_lse=True)
    got = out.double().cpu().numpy()
    B = got.shape[0]
    worst = 0.0
    for b in range(B):
        k = bt["n"][b]
        worst = max(worst, np.abs(got[b, :k] - ref[b, :k]).max())
    assert worst <= TOL[dtype], f"max-abs {worst:.3e} > {TOL[dtype]:.1e}"
    if lse is not None:
        L = lse.double().cpu().numpy()
        for b in range(B):
            k = bt["n"][b]
            np.testing.assert_allclose(L[b, :, :k], ref_lse[b, :, :k], atol=1e-4, rtol=0)
    return worst


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.float16, torch.bfloat16])
@pytest.mark.parametrize("H,Hkv,D", [(4, 4, 64), (2, 2, 8), (4, 2, 32), (2, 1, 128)])
def test_k1_cuda_core_matches_oracle(capi, restatement, dtype, H, Hkv, D):
    rng = np.random.default_rng(11 + H + D)
    bt = make_batch(restatement, rng, 5, H, Hkv, D, dtype=dtype)
    out, lse = run_k1(capi, bt, dtype, force_path=1, lse=True)
    check_k1(restatement, bt, out, dtype, lse)


def test_k1_edge_cases(capi, restatement):
    """Root-only trees, P = 0 (nothing committed), and an empty batch."""
    rng = np.random.default_rng(5)
    trees = [restatement.merge([[3]]), restatement.merge([[4, 1, 2]]),
             restatement.merge([[5, 1], [5, 2], [5, 3]])]
    bt = make_batch(restatement, rng, 3, 2, 2, 64, trees=trees, P_range=(0, 3))
    bt["P"][0] = 0
    out, _ = run_k1(capi, bt, torch.float64, force_path=1)
    check_k1(restatement, bt, out, torch.float64)


def test_k1_deterministic_and_non_ancestor_invariant(capi, restatement):
    """Bitwise: re-running gives identical bits, and perturbing a
    non-ancestor's K/V row never changes a node's output (reference
    transformer_test.cpp:401-423)."""
    rng = np.random.default_rng(9)
    trees = [restatement.merge([[9, 3, 5, 6], [9, 3, 7, 8]])]
    bt = make_batch(restatement, rng, 1, 2, 2, 64, trees=trees, P_range=(7, 7))
    a, _ = run_k1(capi, bt, torch.float64, force_path=1)
    b, _ = run_k1(capi, bt, torch.float64, force_path=1)
    assert torch.equal(a, b)
    # nodes 0..3 = [9,3,5,6]; nodes 4,5 = [7,8] are non-ancestors of 0..3
    P = int(bt["P"][0])
    bt["kc"][0, :, P + 4:P + 6] += 3.0
    bt["vc"][0, :, P + 4:P + 6] -= 2.0
    c, _ = run_k1(capi, bt, torch.float64, force_path=1)
    assert torch.equal(a[0, :4], c[0, :4])
    assert not torch.equal(a[0, 4:6], c[0, 4:6])


@pytest.mark.parametrize("early", [False, True])
def test_build_masks_matches_oracle(capi, restatement, early):
    rng = np.random.default_rng(3)
    trees = [restatement.merge(random_seqs(rng, 1, 20, 12, 20), 4096) for _ in range(4)]
    tok, par, dep, n = pack(trees, 150)
    W = 3
    ref = masks(restatement, par, n, W)
    got = capi.build_masks(torch.tensor(par, device="cuda"), torch.tensor(n, device="cuda"), W,
                           early=early)
    got = got.cpu().numpy().view(np.uint64)
    for b in range(4):
        np.testing.assert_array_equal(got[b, : n[b]], ref[b, : n[b]])


@pytest.mark.parametrize("dtype", [torch.float16, torch.float64])
def test_k2_append_and_compact(capi, restatement, dtype):
    rng = np.random.default_rng(21)
    B, T, Hkv, D, Lmax, layers = 3, 16, 4, 64, 96, 2
    kc = torch.tensor(rng.uniform(-1, 1, (layers, B, Hkv, Lmax, D)), device="cuda").to(dtype)
    vc = torch.tensor(rng.uniform(-1, 1, (layers, B, Hkv, Lmax, D)), device="cuda").to(dtype)
    knew = torch.tensor(rng.uniform(-1, 1, (B, T, Hkv, D)), device="cuda").to(dtype)
    vnew = torch.tensor(rng.uniform(-1, 1, (B, T, Hkv, D)), device="cuda").to(dtype)
    P = torch.tensor([5, 40, 0], dtype=torch.int32, device="cuda")
    n = torch.tensor([16, 7, 1], dtype=torch.int32, device="cuda")
    k0, v0 = kc.clone(), vc.clone()
    capi.kv_append(knew, vnew, P, n, kc[1], vc[1])
    exp_k, exp_v = k0.clone(), v0.clone()
    for b, (p, m) in enumerate(zip(P.tolist(), n.tolist())):
        exp_k[1, b, :, p:p + m] = knew[b, :m].transpose(0, 1)
        exp_v[1, b, :, p:p + m] = vnew[b, :m].transpose(0, 1)
    torch.cuda.synchronize()
    assert torch.equal(kc, exp_k) and torch.equal(vc, exp_v)

    ids = torch.tensor([[0, 2, 3, 7, 11, -1], [0, 1, 4, -1, -1, -1], [0, -1, -1, -1, -1, -1]],
                       dtype=torch.int32, device="cuda")
    keep = torch.tensor([5, 3, 1], dtype=torch.int32, device="cuda")
    newP = torch.zeros(3, dtype=torch.int32, device="cuda")
    before_k, before_v = kc.clone(), vc.clone()
    capi.kv_compact(ids, keep, P, kc, vc, newP)
    torch.cuda.synchronize()
    for b, (p, m) in enumerate(zip(P.tolist(), keep.tolist())):
        for k in range(m):
            src = ids[b, k].item()
            assert torch.equal(kc[:, b, :, p + k], before_k[:, b, :, p + src])
            assert torch.equal(vc[:, b, :, p + k], before_v[:, b, :, p + src])
        assert torch.equal(kc[:, b, :, :p], before_k[:, b, :, :p])  # committed rows untouched
    assert newP.tolist() == [P[0].item() + 5, P[1].item() + 3, P[2].item() + 1]


def _verify_case(capi, restatement, logits, tok, par, n, budget=None, eos=-1):
    dev = "cuda"
    am, ver, ids, ln = capi.verify_greedy(torch.tensor(logits, device=dev),
                                          torch.tensor(tok, device=dev),
                                          torch.tensor(par, device=dev),
                                          torch.tensor(n, device=dev),
                                          None if budget is None else torch.tensor(budget, device=dev),
                                          eos)
    am, ver, ids, ln = am.cpu().numpy(), ver.cpu().numpy(), ids.cpu().numpy(), ln.cpu().numpy()
    for b in range(len(n)):
        k = n[b]
        outs, rv, rids = restatement.greedy_verify(logits[b, :k], tok[b, :k], par[b, :k])
        np.testing.assert_array_equal(am[b, :k], outs)
        L = len(rv)
        if budget is not None:
            L = min(L, budget[b])
        if eos >= 0:
            hit = np.nonzero(rv[:L] == eos)[0]
            if hit.size:
                L = hit[0] + 1
        assert ln[b] == L
        np.testing.assert_array_equal(ver[b, :L], rv[:L])
        np.testing.assert_array_equal(ids[b, :L], rids[:L])
    # the same walk through the fused walk+commit path (the C2 step's K3):
    # bit-exact with the above, twice in a row on one workspace
    B, T = tok.shape
    kc = torch.zeros((B, 1, T + 1, 8), dtype=torch.float16, device=dev)
    ws = capi.verify_workspace(B, T, dev)
    for _ in range(2):
        am2, ver2, ids2, ln2 = capi.verify_greedy_compact(
            torch.tensor(logits, device=dev), torch.tensor(tok, device=dev),
            torch.tensor(par, device=dev), torch.tensor(n, device=dev),
            torch.zeros(B, dtype=torch.int32, device=dev), kc, kc.clone(),
            None if budget is None else torch.tensor(budget, device=dev), eos, workspace=ws)
        np.testing.assert_array_equal(ln2.cpu().numpy(), ln)
        for b in range(len(n)):
            np.testing.assert_array_equal(ver2[b, : ln[b]].cpu().numpy(), ver[b, : ln[b]])
            np.testing.assert_array_equal(ids2[b, : ln[b]].cpu().numpy(), ids[b, : ln[b]])


def test_k3_greedy_verify_matches_oracle(capi, restatement):
    rng = np.random.default_rng(77)
    V = 1003
    trees = []
    for _ in range(6):
        seqs = width_depth_seqs(rng, int(rng.integers(0, 8)), 8, 4, 6)
        trees.append(restatement.merge(seqs, 1024))
    tok, par, dep, n = pack(trees)
    B, T = tok.shape
    logits = rng.standard_normal((B, T, V)).astype(np.float32)
    # force long accepted walks: make each node's argmax its first child's token
    for b in range(B):
        for u in range(n[b]):
            kids = [v for v in range(n[b]) if par[b, v] == u]
            if kids and rng.random() < 0.8:
                logits[b, u, tok[b, kids[-1]]] = 10.0
    _verify_case(capi, restatement, logits, tok, par, n)
    _verify_case(capi, restatement, logits, tok, par, n, budget=np.array([1, 2, 3, 9, 2, 1], np.int32))
    _verify_case(capi, restatement, logits, tok, par, n, eos=int(tok[0, 1]))


def test_k3_tie_and_nan_rules(capi, restatement):
    """Lowest id wins ties; NaN never wins; NaN at index 0 is never replaced
    (argmax_token, reference transformer.cpp:116-122)."""
    tok, par, dep = restatement.merge([[0, 1], [0, 2]])
    T, V = len(tok), 4100
    logits = np.zeros((11, T, V), np.float32)
    logits[0, :, 7] = logits[0, :, 3000] = 5.0       # tie -> 7
    logits[1, :, 1] = np.nan
    logits[1, :, 2] = 1.0                            # NaN skipped -> 2
    logits[2, :, 0] = np.nan
    logits[2, :, 5] = 9.0                            # NaN at 0 -> 0
    logits[3, :, :] = -np.inf                        # all -inf -> 0
    logits[4, :, :] = np.nan                         # -inf at 0, NaN elsewhere but one
    logits[4, :, 0] = -np.inf
    logits[4, :, 3999] = -5.0                        # -> 3999 (last slice)
    logits[5, :, [2050, 2051, 4099]] = 2.0           # tie inside one float4 -> 2050
    logits[6, :, :] = -np.inf
    logits[6, :, 4000] = np.nan                      # -> 0
    logits[7] = np.random.default_rng(3).standard_normal((T, V)).astype(np.float32)
    # +0.0 and -0.0 compare equal under the reference's '>': the lower id wins
    logits[8, :, :] = -1.0
    logits[8, :, 5] = -0.0                           # -0 low (slice 0), +0 high (slice 6)
    logits[8, :, 3000] = 0.0                         # -> 5
    logits[9, :, :] = -1.0
    logits[9, :, 1030] = 0.0                         # +0 low, -0 high, other slices
    logits[9, :, 4000] = -0.0                        # -> 1030
    logits[10, :, :] = -1.0
    logits[10, :, 2049] = -0.0                       # same thread / same float4
    logits[10, :, 2050] = 0.0                        # -> 2049
    for b in (8, 9, 10):
        assert restatement.argmax(logits[b, 0]) == {8: 5, 9: 1030, 10: 2049}[b]
    tok4, par4, _, n4 = pack([(tok, par, dep)] * 11)
    _verify_case(capi, restatement, logits, tok4, par4, n4)
    # V % 4 == 0 (the vectorised argmax), ragged trees with dead rows (n < T)
    # and the slice boundaries of V = 4096
    lg2 = np.full((11, T, 4096), -1.0, np.float32)
    lg2[:, :, :4096] = logits[:, :, :4096]
    lg2[4, :, 3999] = -5.0
    n5 = n4.copy()
    n5[1] = 1
    _verify_case(capi, restatement, lg2, tok4, par4, n5)


def test_library_fails_loudly_without_device_path(capi):
    """Argument validation surfaces as SpectreeError with the Errc name."""
    with pytest.raises(capi.SpectreeError) as e:
        capi.build_masks(torch.zeros((1, 100), dtype=torch.int32, device="cuda"),
                         torch.ones(1, dtype=torch.int32, device="cuda"), W=1)
    assert e.value.code == "shape_mismatch"


def test_heads_gather_layout(capi):
    """C4: [world,B,T,Hl,D] -> [B,T,world*Hl,D] equals a torch permute."""
    g = torch.randn(4, 3, 7, 8, 128, device="cuda").half()
    out = capi.heads_gather_layout(g, 4)
    torch.cuda.synchronize()
    ref = g.permute(1, 2, 0, 3, 4).reshape(3, 7, 32, 128)
    assert torch.equal(out, ref)


def test_tree_prepare_matches_append_and_masks(capi, restatement):
    """st_tree_prepare (one launch) == st_kv_append + st_build_masks, bitwise."""
    rng = np.random.default_rng(5)
    trees = [restatement.merge(random_seqs(rng, 1, 20, 12, 20), 4096) for _ in range(3)]
    tok, par, dep, n = pack(trees, 150)
    B, T, Hkv, D, Lmax = 3, 150, 4, 128, 600
    dev = "cuda"
    kc = torch.randn(B, Hkv, Lmax, D, device=dev).half()
    vc = torch.randn(B, Hkv, Lmax, D, device=dev).half()
    knew = torch.randn(B, T, Hkv, D, device=dev).half()
    vnew = torch.randn(B, T, Hkv, D, device=dev).half()
    P = torch.tensor([5, 300, 0], dtype=torch.int32, device=dev)
    nd, pd = torch.tensor(n, device=dev), torch.tensor(par, device=dev)
    k1, v1 = kc.clone(), vc.clone()
    capi.kv_append(knew, vnew, P, nd, k1, v1)
    m1 = capi.build_masks(pd, nd, 3)
    k2, v2 = kc.clone(), vc.clone()
    m2 = capi.tree_prepare(knew, vnew, P, nd, k2, v2, pd, W=3)
    torch.cuda.synchronize()
    assert torch.equal(k1, k2) and torch.equal(v1, v2)
    for b in range(B):
        assert torch.equal(m1[b, : n[b]], m2[b, : n[b]])


@pytest.mark.parametrize("layers,Hkv", [(1, 32), (2, 6)])
def test_verify_greedy_compact_matches_separate(capi, restatement, layers, Hkv):
    """st_verify_greedy_compact (walk fused into the compaction) == st_verify_greedy
    followed by st_kv_compact(ids, len): outputs, argmax, caches and new prefix
    lengths bitwise; long accepted paths exercise the chunked in-place move."""
    rng = np.random.default_rng(9 + layers)
    V, D, Lmax = 777, 128, 256
    trees = []
    for i in range(5):
        seqs = width_depth_seqs(rng, int(rng.integers(0, 8)), 8, 2 if i else 1, 30 if i < 3 else 6)
        trees.append(restatement.merge(seqs, 1024))
    tok, par, dep, n = pack(trees)
    B, T = tok.shape
    logits = rng.standard_normal((B, T, V)).astype(np.float32)
    for b in range(B):
        for u in range(n[b]):
            kids = [v for v in range(n[b]) if par[b, v] == u]
            if kids and (b == 0 or rng.random() < 0.95):
                logits[b, u, tok[b, kids[0]]] = 10.0
    dev = "cuda"
    lg, tk, pr, nd = (torch.tensor(x, device=dev) for x in (logits, tok, par, n))
    P = torch.tensor(rng.integers(0, 100, B), dtype=torch.int32, device=dev)
    kc = torch.randn(layers, B, Hkv, Lmax, D, device=dev).half()
    vc = torch.randn(layers, B, Hkv, Lmax, D, device=dev).half()
    for budget, eos in [(None, -1), (np.array([3, 40, 1, 2, 9], np.int32), -1), (None, int(tok[1, 2]))]:
        bud = None if budget is None else torch.tensor(budget[:B], device=dev)
        k1, v1, k2, v2 = kc.clone(), vc.clone(), kc.clone(), vc.clone()
        a1, ver1, ids1, ln1 = capi.verify_greedy(lg, tk, pr, nd, bud, eos)
        np1 = torch.zeros(B, dtype=torch.int32, device=dev)
        capi.kv_compact(ids1, ln1, P, k1, v1, np1)
        np2 = torch.zeros(B, dtype=torch.int32, device=dev)
        a2, ver2, ids2, ln2 = capi.verify_greedy_compact(lg, tk, pr, nd, P, k2, v2, bud, eos,
                                                         new_prefix_len=np2)
        torch.cuda.synchronize()
        assert torch.equal(ln1, ln2)
        for b in range(B):   # argmax rows are defined for live nodes only
            assert torch.equal(a1[b, : n[b]], a2[b, : n[b]])
        assert torch.equal(ver1, ver2) and torch.equal(ids1, ids2)
        assert torch.equal(np1, np2)
        assert torch.equal(k1, k2) and torch.equal(v1, v2)
        if budget is None and eos < 0:
            assert int(ln1.max()) > 20  # several row chunks moved
