"""Parity of the BENCHMARKED steps at their full shapes.

* C2 (bench.py's default step, class ``bench.VerifyStep``: B=8, T=64, L=2048,
  H=32, D=128, V=32000, fp16): masks -> K1 (tree rows from ``k_tree``,
  ``early_kv``) -> K3 argmax -> walk + K2 commit from ``k_tree``, run through
  the same CUDA-graph runner the bench times. Checked: K1 outputs of ALL 256
  (request, head) pairs within 2e-3 max-abs of the f64 restatement; accepted
  tokens, node ids and lengths bit-exact vs the restatement's greedy verify
  (reference argmax_token + verify); committed cache rows [P, P+len) equal to
  the accepted tree rows, rows [0, P) untouched. Also the reference cache
  discipline (``--tree-rows cache``: K2 append, in-place compaction).
* C5 corners (B=16, L=32768, T=16 and T=128, the M=128 "dual" path) and the
  GQA sweep shape (H=64, Hkv=8, B=16, L=16384, T=8/16): K1 on every request,
  checked on one (request, head) pair per request against the C restatement
  (each pair is a B=1, H=1 oracle problem; pairs run on a thread pool — the
  oracle is C behind ctypes, which releases the GIL).
* C4 (bench.py --config c4: 65B shape, B=8, merged 3-SSM trees of 61 nodes,
  KV 2048) on one rank of 1 or of 8 head shards — the latter is the per-rank
  slice on the two-piece DSMEM merge: every pair's K1 output, the head-output
  layout and the greedy verify at V=32000.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from tests.treegen import masks, pack, width_depth_seqs

pytestmark = pytest.mark.gpu

TOL16 = 2e-3


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    return _capi


def _pool():
    import os
    return ThreadPoolExecutor(max_workers=max(2, min(16, os.cpu_count() or 2)))


def oracle_pairs(R, q, kc, vc, mask, P, n, pairs, kt=None, vt=None):
    """f64 restatement of K1 for selected (request, query head) pairs.
    q [B,T,H,D], caches [B,Hkv,Lmax,D], tree rows from kt/vt [B,T,Hkv,D] when
    given (k_tree mode) else from cache rows [P, P+n). Returns {pair: [n,D]}."""
    B, T, H, D = q.shape
    Hkv = kc.shape[1]
    G = H // Hkv
    W = mask.shape[-1]

    def one(pair):
        b, h = pair
        hk = h // G
        Pb, nb = int(P[b]), int(n[b])
        qq = q[b, :, h].double().cpu().numpy().reshape(1, T, 1, D)
        if kt is not None:   # committed rows, then the tree's own rows
            kk = torch.cat([kc[b, hk, :Pb], kt[b, :nb, hk]]).double().cpu().numpy()
            vv = torch.cat([vc[b, hk, :Pb], vt[b, :nb, hk]]).double().cpu().numpy()
        else:
            kk = kc[b, hk, : Pb + nb].double().cpu().numpy()
            vv = vc[b, hk, : Pb + nb].double().cpu().numpy()
        o = R.tree_attention(qq, kk[None, None].copy(), vv[None, None].copy(),
                             np.ascontiguousarray(mask[b:b + 1]), np.array([Pb], np.int32),
                             np.array([nb], np.int32), D ** -0.5)
        return pair, o[0, :nb, 0]

    with _pool() as ex:
        return dict(ex.map(one, pairs))


def worst_err(out, ref):
    return max(np.abs(out[b, : r.shape[0], h].double().cpu().numpy() - r).max()
               for (b, h), r in ref.items())


@pytest.mark.parametrize("tree_rows,native", [("own", True), ("own", False), ("cache", True)])
def test_c2_bench_step_full_shape(capi, restatement, tree_rows, native):
    """native: the step as st_verify_plan_run (what bench.py times); else one
    CUDA-graph replay of the Python-issued launches."""
    import bench
    dev = torch.device("cuda", 0)
    st = bench.VerifyStep(dev, 0, tree_rows=tree_rows)
    assert st.path == 2, "C2 must take the tcgen05 K1 path"
    kc0, vc0 = st.kc.clone(), st.vc.clone()
    runner = bench.DPRunner(st, 1, dev, native=native)
    runner.capture(0)
    # capture() ran the step eagerly 3x: restore the cache, then ONE graph replay
    st.kc.copy_(kc0)
    st.vc.copy_(vc0)
    st.out.zero_()
    for t in st.vout:
        t.fill_(-7)
    runner.step()
    runner.sync()
    torch.cuda.synchronize()

    B, T, H = st.B, st.T, st.H
    par, n = st.batch.parents, st.batch.n_nodes
    m = masks(restatement, par, n, st.W)
    assert torch.equal(st.mask.cpu(), torch.tensor(m.view(np.int64))), "device masks"
    # K1: all 256 (request, head) pairs
    pairs = [(b, h) for b in range(B) for h in range(H)]
    P = st.P.cpu().numpy()
    if tree_rows == "own":
        ref = oracle_pairs(restatement, st.q, kc0, vc0, m, P, n, pairs, st.knew, st.vnew)
    else:   # the append wrote the tree rows into cache rows [P, P+n) before K1
        kca, vca = kc0.clone(), vc0.clone()
        for b in range(B):
            kca[b, :, st.L: st.L + n[b]] = st.knew[b, : n[b]].transpose(0, 1)
            vca[b, :, st.L: st.L + n[b]] = st.vnew[b, : n[b]].transpose(0, 1)
        ref = oracle_pairs(restatement, st.q, kca, vca, m, P, n, pairs)
    err = worst_err(st.out, ref)
    assert err <= TOL16, f"K1 max-abs {err:.3e} over 256 pairs"
    # K3: accepted tokens / ids / lengths, bit-exact
    lg = st.logits.cpu().numpy()
    ver, ids, ln = (x.cpu().numpy() for x in st.vout)
    total = 0
    for b in range(B):
        _, rv, rids = restatement.greedy_verify(lg[b, : n[b]], st.batch.tokens[b, : n[b]],
                                                par[b, : n[b]])
        assert ln[b] == len(rv), b
        np.testing.assert_array_equal(ver[b, : ln[b]], rv)
        np.testing.assert_array_equal(ids[b, : ln[b]], rids)
        total += len(rv)
    assert total > B, "planted acceptance should accept beyond the bonus token"
    # K2: committed rows [P, P+len) = the accepted tree rows; [0, P) untouched
    for b in range(B):
        Pb, k = int(P[b]), int(ln[b])
        rows = torch.tensor(ids[b, :k], device=dev, dtype=torch.long)
        want_k = st.knew[b].index_select(0, rows).transpose(0, 1)
        want_v = st.vnew[b].index_select(0, rows).transpose(0, 1)
        assert torch.equal(st.kc[b, :, Pb: Pb + k], want_k), b
        assert torch.equal(st.vc[b, :, Pb: Pb + k], want_v), b
        assert torch.equal(st.kc[b, :, :Pb], kc0[b, :, :Pb])
        assert torch.equal(st.vc[b, :, :Pb], vc0[b, :, :Pb])
    # the bench's own self-check agrees
    assert st.oracle_check()["greedy_vs_oracle"] == "bit-exact"


def _trees(R, rng, B, T, width, vocab=32000):
    depth = -(-(T - 1) // width)
    out = []
    for _ in range(B):
        while True:
            t = R.merge(width_depth_seqs(rng, int(rng.integers(0, vocab)), vocab, width, depth),
                        1 << 20)
            if len(t[0]) > T:   # trim: keep the first T preorder nodes (a valid subtree)
                t = tuple(a[:T] for a in t)
            out.append(t)
            break
    return out


def _k1_sampled(capi, R, B, T, L, H, Hkv, width, seed, dtype=torch.float16):
    rng = np.random.default_rng(seed)
    trees = _trees(R, rng, B, T, width)
    tok, par, dep, n = pack(trees, T)
    W = (T + 63) // 64
    m = masks(R, par, n, W)
    dev = "cuda"
    Lmax = L + T
    q = torch.empty(B, T, H, 128, dtype=dtype, device=dev).uniform_(-1, 1)
    kc = torch.empty(B, Hkv, Lmax, 128, dtype=dtype, device=dev).uniform_(-1, 1)
    vc = torch.empty(B, Hkv, Lmax, 128, dtype=dtype, device=dev).uniform_(-1, 1)
    kt = torch.empty(B, T, Hkv, 128, dtype=dtype, device=dev).uniform_(-1, 1)
    vt = torch.empty(B, T, Hkv, 128, dtype=dtype, device=dev).uniform_(-1, 1)
    P = np.full(B, L, np.int32)
    P[1] = L - 77       # ragged: a prefix ending mid-tile
    Pd, nd = torch.tensor(P, device=dev), torch.tensor(n, device=dev)
    mask = torch.tensor(m.view(np.int64), device=dev)
    assert capi.tree_attention_path(q, kc, vc, mask, Pd, nd) == 2
    out = capi.tree_attention(q, kc, vc, mask, Pd, nd, k_tree=kt, v_tree=vt)
    torch.cuda.synchronize()
    pairs = [(b, int(rng.integers(0, H))) for b in range(B)]
    pairs[0] = (0, 0)
    pairs[-1] = (B - 1, H - 1)
    ref = oracle_pairs(R, q, kc, vc, m, P, n, pairs, kt, vt)
    return worst_err(out, ref)


@pytest.mark.parametrize("T,width", [(16, 4), (128, 16)])
def test_c5_corner_32k(capi, restatement, T, width):
    """C5 corner: B=16, KV 32768 rows, T=16 (M=64) and T=128 (M=128 dual)."""
    err = _k1_sampled(capi, restatement, 16, T, 32768, 32, 32, width, seed=T)
    assert err <= TOL16, f"max-abs {err:.3e}"


@pytest.mark.parametrize("T", [8, 16])
def test_gqa_sweep_shape(capi, restatement, T):
    """GQA sweep shape (LLaMA-3-70B attention: H=64, Hkv=8, B=16, KV 16384):
    the group's 8 x T query rows share each KV tile."""
    err = _k1_sampled(capi, restatement, 16, T, 16384, 64, 8, 2 if T == 8 else 4, seed=100 + T)
    assert err <= TOL16, f"max-abs {err:.3e}"


def test_decode_loop_prefix_advances_early_kv(capi, restatement):
    """A real decode loop: each step's commit writes rows [P_i, P_i + len_i)
    and sets P_{i+1} on the device; the next step's masks (early) -> K1
    (early_kv) must see those rows. Four steps are launched back to back with
    no host sync (the exact PDL chain commit -> masks -> K1 of the bench),
    then every step's K1 output and acceptance is checked against the oracle
    replayed on the host."""
    import bench
    dev = torch.device("cuda", 0)
    st = bench.VerifyStep(dev, 3)
    kc0, vc0 = st.kc.clone(), st.vc.clone()
    steps = 4
    Ps = [st.P.clone()] + [torch.zeros_like(st.P) for _ in range(steps)]
    outs = [torch.zeros_like(st.out) for _ in range(steps)]
    vouts = [tuple(torch.zeros_like(t) for t in st.vout) for _ in range(steps)]
    a = st.resident
    torch.cuda.synchronize()
    for i in range(steps):
        capi.build_masks(st.par, st.nn, W=st.W, out=st.mask, early=True)
        capi.tree_attention(st.q, st.kc, st.vc, st.mask, Ps[i], st.nn, out=outs[i],
                            workspace=st.ws_attn, k_tree=st.knew, v_tree=st.vnew, early_kv=True)
        capi.verify_greedy_compact(st.logits, st.tok, st.par, st.nn, Ps[i], st.kc, st.vc,
                                   workspace=st.ws_ver, want_argmax=False, out=vouts[i],
                                   new_prefix_len=Ps[i + 1], k_tree=st.knew, v_tree=st.vnew)
    torch.cuda.synchronize()
    del a
    par, n = st.batch.parents, st.batch.n_nodes
    m = masks(restatement, par, n, st.W)
    kc, vc = kc0.clone(), vc0.clone()
    lg = st.logits.cpu().numpy()
    for i in range(steps):
        P = Ps[i].cpu().numpy()
        pairs = [(b, (7 * b + i) % st.H) for b in range(st.B)]
        ref = oracle_pairs(restatement, st.q, kc, vc, m, P, n, pairs, st.knew, st.vnew)
        err = worst_err(outs[i], ref)
        assert err <= TOL16, f"step {i}: K1 max-abs {err:.3e}"
        ver, ids, ln = (x.cpu().numpy() for x in vouts[i])
        for b in range(st.B):
            _, rv, rids = restatement.greedy_verify(lg[b, : n[b]], st.batch.tokens[b, : n[b]],
                                                    par[b, : n[b]])
            assert ln[b] == len(rv)
            np.testing.assert_array_equal(ids[b, : ln[b]], rids)
            assert int(Ps[i + 1][b]) == P[b] + ln[b]
            rows = torch.tensor(ids[b, : ln[b]], device=dev, dtype=torch.long)
            kc[b, :, P[b]: P[b] + ln[b]] = st.knew[b].index_select(0, rows).transpose(0, 1)
            vc[b, :, P[b]: P[b] + ln[b]] = st.vnew[b].index_select(0, rows).transpose(0, 1)
    for b in range(st.B):
        Pe = int(Ps[steps][b])
        assert torch.equal(st.kc[b, :, :Pe], kc[b, :, :Pe])
        assert torch.equal(st.vc[b, :, :Pe], vc[b, :, :Pe])


@pytest.mark.parametrize("world", [1, 8])
def test_c4_bench_step_full_shape(capi, restatement, world):
    """C4 as bench.py --config c4 builds it (65B shape: 64 heads, B=8, merged
    3-SSM trees <1,1,3,1,1,1,1,1> of 61 nodes, KV 2048, tree rows in their own
    tensors) for rank 0 of `world` head shards: world=1 runs all 64 heads,
    world=8 rank 0's 8 — the per-rank slice tools/c4_slice.py times, whose 64
    pairs take the two-piece DSMEM merge. K1 on every (request, head) pair
    within 2e-3 of the f64 restatement; the head-output layout of the
    (1-rank) gather; greedy verify at V=32000 bit-exact."""
    import bench
    from paper_2305_09781_b200.dist import gather_head_outputs, head_shard
    from paper_2305_09781_b200.tree import TokenTree, TreeBatch
    dev = torch.device("cuda", 0)
    HT, Bq, D, L, V = 64, 8, 128, 2048, 32000
    h0, h1 = head_shard(HT, world, 0)
    Hl = h1 - h0
    trees = bench.c4_trees(lambda s: TokenTree.merge_sequences(s, 1 << 20), 65, Bq)
    tb = TreeBatch([t for t, _ in trees])
    T = tb.T
    assert T == 61
    g = torch.Generator(device=dev).manual_seed(99)
    q = (torch.rand(Bq, T, Hl, D, device=dev, generator=g) * 2 - 1).half()
    kc = (torch.rand(Bq, Hl, L + T, D, device=dev, generator=g) * 2 - 1).half()
    vc = (torch.rand(Bq, Hl, L + T, D, device=dev, generator=g) * 2 - 1).half()
    kt = (torch.rand(Bq, T, Hl, D, device=dev, generator=g) * 2 - 1).half()
    vt = (torch.rand(Bq, T, Hl, D, device=dev, generator=g) * 2 - 1).half()
    logits = torch.randn(Bq, T, V, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    par = torch.tensor(tb.parents, device=dev)
    tok = torch.tensor(tb.tokens, device=dev)
    nn = torch.tensor(tb.n_nodes, device=dev)
    P = torch.full((Bq,), L, dtype=torch.int32, device=dev)
    mask = capi.build_masks(par, nn)
    out = torch.zeros_like(q)
    ws = capi.tree_attention_workspace(q, kc, vc, mask, P, nn)
    capi.tree_attention(q, kc, vc, mask, P, nn, out=out, workspace=ws, k_tree=kt, v_tree=vt)
    full = gather_head_outputs(out, 1)
    am, ver, ids, ln = capi.verify_greedy(logits, tok, par, nn)
    torch.cuda.synchronize()
    n = np.array(tb.n_nodes)
    m = masks(restatement, np.array(tb.parents), n, (T + 63) // 64)
    pairs = [(b, h) for b in range(Bq) for h in range(Hl)]
    ref = oracle_pairs(restatement, q, kc, vc, m, P.cpu().numpy(), n, pairs, kt, vt)
    err = worst_err(out, ref)
    assert err <= TOL16, f"K1 max-abs {err:.3e} over {len(pairs)} pairs"
    assert torch.equal(full, out), "1-rank gather layout"
    lg = logits.cpu().numpy()
    for b in range(Bq):
        k = int(n[b])
        _, rv, rids = restatement.greedy_verify(lg[b, :k], np.array(tb.tokens)[b, :k],
                                                np.array(tb.parents)[b, :k])
        assert int(ln[b]) == len(rv)
        assert ver[b, : len(rv)].cpu().tolist() == list(rv)
        assert ids[b, : len(rv)].cpu().tolist() == list(rids)
