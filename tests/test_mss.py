"""K4 — multi-step speculative sampling (MSS).

Parity note: the reference has NO stochastic verification,
so parity is unpinned against the reference. The pin is the fp32 CPU oracle
oracle/restate_mss.c (contract: DESIGN.md §5); K4 must match it bit-exactly
given the same host-supplied uniforms. The CPU tests below check the oracle's
own invariants (greedy limit, distribution sanity); the gpu tests check K4
against it.
"""
import numpy as np
import pytest

from tests.treegen import pack, width_depth_seqs


def softmax(x):
    e = np.exp(x - x.max(-1, keepdims=True))
    return (e / e.sum(-1, keepdims=True)).astype(np.float32)


def make_case(restatement, rng, V, width=3, depth=4, n_req=1, peaked=3.0):
    trees = [restatement.merge(width_depth_seqs(rng, int(rng.integers(0, V)), V, width, depth), 1024)
             for _ in range(n_req)]
    tok, par, dep, n = pack(trees)
    Bq, T = tok.shape
    logits = (rng.standard_normal((Bq, T, V)) * peaked).astype(np.float32)
    q = softmax(rng.standard_normal((Bq, T, V)).astype(np.float32) * peaked)
    # make drafts plausible: the proposing SSM favours its own token, and the
    # LLM agrees with the first child half of the time
    for b in range(Bq):
        for v in range(1, n[b]):
            q[b, v] *= 0.3
            q[b, v, tok[b, v]] += 0.7
            if rng.random() < 0.5:
                logits[b, par[b, v], tok[b, v]] += 6.0 * peaked
    return tok, par, n, logits, q


def test_oracle_greedy_limit(restatement):
    """One-hot drafts and near-one-hot targets: MSS == greedy walk (Appendix B)."""
    rng = np.random.default_rng(3)
    V = 300
    for _ in range(20):
        tok, par, n, logits, _ = make_case(restatement, rng, V)
        t, p_, k = tok[0], par[0], n[0]
        lg = logits[0, :k] * 50.0  # peaked: softmax is one-hot in fp32
        q = np.zeros((k, V), np.float32)
        q[np.arange(k), t[:k]] = 1.0
        U = rng.uniform(0.01, 0.99, k + 1).astype(np.float32)
        ver, ids = restatement.mss_verify(lg, q, t[:k], p_[:k], 1.0, U)
        _, gver, gids = restatement.greedy_verify(lg, t[:k], p_[:k])
        assert ver.tolist() == gver.tolist()
        assert ids.tolist() == gids.tolist()


def test_oracle_outputs_are_a_tree_walk(restatement):
    rng = np.random.default_rng(5)
    V = 257
    for _ in range(30):
        tok, par, n, logits, q = make_case(restatement, rng, V)
        k = n[0]
        U = rng.uniform(0, 1, k + 1).astype(np.float32)
        ver, ids = restatement.mss_verify(logits[0, :k], q[0, :k], tok[0, :k], par[0, :k],
                                          float(rng.choice([0.5, 1.0, 2.0])), U)
        assert ids[0] == 0 and len(ids) == len(ver)
        for j in range(1, len(ids)):
            assert par[0, ids[j]] == ids[j - 1] and tok[0, ids[j]] == ver[j - 1]
        assert 0 <= ver[-1] < V


@pytest.mark.gpu
@pytest.mark.parametrize("V,tau", [(1000, 1.0), (32000, 0.7), (4099, 2.0), (1, 1.0)])
def test_k4_bitexact_vs_oracle(restatement, V, tau):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    rng = np.random.default_rng(V)
    if V == 1:
        tok, par, n = pack([restatement.merge([[0, 0, 0]])])[0::2][0], None, None
        tok, par, dep, n = pack([restatement.merge([[0, 0, 0]])])
        logits = np.zeros((1, 3, 1), np.float32)
        q = np.ones((1, 3, 1), np.float32)
    else:
        tok, par, n, logits, q = make_case(restatement, rng, V, width=4, depth=5, n_req=6)
    Bq, T = tok.shape
    U = rng.uniform(0, 1, (Bq, T + 1)).astype(np.float32)
    dev = "cuda"
    ver, ids, ln = _capi.verify_mss(torch.tensor(logits, device=dev), torch.tensor(q, device=dev),
                                    torch.tensor(tok, device=dev), torch.tensor(par, device=dev),
                                    torch.tensor(n, device=dev), tau, torch.tensor(U, device=dev))
    ver, ids, ln = ver.cpu().numpy(), ids.cpu().numpy(), ln.cpu().numpy()
    accepted = 0
    for b in range(Bq):
        k = n[b]
        rv, rids = restatement.mss_verify(logits[b, :k], q[b, :k], tok[b, :k], par[b, :k], tau,
                                          U[b])
        assert ln[b] == len(rv)
        np.testing.assert_array_equal(ver[b, : ln[b]], rv)
        np.testing.assert_array_equal(ids[b, : ln[b]], rids)
        accepted += len(rv) - 1
    if V > 1:
        assert accepted > 0  # the planted agreement must produce some acceptances


@pytest.mark.gpu
def test_k4_c3_bench_shape(restatement):
    """K4 exactly as bench.py --config c3 runs it — 32 requests x 64-node trees
    built like the bench's (bench.c2_trees), V = 32000, tau = 1.0, drafts
    softmax(3 z) — bit-exact against the oracle for every request, with
    planted agreement so acceptance chains (and rejections with residual
    resampling) both occur."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    from paper_2305_09781_b200 import _capi
    from paper_2305_09781_b200.tree import TokenTree, TreeBatch
    V, Bq, T, tau = 32000, 32, 64, 1.0
    rng = np.random.default_rng(3000)
    trees = bench.c2_trees(lambda s_: TokenTree.merge_sequences(s_, 1 << 20), 3000, V, n_req=Bq)
    tb = TreeBatch([t for t, _ in trees], T)
    tok, par, n = np.array(tb.tokens), np.array(tb.parents), np.array(tb.n_nodes)
    logits = (rng.standard_normal((Bq, T, V)) * 3.0).astype(np.float32)
    q = softmax(rng.standard_normal((Bq, T, V)).astype(np.float32) * 3.0)
    for b in range(Bq):
        for v in range(1, n[b]):
            q[b, v] *= 0.3
            q[b, v, tok[b, v]] += 0.7
            if rng.random() < 0.5:
                logits[b, par[b, v], tok[b, v]] += 18.0
    U = rng.uniform(0, 1, (Bq, T + 1)).astype(np.float32)
    dev = "cuda"
    ver, ids, ln = _capi.verify_mss(torch.tensor(logits, device=dev), torch.tensor(q, device=dev),
                                    torch.tensor(tok, device=dev), torch.tensor(par, device=dev),
                                    torch.tensor(n, device=dev), tau, torch.tensor(U, device=dev))
    ver, ids, ln = ver.cpu().numpy(), ids.cpu().numpy(), ln.cpu().numpy()
    longest = 0
    for b in range(Bq):
        k = n[b]
        rv, rids = restatement.mss_verify(logits[b, :k], q[b, :k], tok[b, :k], par[b, :k], tau, U[b])
        assert ln[b] == len(rv)
        np.testing.assert_array_equal(ver[b, : ln[b]], rv)
        np.testing.assert_array_equal(ids[b, : ln[b]], rids)
        longest = max(longest, len(rv))
    assert longest > 2


@pytest.mark.gpu
@pytest.mark.parametrize("V,width", [(32000, 40), (4099, 36), (2048, 70)])
def test_k4_wide_nodes(restatement, V, width):
    """Nodes with more children than K4 prefetches test scalars for (32): the
    later children's scalars are loaded at test time; long rejection chains
    (drafts that the target mostly disagrees with) end in the residual
    sample. Both the float4 (V % 4 == 0) and the scalar slice paths."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    rng = np.random.default_rng(width)
    trees = []
    for _ in range(4):
        root = int(rng.integers(0, V))
        toks = rng.choice(V, size=width, replace=False)
        seqs = [[root, int(t), int(rng.integers(0, V))] for t in toks]
        trees.append(restatement.merge(seqs, 1024))
    tok, par, dep, n = pack(trees)
    Bq, T = tok.shape
    logits = (rng.standard_normal((Bq, T, V)) * 2.0).astype(np.float32)
    q = softmax(rng.standard_normal((Bq, T, V)).astype(np.float32) * 2.0)
    for b in range(Bq):
        for v in range(1, n[b]):
            q[b, v] *= 0.2
            q[b, v, tok[b, v]] += 0.8
    U = rng.uniform(0, 1, (Bq, T + 1)).astype(np.float32)
    dev = "cuda"
    ver, ids, ln = _capi.verify_mss(torch.tensor(logits, device=dev), torch.tensor(q, device=dev),
                                    torch.tensor(tok, device=dev), torch.tensor(par, device=dev),
                                    torch.tensor(n, device=dev), 1.0, torch.tensor(U, device=dev))
    ver, ids, ln = ver.cpu().numpy(), ids.cpu().numpy(), ln.cpu().numpy()
    for b in range(Bq):
        k = n[b]
        rv, rids = restatement.mss_verify(logits[b, :k], q[b, :k], tok[b, :k], par[b, :k], 1.0, U[b])
        assert ln[b] == len(rv)
        np.testing.assert_array_equal(ver[b, : ln[b]], rv)
        np.testing.assert_array_equal(ids[b, : ln[b]], rids)
