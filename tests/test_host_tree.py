"""The product's host C++ TokenTree (csrc/host/token_tree.cpp via st_tree_merge)
against the reference-generated golden fixtures. CPU only."""
import numpy as np
import pytest

from tests.test_oracle_golden import KAT_NAMES, _seqs


@pytest.fixture(scope="module")
def TT():
    from paper_2305_09781_b200.tree import TokenTree
    return TokenTree


@pytest.mark.parametrize("name", KAT_NAMES)
def test_merge_kats(TT, golden, name):
    g = golden("tree_kats.npz")
    t = TT.merge_sequences(_seqs(g[f"{name}_flat"], g[f"{name}_lens"]))
    np.testing.assert_array_equal(t.tokens, g[f"{name}_tok"])
    np.testing.assert_array_equal(t.parents, g[f"{name}_par"])
    np.testing.assert_array_equal(t.depths, g[f"{name}_dep"])
    chains = t.dfs_chains()
    np.testing.assert_array_equal(np.array([i for c in chains for i in c], np.int32),
                                  g[f"{name}_chain_ids"])
    np.testing.assert_array_equal(np.array([len(c) for c in chains], np.int32),
                                  g[f"{name}_chain_lens"])


def test_random_merges(TT, golden):
    g = golden("tree_random.npz")
    fa = la = na = 0
    for c in range(len(g["nseq"])):
        k = int(g["nseq"][c])
        lens = g["lens"][la: la + k]
        flat = g["flat"][fa: fa + int(lens.sum())]
        n = int(g["n_nodes"][c])
        t = TT.merge_sequences(_seqs(flat, lens), 1024)
        np.testing.assert_array_equal(t.tokens, g["tok"][na: na + n])
        np.testing.assert_array_equal(t.parents, g["par"][na: na + n])
        np.testing.assert_array_equal(t.depths, g["dep"][na: na + n])
        fa += int(lens.sum()); la += k; na += n


def test_errors_match_reference_codes(TT):
    from paper_2305_09781_b200 import SpectreeError
    for seqs, mx, code in [([[1, 2], [3, 4]], 64, "root_mismatch"),
                           ([[1, 2, 3, 4, 5]], 3, "tree_too_large"),
                           ([[1, 2], []], 64, "empty_input"),
                           ([], 64, "empty_input")]:
        with pytest.raises(SpectreeError) as e:
            TT.merge_sequences(seqs, mx)
        assert e.value.code == code
    # root-only trees never exceed any cap (reference token_tree.cpp:64 checks on insert)
    assert TT.merge_sequences([[5]], 0).size == 1


def test_merge_is_order_insensitive_and_idempotent(TT):
    """speculator_test.cpp:265-272 (order) and token_tree_test.cpp:99-122 (idempotence)."""
    rng = np.random.default_rng(8)
    for _ in range(50):
        root = int(rng.integers(0, 5))
        seqs = [[root] + rng.integers(0, 5, int(rng.integers(0, 5))).tolist() for _ in range(6)]
        a = TT.merge_sequences(seqs, 1024)
        b = TT.merge_sequences(seqs[::-1], 1024)
        np.testing.assert_array_equal(a.tokens, b.tokens)
        np.testing.assert_array_equal(a.parents, b.parents)
        paths = [a.ancestors(u) for u in range(a.size)]
        c = TT.merge_sequences(paths, 1024)
        np.testing.assert_array_equal(a.tokens, c.tokens)
        np.testing.assert_array_equal(a.parents, c.parents)


def test_ancestor_masks(TT, restatement):
    t = TT.merge_sequences([[2, 3, 4, 5], [2, 3, 6, 7], [2, 3, 8, 9, 1]])
    np.testing.assert_array_equal(t.ancestor_masks(), restatement.ancestor_masks(t.parents))


def _golden_batches(g):
    """The reference-generated random merges, grouped into batches of 8 requests."""
    out, fa, la, na = [], 0, 0, 0
    for c in range(len(g["nseq"])):
        k = int(g["nseq"][c])
        lens = g["lens"][la: la + k]
        flat = g["flat"][fa: fa + int(lens.sum())]
        n = int(g["n_nodes"][c])
        out.append((_seqs(flat, lens), g["tok"][na: na + n], g["par"][na: na + n],
                    g["dep"][na: na + n]))
        fa += int(lens.sum()); la += k; na += n
    return [out[i: i + 8] for i in range(0, len(out), 8)]


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_merge_batch_matches_reference(golden, threads):
    """st_tree_merge_batch (host thread pool, packed [B][T]) equals the
    reference's merge_sequences request by request; padding rows are
    (token 0, parent -1, depth 0)."""
    from paper_2305_09781_b200.tree import merge_batch
    for batch in _golden_batches(golden("tree_random.npz")):
        T = max(len(t) for _, t, _, _ in batch) + 3
        tok, par, dep, n, st = merge_batch([s for s, *_ in batch], T, 1024, n_threads=threads)
        assert (st == 0).all()
        for b, (_, rt, rp, rd) in enumerate(batch):
            k = len(rt)
            assert n[b] == k
            np.testing.assert_array_equal(tok[b, :k], rt)
            np.testing.assert_array_equal(par[b, :k], rp)
            np.testing.assert_array_equal(dep[b, :k], rd)
            assert (tok[b, k:] == 0).all() and (par[b, k:] == -1).all() and (dep[b, k:] == 0).all()


def test_merge_batch_per_request_errors():
    """A failing request reports its own reference error code and gets
    n_nodes = 0; the other requests of the batch are still merged."""
    from paper_2305_09781_b200 import SpectreeError
    from paper_2305_09781_b200.tree import TokenTree, merge_batch
    reqs = [[[1, 2], [1, 3]], [[1, 2], [3, 4]], [[4, 5, 6]], [[1, 2, 3, 4, 5]], [[2], []], [[9, 9]]]
    tok, par, dep, n, st = merge_batch(reqs, T=4, max_nodes=64, raise_on_error=False, n_threads=4)
    names = [SpectreeError(int(s), "").code if s else "ok" for s in st]
    assert names == ["ok", "root_mismatch", "ok", "invalid_argument", "empty_input", "ok"]
    assert list(n) == [3, 0, 3, 0, 0, 2]
    np.testing.assert_array_equal(tok[0, :3], TokenTree.merge_sequences(reqs[0]).tokens)
    with pytest.raises(SpectreeError) as e:
        merge_batch(reqs, T=4)
    assert e.value.code == "root_mismatch"


def test_merge_batch_pool_stress_into_preallocated():
    """Many back-to-back calls through the persistent pool into caller-owned
    (torch CPU) buffers, with varying thread counts."""
    import torch
    from paper_2305_09781_b200.tree import TokenTree, merge_batch
    rng = np.random.default_rng(5)
    B, T = 16, 64
    out = tuple(torch.zeros((B, T), dtype=torch.int32) for _ in range(3)) + (
        torch.zeros(B, dtype=torch.int32),)
    for it in range(200):
        reqs = []
        for _ in range(B):
            root = int(rng.integers(0, 100))
            reqs.append([[root] + rng.integers(0, 100, int(rng.integers(0, 8))).tolist()
                         for _ in range(int(rng.integers(1, 7)))])
        merge_batch(reqs, T, out=out, n_threads=int(it % 5))
        for b in (0, B - 1):
            t = TokenTree.merge_sequences(reqs[b])
            assert int(out[3][b]) == t.size
            np.testing.assert_array_equal(out[0][b, : t.size].numpy(), t.tokens)
            np.testing.assert_array_equal(out[1][b, : t.size].numpy(), t.parents)
