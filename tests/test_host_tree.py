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
