"""Pin the CPU restatement (oracle/restate.c) against golden fixtures that
were produced by the unmodified reference (oracle/gen_golden.py).

These run on CPU only. If the restatement drifts from the reference, every
GPU parity test that uses it as the checker would be meaningless, so this is
the first gate.
"""
import numpy as np
import pytest


def _seqs(flat, lens):
    out, at = [], 0
    for n in lens:
        out.append(flat[at: at + n].tolist())
        at += n
    return out


KAT_NAMES = ["merge6", "linear", "paper", "chain4", "walk", "mismatch", "rootonly"]


@pytest.mark.parametrize("name", KAT_NAMES)
def test_merge_kats(restatement, golden, name):
    g = golden("tree_kats.npz")
    tok, par, dep = restatement.merge(_seqs(g[f"{name}_flat"], g[f"{name}_lens"]))
    np.testing.assert_array_equal(tok, g[f"{name}_tok"])
    np.testing.assert_array_equal(par, g[f"{name}_par"])
    np.testing.assert_array_equal(dep, g[f"{name}_dep"])


@pytest.mark.parametrize("name", ["merge6", "walk", "mismatch", "rootonly"])
def test_verify_kats(restatement, golden, name):
    g = golden("tree_kats.npz")
    ver, ids = restatement.verify(g[f"{name}_tok"], g[f"{name}_par"], g[f"{name}_outputs"])
    np.testing.assert_array_equal(ver, g[f"{name}_verified"])
    # accepted ids walk parent links from the root
    assert ids[0] == 0
    for k in range(1, len(ids)):
        assert g[f"{name}_par"][ids[k]] == ids[k - 1]


def test_published_kat_values(golden):
    """The literal answers the reference's own tests assert."""
    g = golden("tree_kats.npz")
    assert len(g["merge6_tok"]) == 6                               # token_tree_test.cpp:45
    assert g["merge6_verified"].tolist() == [3, 4, 5, 1]           # test_smoke.py:27
    assert g["walk_verified"].tolist() == [1, 3, 7]                # token_tree_test.cpp:227
    assert g["mismatch_verified"].tolist() == [9]                  # token_tree_test.cpp:232
    assert g["paper_chain_lens"].tolist() == [3, 2, 2]             # token_tree_test.cpp:156
    assert dict(zip(g["error_names"].tolist(), g["error_codes"].tolist())) == {
        "root_mismatch": "root_mismatch", "too_large": "tree_too_large",
        "empty_seq": "empty_input"}


def test_merge_errors(restatement):
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        restatement.merge([[1, 2], [3, 4]])
    assert e.value.code == "root_mismatch"
    with pytest.raises(OracleError) as e:
        restatement.merge([[1, 2, 3, 4, 5]], 3)
    assert e.value.code == "tree_too_large"
    with pytest.raises(OracleError) as e:
        restatement.merge([[1, 2], []])
    assert e.value.code == "empty_input"
    with pytest.raises(OracleError) as e:
        restatement.verify([1, 2], [-1, 0], [1])
    assert e.value.code == "missing_output"


def test_random_merges_and_walks(restatement, golden):
    g = golden("tree_random.npz")
    fa = la = na = va = 0
    for c in range(len(g["nseq"])):
        k = int(g["nseq"][c])
        lens = g["lens"][la: la + k]
        flat = g["flat"][fa: fa + int(lens.sum())]
        n = int(g["n_nodes"][c])
        tok, par, dep = restatement.merge(_seqs(flat, lens), 1024)
        np.testing.assert_array_equal(tok, g["tok"][na: na + n])
        np.testing.assert_array_equal(par, g["par"][na: na + n])
        np.testing.assert_array_equal(dep, g["dep"][na: na + n])
        nv = int(g["n_verified"][c])
        ver, _ = restatement.verify(tok, par, g["outputs"][na: na + n])
        np.testing.assert_array_equal(ver, g["verified"][va: va + nv])
        fa += int(lens.sum()); la += k; na += n; va += nv


def test_uniform_stream_matches_reference_weights(restatement, golden):
    """init_random_weights draws every tensor from one UniformStream in
    serialized order (transformer.cpp:71-114), so the whole parameter vector
    is the stream itself."""
    g = golden("weights_toy.npz")
    w = g["weights"]
    ours = restatement.uniform_stream(int(g["seed"]), w.size, -0.08, 0.08)
    np.testing.assert_array_equal(ours, w)


def test_tree_attention_matches_reference_attention(restatement, golden):
    """Masked one-pass tree attention == the reference's attention() with an
    explicit prefix+tree mask (transformer.cpp:160-216), node rows only."""
    g = golden("attention_tree.npz")
    x, par, P, heads = g["x"], g["par"], int(g["P"]), int(g["heads"])
    n = len(par)
    l, d = x.shape
    D = d // heads
    q, k, v = x @ g["wq"], x @ g["wk"], x @ g["wv"]
    Lmax = l + 3
    kc = np.zeros((1, heads, Lmax, D))
    vc = np.zeros((1, heads, Lmax, D))
    for h in range(heads):
        kc[0, h, :l] = k[:, h * D:(h + 1) * D]
        vc[0, h, :l] = v[:, h * D:(h + 1) * D]
    qq = q[P:].reshape(1, n, heads, D)
    mask = restatement.ancestor_masks(par)[None]
    o = restatement.tree_attention(qq, kc, vc, mask, np.array([P], np.int32),
                                   np.array([n], np.int32), 1.0 / np.sqrt(D))
    np.testing.assert_allclose(o.reshape(n, d), g["out"][P:], rtol=0, atol=1e-12)


def test_ancestor_masks_are_ancestor_sets(restatement, golden):
    g = golden("tree_kats.npz")
    par = g["paper_par"]
    m = restatement.ancestor_masks(par)
    for u in range(len(par)):
        anc, v = set(), u
        while v >= 0:
            anc.add(v)
            v = par[v]
        bits = {i for i in range(len(par)) if (int(m[u, i // 64]) >> (i % 64)) & 1}
        assert bits == anc


def test_greedy_verify_tie_rule(restatement):
    """Lowest token id wins ties (transformer.cpp:116-122, transformer_test.cpp:259-262)."""
    assert restatement.argmax(np.array([1.0, 3.0, 3.0, 2.0])) == 1
    assert restatement.argmax(np.array([1.0, 3.0, 3.0, 2.0], np.float32)) == 1
    assert restatement.argmax(np.array([np.nan, 3.0], np.float32)) == 0
    assert restatement.argmax(np.array([1.0, np.nan, 3.0], np.float32)) == 2
