"""The reference-facing Python API (paper_2305_09781_b200.tree, mirroring
proj/python/bindings.cpp:47-64) on the GPU: merge on the host C++ library,
verify through the K3 walk. KATs from proj/tests/python/test_smoke.py:17-27 and
proj/tests/token_tree_test.cpp:203-235, plus the 200 reference-generated
random walks."""
import numpy as np
import pytest

from tests.test_oracle_golden import _seqs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import tree
    return tree


def test_smoke_kat(api):
    t = api.TokenTree.merge_sequences([[2, 3, 4, 5], [2, 3, 8, 9]])
    assert t.size == 6
    assert t.ancestors(t.size - 1) == [2, 3, 8, 9]
    assert len(api.TokenTree.merge_sequences([[2, 3, 4, 5], [2, 3, 6, 7], [2, 3, 8, 9]]).dfs_chains()) == 3
    assert api.verify(t, [3, 4, 5, 1, 0, 0]) == [3, 4, 5, 1]


def test_verify_kats(api):
    assert api.verify(api.TokenTree.merge_sequences([[5]]), [9]) == [9]
    assert api.verify(api.TokenTree.merge_sequences([[0, 1, 3], [0, 2]]), [1, 3, 7, 0]) == [1, 3, 7]
    assert api.verify(api.TokenTree.merge_sequences([[0, 1], [0, 2]]), [9, 0, 0]) == [9]
    from paper_2305_09781_b200 import SpectreeError
    with pytest.raises(SpectreeError) as e:
        api.verify(api.TokenTree.merge_sequences([[0, 1]]), [1])
    assert e.value.code == "missing_output"


def test_random_walks_match_reference(api, golden):
    g = golden("tree_random.npz")
    fa = la = na = va = 0
    for c in range(len(g["nseq"])):
        k = int(g["nseq"][c])
        lens = g["lens"][la: la + k]
        flat = g["flat"][fa: fa + int(lens.sum())]
        n = int(g["n_nodes"][c])
        nv = int(g["n_verified"][c])
        t = api.TokenTree.merge_sequences(_seqs(flat, lens), 1024)
        assert api.verify(t, g["outputs"][na: na + n]) == g["verified"][va: va + nv].tolist()
        fa += int(lens.sum()); la += k; na += n; va += nv
