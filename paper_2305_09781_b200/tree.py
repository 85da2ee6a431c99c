"""Python mirror of the reference's tree API (reference proj/python/bindings.cpp:47-64:
``TokenTree.merge_sequences``, ``size``, ``ancestors``, ``dfs_chains`` and
``verify``) over this package's C++ host library and GPU walk.

* Tree construction is the C++ ``TokenTree::merge_sequences``
  (csrc/host/token_tree.cpp) through ``st_tree_merge``.
* ``verify`` runs the K3 walk on the GPU through ``st_verify_outputs``.
* ``TreeBatch`` packs several trees into the device layout
  (include/spectree_capi.h) for the batched kernels; ``merge_batch`` merges
  and packs a whole batch on the host thread pool (``st_tree_merge_batch``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._capi import SpectreeError, check, lib


class TokenTree:
    __slots__ = ("tokens", "parents", "depths", "_children")

    def __init__(self, tokens, parents, depths):
        self.tokens = np.asarray(tokens, np.int32)
        self.parents = np.asarray(parents, np.int32)
        self.depths = np.asarray(depths, np.int32)
        self._children = None

    @staticmethod
    def merge_sequences(sequences, max_nodes: int = 64) -> "TokenTree":
        seqs = [list(map(int, s)) for s in sequences]
        lens = np.array([len(s) for s in seqs], np.int32)
        flat = np.array([t for s in seqs for t in s] or [0], np.int32)
        cap = int(lens.sum()) + 1 if len(seqs) else 1
        tok = np.zeros(cap, np.int32)
        par = np.zeros(cap, np.int32)
        dep = np.zeros(cap, np.int32)
        n = C.c_int(0)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        st = lib().st_tree_merge(p(flat), p(lens) if len(seqs) else None, len(seqs), int(max_nodes),
                                 p(tok), p(par), p(dep), cap, C.byref(n))
        if st != 0:
            raise SpectreeError(st, "merge_sequences")
        k = n.value
        return TokenTree(tok[:k].copy(), par[:k].copy(), dep[:k].copy())

    @property
    def size(self) -> int:
        return int(self.tokens.size)

    def __len__(self):
        return self.size

    @property
    def max_depth(self) -> int:
        return int(self.depths.max())

    def _check(self, node):
        if not 0 <= node < self.size:
            raise SpectreeError(3, f"node {node} not in tree of size {self.size}")

    def token(self, node):
        self._check(node)
        return int(self.tokens[node])

    def parent(self, node):
        self._check(node)
        return int(self.parents[node])

    def depth(self, node):
        self._check(node)
        return int(self.depths[node])

    def children(self, node):
        self._check(node)
        if self._children is None:
            ch = [[] for _ in range(self.size)]
            for v in range(1, self.size):
                ch[self.parents[v]].append(v)
            self._children = ch
        return list(self._children[node])

    def ancestors(self, node):
        self._check(node)
        out = []
        while node >= 0:
            out.append(int(self.tokens[node]))
            node = int(self.parents[node])
        return out[::-1]

    def dfs_chains(self):
        chains = []
        for v in range(1, self.size):
            if not chains or self.parents[v] != v - 1:
                chains.append([])
            chains[-1].append(v)
        return chains

    def ancestor_masks(self, W=None) -> np.ndarray:
        W = W or (self.size + 63) // 64
        m = np.zeros((self.size, W), np.uint64)
        for u in range(self.size):
            if self.parents[u] >= 0:
                m[u] = m[self.parents[u]]
            m[u, u // 64] |= np.uint64(1) << np.uint64(u % 64)
        return m


def verify(tree: TokenTree, outputs, device="cuda"):
    """Alg.-2 walk (reference token_tree.cpp:153-175) on the GPU."""
    import torch

    outputs = list(map(int, outputs))
    if len(outputs) != tree.size:
        raise SpectreeError(4, f"verify: got {len(outputs)} outputs for {tree.size} nodes")
    from . import _capi

    T = tree.size
    out = torch.tensor([outputs], dtype=torch.int32, device=device)
    tok = torch.tensor(tree.tokens[None], device=device)
    par = torch.tensor(tree.parents[None], device=device)
    n = torch.tensor([T], dtype=torch.int32, device=device)
    ver = torch.zeros((1, T + 1), dtype=torch.int32, device=device)
    ids = torch.zeros((1, T + 1), dtype=torch.int32, device=device)
    ln = torch.zeros(1, dtype=torch.int32, device=device)
    check(lib().st_verify_outputs(_capi._ptr(out), 1, T, _capi._ptr(tok), _capi._ptr(par),
                                  _capi._ptr(n), None, -1, _capi._ptr(ver), _capi._ptr(ids),
                                  _capi._ptr(ln), _capi._stream()))
    k = int(ln.item())
    return ver[0, :k].tolist()


class TreeBatch:
    """B trees padded to T nodes in the device layout of include/spectree_capi.h."""

    def __init__(self, trees, T=None):
        self.B = len(trees)
        self.T = T or max(t.size for t in trees)
        self.W = (self.T + 63) // 64
        self.tokens = np.zeros((self.B, self.T), np.int32)
        self.parents = np.full((self.B, self.T), -1, np.int32)
        self.depths = np.zeros((self.B, self.T), np.int32)
        self.n_nodes = np.zeros(self.B, np.int32)
        for b, t in enumerate(trees):
            if t.size > self.T:
                raise SpectreeError(5, f"tree of {t.size} nodes > T={self.T}")
            k = t.size
            self.tokens[b, :k], self.parents[b, :k], self.depths[b, :k] = t.tokens, t.parents, t.depths
            self.n_nodes[b] = k


class MergeInputs:
    """Flattened candidate sequences of a batch (request b's sequences are the
    next nseq[b] entries of lens, their tokens the next sum(lens) of flat) —
    the argument layout of st_tree_merge_batch."""

    def __init__(self, batch_sequences):
        seqs = [[list(map(int, s)) for s in req] for req in batch_sequences]
        self.B = len(seqs)
        self.nseq = np.array([len(r) for r in seqs], np.int32)
        self.lens = np.array([len(s) for r in seqs for s in r] or [0], np.int32)
        self.flat = np.array([t for r in seqs for s in r for t in s] or [0], np.int32)


def merge_batch(batch_sequences, T: int, max_nodes: int = 64, out=None, n_threads: int = 0,
                raise_on_error: bool = True):
    """TokenTree.merge_sequences for every request of a batch on the host
    thread pool, packed into padded [B][T] arrays. ``out`` may be a tuple of
    preallocated (tok, parent, depth, n_nodes) arrays — numpy, or pinned torch
    CPU tensors so a single H2D copy follows. Returns (tok, parent, depth,
    n_nodes, status)."""
    mi = batch_sequences if isinstance(batch_sequences, MergeInputs) else MergeInputs(batch_sequences)
    B = mi.B
    if out is None:
        out = (np.zeros((B, T), np.int32), np.zeros((B, T), np.int32), np.zeros((B, T), np.int32),
               np.zeros(B, np.int32))
    tok, par, dep, n = out
    status = np.zeros(max(B, 1), np.int32)

    def ptr(a):
        if isinstance(a, np.ndarray):
            assert a.dtype == np.int32 and a.flags.c_contiguous
            return a.ctypes.data_as(C.c_void_p)
        assert a.dtype.__str__() == "torch.int32" and a.is_contiguous() and a.device.type == "cpu"
        return C.c_void_p(a.data_ptr())

    st = lib().st_tree_merge_batch(B, ptr(mi.flat), ptr(mi.lens), ptr(mi.nseq), int(max_nodes), int(T),
                                   ptr(tok), ptr(par), None if dep is None else ptr(dep), ptr(n),
                                   ptr(status), int(n_threads))
    if st != 0 and raise_on_error:
        bad = int(np.nonzero(status[:B])[0][0])
        raise SpectreeError(int(status[bad]), f"merge_batch: request {bad}")
    return tok, par, dep, n, status[:B]
