"""Seeded synthetic token trees and packed batches for the parity tests."""
import numpy as np


def random_seqs(rng, root, vocab, n_seqs, max_extra):
    return [[root] + rng.integers(0, vocab, int(rng.integers(0, max_extra + 1))).tolist()
            for _ in range(n_seqs)]


def width_depth_seqs(rng, root, vocab, width, depth):
    """SURVEY.md §8(d) construction: W root-to-leaf paths of one depth."""
    return [[root] + rng.integers(0, vocab, depth).tolist() for _ in range(width)]


def pack(trees, T=None):
    """trees: list of (tok, par, dep) -> padded int32 arrays [B,T] + n_nodes."""
    B = len(trees)
    T = T or max(len(t[0]) for t in trees)
    tok = np.zeros((B, T), np.int32)
    par = np.full((B, T), -1, np.int32)
    dep = np.zeros((B, T), np.int32)
    n = np.zeros(B, np.int32)
    for b, (t, p, d) in enumerate(trees):
        k = len(t)
        tok[b, :k], par[b, :k], dep[b, :k], n[b] = t, p, d, k
    return tok, par, dep, n


def masks(restatement, par, n, W):
    B, T = par.shape
    out = np.zeros((B, T, W), np.uint64)
    for b in range(B):
        out[b, : n[b]] = restatement.ancestor_masks(par[b, : n[b]], W)
    return out


def expansion_seqs(rng, root, vocab, n_ssm, expansion):
    """SpecInfer expansion trees: each SSM keeps the
    top-e_i children per frontier node at depth i (here: random tokens); the
    SSMs' root-to-leaf paths are returned for merge_sequences. With
    expansion <1,1,3,1,1,1,1,1> and 3 SSMs this gives the 61-node C4 tree."""
    seqs = []
    for _ in range(n_ssm):
        frontier = [[root]]
        for e in expansion:
            frontier = [p + [int(t)] for p in frontier for t in rng.integers(0, vocab, e)]
        seqs.extend(frontier)
    return seqs
