"""K4 — the MSS GUARANTEE, tested statistically (not only self-consistency).

SpecInfer's multi-step speculative sampling promises that the tokens it emits
follow the LLM's own distribution p = softmax(z / tau) whatever the drafts are,
provided every drafted child token was drawn from the draft distribution q of
the edge that proposed it. The reference has no stochastic path,
so this is the independent check of K4 (and of its oracle) that the
bit-exact tests cannot give: chi-square goodness of fit over 2*10^5 trials.

Trees (T = 4, one request per trial, fresh draft tokens every trial):
  node 0 = root; node 1 ~ q1 and node 2 ~ q2 are the root's children (q1 and
  q2 have disjoint supports, so the two drafts never collide and the
  rejection chain root -> child 1 -> residual -> child 2 -> residual is
  exercised); node 3 ~ q3 is child 1's child.
Checked:
  * first emitted token ~ p_root                       (all trials)
  * second token ~ p_node1  given first == tok(node 1)  (accepted at depth 1)
"""
import numpy as np
import pytest

V, TAU, TRIALS = 24, 0.8, 200_000
P_MIN = 1e-4   # fixed seeds: a wrong residual rule gives p-values ~1e-100


def softmax(x):
    e = np.exp(x - x.max(-1, keepdims=True))
    return e / e.sum(-1, keepdims=True)


def setup(rng):
    z = rng.standard_normal((4, V)).astype(np.float32) * 1.5
    z[0, 3] += 2.0          # the LLM likes a token child 1 may propose
    q = np.zeros((4, V), np.float32)
    half = V // 2
    q[1, :half] = softmax(rng.standard_normal(half) * 1.2)
    q[2, half:] = softmax(rng.standard_normal(V - half) * 1.2)
    q[3] = softmax(rng.standard_normal(V) * 1.2)
    q[1] /= q[1].sum(dtype=np.float64)
    q[2] /= q[2].sum(dtype=np.float64)
    q[3] /= q[3].sum(dtype=np.float64)
    return z, q


def draws(rng, q, n):
    """Per trial: child tokens t1 ~ q1, t2 ~ q2, t3 ~ q3; the tree in preorder
    with children ascending by token: root, then the smaller of (t1, t2)..."""
    def pr(row):   # the fp32 draft row as a float64 distribution
        x = row.astype(np.float64)
        return x / x.sum()
    t1 = rng.choice(V, n, p=pr(q[1]))
    t2 = rng.choice(V, n, p=pr(q[2]))
    t3 = rng.choice(V, n, p=pr(q[3]))
    return t1, t2, t3


def pack_trial(t1, t2, t3):
    """t1 < V/2 <= t2 always, so preorder is root, node(t1), node(t3), node(t2):
    tok [r, t1, t3, t2], parent [-1, 0, 1, 0], draft rows [-, q1, q3, q2]."""
    n = t1.size
    tok = np.stack([np.zeros(n, np.int32), t1, t3, t2], 1).astype(np.int32)
    par = np.tile(np.array([-1, 0, 1, 0], np.int32), (n, 1))
    return tok, par


def chi2_p(counts, probs):
    from scipy.stats import chisquare
    exp = probs * counts.sum()
    keep = exp >= 5
    obs = np.append(counts[keep], counts[~keep].sum())
    ex = np.append(exp[keep], exp[~keep].sum())
    if ex[-1] == 0:
        obs, ex = obs[:-1], ex[:-1]
    return chisquare(obs, ex * obs.sum() / ex.sum()).pvalue


def check(first, second, t1, z):
    p_root = softmax(z[0].astype(np.float64) / TAU)
    p1 = softmax(z[1].astype(np.float64) / TAU)
    c0 = np.bincount(first, minlength=V)
    assert chi2_p(c0, p_root) > P_MIN, "first token does not follow softmax(z_root / tau)"
    acc = (first == t1) & (second >= 0)
    assert acc.sum() > 2000
    c1 = np.bincount(second[acc], minlength=V)
    assert chi2_p(c1, p1) > P_MIN, "second token does not follow softmax(z_1 / tau)"
    # the acceptance actually happens at the empirical rate sum_x min(p, q1)
    q1_rate = np.minimum(p_root, softmax_q1_cache[0]).sum()
    assert abs(acc.mean() - q1_rate) < 5 * np.sqrt(q1_rate * (1 - q1_rate) / first.size)


softmax_q1_cache = [None]


def test_oracle_mss_follows_target_distribution(restatement):
    rng = np.random.default_rng(11)
    z, q = setup(rng)
    softmax_q1_cache[0] = q[1].astype(np.float64)
    n = TRIALS // 4      # the C oracle through ctypes: 5e4 trials ~ seconds
    t1, t2, t3 = draws(rng, q, n)
    tok, par = pack_trial(t1, t2, t3)
    qrows = np.stack([q[0], q[1], q[3], q[2]])     # draft row per preorder node
    zrows = np.stack([z[0], z[1], z[3], z[2]])
    U = rng.random((n, 5)).astype(np.float32)
    first = np.zeros(n, np.int64)
    second = np.full(n, -1, np.int64)
    for i in range(n):
        ver, _ = restatement.mss_verify(zrows, qrows, tok[i], par[i], TAU, U[i])
        first[i] = ver[0]
        if len(ver) > 1:
            second[i] = ver[1]
    check(first, second, t1, z)


@pytest.mark.gpu
def test_k4_mss_follows_target_distribution():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    rng = np.random.default_rng(12)
    z, q = setup(rng)
    softmax_q1_cache[0] = q[1].astype(np.float64)
    t1, t2, t3 = draws(rng, q, TRIALS)
    tok, par = pack_trial(t1, t2, t3)
    dev = "cuda"
    zrows = torch.tensor(np.stack([z[0], z[1], z[3], z[2]]), device=dev)
    qrows = torch.tensor(np.stack([q[0], q[1], q[3], q[2]]), device=dev)
    first = np.zeros(TRIALS, np.int64)
    second = np.full(TRIALS, -1, np.int64)
    chunk = 50_000
    for s in range(0, TRIALS, chunk):
        e = min(TRIALS, s + chunk)
        nb = e - s
        logits = zrows.expand(nb, 4, V).contiguous()
        qd = qrows.expand(nb, 4, V).contiguous()
        U = torch.tensor(rng.random((nb, 5)).astype(np.float32), device=dev)
        ver, ids, ln = _capi.verify_mss(logits, qd, torch.tensor(tok[s:e], device=dev),
                                        torch.tensor(par[s:e], device=dev),
                                        torch.full((nb,), 4, dtype=torch.int32, device=dev), TAU, U)
        ver, ln = ver.cpu().numpy(), ln.cpu().numpy()
        first[s:e] = ver[:, 0]
        second[s:e] = np.where(ln > 1, ver[:, 1], -1)
    check(first, second, t1, z)
