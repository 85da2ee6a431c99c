"""N>1 host logic on CPU: world_size-2 gloo processes partition a global batch
of requests, verify their shard (the CPU restatement stands in for the GPU
kernels here: this test covers partitioning + the all-gather exchange only),
and all-gather the accepted tokens; the gathered result must equal the
single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_09781_b200.dist import gather_accepted, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch(seed=0, B=6, V=97):
    from oracle.oracle import Restatement
    from tests.treegen import pack, width_depth_seqs
    R = Restatement()
    rng = np.random.default_rng(seed)
    trees = [R.merge(width_depth_seqs(rng, int(rng.integers(0, V)), V, 3, 4), 1024) for _ in range(B)]
    tok, par, dep, n = pack(trees)
    logits = rng.standard_normal((B, tok.shape[1], V)).astype(np.float32)
    for b in range(B):
        for u in range(n[b]):
            kids = np.nonzero(par[b] == u)[0]
            if kids.size and rng.random() < 0.7:
                logits[b, u, tok[b, kids[0]]] = 9.0
    return R, tok, par, n, logits


def _verify_shard(R, tok, par, n, logits, lo, hi):
    T = tok.shape[1]
    ver = np.full((hi - lo, T + 1), -1, np.int32)
    ln = np.zeros(hi - lo, np.int32)
    for i, b in enumerate(range(lo, hi)):
        _, v, _ = R.greedy_verify(logits[b, : n[b]], tok[b, : n[b]], par[b, : n[b]])
        ver[i, : len(v)] = v
        ln[i] = len(v)
    return ver, ln


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    R, tok, par, n, logits = _batch()
    lo, hi = shard_range(len(n), world, rank)
    ver, ln = _verify_shard(R, tok, par, n, logits, lo, hi)
    g_ver, g_ln = gather_accepted(torch.tensor(ver), torch.tensor(ln), world)
    if rank == 0:
        q.put((g_ver.numpy(), g_ln.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_exactly():
    for n in range(0, 20):
        for w in range(1, 9):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_two_rank_gather_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got_ver, got_ln = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    R, tok, par, n, logits = _batch()
    ref_ver, ref_ln = _verify_shard(R, tok, par, n, logits, 0, len(n))
    np.testing.assert_array_equal(got_ln, ref_ln)
    np.testing.assert_array_equal(got_ver, ref_ver)


def _head_worker(rank, world, port, q):
    """C4 plumbing: each rank owns heads head_shard(H, world, rank), computes its
    slice of a (toy, CPU) attention output, and all-gathers; the gathered chunks
    re-laid out [B,T,world*Hl,D] must equal the unsharded result."""
    from paper_2305_09781_b200.dist import head_shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(0)
    B, T, H, D = 2, 5, 8, 16
    full = torch.randn(B, T, H, D, generator=g)
    h0, h1 = head_shard(H, world, rank)
    mine = full[:, :, h0:h1].contiguous()
    gathered = torch.empty(world * mine.numel())
    dist.all_gather_into_tensor(gathered, mine.view(-1))
    out = gathered.view(world, B, T, h1 - h0, D).permute(1, 2, 0, 3, 4).reshape(B, T, H, D)
    if rank == 0:
        q.put(bool(torch.equal(out, full)))
    dist.barrier()
    dist.destroy_process_group()


def test_head_sharded_gather_layout_two_ranks():
    from paper_2305_09781_b200.dist import head_shard
    assert head_shard(64, 8, 3) == (24, 32)
    with pytest.raises(ValueError):
        head_shard(10, 4, 0)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_head_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    assert q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
