"""Head-sharded K1 with the all-gather fused into the epilogue (C4, SURVEY.md
§8(e)): st_tree_attention_allgather + st_peer_signal / st_peer_wait through
dist.PeerHeadGather, with `world` ranks simulated on one device (one output
slot and one signal array per simulated rank; the kernels only see pointer
tables, exactly as with peer-mapped symmetric memory on 8 GPUs).

Checked: every rank's gathered buffer equals the f64 oracle over ALL heads
(north-star tolerance 2e-3) and the buffers are bitwise identical across
ranks; three epochs exercise the slot alternation and the epoch compare.
"""
import numpy as np
import pytest
import torch

from tests.test_gpu_kernels import check_k1, make_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    return _capi


@pytest.mark.parametrize("world,Hl,T", [(4, 2, 32), (8, 1, 61), (2, 4, 64)])
def test_fused_head_allgather_simulated_ranks(capi, restatement, world, Hl, T):
    from paper_2305_09781_b200.dist import PeerHeadGather
    dev, dt = "cuda", torch.float16
    H = world * Hl
    rng = np.random.default_rng(world * 10 + T)
    bt = make_batch(restatement, rng, 3, H, H, 128, T=T, dtype=dt, P_range=(30, 400))
    B, D = 3, 128
    q = torch.tensor(bt["q"], device=dev).to(dt)
    kc = torch.tensor(bt["kc"], device=dev).to(dt)
    vc = torch.tensor(bt["vc"], device=dev).to(dt)
    mask = torch.tensor(bt["mask"].view(np.int64), device=dev)
    P = torch.tensor(bt["P"], device=dev)
    n = torch.tensor(bt["n"], device=dev)
    Tb = q.shape[1]
    bufs = [torch.full((2 * B * Tb * H * D,), float("nan"), dtype=dt, device=dev)
            for _ in range(world)]
    sigs = [torch.zeros(2 * world, dtype=torch.int32, device=dev) for _ in range(world)]
    ranks = [PeerHeadGather(B, Tb, Hl, D, dt, dev, world, r, buffers=bufs, signals=sigs)
             for r in range(world)]
    shards = [(q[:, :, r * Hl:(r + 1) * Hl].contiguous(), kc[:, r * Hl:(r + 1) * Hl].contiguous(),
               vc[:, r * Hl:(r + 1) * Hl].contiguous()) for r in range(world)]
    for epoch in range(3):
        for r in range(world):
            qr, kr, vr = shards[r]
            ranks[r].attention(qr, kr, vr, mask, P, n)
        outs = [g.wait() for g in ranks]
        torch.cuda.synchronize()
        for r in range(1, world):   # rows past each tree are never written (NaN fill)
            for b in range(B):
                k = int(bt["n"][b])
                assert torch.equal(outs[r][b, :k], outs[0][b, :k]), f"rank {r} differs (epoch {epoch})"
        check_k1(restatement, bt, outs[0], dt)
        for g in ranks:
            assert (g.signal[g.epoch % 2] == g.epoch).all()


def test_peer_wait_traps_instead_of_hanging(capi):
    """A missing peer signal must fail loudly (device trap after ~10 s), not
    hang the stream forever — run in a subprocess so the context loss stays
    there."""
    import subprocess
    import sys
    code = ("import torch; from paper_2305_09781_b200 import _capi; "
            "s = torch.zeros(2, dtype=torch.int32, device='cuda'); "
            "_capi.peer_wait(s, 2, 1); torch.cuda.synchronize()")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert r.returncode != 0
