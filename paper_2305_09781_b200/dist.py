"""Multi-GPU plumbing for the verification path.

Requests are independent (each owns its KV cache and tree, reference
proj/include/spectree/transformer.hpp:64-67), so a global batch is partitioned
by request across ranks with no collective inside any kernel. The one exchange
step is an all-gather of every rank's accepted tokens and lengths after each
verification step, so every rank (and its host) sees the new sequences.
torch.distributed is plumbing only: NCCL over NVLink on GPUs, gloo on CPU
(tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n_items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_accepted(verified: torch.Tensor, lengths: torch.Tensor) -> torch.Tensor:
    """[B, T+1] tokens + [B] lengths -> one int32 vector [B*(T+2)]."""
    return torch.cat([verified.reshape(-1), lengths.reshape(-1)]).to(torch.int32)


def gather_accepted(verified: torch.Tensor, lengths: torch.Tensor, world: int,
                    out: torch.Tensor | None = None):
    """All-gather every rank's accepted tokens (equal B per rank).
    Returns (verified [world*B, T+1], lengths [world*B])."""
    B, T1 = verified.shape
    mine = pack_accepted(verified, lengths)
    if out is None:
        out = torch.empty(world * mine.numel(), dtype=torch.int32, device=mine.device)
    if world > 1:
        dist.all_gather_into_tensor(out, mine)
    else:
        out.copy_(mine)
    parts = out.view(world, -1)
    ver = parts[:, : B * T1].reshape(world * B, T1)
    ln = parts[:, B * T1:].reshape(world * B)
    return ver, ln


def head_shard(n_heads: int, world: int, rank: int) -> tuple[int, int]:
    """Heads [h0, h1) owned by `rank` for head-sharded attention (C4). The
    Q/K/V projections are column-sharded the same way, so each rank's KV cache
    holds only its heads and K1 runs unchanged on H = n_heads / world."""
    if n_heads % world:
        raise ValueError(f"{n_heads} heads do not split over {world} ranks")
    per = n_heads // world
    return rank * per, (rank + 1) * per


def gather_head_outputs(o_local: torch.Tensor, world: int, gathered: torch.Tensor | None = None,
                        out: torch.Tensor | None = None):
    """All-gather every rank's K1 output [B, T, Hl, D] (NCCL, one contiguous
    chunk per rank) and lay it out as [B, T, world*Hl, D] with the CUDA layout
    kernel (st_heads_gather_layout)."""
    from . import _capi
    B, T, Hl, D = o_local.shape
    if gathered is None:
        gathered = torch.empty((world, B, T, Hl, D), dtype=o_local.dtype, device=o_local.device)
    if world > 1:
        dist.all_gather_into_tensor(gathered.view(-1), o_local.contiguous().view(-1))
    else:
        gathered[0].copy_(o_local)
    return _capi.heads_gather_layout(gathered, world, out=out)


class PeerHeadGather:
    """Head-sharded attention with the all-gather fused into K1 (C4).

    Every rank owns one symmetric-memory allocation holding two full-head
    output slots [2][B, T, world*Hl, D] and two signal arrays uint32[2][world].
    ``attention`` runs K1 over this rank's heads with st_tree_attention_allgather
    (its epilogue stores each output row into every rank's slot over NVLink)
    and then publishes the call's epoch with st_peer_signal; ``wait`` holds the
    stream until every rank's epoch has arrived and returns the gathered
    [B, T, world*Hl, D] slot. Slots alternate by epoch: a rank that has
    received epoch e from every peer knows each peer has finished reading slot
    (e-1)%2, so rank r's epoch e+1 writes into it are safe.

    ``buffers`` / ``signals`` (lists of per-"rank" tensors on one device) make
    a single-process simulation of ``world`` ranks possible for tests.
    """

    def __init__(self, B, T, Hl, D, dtype, device, world, rank, group=None,
                 buffers=None, signals=None):
        self.world, self.rank, self.epoch = world, rank, 0
        shape = (2, B, T, world * Hl, D)
        esz = torch.empty((), dtype=dtype).element_size()
        obytes = 2 * B * T * world * Hl * D * esz
        if buffers is None:
            import torch.distributed._symmetric_memory as symm
            raw = symm.empty(obytes + 2 * world * 4, dtype=torch.uint8, device=device)
            raw[obytes:].zero_()
            hdl = symm.rendezvous(raw, group or dist.group.WORLD)
            bases = list(hdl.buffer_ptrs)
            self.out = raw[:obytes].view(dtype).view(shape)
            self.signal = raw[obytes:].view(torch.int32).view(2, world)
            out_bases, sig_bases = bases, [b + obytes for b in bases]
            dist.barrier(group)   # every signal array is zeroed before anyone signals
        else:
            self.out = buffers[rank].view(shape)
            self.signal = signals[rank].view(2, world)
            out_bases = [t.data_ptr() for t in buffers]
            sig_bases = [t.data_ptr() for t in signals]
        slot = B * T * world * Hl * D * esz
        self._out_ptrs = [torch.tensor([b + s * slot for b in out_bases], dtype=torch.int64,
                                       device=device) for s in range(2)]
        self._sig_ptrs = [torch.tensor([b + s * world * 4 for b in sig_bases], dtype=torch.int64,
                                       device=device) for s in range(2)]

    def attention(self, q, k_cache, v_cache, mask, prefix_len, n_nodes, workspace=None,
                  stream=None):
        from . import _capi
        self.epoch += 1
        s = self.epoch % 2
        _capi.tree_attention_allgather(q, k_cache, v_cache, mask, prefix_len, n_nodes,
                                       self._out_ptrs[s], self.world, self.rank,
                                       workspace=workspace, stream=stream)
        _capi.peer_signal(self._sig_ptrs[s], self.world, self.rank, self.epoch, stream=stream)

    def wait(self, stream=None):
        from . import _capi
        s = self.epoch % 2
        _capi.peer_wait(self.signal[s], self.world, self.epoch, stream=stream)
        return self.out[s]
