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
