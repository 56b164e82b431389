"""Batch x KV-head partitioning across GPUs.

Every (batch, kv-head) unit of the OTT cache is independent (cache.py:17-18,
outlier.py:10-11): flush, prefill and attention need no cross-GPU exchange. A
rank therefore owns whole sequences — a contiguous slice of the batch with all
of its kv heads, so GQA groups stay intact and q never moves — and the only
collective is the all-gather of head outputs [B_local, H_q, d] -> [B, H_q, d]
that the next layer's consumers expect (north star: "NCCL over NVLink used
only to all-gather head outputs").
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous batch slice [lo, hi) owned by `rank` (equal shards; batch % world == 0)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if batch % world:
        raise ValueError(f"batch {batch} is not divisible by world size {world}")
    per = batch // world
    return rank * per, (rank + 1) * per


def all_gather_heads(local: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """All-gather head outputs along the batch axis (rank order = batch order)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((local.shape[0] * world, *local.shape[1:]), dtype=local.dtype, device=local.device)
    if world == 1:
        out.copy_(local)
        return out
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    else:  # gloo (CPU tests): list form
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local.contiguous(), group=group)
    return out
