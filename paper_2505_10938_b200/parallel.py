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


def gather_row_offset(layer: int, rank: int, batch_local: int, world: int, n_q_heads: int, head_dim: int) -> int:
    """Byte offset of `rank`'s rows [batch_local, H_q, d] inside layer `layer` of a
    [L, batch_local * world, H_q, d] fp16 gather buffer (rank order = batch order)."""
    row = n_q_heads * head_dim * 2
    return (layer * batch_local * world + rank * batch_local) * row


def peer_destinations(buffer_ptrs, rank: int, layer: int, batch_local: int, n_q_heads: int, head_dim: int):
    """Addresses at which `rank` stores its layer-`layer` outputs in every OTHER rank's
    gather buffer (`buffer_ptrs[p]` = base of rank p's buffer as mapped on this GPU)."""
    world = len(buffer_ptrs)
    off = gather_row_offset(layer, rank, batch_local, world, n_q_heads, head_dim)
    return [int(buffer_ptrs[p]) + off for p in range(world) if p != rank]


class PeerGather:
    """Head-output all-gather fused into the attention epilogue over NVLink.

    One symmetric fp16 buffer [L, B, H_q, d] per rank (torch symmetric memory: every
    peer's buffer is mapped into this GPU's address space). Layer l's cache gets the
    peer addresses of this rank's rows (`OTTCache.set_output_peers`), so the combine
    kernel that produces the outputs also stores them into all peers' buffers: no
    separate collective kernel and no staging copy. `out(l)` is the local slice to pass
    as the attention's `out`; `wait(l)` (a device-side barrier over the signal pads)
    orders every rank's stores before this rank reads `gathered(l)`."""

    def __init__(self, caches, n_q_heads: int, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world - 1 > 7:
            raise ValueError("PeerGather supports up to 8 ranks (OTT_MAX_OUT_PEERS = 7)")
        c0 = caches[0]
        self.L, self.b_local, self.hq, self.d = len(caches), c0.batch, n_q_heads, c0.config.head_dim
        pg = group or dist.group.WORLD
        self.buf = symm_mem.empty(self.L, self.b_local * self.world, n_q_heads, self.d, dtype=torch.float16,
                                  device=c0.device)
        self.handle = symm_mem.rendezvous(self.buf, pg)
        ptrs = list(self.handle.buffer_ptrs)
        for l, c in enumerate(caches):
            c.set_output_peers(peer_destinations(ptrs, self.rank, l, self.b_local, n_q_heads, self.d))
        self.caches = caches

    def out(self, layer: int) -> torch.Tensor:
        lo = self.rank * self.b_local
        return self.buf[layer, lo:lo + self.b_local]

    def wait(self, layer: int) -> None:
        self.handle.barrier(channel=0)

    def gathered(self, layer: int) -> torch.Tensor:
        return self.buf[layer]

    def close(self) -> None:
        for c in self.caches:
            c.set_output_peers([])
