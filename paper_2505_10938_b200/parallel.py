"""Batch x KV-head partitioning across GPUs.

Every (batch, kv-head) unit of the OTT cache is independent (cache.py:17-18,
outlier.py:10-11): flush, prefill and attention need no cross-GPU
exchange. The U = B * H_kv units are split into equal contiguous ranges in
batch-major order, one per rank. A unit carries its own n_rep query heads (GQA
groups stay whole), so a rank's shard is an OTTCache of `U / world` units with one
kv head each, its query rows are the contiguous slice q.view(U, n_rep, d)[u0:u1],
and its head outputs are the same slice of [B, H_q, d]. Shards may split a
sequence's kv heads across ranks, so configs with few sequences (config 0: B=1,
H=32; config 2: B=4) still use 8 GPUs. The only collective is the all-gather of
head outputs [U/world, n_rep, d] -> [U, n_rep, d] (north star: "NCCL over NVLink
used only to all-gather head outputs").
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def unit_bounds(n_units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous unit range [lo, hi) owned by `rank` (equal shards: n_units % world == 0,
    so the head outputs gather into [U, n_rep, d] with one all_gather_into_tensor)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if n_units % world:
        raise ValueError(f"{n_units} (batch x kv-head) units do not split evenly over {world} ranks")
    per = n_units // world
    return rank * per, (rank + 1) * per


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Whole-sequence shards: the batch slice [lo, hi) of `rank` (batch % world == 0)."""
    return unit_bounds(batch, world, rank)


def shard_queries(q: torch.Tensor, n_kv_heads: int, lo: int, hi: int) -> torch.Tensor:
    """Query rows [B, H_q, d] of units [lo, hi) as [hi - lo, n_rep, d] (a view)."""
    B, Hq, d = q.shape
    return q.view(B * n_kv_heads, Hq // n_kv_heads, d)[lo:hi]


def all_gather_heads(local: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """All-gather head outputs along the unit axis (rank order = unit order)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((local.shape[0] * world, *local.shape[1:]), dtype=local.dtype, device=local.device)
    if world == 1:
        out.copy_(local)
        return out
    if local.is_cuda and dist.get_backend(group) != "gloo":
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    elif local.is_cuda:  # gloo process group over CUDA tensors (multi-rank tests on one GPU): via host
        parts = list(torch.empty((world, *local.shape), dtype=local.dtype).unbind(0))
        dist.all_gather(parts, local.cpu(), group=group)
        out.copy_(torch.cat(parts, dim=0))
    else:  # gloo (CPU tests): list form
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local.contiguous(), group=group)
    return out


def gather_row_offset(layer: int, rank: int, units_local: int, world: int, n_rep: int, head_dim: int,
                      slot: int = 0, n_layers: int = 1) -> int:
    """Byte offset of `rank`'s rows [units_local, n_rep, d] inside layer `layer` (buffer
    `slot`) of a [2, L, units_local * world, n_rep, d] fp16 gather buffer."""
    row = n_rep * head_dim * 2
    return ((slot * n_layers + layer) * units_local * world + rank * units_local) * row


def peer_destinations(buffer_ptrs, rank: int, layer: int, units_local: int, n_rep: int, head_dim: int,
                      slot: int = 0, n_layers: int = 1):
    """Addresses at which `rank` stores its layer-`layer` outputs in every OTHER rank's
    gather buffer (`buffer_ptrs[p]` = base of rank p's buffer as mapped on this GPU)."""
    world = len(buffer_ptrs)
    off = gather_row_offset(layer, rank, units_local, world, n_rep, head_dim, slot, n_layers)
    return [int(buffer_ptrs[p]) + off for p in range(world) if p != rank]


class PeerGather:
    """Head-output all-gather fused into the attention epilogue over NVLink.

    One symmetric fp16 buffer [2, L, U, n_rep, d] per rank (torch symmetric memory: every
    peer's buffer is mapped into this GPU's address space). Layer l's cache gets the
    peer addresses of this rank's rows (`OTTCache.set_output_peers`), so the combine
    kernel that produces the outputs also stores them into all peers' buffers: no
    separate collective kernel and no staging copy. `out(l)` is the local slice to pass
    as the attention's `out`; `wait(l)` (a device-side barrier over the signal pads)
    orders every rank's stores before this rank reads `gathered(l)`. The buffer is double
    buffered by step parity (`next_step()` flips it and re-points the caches): a rank's
    step-s stores never land in the slot a peer may still be reading from step s - 1
    (the barrier of step s - 1 layer L-1 is past before anyone starts step s + 1)."""

    def __init__(self, caches, n_rep: int, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world - 1 > 7:
            raise ValueError("PeerGather supports up to 8 ranks (OTT_MAX_OUT_PEERS = 7)")
        c0 = caches[0]
        self.L, self.u_local, self.n_rep, self.d = len(caches), c0.batch * c0.n_kv_heads, n_rep, c0.config.head_dim
        pg = group or dist.group.WORLD
        self.buf = symm_mem.empty(2, self.L, self.u_local * self.world, n_rep, self.d, dtype=torch.float16,
                                  device=c0.device)
        self.handle = symm_mem.rendezvous(self.buf, pg)
        self.ptrs = list(self.handle.buffer_ptrs)
        self.caches = caches
        self.slot = 1
        self.next_step()

    def next_step(self) -> None:
        """Switch to the other buffer slot for the next decode step."""
        self.slot ^= 1
        for l, c in enumerate(self.caches):
            c.set_output_peers(peer_destinations(self.ptrs, self.rank, l, self.u_local, self.n_rep, self.d,
                                                 self.slot, self.L))

    def out(self, layer: int) -> torch.Tensor:
        """This rank's rows of the layer, shaped like the caches' query [batch, H_kv * n_rep, d]."""
        lo = self.rank * self.u_local
        c = self.caches[0]
        return self.buf[self.slot, layer, lo:lo + self.u_local].view(c.batch, c.n_kv_heads * self.n_rep, self.d)

    def wait(self, layer: int) -> None:
        self.handle.barrier(channel=0)

    def gathered(self, layer: int) -> torch.Tensor:
        """All ranks' rows [world * batch, H_kv * n_rep, d] (after wait(layer))."""
        c = self.caches[0]
        return self.buf[self.slot, layer].view(c.batch * self.world, c.n_kv_heads * self.n_rep, self.d)

    def close(self) -> None:
        for c in self.caches:
            c.set_output_peers([])
