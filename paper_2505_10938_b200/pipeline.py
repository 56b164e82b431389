"""Host-buffer decode step over a stack of per-layer caches.

The reference is driven with host rows (`TieredCache.append(k_row, v_row)`,
`attend_mixed(q, cache)` on numpy arrays, cache.py:124, attention.py:79). This
is the batched equivalent for a whole model step: every layer's new K/V rows
and query heads come from pinned host memory and every layer's head outputs
go back to it, with the copies overlapped with the kernels:

    H2D stream : copy(l+1) ............ copy(l+2) ...
    compute    :      append(l), attend(l)      append(l+1), attend(l+1) ...
    D2H stream :                    read(l)                          read(l+1)

Device staging is double buffered per layer parity; cross-stream order is kept
with CUDA events only (no host synchronisation inside a step).
"""

from __future__ import annotations

import torch

from .errors import ContractViolation


class HostDecodePipeline:
    """Runs `step(k_h, v_h, q_h, out_h)` for caches[0..L): per layer l, append
    (k_h[l], v_h[l]) [B, H_kv, d] and attend q_h[l] [B, H_q, d] -> out_h[l] ([world * B,
    H_q, d] with a gather: every rank's head outputs).
    Host tensors must be pinned fp16. Work is enqueued on the current stream;
    `step` returns without waiting (use `torch.cuda.current_stream().synchronize()`
    or the returned event)."""

    def __init__(self, caches, n_q_heads: int, gather=None, peer_gather=None, world: int = 1):
        if not caches:
            raise ContractViolation("need at least one layer cache")
        c0 = caches[0]
        self.caches = list(caches)
        self.device = c0.device
        # multi-GPU: the step reads back every rank's rows ([world * batch, H_q, d] per layer),
        # all-gathered by `gather` (callable(out_local, layer) -> gathered rows, NCCL) or by
        # `peer_gather` (parallel.PeerGather: P2P stores fused into the attention)
        self.gather = gather
        self.peer_gather = peer_gather
        self.world = world if (gather is not None or peer_gather is not None) else 1
        B, H, d = c0.batch, c0.n_kv_heads, c0.config.head_dim
        if n_q_heads % H:
            raise ContractViolation("H_q must be a multiple of n_kv_heads")
        kw = dict(dtype=torch.float16, device=self.device)
        self.k_d = [torch.empty((B, H, d), **kw) for _ in range(2)]
        self.v_d = [torch.empty((B, H, d), **kw) for _ in range(2)]
        self.q_d = [torch.empty((B, n_q_heads, d), **kw) for _ in range(2)]
        self.o_d = [torch.empty((B, n_q_heads, d), **kw) for _ in range(2)]
        self.out_shape = (B * self.world, n_q_heads, d)
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.splits = [c.splits(n_q_heads // H) for c in self.caches]
        self.launches = 0

    def _check(self, t, shape, name):
        if t.dtype != torch.float16 or t.is_cuda or tuple(t.shape) != shape:
            raise ContractViolation(f"{name} must be a host float16 tensor of shape {shape}")
        if not t.is_pinned():
            raise ContractViolation(f"{name} must be in pinned host memory")

    def step(self, k_h: torch.Tensor, v_h: torch.Tensor, q_h: torch.Tensor, out_h: torch.Tensor) -> torch.cuda.Event:
        L = len(self.caches)
        self._check(k_h, (L, *self.k_d[0].shape), "k_h")
        self._check(v_h, (L, *self.v_d[0].shape), "v_h")
        self._check(q_h, (L, *self.q_d[0].shape), "q_h")
        self._check(out_h, (L, *self.out_shape), "out_h")
        main = torch.cuda.current_stream(self.device)
        if self.peer_gather is not None:
            self.peer_gather.next_step()  # the other slot of the symmetric gather buffer
        start = torch.cuda.Event()
        start.record(main)
        loaded = [torch.cuda.Event() for _ in range(L)]
        computed = [torch.cuda.Event() for _ in range(L)]
        read = [torch.cuda.Event() for _ in range(L)]

        def load(l):
            b = l % 2
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(computed[l - 2] if l >= 2 else start)  # buffer b free again
                self.k_d[b].copy_(k_h[l], non_blocking=True)
                self.v_d[b].copy_(v_h[l], non_blocking=True)
                self.q_d[b].copy_(q_h[l], non_blocking=True)
                loaded[l].record(self.h2d)

        load(0)
        for l, c in enumerate(self.caches):
            b = l % 2
            if l + 1 < L:
                load(l + 1)
            main.wait_event(loaded[l])
            if l >= 2:
                main.wait_event(read[l - 2])  # o_d[b] drained
            before = c.quantized_tokens
            out_d = self.o_d[b] if self.peer_gather is None else self.peer_gather.out(l)
            c.append_attend(self.k_d[b], self.v_d[b], self.q_d[b], out=out_d, n_splits=self.splits[l])
            self.launches += 2 + (1 if c.quantized_tokens != before else 0)
            if self.peer_gather is not None:
                self.peer_gather.wait(l)  # every rank's rows are in this rank's gather buffer
                src = self.peer_gather.gathered(l)
            else:
                src = out_d if self.gather is None else self.gather(out_d, l)
            computed[l].record(main)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(computed[l])
                out_h[l].copy_(src, non_blocking=True)
                read[l].record(self.d2h)
        for l in range(max(0, L - 2), L):
            main.wait_event(read[l])
        done = torch.cuda.Event()
        done.record(main)
        return done
