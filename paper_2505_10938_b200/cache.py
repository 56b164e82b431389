"""Batched GPU tiered KV cache — the reference's TieredCache (kvtrace/cache.py:90-203)
for all (batch, kv-head) units of one layer at once, resident in HBM.

State lives in torch CUDA tensors (allocation/streams only); every byte of it is
produced and consumed by the sm_100a kernels in ``csrc/`` via the C ABI in
``include/ott_b200.h``. There is no CPU fallback: without a CUDA device and
``libott_b200.so`` every method raises.

HBM layout per unit (u = b * H_kv + h), see DESIGN.md §3:
  blocks     uint8 [U, max_groups, record]  K codes | V codes | K step halves | V step,x_min f32[G] | K e hi/lo
  pend_k/v   fp16  [U, G+R, d]              pending ring, slot = position % (G+R)
  pool_*     slot-stable pool.entries (pos, score f64, K/V rows fp16), aux ledger, meta
  pool_mask  uint32 [U, max_tokens/32]      1 bit per position currently in pool.entries
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .config import EngineConfig, MemoryBreakdown
from .errors import ContractViolation
from .views import (FP16_BITS, AttentionResult, GroupAxis, OutlierEntry, OutlierPoolView, QuantizedBlock, QuantParams,
                    require)


def _stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def _on_device(fn):
    """Run a cache method with the cache's GPU as the current device, so the C ABI
    launches on that device's current stream (multi-GPU processes)."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        with torch.cuda.device(self.device):
            return fn(self, *args, **kwargs)

    return wrapper


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()



def kpair_index(c, d=128):
    """Index of channel c in the record's fp16 K step halves (ott_b200.h): pair order
    when d % 16 == 0, channel order otherwise."""
    c = np.asarray(c)
    c = np.asarray(c)
    return c if d % 16 else 16 * (c // 16) + 2 * (c % 8) + (c % 16) // 8


def code_bits(bits, d, G):
    """Stored code width (ott_common.cuh code_bits): at the tensor-core shapes 1-bit codes live
    in 2-bit fields, 3-bit in 4-bit and 5..7-bit in 8-bit fields (levels stay 2^bits - 1)."""
    if d != 128 or G not in (32, 64, 128):
        return bits
    if bits == 1:
        return 2
    if bits == 3:
        return 4
    if 5 <= bits <= 7:
        return 8
    return bits


def record_code_bytes(d, G, bits):
    """Bytes of one code field of a block record: ceil(G d code_bits / 8) padded to 16."""
    return ((G * d * code_bits(bits, d, G) + 7) // 8 + 15) & ~15


def repack_codes(buf, n, from_bits, to_bits, shift=0):
    """pack_codes stream (quant.py:241-256, LSB first) of n codes re-packed at another width
    (codes stored shifted left by `shift` in their container are shifted back)."""
    if from_bits == to_bits:
        return bytes(buf[:(n * to_bits + 7) // 8])
    bits = np.unpackbits(np.frombuffer(bytes(buf), np.uint8), bitorder="little")[: n * from_bits]
    codes = bits.reshape(n, from_bits)[:, shift:shift + to_bits]  # the other container bits are zero
    return np.packbits(codes.reshape(-1), bitorder="little").tobytes()


def kpair4_index(c):
    """4-bit pair order: half2 pairs (8w+k, 8w+k+4) of the nibble unpack (ott_common.cuh)."""
    c = np.asarray(c)
    return 8 * (c // 8) + 2 * (c % 4) + (c % 8) // 4


def kpair_u(c):
    """Position scale u(c) = 4^(4 - P(c % 8)) of the decode kernels' code-pair unpack."""
    P = np.array([3, 4, 2, 3, 4, 2, 3, 4])[np.asarray(c) % 8]
    return (4.0 ** (4 - P)).astype(np.float32)


class OTTCache:
    """One layer's OTT cache for ``batch * n_kv_heads`` independent units.

    All units advance in lock step (one token per unit per ``append``), so the
    flush trigger ``pending - R >= G`` (cache.py:138) is decided on the host
    from the shared token count with no device synchronisation.

    Args:
        config: EngineConfig (same fields as the reference). bits in [1, 8]
            (2-bit uses the tensor-core kernels, other widths the CUDA-core kernel);
            head_dim in [1, 256] and group_size in [1, 128] (d = 128 with G % 32 == 0 runs the
            tensor-core kernels; other shapes, e.g. the reference tests' d = 2..16,
            G = 4..16, run a generic CUDA-core kernel).
        batch, n_kv_heads: unit grid.
        max_tokens: capacity of the quantized store per unit.
        layer: layer index; pool capacity is ``config.outlier_capacity(layer)``.
        keep_f64_params: also store the exact float64 (x_min, step) of every
            parameter line (parity/debug; 2.5x the param bytes).
        validate: check inputs for NaN/Inf on every call (costs a device sync;
            the reference raises ContractViolation, cache.py:131-132).
    """

    def __init__(self, config: EngineConfig, batch: int, n_kv_heads: int, max_tokens: int, layer: int = 0,
                 device=None, keep_f64_params: bool = False, validate: bool = False):
        if not torch.cuda.is_available():
            raise _native.NativeError("OTTCache needs a CUDA device (B200); there is no CPU path")
        require(1 <= config.bits <= 8, "bits must be in [1, 8]")
        require(1 <= config.head_dim <= 256, "head_dim must be in [1, 256] on the GPU path")
        require(1 <= config.group_size <= 128, "group_size must be in [1, 128] on the GPU path")
        require(batch >= 1 and n_kv_heads >= 1 and max_tokens >= 1, "batch, n_kv_heads, max_tokens must be >= 1")
        self.config = config
        self.layer = layer
        self.batch, self.n_kv_heads = batch, n_kv_heads
        self.n_units = batch * n_kv_heads
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.validate = validate
        d, G, R = config.head_dim, config.group_size, config.residual
        self.N = config.outlier_capacity(layer)
        self.A = config.aux_capacity
        require(self.N <= 128, "outlier_num must be <= 128 on the GPU path")
        require(self.A <= 1024, "aux_capacity must be <= 1024 on the GPU path")
        self.max_groups = (max_tokens + G - 1) // G
        self.max_tokens = max_tokens
        L = _native.lib()
        self.record_bytes = int(L.ott_record_bytes(d, G, config.bits))
        U, dev = self.n_units, self.device
        kw = dict(device=dev)
        self.blocks = torch.zeros((U, self.max_groups, self.record_bytes), dtype=torch.uint8, **kw)
        self.pend_k = torch.zeros((U, G + R, d), dtype=torch.float16, **kw)
        self.pend_v = torch.zeros((U, G + R, d), dtype=torch.float16, **kw)
        words = (self.max_groups * G + 31) // 32
        self.pool_mask = torch.zeros((U, words), dtype=torch.int32, **kw)
        self.subst_mask = torch.zeros((U, words), dtype=torch.int32, **kw)
        n, a = max(self.N, 1), max(self.A, 1)
        self.pool_pos = torch.full((U, n), -1, dtype=torch.int32, **kw)
        self.pool_score = torch.zeros((U, n), dtype=torch.float64, **kw)
        self.pool_k = torch.zeros((U, n, d), dtype=torch.float16, **kw)
        self.pool_v = torch.zeros((U, n, d), dtype=torch.float16, **kw)
        self.aux_pos = torch.full((U, a), -1, dtype=torch.int32, **kw)
        self.aux_score = torch.zeros((U, a), dtype=torch.float64, **kw)
        self.aux_k = torch.zeros((U, a, d), dtype=torch.float16, **kw)
        self.aux_v = torch.zeros((U, a, d), dtype=torch.float16, **kw)
        self.pool_meta = torch.zeros((U, 4), dtype=torch.int32, **kw)
        if self.A == 0:
            self.pool_meta[:, 2] = 1  # outlier.py:77-78: aux_capacity 0 freezes at construction
        self.params64 = (torch.zeros((U, self.max_groups, 2 * (d + G)), dtype=torch.float64, **kw)
                         if keep_f64_params else None)
        self._c = _native.OttCacheT(
            n_units=U, head_dim=d, group_size=G, residual=R, capacity=self.N, aux_capacity=self.A, bits=config.bits,
            max_groups=self.max_groups, blocks=_ptr(self.blocks), pend_k=_ptr(self.pend_k), pend_v=_ptr(self.pend_v),
            pool_mask=_ptr(self.pool_mask), subst_mask=_ptr(self.subst_mask), pool_pos=_ptr(self.pool_pos),
            pool_score=_ptr(self.pool_score), pool_k=_ptr(self.pool_k), pool_v=_ptr(self.pool_v),
            aux_pos=_ptr(self.aux_pos), aux_score=_ptr(self.aux_score), aux_k=_ptr(self.aux_k),
            aux_v=_ptr(self.aux_v), pool_meta=_ptr(self.pool_meta), params64=_ptr(self.params64))
        self._cref = ctypes.byref(self._c)
        self.total_tokens = 0
        self.quantized_tokens = 0
        # device copy of (quantized_tokens, total_tokens) for graph-capturable decode steps
        self.counters = torch.zeros(3, dtype=torch.int64, device=dev)  # quantized, total, error
        self._ws = None
        self._ws_key = None

    # ------------------------------------------------------------------ helpers
    @property
    def pending_rows(self) -> int:
        return self.total_tokens - self.quantized_tokens

    def _check_out(self, out: torch.Tensor | None, q: torch.Tensor) -> torch.Tensor:
        """Caller-supplied output buffer: the kernels write it through a raw pointer (and, with
        output peers set, the same offsets into the peers' gather buffers), so it must be
        exactly q's shape, fp16, contiguous and on the cache device."""
        if out is None:
            return torch.empty_like(q)
        require(tuple(out.shape) == tuple(q.shape) and out.dtype == torch.float16 and out.device == self.device
                and out.is_contiguous(), "out must be a contiguous float16 tensor of q's shape on the cache device")
        return out

    def _check_rows(self, x: torch.Tensor, name: str, T: int | None = None) -> torch.Tensor:
        d = self.config.head_dim
        shape = (self.batch, self.n_kv_heads, d) if T is None else (self.batch, self.n_kv_heads, T, d)
        if tuple(x.shape) != shape:
            if T is None and tuple(x.shape) == (self.n_units, d):
                pass
            else:
                raise ContractViolation(f"{name} must have shape {shape}, got {tuple(x.shape)}")
        require(x.dtype == torch.float16, f"{name} must be float16")
        require(x.device == self.device, f"{name} must live on {self.device}")
        x = x.contiguous()
        if self.validate and not bool(torch.isfinite(x).all()):
            raise ContractViolation("rows contain NaN or Inf")  # cache.py:131-132
        return x

    # --------------------------------------------------------------- write path
    @_on_device
    def append(self, k: torch.Tensor, v: torch.Tensor) -> None:
        """cache.py:124-139: add one token per unit; quantize a group when due."""
        k = self._check_rows(k, "k")
        v = self._check_rows(v, "v")
        _native.check(_native.lib().ott_ring_write(self._cref, k.data_ptr(), v.data_ptr(), self.config.head_dim,
                                                   self.total_tokens, self.total_tokens, 1, _stream_handle()))
        self.total_tokens += 1
        if self.pending_rows - self.config.residual >= self.config.group_size:  # cache.py:138
            self.quantize_oldest_group()

    @_on_device
    def quantize_oldest_group(self) -> None:
        """cache.py:141-186 for every unit (one launch of the flush kernel)."""
        G = self.config.group_size
        if self.pending_rows < G:
            raise ContractViolation(f"need {G} pending rows to quantize, have {self.pending_rows}")
        self._flush(1, ring_end=self.total_tokens)

    def _flush(self, n_groups: int, ring_end: int, in_k=None, in_v=None, in_stride: int = 0,
               in_first: int = 0) -> None:
        require(self.quantized_tokens // self.config.group_size + n_groups <= self.max_groups,
                "cache capacity (max_tokens) exceeded")
        _native.check(_native.lib().ott_flush(self._cref, self.quantized_tokens, n_groups, ring_end, _ptr(in_k),
                                              _ptr(in_v), in_stride, in_first, _stream_handle()))
        self.quantized_tokens += n_groups * self.config.group_size

    @_on_device
    def update(self, k: torch.Tensor, v: torch.Tensor) -> None:
        """Bulk insert of T tokens per unit, numerically identical to T sequential
        ``append`` calls: full groups are flushed straight from the
        input (one launch; the pool competition runs group by group inside it),
        the newest rows land in the pending ring."""
        require(k.dim() == 4, "k must be [batch, n_kv_heads, T, d]")
        T = k.shape[2]
        k = self._check_rows(k, "k", T)
        v = self._check_rows(v, "v", T)
        if T == 0:
            return
        G, R, d = self.config.group_size, self.config.residual, self.config.head_dim
        t0 = self.total_tokens
        n_groups = max(0, (self.pending_rows + T - R) // G)
        if n_groups:
            self._flush(n_groups, ring_end=t0, in_k=k, in_v=v, in_stride=T * d, in_first=t0)
        self.total_tokens = t0 + T
        first = max(self.quantized_tokens, t0)
        n_rows = self.total_tokens - first
        if n_rows:
            _native.check(_native.lib().ott_ring_write(self._cref, k.data_ptr(), v.data_ptr(), T * d, t0, first,
                                                       n_rows, _stream_handle()))

    # ---------------------------------------------------------------- read path
    def splits(self, n_rep: int) -> int:
        return int(_native.lib().ott_pick_splits(self._cref, n_rep, self.total_tokens))

    def workspace(self, n_rep: int, n_splits: int) -> torch.Tensor:
        n = int(_native.lib().ott_attend_workspace_floats(self._cref, n_rep, n_splits))
        if self._ws is None or self._ws.numel() < n:
            self._ws = torch.empty(n, dtype=torch.float32, device=self.device)
        return self._ws

    @_on_device
    def append_attend(self, k: torch.Tensor, v: torch.Tensor, q: torch.Tensor, out: torch.Tensor | None = None,
                      n_splits: int | None = None) -> torch.Tensor:
        """``append(k, v)`` then ``attend(q)`` in one call (the decode step of cli.py:211-213):
        a due flush is launched first (it never needs the new row when R >= 1), and on the
        tensor-core path the attention kernel writes the new row into the pending ring
        itself, saving the ring-write launch. Same results as the two calls."""
        k = self._check_rows(k, "k")
        v = self._check_rows(v, "v")
        require(q.dim() == 3 and q.shape[0] == self.batch and q.shape[2] == self.config.head_dim,
                f"query must have shape (batch, H_q, {self.config.head_dim})")
        require(q.shape[1] % self.n_kv_heads == 0, "H_q must be a multiple of n_kv_heads")
        require(q.dtype == torch.float16 and q.device == self.device, "query must be float16 on the cache device")
        if self.config.residual == 0:  # the new row may belong to the flushed group
            self.append(k, v)
            return self.attend(q, out=out, n_splits=n_splits)
        n_rep = q.shape[1] // self.n_kv_heads
        q = q.contiguous()
        out = self._check_out(out, q)
        G, R = self.config.group_size, self.config.residual
        due = self.total_tokens + 1 - self.quantized_tokens - R >= G  # cache.py:138
        require(not due or self.quantized_tokens // G + 1 <= self.max_groups, "cache capacity (max_tokens) exceeded")
        self.total_tokens += 1
        if due:
            self._flush(1, ring_end=self.total_tokens)
        s = n_splits or self.splits(n_rep)
        ws = self.workspace(n_rep, s)
        _native.check(_native.lib().ott_append_attend(self._cref, k.data_ptr(), v.data_ptr(), q.data_ptr(),
                                                      out.data_ptr(), n_rep, self.quantized_tokens,
                                                      self.total_tokens, ws.data_ptr(), s, _stream_handle()))
        return out

    def set_output_peers(self, ptrs) -> None:
        """Fuse the head-output all-gather into the attention epilogue: every
        output row this cache's attention writes to `out` is also stored at the same offset
        from each address in `ptrs` (device pointers, e.g. this rank's rows of the peer GPUs'
        symmetric gather buffers; at most OTT_MAX_OUT_PEERS). Empty = off."""
        ptrs = [int(p) for p in ptrs]
        require(len(ptrs) <= _native.MAX_OUT_PEERS, f"at most {_native.MAX_OUT_PEERS} output peers")
        require(all(p != 0 for p in ptrs), "null output peer pointer")
        for i in range(_native.MAX_OUT_PEERS):
            self._c.out_peer[i] = ptrs[i] if i < len(ptrs) else None
        self._c.n_out_peers = len(ptrs)

    @_on_device
    def sync_counters(self) -> None:
        """Copy the host token counts into `counters` (before capturing `decode_step`)."""
        self.counters.copy_(torch.tensor([self.quantized_tokens, self.total_tokens, 0], dtype=torch.int64))

    def device_error(self) -> None:
        """Raise if a device-counter step ran out of group records (the combine kernel sets
        counters[2] and stops advancing; the host mirror normally refuses such a step first)."""
        if int(self.counters[2].item()):
            raise ContractViolation("cache capacity (max_tokens) exceeded in a device-counter decode step")

    @_on_device
    def decode_step(self, k: torch.Tensor, v: torch.Tensor, q: torch.Tensor, out: torch.Tensor,
                    n_splits: int) -> torch.Tensor:
        """append(k, v) + attend(q) -> out with the token counts read from and advanced
        in device memory (`counters`), so the launches can be captured in a CUDA graph
        and replayed once per step (ott_decode_step). The host counts advance too; call
        `sync_counters()` once before the first device-counter step."""
        k = self._check_rows(k, "k")
        v = self._check_rows(v, "v")
        require(q.dim() == 3 and q.shape[0] == self.batch and q.shape[2] == self.config.head_dim
                and q.shape[1] % self.n_kv_heads == 0 and q.dtype == torch.float16 and q.is_contiguous(),
                "query must be contiguous float16 (batch, H_q, head_dim)")
        require(q.device == self.device, "query must be on the cache device")
        self._check_out(out, q)
        G, R = self.config.group_size, self.config.residual
        due = self.total_tokens + 1 - self.quantized_tokens - R >= G
        require(not due or self.quantized_tokens // G + 1 <= self.max_groups, "cache capacity (max_tokens) exceeded")
        n_rep = q.shape[1] // self.n_kv_heads
        ws = self.workspace(n_rep, n_splits)
        _native.check(_native.lib().ott_decode_step(self._cref, k.data_ptr(), v.data_ptr(), q.data_ptr(),
                                                    out.data_ptr(), n_rep, self.counters.data_ptr(), ws.data_ptr(),
                                                    n_splits, _stream_handle()))
        self.advance_host_counts()
        return out

    def advance_host_counts(self) -> None:
        """Host mirror of one device-counter step (what the combine kernel does to
        `counters`); used by callers that replay a captured `decode_step`."""
        G, R = self.config.group_size, self.config.residual
        self.total_tokens += 1
        if self.total_tokens - self.quantized_tokens - R >= G:
            require(self.quantized_tokens // G + 1 <= self.max_groups, "cache capacity (max_tokens) exceeded")
            self.quantized_tokens += G

    @_on_device
    def attend(self, q: torch.Tensor, out: torch.Tensor | None = None, n_splits: int | None = None) -> torch.Tensor:
        """attend_mixed (attention.py:79-92) for every query head.

        q: fp16 [batch, H_q, d] with H_q = n_kv_heads * n_rep; query head h reads
        kv head h // n_rep. Returns fp16 [batch, H_q, d]."""
        require(q.dim() == 3 and q.shape[0] == self.batch and q.shape[2] == self.config.head_dim,
                f"query must have shape (batch, H_q, {self.config.head_dim})")
        require(q.shape[1] % self.n_kv_heads == 0, "H_q must be a multiple of n_kv_heads")
        require(q.dtype == torch.float16 and q.device == self.device, "query must be float16 on the cache device")
        if self.total_tokens == 0:
            raise ContractViolation("cannot attend over an empty cache")  # attention.py:89-90
        n_rep = q.shape[1] // self.n_kv_heads
        q = q.contiguous()
        out = self._check_out(out, q)
        s = n_splits or self.splits(n_rep)
        ws = self.workspace(n_rep, s)
        _native.check(_native.lib().ott_attend(self._cref, q.data_ptr(), out.data_ptr(), n_rep, self.quantized_tokens,
                                               self.total_tokens, ws.data_ptr(), s, _stream_handle()))
        return out

    def logits(self, q: torch.Tensor) -> torch.Tensor:
        """Debug: AttentionResult.scores for every unit/head, float32 [batch, H_q, T]."""
        n_rep = q.shape[1] // self.n_kv_heads
        out = torch.empty((self.batch, q.shape[1], self.total_tokens), dtype=torch.float32, device=self.device)
        _native.check(_native.lib().ott_logits(self._cref, q.contiguous().data_ptr(), out.data_ptr(), n_rep,
                                               self.quantized_tokens, self.total_tokens, _stream_handle()))
        return out

    # ------------------------------------------------------------- accounting
    def memory_usage(self, b: int = 0, h: int = 0) -> MemoryBreakdown:
        """cache.py:188-203 for unit (b, h), identical bit counts."""
        G, d = self.config.group_size, self.config.head_dim
        nb = self.quantized_tokens // G
        meta = self.pool_meta[b * self.n_kv_heads + h].tolist() if self.N > 0 else [0, 0, 0, 0]
        return MemoryBreakdown(
            quantized_bits=2 * nb * G * d * self.config.bits,
            param_bits=nb * (d + G) * 2 * FP16_BITS,
            pending_bits=self.pending_rows * d * FP16_BITS * 2,
            pool_bits=(meta[0] + meta[1]) * d * FP16_BITS * 2,
        )

    def hbm_bytes(self) -> int:
        """Bytes of device state actually allocated for this layer."""
        ts = [self.blocks, self.pend_k, self.pend_v, self.pool_mask, self.subst_mask, self.pool_pos, self.pool_score,
              self.pool_k, self.pool_v, self.aux_pos, self.aux_score, self.aux_k, self.aux_v, self.pool_meta]
        if self.params64 is not None:
            ts.append(self.params64)
        return sum(t.numel() * t.element_size() for t in ts)

    # --------------------------------------------------------------- snapshots
    def unit(self, b: int, h: int) -> "UnitView":
        """Reference-shaped snapshot of one (batch, kv-head) unit."""
        return UnitView(self, b * self.n_kv_heads + h)


class UnitView:
    """Read-only host snapshot of one unit with the reference TieredCache's
    attribute names (quantized_k/v, pool, substituted_positions, pending_k/v)."""

    def __init__(self, cache: OTTCache, u: int):
        torch.cuda.synchronize(cache.device)
        cfg = cache.config
        d, G = cfg.head_dim, cfg.group_size
        self.config = cfg
        self.total_tokens = cache.total_tokens
        self.quantized_tokens = cache.quantized_tokens
        nb = cache.quantized_tokens // G
        rec = cache.blocks[u, :nb].cpu().numpy()
        code_b = record_code_bytes(d, G, cfg.bits)  # padded field (ott_b200.h)
        pb = code_bits(cfg.bits, d, G)  # stored width; the views re-pack at cfg.bits
        code_n = (G * d * pb + 7) // 8
        # K params are stored in the decode kernels' encoding (ott_b200.h): fp16 halves
        # sh + sl of the step in pair order and e = x_min - 4 u step; the float32 views
        # below are reconstructions, the exact values come from params64
        self.k_sh16 = rec[:, 2 * code_b: 2 * code_b + 2 * d].copy().view(np.float16)
        self.k_sl16 = rec[:, 2 * code_b + 2 * d: 2 * code_b + 4 * d].copy().view(np.float16)
        if pb == 2:  # ... sl | V step | V x_min | e hi | e lo (e last, ott_common.cuh RecordLayout)
            vo = 2 * code_b + 4 * d
            eo = vo + 8 * G
            self.k_ehi16 = rec[:, eo: eo + 2 * d].copy().view(np.float16)
            self.k_elo16 = rec[:, eo + 2 * d: eo + 4 * d].copy().view(np.float16)
        else:
            vo = 2 * code_b + 8 * d
            self.k_e32 = rec[:, 2 * code_b + 4 * d: 2 * code_b + 8 * d].copy().view(np.float32)
        vst = rec[:, vo: vo + 4 * G].copy().view(np.float32)
        vmn = rec[:, vo + 4 * G: vo + 8 * G].copy().view(np.float32)
        kshift = 1 if (cfg.bits == 1 and pb == 2) else 0  # 1-bit K: doubled codes, halved step
        if pb == 2:  # tensor-core encoding: step = sh + sl, e / (8 u) = hi + lo (pair order), e = x_min - 4 u step
            pidx = kpair_index(np.arange(d), d)
            kst = self.k_sh16[:, pidx].astype(np.float32) + self.k_sl16[:, pidx].astype(np.float32)
            uf = kpair_u(np.arange(d)).astype(np.float32)
            self.k_e32 = ((self.k_ehi16[:, pidx].astype(np.float32) + self.k_elo16[:, pidx].astype(np.float32))
                          * (np.float32(8) * uf)).astype(np.float32)
            kmn = (self.k_e32 + np.float32(4) * uf * kst).astype(np.float32)
            kst = kst * np.float32(2 ** kshift)
        elif pb == 4 and d % 8 == 0:  # 4-bit tensor-core encoding: pair4 order, e = x_min - 64 step
            pidx = kpair4_index(np.arange(d))
            kst = self.k_sh16[:, pidx].astype(np.float32) + self.k_sl16[:, pidx].astype(np.float32)
            kmn = (self.k_e32 + np.float32(64) * kst).astype(np.float32)
        elif pb == 8 and d % 8 == 0:  # 8-bit tensor-core encoding: channel order, e = x_min - 1024 step
            kst = self.k_sh16.astype(np.float32) + self.k_sl16.astype(np.float32)
            kmn = (self.k_e32 + np.float32(1024) * kst).astype(np.float32)
        else:  # other widths: float32 step[d] in the sh/sl bytes, x_min in e
            kst = rec[:, 2 * code_b: 2 * code_b + 4 * d].copy().view(np.float32)
            kmn = self.k_e32.copy()
        self.k_step32, self.k_xmin32, self.v_step32, self.v_xmin32 = kst, kmn, vst, vmn
        if cache.params64 is not None:
            p = cache.params64[u, :nb].cpu().numpy()
            kmn64, kst64, vmn64, vst64 = p[:, :d], p[:, d:2 * d], p[:, 2 * d:2 * d + G], p[:, 2 * d + G:]
        else:
            kmn64, kst64, vmn64, vst64 = kmn, kst, vmn, vst
        self.quantized_k, self.quantized_v = [], []
        for i in range(nb):
            b = cfg.bits
            self.quantized_k.append(QuantizedBlock(repack_codes(rec[i, :code_n], G * d, pb, b, kshift), GroupAxis.PER_CHANNEL,
                                                   [QuantParams(float(kmn64[i, c]), float(kst64[i, c]), b)
                                                    for c in range(d)], G, d, b))
            self.quantized_v.append(QuantizedBlock(repack_codes(rec[i, code_b:code_b + code_n], G * d, pb, b),
                                                   GroupAxis.PER_TOKEN,
                                                   [QuantParams(float(vmn64[i, t]), float(vst64[i, t]), b)
                                                    for t in range(G)], G, d, b))
        cap = G + cfg.residual
        pos = np.arange(cache.quantized_tokens, cache.total_tokens)
        pk = cache.pend_k[u].float().cpu().numpy()
        pv = cache.pend_v[u].float().cpu().numpy()
        self.pending_k = pk[pos % cap] if len(pos) else np.zeros((0, d), np.float32)
        self.pending_v = pv[pos % cap] if len(pos) else np.zeros((0, d), np.float32)
        pool = OutlierPoolView(capacity=cache.N, aux_capacity=cache.A)
        if cache.N > 0:
            meta = cache.pool_meta[u].tolist()
            ppos = cache.pool_pos[u].cpu().numpy()
            psc = cache.pool_score[u].cpu().numpy()
            pkr = cache.pool_k[u].float().cpu().numpy()
            pvr = cache.pool_v[u].float().cpu().numpy()
            ents = [OutlierEntry(int(ppos[s]), pkr[s], pvr[s], float(psc[s])) for s in range(cache.N) if ppos[s] >= 0]
            pool.entries = sorted(ents, key=lambda e: (e.score, e.position))  # outlier.py:102-103 order
            apos = cache.aux_pos[u].cpu().numpy()
            asc = cache.aux_score[u].cpu().numpy()
            akr = cache.aux_k[u].float().cpu().numpy()
            avr = cache.aux_v[u].float().cpu().numpy()
            pool.aux = [OutlierEntry(int(apos[s]), akr[s], avr[s], float(asc[s])) for s in range(meta[1])]
            pool.frozen = bool(meta[2])
        else:
            pool.frozen = cache.A == 0
        self.pool = pool
        sm = cache.subst_mask[u].cpu().numpy().view(np.uint32)
        bits = np.unpackbits(sm.view(np.uint8), bitorder="little")
        self.substituted_positions = set(np.nonzero(bits)[0].tolist())
        pm = cache.pool_mask[u].cpu().numpy().view(np.uint32)
        self.pool_mask_positions = set(np.nonzero(np.unpackbits(pm.view(np.uint8), bitorder="little"))[0].tolist())

    @property
    def pending_rows(self) -> int:
        return self.total_tokens - self.quantized_tokens


class TieredCache:
    """Drop-in for ``kvtrace.TieredCache(config, layer, passthrough)`` (cache.py:90-203):
    one (layer, head) cache with the reference's numpy row interface and attribute
    names (quantized_k/v, pool, substituted_positions, pending_k/v, memory_usage),
    backed by a one-unit OTTCache on the GPU. Rows must be fp16-representable (the
    GPU stores fp16, as the reference's traces are fp16 in practice) unless
    ``round_rows_to_fp16`` is set, which rounds them instead of raising."""

    def __init__(self, config: EngineConfig, layer: int = 0, passthrough: bool = False, max_tokens: int = 65536,
                 device=None, keep_f64_params: bool = True, round_rows_to_fp16: bool = False):
        if passthrough:
            raise ContractViolation("passthrough (lossless test fixture, quant.py:166-198) is not a GPU mode")
        self.config = config
        self.layer = layer
        self.round_rows_to_fp16 = round_rows_to_fp16
        self._c = OTTCache(config, 1, 1, max_tokens, layer=layer, device=device, keep_f64_params=keep_f64_params)
        self._snap = None

    def _row(self, x, name):
        a = np.asarray(x, dtype=np.float32)
        d = self.config.head_dim
        if a.shape != (d,):
            raise ContractViolation(f"rows must have shape ({d},)")  # cache.py:129-130
        if not np.isfinite(a).all():
            raise ContractViolation("rows contain NaN or Inf")  # cache.py:131-132
        h = a.astype(np.float16)
        if not self.round_rows_to_fp16 and not np.array_equal(h.astype(np.float32), a):
            raise ContractViolation(f"{name} row is not fp16-representable")
        return torch.from_numpy(h).to(self._c.device).view(1, 1, d)

    def append(self, k_row, v_row) -> None:
        k, v = self._row(k_row, "key"), self._row(v_row, "value")
        self._snap = None
        self._c.append(k, v)

    def extend(self, keys, values) -> None:
        """Bulk append (prefill), identical to appending row by row."""
        k = np.asarray(keys, dtype=np.float32)
        v = np.asarray(values, dtype=np.float32)
        require(k.ndim == 2 and k.shape == v.shape and k.shape[1] == self.config.head_dim, "bad prefill shape")
        require(np.isfinite(k).all() and np.isfinite(v).all(), "rows contain NaN or Inf")
        kh, vh = k.astype(np.float16), v.astype(np.float16)
        require(self.round_rows_to_fp16 or (np.array_equal(kh.astype(np.float32), k)
                                            and np.array_equal(vh.astype(np.float32), v)),
                "rows are not fp16-representable (TieredCache(round_rows_to_fp16=True) rounds them)")
        dev = self._c.device
        self._snap = None
        self._c.update(torch.from_numpy(kh).to(dev)[None, None], torch.from_numpy(vh).to(dev)[None, None])

    def quantize_oldest_group(self) -> None:
        self._snap = None
        self._c.quantize_oldest_group()

    def memory_usage(self) -> MemoryBreakdown:
        return self._c.memory_usage(0, 0)

    def snapshot(self) -> UnitView:
        """Host copy of the unit's state (taken once per mutation, then reused)."""
        if self._snap is None:
            self._snap = self._c.unit(0, 0)
        return self._snap

    # the reference's state attributes (cache.py:93-122), read from the snapshot
    @property
    def quantized_k(self) -> list:
        return self.snapshot().quantized_k

    @property
    def quantized_v(self) -> list:
        return self.snapshot().quantized_v

    @property
    def pool(self) -> OutlierPoolView:
        return self.snapshot().pool

    @property
    def substituted_positions(self) -> set:
        return self.snapshot().substituted_positions

    @property
    def pending_k(self) -> np.ndarray:
        return self.snapshot().pending_k

    @property
    def pending_v(self) -> np.ndarray:
        return self.snapshot().pending_v

    @property
    def total_tokens(self) -> int:
        return self._c.total_tokens

    @property
    def quantized_tokens(self) -> int:
        return self._c.quantized_tokens

    @property
    def pending_rows(self) -> int:
        return self._c.pending_rows

    @property
    def gpu(self) -> OTTCache:
        return self._c


def attend_mixed(q, cache, with_weights: bool = True):
    """attention.py:79-92. With a TieredCache (numpy interface) returns an
    AttentionResult (weights and scores too, as the reference does, unless
    with_weights=False); with an OTTCache, q is fp16 [B, H_q, d] and the fp16
    output tensor is returned."""
    if isinstance(cache, OTTCache):
        return cache.attend(q)
    require(isinstance(cache, TieredCache), "cache must be a TieredCache or OTTCache")
    d = cache.config.head_dim
    qa = np.asarray(q, dtype=np.float32)
    if qa.shape != (d,):
        raise ContractViolation(f"query must have shape ({d},)")  # attention.py:87-88
    if cache.total_tokens == 0:
        raise ContractViolation("cannot attend over an empty cache")
    qh = qa.astype(np.float16)
    require(cache.round_rows_to_fp16 or np.array_equal(qh.astype(np.float32), qa), "query is not fp16-representable")
    qt = torch.from_numpy(qh).to(cache.gpu.device).view(1, 1, d)
    out = cache.gpu.attend(qt)
    res = AttentionResult(output=out.float().cpu().numpy().reshape(d))
    if with_weights:
        s = cache.gpu.logits(qt).cpu().numpy().reshape(-1).astype(np.float64)
        w = np.exp(s - s.max())
        res.weights = (w / w.sum()).astype(np.float32)  # tensor.py:45-57
        res.scores = s.astype(np.float32)
    return res
