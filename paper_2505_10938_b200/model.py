"""Llama-2-7B-shaped random-init decoder with the OTT cache (BASELINE configs[1]).

SURVEY §8(f) rank 2: turns the cache kernels' bandwidth into model decode
tokens/s. The reference has no model (it replays recorded traces,
cli.py:189-236); the paper's throughput setting is a
Llama-2-7B decoder with the OTT cache. This module is that decoder with
random N(0, 0.02) fp16 weights (no checkpoints are available offline):

* projections, MLP and LM head are plain library GEMMs (torch.matmul ->
  cuBLAS), RMSNorm / RoPE / SiLU are torch elementwise ops;
* prefill runs causal attention over the exact fp16 prompt K/V (flash SDPA)
  and inserts the post-RoPE keys and values into each layer's OTT cache with
  the bulk `OTTCache.update`;
* each greedy decode step appends one post-RoPE K/V row per (batch, kv head)
  and attends through the OTT cache kernels (K4 ring write, K1 flush when due,
  K2/K3 attention);
* `kv="fp16"` swaps the OTT cache for a plain fp16 KV cache attended with
  torch SDPA: the accuracy/throughput baseline the paper compares against;
* `kv="flash"` is an independent fp16 throughput baseline: a plain fp16 KV cache attended with
  FlashAttention-2's decode kernel (`flash_attn_with_kvcache`, library code, device-side
  sequence lengths), captured in the same CUDA graph step.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import _native
from .cache import OTTCache, _stream_handle
from .config import EngineConfig
from .errors import ContractViolation


@dataclass(frozen=True)
class DecoderConfig:
    n_layers: int = 32
    hidden: int = 4096
    n_heads: int = 32
    n_kv_heads: int = 32
    head_dim: int = 128
    mlp: int = 11008
    vocab: int = 32000
    rope_theta: float = 10000.0
    eps: float = 1e-5


LLAMA2_7B = DecoderConfig()


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


def rope_tables(d: int, max_pos: int, theta: float, device) -> tuple[torch.Tensor, torch.Tensor]:
    inv = 1.0 / (theta ** (torch.arange(0, d, 2, device=device, dtype=torch.float32) / d))
    ang = torch.outer(torch.arange(max_pos, device=device, dtype=torch.float32), inv)
    ang = torch.cat([ang, ang], dim=-1)
    return ang.cos(), ang.sin()


def apply_rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [..., T, d] (or [..., d] with cos/sin [.., d]); rotate-half convention."""
    d = x.shape[-1]
    xf = x.float()
    rot = torch.cat([-xf[..., d // 2:], xf[..., : d // 2]], dim=-1)
    return (xf * cos + rot * sin).to(x.dtype)


class Decoder:
    """Random-init decoder; `generate(prompt, steps)` = prefill + greedy decode."""

    def __init__(self, cfg: DecoderConfig, batch: int, max_tokens: int, kv: str = "ott",
                 ott: EngineConfig | None = None, device=None, seed: int = 0, k_outliers: int = 0,
                 track_exact: bool = False):
        """k_outliers > 0: per kv head, that many seeded outlier channels in the cached keys (an
        offset of 6x the channel's spread with a tight spread around it), missing on a seeded 1%
        of token ids (outlier tokens); plain random-init keys are isotropic, so 2-bit schemes
        would all look alike. track_exact: keep an fp16 shadow of every K/V row and,
        in eager decode steps, record the reference's fidelity metric (cli.py:208-218): per step
        the mean over (layer, batch, head) of the L1 distance between the cache's attention
        output and exact float32 attention over the same rows (`attn_l1`)."""
        if kv not in ("ott", "fp16", "flash"):
            raise ContractViolation("kv must be 'ott', 'fp16' or 'flash'")
        self.cfg, self.batch, self.max_tokens, self.kv = cfg, batch, max_tokens, kv
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dev, H, Hkv, d, D = self.device, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.hidden
        g = torch.Generator(device=dev).manual_seed(seed)

        def w(*shape):
            return (torch.randn(shape, generator=g, device=dev, dtype=torch.float32) * 0.02).half()

        self.embed = w(cfg.vocab, D)
        self.layers = []
        self.k_struct = []
        for _ in range(cfg.n_layers):
            wqkv = w(D, (H + 2 * Hkv) * d)
            if k_outliers:
                # outlier-channel structure of the cache input (made one-sided
                # as massive-activation channels are): per kv head, k_outliers channels carry a
                # large offset (6x the channel's natural spread) with a tight spread around it;
                # "outlier tokens" (a seeded 1% of the vocabulary, e.g. sink-like tokens) lack it
                # (x0.05), so they stretch their group's quantization range (PAPER.md motivation)
                ch = torch.rand((Hkv, d), generator=g, device=dev).argsort(dim=1)[:, :k_outliers]
                cols = (H * d + torch.arange(Hkv, device=dev)[:, None] * d + ch).reshape(-1)
                spread = wqkv[:, cols].float().norm(dim=0)  # std of norm(x) @ w_c
                self.k_struct.append((ch, (6.0 * spread).view(Hkv, k_outliers)))
            self.layers.append({
                "wqkv": wqkv, "wo": w(H * d, D), "wgu": w(D, 2 * cfg.mlp), "wd": w(cfg.mlp, D),
                "n1": torch.ones(D, dtype=torch.float16, device=dev), "n2": torch.ones(D, dtype=torch.float16, device=dev),
            })
        self.norm = torch.ones(D, dtype=torch.float16, device=dev)
        self.lm_head = w(D, cfg.vocab)
        self.cos, self.sin = rope_tables(d, max_tokens, cfg.rope_theta, dev)
        self.special = (torch.rand(cfg.vocab, generator=g, device=dev) < 0.01) if k_outliers else None
        if kv == "ott":
            ott = ott or EngineConfig(bits=2, group_size=32, residual=128, outlier_num=32, aux_capacity=32,
                                      n_layers=cfg.n_layers, n_heads=Hkv, head_dim=d)
            self.caches = [OTTCache(ott, batch, Hkv, max_tokens, layer=l, device=dev) for l in range(cfg.n_layers)]
        elif kv == "flash":  # [layer, batch, token, kv head, d] (flash_attn_with_kvcache's layout)
            self.k_cache = torch.zeros((cfg.n_layers, batch, max_tokens, Hkv, d), dtype=torch.float16, device=dev)
            self.v_cache = torch.zeros_like(self.k_cache)
            self.seqlens = torch.zeros(batch, dtype=torch.int32, device=dev)
        else:
            self.k_cache = torch.zeros((cfg.n_layers, batch, Hkv, max_tokens, d), dtype=torch.float16, device=dev)
            self.v_cache = torch.zeros_like(self.k_cache)
        self.pos = 0
        self.graph = None
        self.track_exact = track_exact and kv == "ott"
        self.attn_l1 = []
        if self.track_exact:
            self.sk = torch.zeros((cfg.n_layers, batch, Hkv, max_tokens, d), dtype=torch.float16, device=dev)
            self.sv = torch.zeros_like(self.sk)

    # ------------------------------------------------------------------ blocks
    def _qkv(self, x, lw, pos0, cos=None, sin=None):
        cfg, B = self.cfg, x.shape[0]
        H, Hkv, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        T = x.shape[1]
        qkv = rms_norm(x, lw["n1"], cfg.eps) @ lw["wqkv"]
        q, k, v = qkv.split([H * d, Hkv * d, Hkv * d], dim=-1)
        q = q.view(B, T, H, d).transpose(1, 2)
        k = k.view(B, T, Hkv, d).transpose(1, 2)
        v = v.view(B, T, Hkv, d).transpose(1, 2)
        if cos is None:
            cos, sin = self.cos[pos0:pos0 + T], self.sin[pos0:pos0 + T]
        return apply_rope(q, cos, sin), apply_rope(k, cos, sin), v.contiguous()

    def _apply_kstruct(self, l, k, tok):
        """k [B, Hkv, (T,) d] post-RoPE in place: outlier channels -> offset + 0.1 k, or 0.05 k for
        the outlier tokens `tok` ([B] or [B, T] ids)."""
        if not self.k_struct:
            return
        ch, off = self.k_struct[l]
        sp = self.special[tok].to(k.dtype)  # [B] or [B, T]
        B, Hkv = k.shape[0], k.shape[1]
        idx = ch.view(1, Hkv, -1)
        if k.dim() == 4:
            kc = k.gather(3, idx[:, :, None, :].expand(B, Hkv, k.shape[2], -1)).float()
            spb = sp[:, None, :, None].float()
            new = spb * 0.05 * kc + (1 - spb) * (off[None, :, None, :] + 0.1 * kc)
            k.scatter_(3, idx[:, :, None, :].expand(B, Hkv, k.shape[2], -1), new.to(k.dtype))
        else:
            kc = k.gather(2, idx.expand(B, Hkv, -1)).float()
            spb = sp[:, None, None].float()
            new = spb * 0.05 * kc + (1 - spb) * (off[None] + 0.1 * kc)
            k.scatter_(2, idx.expand(B, Hkv, -1), new.to(k.dtype))

    def _mlp(self, x, lw):
        h = rms_norm(x, lw["n2"], self.cfg.eps) @ lw["wgu"]
        a, b = h.chunk(2, dim=-1)
        return (F.silu(a.float()) * b.float()).half() @ lw["wd"]

    def _logits(self, x):
        return rms_norm(x, self.norm, self.cfg.eps) @ self.lm_head

    # ------------------------------------------------------------------ phases
    @torch.no_grad()
    def prefill(self, tokens: torch.Tensor) -> torch.Tensor:
        """tokens int64 [B, T] -> next greedy tokens [B]."""
        cfg = self.cfg
        B, T = tokens.shape
        if B != self.batch or T + 1 > self.max_tokens or self.pos:
            raise ContractViolation("prefill needs a fresh decoder, batch rows and room for T + 1 tokens")
        x = self.embed[tokens]
        rep = cfg.n_heads // cfg.n_kv_heads
        for l, lw in enumerate(self.layers):
            q, k, v = self._qkv(x, lw, 0)
            k = k.contiguous()
            self._apply_kstruct(l, k, tokens)
            kk = k.repeat_interleave(rep, dim=1) if rep > 1 else k
            vv = v.repeat_interleave(rep, dim=1) if rep > 1 else v
            o = F.scaled_dot_product_attention(q, kk, vv, is_causal=True)
            if self.kv == "ott":
                self.caches[l].update(k.contiguous(), v)
                if self.track_exact:
                    self.sk[l, :, :, :T] = k
                    self.sv[l, :, :, :T] = v
            elif self.kv == "flash":
                self.k_cache[l, :, :T] = k.transpose(1, 2)
                self.v_cache[l, :, :T] = v.transpose(1, 2)
            else:
                self.k_cache[l, :, :, :T] = k
                self.v_cache[l, :, :, :T] = v
            x = x + o.transpose(1, 2).reshape(B, T, -1) @ lw["wo"]
            x = x + self._mlp(x, lw)
        self.pos = T
        if self.kv == "flash":
            self.seqlens.fill_(T)
        self.last_logits = self._logits(x[:, -1])
        return self.last_logits.argmax(-1)

    # ------------------------------------------------------------------ decode step
    def _decode_buffers(self):
        if getattr(self, "_dbuf", None) is None:
            cfg, B, dev = self.cfg, self.batch, self.device
            H, Hkv, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
            kw = dict(dtype=torch.float16, device=dev)
            self._dbuf = {
                "h": torch.empty((B, cfg.hidden), **kw), "qkv": torch.empty((B, (H + 2 * Hkv) * d), **kw),
                "q": torch.empty((B, H, d), **kw), "k": torch.empty((B, Hkv, d), **kw),
                "v": torch.empty((B, Hkv, d), **kw), "o": torch.empty((B, H, d), **kw),
                "gu": torch.empty((B, 2 * cfg.mlp), **kw), "act": torch.empty((B, cfg.mlp), **kw),
                "logits": torch.empty((B, cfg.vocab), **kw),
            }
        return self._dbuf

    def _layers_step(self, x, pos_host: int, pos_dev=None, graph: bool = False, tok=None):
        """One decode step over all layers on the residual stream x [B, D] (updated in
        place): fused RMSNorm / RoPE+split / SiLU-gate kernels (ott_model.h), cuBLAS
        GEMMs with the residual adds in their epilogues (addmm_), and the OTT cache
        (device-counter `decode_step` when graph=True, host-count append+attend otherwise)."""
        cfg, B, lib, st = self.cfg, self.batch, _native.lib(), _stream_handle()
        H, Hkv, d, D = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.hidden
        bf = self._decode_buffers()
        h, qkv, q, k, v, o, gu, act = (bf[n] for n in ("h", "qkv", "q", "k", "v", "o", "gu", "act"))
        pos_ptr = pos_dev.data_ptr() if pos_dev is not None else None
        l1_sum = 0.0
        for l, lw in enumerate(self.layers):
            _native.check(lib.ott_model_rmsnorm(x.data_ptr(), lw["n1"].data_ptr(), h.data_ptr(), B, D, cfg.eps, st))
            torch.mm(h, lw["wqkv"], out=qkv)
            _native.check(lib.ott_model_rope_qkv(qkv.data_ptr(), self.cos.data_ptr(), self.sin.data_ptr(), pos_ptr,
                                                 pos_host, q.data_ptr(), k.data_ptr(), v.data_ptr(), B, H, Hkv, d, st))
            if self.k_struct:
                self._apply_kstruct(l, k, tok)
            if self.kv == "ott":
                c = self.caches[l]
                if graph:
                    c.decode_step(k, v, q, o, self.g_splits[l])
                else:
                    c.append(k, v)
                    c.attend(q, out=o)
                    if self.track_exact:
                        l1_sum += self._exact_l1(l, k, v, q, o, pos_host)
            elif self.kv == "flash":
                from flash_attn import flash_attn_with_kvcache

                # appends k, v at seqlens[b] and attends over seqlens[b] + 1 rows (device lengths)
                o.copy_(flash_attn_with_kvcache(q.view(B, 1, H, d), self.k_cache[l], self.v_cache[l],
                                                k=k.view(B, 1, Hkv, d), v=v.view(B, 1, Hkv, d),
                                                cache_seqlens=self.seqlens).view(B, H, d))
            else:
                p = pos_host
                self.k_cache[l, :, :, p] = k
                self.v_cache[l, :, :, p] = v
                rep = H // Hkv
                kk, vv = self.k_cache[l, :, :, : p + 1], self.v_cache[l, :, :, : p + 1]
                if rep > 1:
                    kk, vv = kk.repeat_interleave(rep, dim=1), vv.repeat_interleave(rep, dim=1)
                o.copy_(F.scaled_dot_product_attention(q[:, :, None], kk, vv)[:, :, 0])
            x.addmm_(o.view(B, H * d), lw["wo"])
            _native.check(lib.ott_model_rmsnorm(x.data_ptr(), lw["n2"].data_ptr(), h.data_ptr(), B, D, cfg.eps, st))
            torch.mm(h, lw["wgu"], out=gu)
            _native.check(lib.ott_model_silu_mul(gu.data_ptr(), act.data_ptr(), B, cfg.mlp, st))
            x.addmm_(act, lw["wd"])
        _native.check(lib.ott_model_rmsnorm(x.data_ptr(), self.norm.data_ptr(), h.data_ptr(), B, D, cfg.eps, st))
        torch.mm(h, self.lm_head, out=bf["logits"])
        if self.track_exact and not graph:
            self.attn_l1.append(float(l1_sum) / cfg.n_layers)
        return bf["logits"]

    def _exact_l1(self, l, k, v, q, o, p):
        """Mean over (batch, head) of sum_d |o - exact| for layer l at position p: exact float32
        attention (attend_full_precision, attention.py:35-59) over the fp16 shadow rows."""
        cfg = self.cfg
        self.sk[l, :, :, p] = k
        self.sv[l, :, :, p] = v
        rep = cfg.n_heads // cfg.n_kv_heads
        kk = self.sk[l, :, :, : p + 1].float()
        vv = self.sv[l, :, :, : p + 1].float()
        if rep > 1:
            kk, vv = kk.repeat_interleave(rep, dim=1), vv.repeat_interleave(rep, dim=1)
        s = torch.einsum("bhd,bhtd->bht", q.float(), kk) / float(cfg.head_dim) ** 0.5
        ex = torch.einsum("bht,bhtd->bhd", torch.softmax(s.double(), dim=-1).float(), vv)
        return (o.float() - ex).abs().sum(-1).mean()

    @torch.no_grad()
    def decode(self, tokens: torch.Tensor) -> torch.Tensor:
        """One greedy step: tokens int64 [B] at position self.pos -> next tokens [B]."""
        if self.pos + 1 > self.max_tokens:
            raise ContractViolation("decoder is full")
        x = self.embed.index_select(0, tokens)
        logits = self._layers_step(x, self.pos, tok=tokens)
        if self.kv == "flash":
            self.seqlens.add_(1)
        self.pos += 1
        self.last_logits = logits.clone()
        return logits.argmax(-1)

    # ------------------------------------------------------------------ CUDA graph decode
    def _graph_body(self):
        """One decode step on static buffers: token ids g_tok, position g_pos (device),
        OTT decode steps with device token counters; writes g_next, advances g_pos."""
        self.g_x.copy_(self.embed.index_select(0, self.g_tok))
        logits = self._layers_step(self.g_x, 0, pos_dev=self.g_pos, graph=True, tok=self.g_tok)
        self.g_logits.copy_(logits)
        self.g_next.copy_(logits.argmax(-1))
        self.g_pos.add_(1)
        if self.kv == "flash":
            self.seqlens.add_(1)

    @torch.no_grad()
    def capture_decode_graph(self) -> None:
        """Capture one OTT decode step (all layers: GEMMs, RoPE, ring write, flush-if-due,
        attention, combine) in a CUDA graph; `decode_graph` then replays it per step."""
        if self.kv == "fp16":
            raise ContractViolation("graph decode needs device-side lengths (kv='ott' or 'flash')")
        cfg, B, dev = self.cfg, self.batch, self.device
        self.g_tok = torch.zeros(B, dtype=torch.int64, device=dev)
        self.g_next = torch.zeros(B, dtype=torch.int64, device=dev)
        self.g_pos = torch.full((1,), self.pos, dtype=torch.int64, device=dev)
        self.g_x = torch.zeros((B, cfg.hidden), dtype=torch.float16, device=dev)
        self._decode_buffers()
        self.g_logits = torch.zeros((B, cfg.vocab), dtype=torch.float16, device=dev)
        n_rep = cfg.n_heads // cfg.n_kv_heads
        caches = self.caches if self.kv == "ott" else []
        # splits sized for the longest context of the run; workspaces allocated before capture
        self.g_splits = [c.splits(n_rep) for c in caches]
        saved = []
        for c, s in zip(caches, self.g_splits):
            c.workspace(n_rep, s)
            c.sync_counters()
            saved.append((c.total_tokens, c.quantized_tokens))
        if self.kv == "flash":
            saved_len = self.seqlens.clone()
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._graph_body()
        for c, (t, q) in zip(caches, saved):  # capture ran the host side once, not the kernels
            c.total_tokens, c.quantized_tokens = t, q
        if self.kv == "flash":
            self.seqlens.copy_(saved_len)

    @torch.no_grad()
    def decode_graph(self, tokens: torch.Tensor) -> torch.Tensor:
        """`decode` through the captured graph (captured on first use)."""
        if self.graph is None:
            self.capture_decode_graph()
        if self.pos + 1 > self.max_tokens:
            raise ContractViolation("decoder is full")
        for c in (self.caches if self.kv == "ott" else []):
            c.advance_host_counts()  # checks capacity before the replay writes
        self.g_tok.copy_(tokens)
        self.graph.replay()
        self.pos += 1
        self.last_logits = self.g_logits
        return self.g_next.clone()

    @torch.no_grad()
    def generate(self, prompt: torch.Tensor, steps: int) -> torch.Tensor:
        """Prefill + `steps` greedy decode steps; returns generated ids [B, steps + 1]."""
        out = [self.prefill(prompt)]
        for _ in range(steps):
            out.append(self.decode(out[-1]))
        return torch.stack(out, dim=1)
