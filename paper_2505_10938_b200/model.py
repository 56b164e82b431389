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
  torch SDPA: the accuracy/throughput baseline the paper compares against.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .cache import OTTCache
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
                 ott: EngineConfig | None = None, device=None, seed: int = 0):
        if kv not in ("ott", "fp16"):
            raise ContractViolation("kv must be 'ott' or 'fp16'")
        self.cfg, self.batch, self.max_tokens, self.kv = cfg, batch, max_tokens, kv
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dev, H, Hkv, d, D = self.device, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.hidden
        g = torch.Generator(device=dev).manual_seed(seed)

        def w(*shape):
            return (torch.randn(shape, generator=g, device=dev, dtype=torch.float32) * 0.02).half()

        self.embed = w(cfg.vocab, D)
        self.layers = []
        for _ in range(cfg.n_layers):
            self.layers.append({
                "wqkv": w(D, (H + 2 * Hkv) * d), "wo": w(H * d, D), "wgu": w(D, 2 * cfg.mlp), "wd": w(cfg.mlp, D),
                "n1": torch.ones(D, dtype=torch.float16, device=dev), "n2": torch.ones(D, dtype=torch.float16, device=dev),
            })
        self.norm = torch.ones(D, dtype=torch.float16, device=dev)
        self.lm_head = w(D, cfg.vocab)
        self.cos, self.sin = rope_tables(d, max_tokens, cfg.rope_theta, dev)
        if kv == "ott":
            ott = ott or EngineConfig(bits=2, group_size=32, residual=128, outlier_num=32, aux_capacity=32,
                                      n_layers=cfg.n_layers, n_heads=Hkv, head_dim=d)
            self.caches = [OTTCache(ott, batch, Hkv, max_tokens, layer=l, device=dev) for l in range(cfg.n_layers)]
        else:
            self.k_cache = torch.zeros((cfg.n_layers, batch, Hkv, max_tokens, d), dtype=torch.float16, device=dev)
            self.v_cache = torch.zeros_like(self.k_cache)
        self.pos = 0
        self.graph = None

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
            kk = k.repeat_interleave(rep, dim=1) if rep > 1 else k
            vv = v.repeat_interleave(rep, dim=1) if rep > 1 else v
            o = F.scaled_dot_product_attention(q, kk, vv, is_causal=True)
            if self.kv == "ott":
                self.caches[l].update(k.contiguous(), v)
            else:
                self.k_cache[l, :, :, :T] = k
                self.v_cache[l, :, :, :T] = v
            x = x + o.transpose(1, 2).reshape(B, T, -1) @ lw["wo"]
            x = x + self._mlp(x, lw)
        self.pos = T
        self.last_logits = self._logits(x[:, -1])
        return self.last_logits.argmax(-1)

    @torch.no_grad()
    def decode(self, tokens: torch.Tensor) -> torch.Tensor:
        """One greedy step: tokens int64 [B] at position self.pos -> next tokens [B]."""
        cfg, B = self.cfg, self.batch
        if self.pos + 1 > self.max_tokens:
            raise ContractViolation("decoder is full")
        x = self.embed[tokens][:, None]  # [B, 1, D]
        p = self.pos
        for l, lw in enumerate(self.layers):
            q, k, v = self._qkv(x, lw, p)  # [B, h, 1, d]
            if self.kv == "ott":
                c = self.caches[l]
                c.append(k[:, :, 0].contiguous(), v[:, :, 0].contiguous())
                o = c.attend(q[:, :, 0].contiguous())  # [B, H, d]
            else:
                self.k_cache[l, :, :, p] = k[:, :, 0]
                self.v_cache[l, :, :, p] = v[:, :, 0]
                rep = cfg.n_heads // cfg.n_kv_heads
                kk, vv = self.k_cache[l, :, :, : p + 1], self.v_cache[l, :, :, : p + 1]
                if rep > 1:
                    kk, vv = kk.repeat_interleave(rep, dim=1), vv.repeat_interleave(rep, dim=1)
                o = F.scaled_dot_product_attention(q, kk, vv)[:, :, 0]
            x = x + o.reshape(B, 1, -1) @ lw["wo"]
            x = x + self._mlp(x, lw)
        self.pos = p + 1
        self.last_logits = self._logits(x[:, 0])
        return self.last_logits.argmax(-1)

    # ------------------------------------------------------------------ CUDA graph decode
    def _graph_body(self):
        """One decode step on static buffers: token ids g_tok, position g_pos (device),
        OTT decode steps with device token counters; writes g_next, advances g_pos."""
        cfg, B = self.cfg, self.batch
        x = self.embed.index_select(0, self.g_tok)[:, None]
        cos, sin = self.cos.index_select(0, self.g_pos), self.sin.index_select(0, self.g_pos)
        for l, lw in enumerate(self.layers):
            q, k, v = self._qkv(x, lw, 0, cos, sin)
            c = self.caches[l]
            self.g_q[l].copy_(q[:, :, 0])
            c.decode_step(k[:, :, 0], v[:, :, 0], self.g_q[l], self.g_o[l], self.g_splits[l])
            x = x + self.g_o[l].view(B, 1, -1) @ lw["wo"]
            x = x + self._mlp(x, lw)
        self.g_logits.copy_(self._logits(x[:, 0]))
        self.g_next.copy_(self.g_logits.argmax(-1))
        self.g_pos.add_(1)

    @torch.no_grad()
    def capture_decode_graph(self) -> None:
        """Capture one OTT decode step (all layers: GEMMs, RoPE, ring write, flush-if-due,
        attention, combine) in a CUDA graph; `decode_graph` then replays it per step."""
        if self.kv != "ott":
            raise ContractViolation("graph decode needs the OTT cache (device token counters)")
        cfg, B, dev = self.cfg, self.batch, self.device
        self.g_tok = torch.zeros(B, dtype=torch.int64, device=dev)
        self.g_next = torch.zeros(B, dtype=torch.int64, device=dev)
        self.g_pos = torch.full((1,), self.pos, dtype=torch.int64, device=dev)
        self.g_q = torch.zeros((cfg.n_layers, B, cfg.n_heads, cfg.head_dim), dtype=torch.float16, device=dev)
        self.g_o = torch.zeros_like(self.g_q)
        self.g_logits = torch.zeros((B, cfg.vocab), dtype=torch.float16, device=dev)
        n_rep = cfg.n_heads // cfg.n_kv_heads
        # splits sized for the longest context of the run; workspaces allocated before capture
        self.g_splits = [c.splits(n_rep) for c in self.caches]
        saved = []
        for c, s in zip(self.caches, self.g_splits):
            c.workspace(n_rep, s)
            c.sync_counters()
            saved.append((c.total_tokens, c.quantized_tokens))
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._graph_body()
        for c, (t, q) in zip(self.caches, saved):  # capture ran the host side once, not the kernels
            c.total_tokens, c.quantized_tokens = t, q

    @torch.no_grad()
    def decode_graph(self, tokens: torch.Tensor) -> torch.Tensor:
        """`decode` through the captured graph (captured on first use)."""
        if self.graph is None:
            self.capture_decode_graph()
        if self.pos + 1 > self.max_tokens:
            raise ContractViolation("decoder is full")
        for c in self.caches:
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
