"""Seeded synthetic KV workloads of BASELINE.json's configs, generated on the GPU.

BASELINE names no dataset: every config is "synthetic KV with the outlier
structure of config 0": K ~ N(0,1) with 4 seeded outlier channels
per (batch, kv-head) unit scaled x15, and seeded outlier tokens whose values in
those channels are scaled x0.05; V ~ N(0,1); q ~ N(0,1). All values fp16.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Workload:
    name: str
    n_layers: int
    batch: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    context: int
    group_size: int = 32
    residual: int = 128
    outlier_num: int = 32
    aux_capacity: int = 32
    skip_layers: tuple = ()
    bits: int = 2

    @property
    def n_rep(self) -> int:
        return self.n_q_heads // self.n_kv_heads


WORKLOADS = {
    # BASELINE configs[0]: single layer, B=1, 32 heads, T=1024
    "c0": Workload("config0-single-layer-B1-H32-T1024", 1, 1, 32, 32, 128, 1024),
    # configs[2]: streaming stress, single layer, B=4, H=32, prefill 32768
    "c2": Workload("config2-stream-B4-H32-T32768", 1, 4, 32, 32, 128, 32768),
    # configs[3]: Llama-3-8B GQA sweep corner (largest point)
    "c3": Workload("config3-llama3-8b-gqa-B64-T8192", 1, 64, 32, 8, 128, 8192),
    "c3s": Workload("config3-llama3-8b-gqa-B16-T4096", 1, 16, 32, 8, 128, 4096),
    # configs[4]: Llama-3-70B-shaped KV cache, 80 layers, paper default skip_layers (0, 1)
    "c4": Workload("config4-llama3-70b-kv-80L-B128-Hq64-Hkv8-T16384", 80, 128, 64, 8, 128, 16384,
                   skip_layers=(0, 1)),
}


def _unit_structure(gen: torch.Generator, U: int, d: int, n_ch: int, device) -> torch.Tensor:
    """Per-unit channel scale vector [U, d]: 15 on n_ch seeded channels, else 1."""
    ch = torch.rand((U, d), generator=gen, device=device).argsort(dim=1)[:, :n_ch]
    scale = torch.ones((U, d), device=device)
    scale.scatter_(1, ch, 15.0)
    return scale


def fill_prefill(gen: torch.Generator, k_out: torch.Tensor, v_out: torch.Tensor, n_out_tok: int = 8,
                 chunk_units: int = 64) -> torch.Tensor:
    """Fill fp16 k_out/v_out [B, H, T, d] with the config-0 recipe; returns the
    per-unit channel scale [U, d] so decode rows can follow the same structure."""
    B, H, T, d = k_out.shape
    U = B * H
    dev = k_out.device
    scale = _unit_structure(gen, U, d, 4, dev)
    kf = k_out.view(U, T, d)
    vf = v_out.view(U, T, d)
    for u0 in range(0, U, chunk_units):
        u1 = min(U, u0 + chunk_units)
        n = u1 - u0
        k = torch.randn((n, T, d), generator=gen, device=dev) * scale[u0:u1, None, :]
        tok = torch.rand((n, T), generator=gen, device=dev).argsort(dim=1)[:, :n_out_tok]
        tmask = torch.zeros((n, T), dtype=torch.bool, device=dev)
        tmask.scatter_(1, tok, True)
        damp = torch.where(tmask[:, :, None] & (scale[u0:u1, None, :] > 1.0), 0.05, 1.0)
        kf[u0:u1] = (k * damp).half()
        vf[u0:u1] = torch.randn((n, T, d), generator=gen, device=dev).half()
    return scale


def decode_rows(gen: torch.Generator, scale: torch.Tensor, B: int, H: int, outlier_rate: float = 0.008):
    """One new token per unit with the same channel structure; a fraction of
    tokens are outlier tokens (x0.05 in the outlier channels)."""
    U, d = scale.shape
    dev = scale.device
    k = torch.randn((U, d), generator=gen, device=dev) * scale
    hit = torch.rand((U, 1), generator=gen, device=dev) < outlier_rate
    k = torch.where(hit & (scale > 1.0), k * 0.05, k)
    v = torch.randn((U, d), generator=gen, device=dev)
    return k.half().view(B, H, d), v.half().view(B, H, d)
