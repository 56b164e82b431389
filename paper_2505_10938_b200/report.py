"""Compression-ratio curve on the GPU cache (reference report.py:159-216).

`ratio_curve` replays one representative unit (the lowest layer with an active
outlier pool, as the reference picks it) with N(0, 1) rows and snapshots the
cache's memory accounting (cache.py:188-203) at ascending lengths. The product
consumes fp16, so rows are rounded to fp16 (the reference keeps float32 rows);
bit counts depend on the data only through the pool/aux occupancy.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import EngineConfig
from .errors import ContractViolation

FP16_BITS = 16


@dataclass(frozen=True)
class ExperimentRow:  # report.py ExperimentRow fields used by ratio_curve
    mode: str
    bits: int
    group_size: int
    residual: int
    outlier_num: int
    seq_len: int
    l1_output_error: float | None
    total_bits: int
    ratio_vs_fp16: float


def ratio_curve(config: EngineConfig, seq_lens, *, layer: int | None = None, seed: int = 0, device=None):
    import torch

    from .cache import OTTCache

    seq_lens = list(seq_lens)
    if seq_lens != sorted(seq_lens) or any(s < 1 for s in seq_lens):
        raise ContractViolation("seq_lens must be positive and sorted ascending")
    if layer is None:
        layer = 0
        while layer in config.skip_layers:
            layer += 1
    d, T = config.head_dim, seq_lens[-1]
    cache = OTTCache(config, 1, 1, T, layer=layer, device=device)
    mode = "ott" if cache.N > 0 else "baseline"
    rows = np.random.default_rng(seed).standard_normal((T, 2, d)).astype(np.float16)  # k_t, v_t per token
    kv = torch.from_numpy(rows).to(cache.device)
    out, tok = [], 0
    for target in seq_lens:
        if target > tok:
            cache.update(kv[None, None, tok:target, 0].contiguous(), kv[None, None, tok:target, 1].contiguous())
            tok = target
        u = cache.memory_usage()
        out.append(ExperimentRow(mode, config.bits, config.group_size, config.residual, cache.N, target, None,
                                 u.total_bits, 2 * target * d * FP16_BITS / u.total_bits))
    return out
