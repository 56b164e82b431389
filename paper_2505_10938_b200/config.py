"""Engine configuration and the memory accounting record: the drop-in surface of the
reference's `EngineConfig` / `MemoryBreakdown` (kvtrace/cache.py:37-87). Field names,
defaults, the per-layer pool rule and the ContractViolation cases are the reference's
contract; the implementation here is table-driven."""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

from .errors import ContractViolation


@dataclass(frozen=True)
class EngineConfig:
    """Quantization settings of one cache. The defaults are the paper's setting: 2-bit codes,
    groups of 128 tokens, a 32-token full-precision window, a pool of 3 outlier tokens per
    (layer, head) that is off on layers 0 and 1, and an auxiliary pool of 32."""

    bits: int = 2                 # code width, 1..8 (quant.py:53-54)
    group_size: int = 128         # G: tokens quantized together
    residual: int = 32            # R: newest tokens kept in full precision
    outlier_num: int = 3          # N: outlier-pool capacity on pooled layers
    skip_layers: tuple = (0, 1)   # layers without a pool
    aux_capacity: int = 32        # A: auxiliary (evicted-entry) pool
    n_layers: int = 1
    n_heads: int = 1
    head_dim: int = 64

    def __post_init__(self):
        for broken, message in (
            (not 1 <= self.bits <= 8, f"bits must be in [1, 8], got {self.bits}"),
            (self.group_size < 1, "group_size must be >= 1"),
            (min(self.residual, self.outlier_num, self.aux_capacity) < 0,
             "residual, outlier_num, aux_capacity must be >= 0"),
            (min(self.n_layers, self.n_heads, self.head_dim) < 1, "dimensions must be >= 1"),
        ):
            if broken:
                raise ContractViolation(message)

    def outlier_capacity(self, layer: int) -> int:
        """N for `layer`, 0 where pooling is skipped (cache.py:66-68)."""
        return self.outlier_num * (layer not in self.skip_layers)


class MemoryBreakdown(NamedTuple):
    """A cache's footprint in bits (fp16-equivalent accounting, cache.py:71-87 / 188-203): codes
    at their width, two 16-bit parameters per quantized line, 16 bits per full-precision value
    (pending window, outlier and aux pools)."""

    quantized_bits: int
    param_bits: int
    pending_bits: int
    pool_bits: int

    @property
    def total_bits(self) -> int:
        return sum(self)
