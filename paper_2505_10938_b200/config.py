"""EngineConfig / MemoryBreakdown — same fields, defaults and validation as the
reference (kvtrace/cache.py:37-87)."""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ContractViolation


@dataclass(frozen=True)
class EngineConfig:
    """Quantization engine settings (cache.py:37-68). Defaults are the paper
    setting: 2-bit, G=128, R=32, N=3 outliers with layers 0/1 skipped, A=32."""

    bits: int = 2
    group_size: int = 128
    residual: int = 32
    outlier_num: int = 3
    skip_layers: tuple = (0, 1)
    aux_capacity: int = 32
    n_layers: int = 1
    n_heads: int = 1
    head_dim: int = 64

    def __post_init__(self):
        if not 1 <= self.bits <= 8:
            raise ContractViolation(f"bits must be in [1, 8], got {self.bits}")
        if self.group_size < 1:
            raise ContractViolation("group_size must be >= 1")
        if self.residual < 0 or self.outlier_num < 0 or self.aux_capacity < 0:
            raise ContractViolation("residual, outlier_num, aux_capacity must be >= 0")
        if self.n_layers < 1 or self.n_heads < 1 or self.head_dim < 1:
            raise ContractViolation("dimensions must be >= 1")

    def outlier_capacity(self, layer: int) -> int:
        """Pool capacity for one layer (0 on skipped layers), cache.py:66-68."""
        return 0 if layer in self.skip_layers else self.outlier_num


@dataclass(frozen=True)
class MemoryBreakdown:
    """Footprint in bits under fp16-equivalent accounting (cache.py:71-87)."""

    quantized_bits: int
    param_bits: int
    pending_bits: int
    pool_bits: int

    @property
    def total_bits(self) -> int:
        return self.quantized_bits + self.param_bits + self.pending_bits + self.pool_bits
