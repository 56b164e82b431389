"""Host-side views of GPU cache state in the reference's own types.

These mirror kvtrace's value types (quant.py:34-163, outlier.py:24-117,
attention.py:26-32) so a reference user (or a parity test) can inspect one
(layer, head) unit of the batched GPU cache exactly as it would inspect a
``kvtrace.TieredCache``. They are read-only snapshots copied from device
memory; nothing here computes on the hot path.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from .errors import ContractViolation

FP16_BITS = 16  # quant.py:31


class GroupAxis(enum.Enum):
    PER_CHANNEL = "per_channel"
    PER_TOKEN = "per_token"


@dataclass(frozen=True)
class QuantParams:
    """quant.py:39-56. x_min/step are the exact float64 values when the cache
    keeps float64 params (keep_f64_params=True), else the stored float32."""

    x_min: float
    step: float
    bits: int


def unpack_codes(data: bytes, bits: int, count: int) -> np.ndarray:
    """The `count` codes of a little-endian (LSB-first) stream of `bits`-bit fields, as int64
    (the layout of the reference's pack_codes, quant.py:241-273). Code i starts at bit i * bits;
    a field of <= 8 bits lies inside the 16-bit window starting at its first byte."""
    if count == 0:
        return np.zeros(0, dtype=np.int64)
    window = np.frombuffer(bytes(data) + b"\0", dtype=np.uint8).astype(np.int64)
    first = np.arange(count, dtype=np.int64) * bits
    lo = first >> 3
    return ((window[lo] | (window[lo + 1] << 8)) >> (first & 7)) & ((1 << bits) - 1)


@dataclass
class QuantizedBlock:
    """quant.py:114-163: packed codes (reference byte order) + per-line params."""

    codes: bytes
    group_axis: GroupAxis
    params: list
    n_tokens: int
    n_channels: int
    bits: int

    @property
    def code_bits(self) -> int:
        return self.n_tokens * self.n_channels * self.bits

    @property
    def param_bits(self) -> int:
        return len(self.params) * 2 * FP16_BITS

    def code_matrix(self) -> np.ndarray:
        return unpack_codes(self.codes, self.bits, self.n_tokens * self.n_channels).reshape(self.n_tokens,
                                                                                           self.n_channels)

    def to_matrix(self) -> np.ndarray:
        """codes * step + x_min in float64 per line (a column per channel, a row per token),
        rounded once to float32 (quant.py:105-111, 154-163)."""
        line = np.array([(p.step, p.x_min) for p in self.params], dtype=np.float64)
        bcast = (1, -1) if self.group_axis is GroupAxis.PER_CHANNEL else (-1, 1)
        return (self.code_matrix() * line[:, 0].reshape(bcast) + line[:, 1].reshape(bcast)).astype(np.float32)


@dataclass
class OutlierEntry:
    """outlier.py:24-42."""

    position: int
    key: np.ndarray
    value: np.ndarray
    score: float

    @classmethod
    def from_rows(cls, position: int, key, value) -> "OutlierEntry":
        """outlier.py:37-42 (the float64 L1 score is computed by the library, pool.py)."""
        from .pool import entry_from_rows

        return entry_from_rows(position, key, value)


@dataclass
class OutlierPoolView:
    """Snapshot of one unit's OutlierPool (outlier.py:57-117)."""

    capacity: int
    aux_capacity: int
    entries: list = field(default_factory=list)
    aux: list = field(default_factory=list)
    frozen: bool = False

    @property
    def positions(self) -> set:
        return {e.position for e in self.entries}


@dataclass
class AttentionResult:
    """attention.py:26-32. ``weights``/``scores`` are filled only when asked
    for (they cost a T-length D2H copy per call)."""

    output: np.ndarray
    weights: np.ndarray | None = None
    scores: np.ndarray | None = None


def require(cond: bool, msg: str) -> None:
    if not cond:
        raise ContractViolation(msg)
