"""B200-native OTT quantized-KV decode path (arXiv 2505.10938), drop-in for the
reference package's cache/attention API (kvtrace: EngineConfig, TieredCache,
attend_mixed, ContractViolation, MemoryBreakdown).

Hot path = hand-written sm_100a CUDA kernels behind the C ABI in
include/ott_b200.h (libott_b200.so), driven from PyTorch streams. There is no
CPU fallback.
"""

from .config import EngineConfig, MemoryBreakdown
from .errors import ContractViolation, NativeError
from .views import AttentionResult, GroupAxis, OutlierEntry, OutlierPoolView, QuantizedBlock, QuantParams

__all__ = [
    "AttentionResult", "ContractViolation", "EngineConfig", "GroupAxis", "MemoryBreakdown", "NativeError",
    "OTTCache", "OutlierEntry", "OutlierPool", "OutlierPoolView", "QuantParams", "QuantizedBlock", "TieredCache",
    "attend_full_precision", "attend_mixed", "score_tokens",
]


def __getattr__(name):  # torch-dependent pieces load lazily
    if name in ("OTTCache", "TieredCache", "attend_mixed", "UnitView"):
        from . import cache

        return getattr(cache, name)
    if name in ("OutlierPool", "attend_full_precision", "score_tokens"):
        from . import pool

        return getattr(pool, name)
    raise AttributeError(name)
