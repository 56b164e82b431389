"""Drop-ins for the reference's standalone pool/attention objects (kvtrace outlier.py:24-117,
attention.py:35-59) on the GPU.

The decode hot path never uses these: it runs the pool competition inside the flush kernels
and the mixed-tier attention in K2 (ott_flush.cu, ott_attend.cu). These objects exist so code
written against ``kvtrace.OutlierPool``, ``score_tokens``, ``OutlierEntry.from_rows`` and
``attend_full_precision`` finds the same names, arguments, results and ContractViolations.
The arithmetic runs in the library's kernels (ott_api.cu, C ABI ``ott_pool_rank``,
``ott_score_rows``, ``ott_attend_exact``); the host keeps only the entry bookkeeping.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .errors import ContractViolation
from .views import AttentionResult, OutlierEntry, require


def _dev():
    if not torch.cuda.is_available():
        raise _native.NativeError("no CUDA device: the pool and attention kernels need a GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def score_rows(keys) -> np.ndarray:
    """Per-row L1 norms in float64 (row_l1_norm, tensor.py:38-42) of a float32 (n, d) matrix."""
    k = np.ascontiguousarray(keys, dtype=np.float32)
    if k.ndim != 2 or k.shape[0] < 1:
        raise ContractViolation("score_tokens expects a non-empty 2-D key matrix")  # outlier.py:47-48
    dev = _dev()
    kt = torch.from_numpy(k).to(dev)
    out = torch.empty(k.shape[0], dtype=torch.float64, device=dev)
    _native.check(_native.lib().ott_score_rows(kt.data_ptr(), k.shape[0], k.shape[1], out.data_ptr(), _stream()))
    return out.cpu().numpy()


def score_tokens(keys) -> np.ndarray:
    """outlier.py:45-49."""
    return score_rows(keys)


def entry_from_rows(position: int, key, value) -> OutlierEntry:
    """OutlierEntry.from_rows (outlier.py:37-42): the score is the key row's float64 L1 norm."""
    k = np.asarray(key, dtype=np.float32)
    v = np.asarray(value, dtype=np.float32)
    return OutlierEntry(position=int(position), key=k, value=v, score=float(score_rows(k[None, :])[0]))



def _ranks(items) -> np.ndarray:
    """Ascending (score, position) rank of each item (outlier.py:52-54) on the GPU."""
    dev = _dev()
    s = torch.tensor([float(e.score) for e in items], dtype=torch.float64, device=dev)
    p = torch.tensor([int(e.position) for e in items], dtype=torch.int64, device=dev)
    r = torch.empty(len(items), dtype=torch.int32, device=dev)
    _native.check(_native.lib().ott_pool_rank(s.data_ptr(), p.data_ptr(), len(items), r.data_ptr(), _stream()))
    return r.cpu().numpy()


class OutlierPool:
    """The reference's outlier pool (outlier.py:57-117) with the competition ranked on the GPU.

    The pool holds the ``capacity`` lowest (score, position) tokens presented so far. A member
    that loses its slot is retired to ``aux`` while there is room, and a full ``aux`` freezes the
    pool: later updates change nothing."""

    def __init__(self, capacity: int, aux_capacity: int = 32, entries=None, aux=None, frozen: bool = False):
        if min(capacity, aux_capacity) < 0:
            raise ContractViolation("pool capacities must be nonnegative")  # outlier.py:75-76
        self.capacity, self.aux_capacity = capacity, aux_capacity
        self.entries = list(entries or ())
        self.aux = list(aux or ())
        self.frozen = bool(frozen) or len(self.aux) >= aux_capacity

    def __repr__(self) -> str:
        return (f"OutlierPool(capacity={self.capacity}, aux_capacity={self.aux_capacity}, "
                f"positions={sorted(self.positions)}, aux={len(self.aux)}, frozen={self.frozen})")

    @property
    def positions(self) -> set:
        return {e.position for e in self.entries}

    def update(self, candidates) -> tuple:
        """One competition round of the members and ``candidates``: returns (positions of the
        candidates that won a slot, former members that lost theirs, in member order)."""
        if self.frozen or self.capacity == 0:
            return set(), []
        candidates = list(candidates)
        taken = self.positions
        for c in candidates:  # outlier.py:96-100
            if c.position in taken:
                raise ContractViolation(f"duplicate position {c.position} in pool update")
            taken.add(c.position)
        field = self.entries + candidates
        if not field:
            return set(), []
        kept = np.argsort(_ranks(field), kind="stable")[: self.capacity]
        n_members = len(self.entries)
        kept_set = set(kept.tolist())
        won = {field[i].position for i in kept if i >= n_members}
        lost = [e for i, e in enumerate(self.entries) if i not in kept_set]
        self.entries = [field[i] for i in kept]
        self._retire(lost)
        return won, lost

    def _retire(self, lost) -> None:
        self.aux += lost[: max(0, self.aux_capacity - len(self.aux))]
        if len(self.aux) >= self.aux_capacity:
            self.frozen = True


def attend_full_precision(q, keys, values, with_weights: bool = True) -> AttentionResult:
    """attention.py:35-59 on the GPU (ott_attend_exact): scores = (K q) / f32(sqrt(d)) in
    float32, softmax in float64 (tensor.py:45-57), output = weights V in float32."""
    q = np.asarray(q, dtype=np.float32)
    keys = np.asarray(keys, dtype=np.float32)
    values = np.asarray(values, dtype=np.float32)
    require(q.ndim == 1, "query must be 1-D")
    require(keys.ndim == 2 and values.ndim == 2, "keys and values must be 2-D")
    require(keys.shape[0] == values.shape[0], "keys and values must cover the same tokens")
    require(keys.shape[1] == q.shape[0] and values.shape[1] == q.shape[0], "width mismatch between query and cache rows")
    require(keys.shape[0] > 0, "attention needs at least one cached token")
    n, d = keys.shape
    dev = _dev()
    qt = torch.from_numpy(np.ascontiguousarray(q)).to(dev)
    kt = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    vt = torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    out = torch.empty(d, dtype=torch.float32, device=dev)
    w = torch.empty(n, dtype=torch.float32, device=dev)
    s = torch.empty(n, dtype=torch.float32, device=dev)
    _native.check(_native.lib().ott_attend_exact(qt.data_ptr(), kt.data_ptr(), vt.data_ptr(), n, d, 1, out.data_ptr(),
                                                 w.data_ptr(), s.data_ptr(), _stream()))
    res = AttentionResult(output=out.cpu().numpy())
    if with_weights:
        res.weights = w.cpu().numpy()
        res.scores = s.cpu().numpy()
    return res
