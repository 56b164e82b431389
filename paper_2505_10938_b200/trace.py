"""KVTRACE1 trace ingestion and GPU replay.

File format (the reference's trace.py:1-8, 68-121): 8-byte magic ``KVTRACE1``,
four little-endian uint32 (n_layers, n_heads, head_dim, seq_len), then for each
layer (major) and head (minor) the Q, K, V matrices, each seq_len x head_dim
row-major little-endian float32. Reading validates exactly as the reference
does and raises `TraceFormatError` with the same byte offsets.

`simulate` is the reference's `kvtrace simulate` replay (cli.py:189-236) on the
GPU: every (layer, head) is a unit of one OTTCache per layer; at each step t the
new K/V rows are appended (flushing groups as the reference does), q_t attends
through the OTT kernels, and the result is compared with exact attention over
the full-precision rows 0..t (attention.py:35-59) by the L1 error of the
outputs (attention.py:95-101), averaged over the caches. The product consumes
fp16, so traces must hold fp16-representable values (or be rounded with
``round_fp16=True``, which the reference does not do).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .config import EngineConfig
from .errors import ContractViolation, TraceFormatError

MAGIC = b"KVTRACE1"
_DIMS = ("n_layers", "n_heads", "head_dim", "seq_len")  # header field order
_HEADER = struct.Struct("<4I")
_PAYLOAD = np.dtype("<f4")
FP16_BITS = 16


class TraceHeader(tuple):
    """The four header fields (n_layers, n_heads, head_dim, seq_len); each must fit a non-zero
    uint32 (ContractViolation otherwise). Compares equal to a tuple of the same values."""

    __slots__ = ()

    def __new__(cls, n_layers, n_heads, head_dim, seq_len):
        vals = tuple(int(x) for x in (n_layers, n_heads, head_dim, seq_len))
        for name, val in zip(_DIMS, vals):
            if val < 1 or val > 0xFFFFFFFF:
                raise ContractViolation(f"{name} must be in [1, 2**32), got {val}")
        return super().__new__(cls, vals)

    n_layers = property(lambda self: self[0])
    n_heads = property(lambda self: self[1])
    head_dim = property(lambda self: self[2])
    seq_len = property(lambda self: self[3])

    @property
    def matrix_shape(self):  # (layers, heads, seq, dim): the shape of Trace.q / .k / .v
        return (self[0], self[1], self[3], self[2])

    @property
    def file_bytes(self) -> int:
        return len(MAGIC) + _HEADER.size + self[0] * self[1] * 3 * self[3] * self[2] * _PAYLOAD.itemsize


class Trace:
    """Q/K/V of every (layer, head), held as one float32 block [layers, heads, 3, seq, dim] in
    the file's order (layer-major, head-minor, Q K V per head), so a file maps onto it without a
    copy per matrix; `q`, `k`, `v` are views of shape (layers, heads, seq, dim)."""

    def __init__(self, header: TraceHeader, q, k, v):
        self.header = header
        want = header.matrix_shape
        mats = []
        for name, m in (("q", q), ("k", k), ("v", v)):
            m = np.asarray(m, dtype=np.float32)
            if m.shape != want:
                raise ContractViolation(f"{name} must have shape {want}, got {m.shape}")
            mats.append(m)
        self.qkv = np.stack(mats, axis=2)

    @classmethod
    def _from_block(cls, header: TraceHeader, qkv: np.ndarray) -> "Trace":
        t = cls.__new__(cls)
        t.header, t.qkv = header, qkv
        return t

    q = property(lambda self: self.qkv[:, :, 0])
    k = property(lambda self: self.qkv[:, :, 1])
    v = property(lambda self: self.qkv[:, :, 2])


def write_trace(path, trace: Trace) -> None:
    """Serialize in the KVTRACE1 format (bit-exact round trip): header, then the qkv block."""
    with open(path, "wb") as f:
        f.write(MAGIC + _HEADER.pack(*trace.header))
        f.write(trace.qkv.astype(_PAYLOAD, copy=False).tobytes())


def read_trace(path) -> Trace:
    """Parse a KVTRACE1 file. Damage raises TraceFormatError at the byte offsets (and with the
    messages) the format's reference reader uses, checked in file order."""
    with open(path, "rb") as f:
        data = f.read()
    size, hdr_end = len(data), len(MAGIC) + _HEADER.size
    if size < len(MAGIC):
        raise TraceFormatError("truncated file: magic missing", offset=size)
    if not data.startswith(MAGIC):
        raise TraceFormatError("bad magic", offset=0)
    if size < hdr_end:
        raise TraceFormatError("truncated file: header incomplete", offset=size)
    fields = _HEADER.unpack_from(data, len(MAGIC))
    zero = next((i for i, val in enumerate(fields) if val == 0), None)
    if zero is not None:
        raise TraceFormatError(f"{_DIMS[zero]} must be >= 1, got 0", offset=len(MAGIC))
    header = TraceHeader(*fields)
    expected = header.file_bytes
    if size != expected:
        raise (TraceFormatError("truncated file: payload incomplete", offset=size) if size < expected else
               TraceFormatError("trailing bytes after payload", offset=expected))
    L, H, d, T = fields
    block = np.frombuffer(data, dtype=_PAYLOAD, offset=hdr_end).reshape(L, H, 3, T, d)
    return Trace._from_block(header, block.astype(np.float32))


@dataclass
class SimulateResult:
    step_errors: np.ndarray          # mean L1(mixed, exact) over caches, per step
    usage: dict                      # summed MemoryBreakdown fields + total_bits
    ratio_vs_fp16: float

    @property
    def aggregate_l1_error(self) -> float:
        return float(self.step_errors.mean())


def simulate(trace: Trace, config: EngineConfig, device=None, round_fp16: bool = False) -> SimulateResult:
    """GPU `kvtrace simulate` (mode ott/baseline via config.outlier_num)."""
    import torch

    from .cache import OTTCache

    h = trace.header
    L, H, d, T = h.n_layers, h.n_heads, h.head_dim, h.seq_len
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    arrs = []
    for name in ("q", "k", "v"):
        a = getattr(trace, name)
        a16 = a.astype(np.float16)
        if not round_fp16 and not np.array_equal(a16.astype(np.float32), a):
            raise ContractViolation(f"trace {name} is not fp16-representable (pass round_fp16=True)")
        arrs.append(torch.from_numpy(a16).to(dev))
    q, k, v = arrs  # [L, H, T, d] fp16
    caches = [OTTCache(config, 1, H, T, layer=l, device=dev) for l in range(L)]
    kf, vf = k.double(), v.double()
    scale = 1.0 / float(np.float32(np.sqrt(np.float32(d))))
    errs = torch.zeros(T, dtype=torch.float64, device=dev)
    out = torch.empty((L, H, d), dtype=torch.float16, device=dev)
    for t in range(T):
        for l, c in enumerate(caches):
            c.append(k[l, :, t][None], v[l, :, t][None])
            c.attend(q[l, :, t][None], out=out[l][None])
        # exact attention over rows 0..t for every (layer, head) (attention.py:35-59)
        s = torch.einsum("lhtd,lhd->lht", kf[:, :, : t + 1], q[:, :, t].double()) * scale
        w = torch.softmax(s, dim=-1)
        exact = torch.einsum("lht,lhtd->lhd", w, vf[:, :, : t + 1])
        errs[t] = (out.double() - exact).abs().sum(-1).mean()
    usage = {"quantized_bits": 0, "param_bits": 0, "pending_bits": 0, "pool_bits": 0}
    for c in caches:
        for hh in range(H):
            mu = c.memory_usage(0, hh)
            for key in usage:
                usage[key] += getattr(mu, key)
    usage["total_bits"] = sum(usage.values())
    fp16_bits = L * H * 2 * T * d * FP16_BITS
    return SimulateResult(errs.cpu().numpy(), usage, fp16_bits / usage["total_bits"])


def main(argv=None) -> int:
    """`python -m paper_2505_10938_b200.trace TRACE [--bits 2 --group-size 128 ...]`:
    prints the reference simulate summary (cli.py:222-229)."""
    import argparse

    ap = argparse.ArgumentParser(prog="paper_2505_10938_b200.trace")
    ap.add_argument("trace")
    ap.add_argument("--bits", type=int, default=2)
    ap.add_argument("--group-size", type=int, default=128)
    ap.add_argument("--residual", type=int, default=32)
    ap.add_argument("--outlier-num", type=int, default=3)
    ap.add_argument("--aux-capacity", type=int, default=32)
    ap.add_argument("--skip-layers", default="0,1")
    ap.add_argument("--mode", choices=["ott", "baseline"], default="ott")
    ap.add_argument("--round-fp16", action="store_true")
    ap.add_argument("--out", help="per-step CSV path")
    a = ap.parse_args(argv)
    tr = read_trace(a.trace)
    skip = tuple(int(x) for x in a.skip_layers.split(",") if x.strip())
    cfg = EngineConfig(bits=a.bits, group_size=a.group_size, residual=a.residual,
                       outlier_num=0 if a.mode == "baseline" else a.outlier_num, skip_layers=skip,
                       aux_capacity=a.aux_capacity, n_layers=tr.header.n_layers, n_heads=tr.header.n_heads,
                       head_dim=tr.header.head_dim)
    r = simulate(tr, cfg, round_fp16=a.round_fp16)
    if a.out:
        with open(a.out, "w") as f:
            f.write("step,l1_error\n")
            for t, e in enumerate(r.step_errors):
                f.write(f"{t},{float(e)!r}\n")
    print(f"mode={a.mode} steps={tr.header.seq_len} aggregate_l1_error={r.aggregate_l1_error:.6g}")
    for key in ("quantized_bits", "param_bits", "pending_bits", "pool_bits", "total_bits"):
        print(f"{key}={r.usage[key]}")
    print(f"ratio_vs_fp16={r.ratio_vs_fp16:.6g}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
