"""KVTRACE1 ingestion (reference trace.py:68-121) pinned by a file the reference
itself wrote, damage handling with the reference's byte offsets, and the GPU
`simulate` replay against the reference's per-step L1 errors (cli.py:189-236)."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2505_10938_b200.errors import TraceFormatError
from paper_2505_10938_b200.trace import Trace, TraceHeader, read_trace, write_trace


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "trace.npz"))


def test_reads_reference_written_file_and_writes_it_back(tmp_path, g):
    p = tmp_path / "t.kvt"
    p.write_bytes(g["tiny_bytes"].tobytes())
    tr = read_trace(p)
    assert tr.header == TraceHeader(1, 2, 4, 3)
    for name in ("q", "k", "v"):
        np.testing.assert_array_equal(getattr(tr, name), g["tiny_" + name])
    out = tmp_path / "w.kvt"
    write_trace(out, tr)
    assert out.read_bytes() == g["tiny_bytes"].tobytes()


def test_round_trip_random(tmp_path):
    rng = np.random.default_rng(0)
    tr = Trace(TraceHeader(2, 3, 8, 5), *(rng.standard_normal((2, 3, 5, 8)).astype(np.float32) for _ in range(3)))
    write_trace(tmp_path / "r.kvt", tr)
    back = read_trace(tmp_path / "r.kvt")
    for name in ("q", "k", "v"):
        assert np.array_equal(getattr(back, name), getattr(tr, name))


@pytest.mark.parametrize("case", ["short_magic", "bad_magic", "short_header", "zero_dim", "short_payload",
                                  "trailing"])
def test_damage_offsets(tmp_path, g, case):
    raw = g["tiny_bytes"].tobytes()
    expected_len = 8 + 16 + 1 * 2 * 3 * 3 * 4 * 4
    assert len(raw) == expected_len
    data, off = {
        "short_magic": (raw[:5], 5),
        "bad_magic": (b"KVTRACE2" + raw[8:], 0),
        "short_header": (raw[:13], 13),
        "zero_dim": (raw[:8] + struct.pack("<4I", 1, 0, 4, 3) + raw[24:], 8),
        "short_payload": (raw[:-7], expected_len - 7),
        "trailing": (raw + b"\0\0", expected_len),
    }[case]
    p = tmp_path / "d.kvt"
    p.write_bytes(data)
    with pytest.raises(TraceFormatError) as e:
        read_trace(p)
    assert e.value.offset == off


@pytest.mark.gpu
def test_gpu_simulate_matches_reference_replay(g):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10938_b200 import EngineConfig
    from paper_2505_10938_b200.trace import simulate

    q, k, v = (g[n].astype(np.float32) for n in ("q", "k", "v"))
    L, H, T, d = q.shape
    G, R, N, A = (int(x) for x in g["cfg"])
    cfg = EngineConfig(bits=2, group_size=G, residual=R, outlier_num=N, skip_layers=(), aux_capacity=A,
                       n_layers=L, n_heads=H, head_dim=d)
    res = simulate(Trace(TraceHeader(L, H, d, T), q, k, v), cfg)
    ref = g["step_errors"]
    assert [res.usage[k_] for k_ in ("quantized_bits", "param_bits", "pending_bits", "pool_bits")] == \
        g["usage"].tolist()
    err = np.abs(res.step_errors - ref)
    assert (err <= 0.02 * ref + 0.05).all(), float(err.max())
    assert abs(res.aggregate_l1_error - ref.mean()) <= 0.005 * ref.mean()
