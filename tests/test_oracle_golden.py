"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference itself
(tests/golden/make_golden.py imports /root/reference/pkg/src/kvtrace)."""

import os

import numpy as np
import pytest

import oracle

from conftest import GOLDEN


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def test_quantize_line_matches_reference_bit_exact():
    g = load("quant_lines.npz")
    offs = g["offsets"]
    for i in range(len(g["bits"])):
        x = g["x"][offs[i]:offs[i + 1]]
        codes, mn, st = oracle.quantize_line(x, int(g["bits"][i]))
        assert mn == g["x_min"][i] and st == g["step"][i], i
        np.testing.assert_array_equal(codes, g["codes"][offs[i]:offs[i + 1]])


def test_quantize_line_kats():
    # tests/test_quant.py:35-50 (reference unit-test examples)
    codes, mn, st = oracle.quantize_line([0.0, 1.0, 2.0, 3.0], 2)
    assert st == 1.0 and codes.tolist() == [0, 1, 2, 3]
    codes, mn, st = oracle.quantize_line([5.0, 5.0, 5.0], 4)
    assert st == 0.0 and mn == 5.0 and codes.tolist() == [0, 0, 0]
    codes, mn, st = oracle.quantize_line([0.0, 0.5, 1.0], 1)
    assert st == 1.0 and codes.tolist() == [0, 0, 1]
    with pytest.raises(oracle.OracleError):
        oracle.quantize_line([1.0, float("nan")], 2)
    with pytest.raises(oracle.OracleError):
        oracle.quantize_line([1.0, 2.0], 9)


def test_pack_matches_reference():
    g = load("pack.npz")
    for bits in range(1, 9):
        packed = oracle.pack_codes(g[f"codes_{bits}"], bits)
        assert packed == g[f"packed_{bits}"].tobytes()
        np.testing.assert_array_equal(oracle.unpack_codes(packed, bits, g[f"codes_{bits}"].size), g[f"codes_{bits}"])
    assert oracle.pack_codes([0, 1, 2, 3], 2) == g["kat_a"].tobytes() == b"\xe4"
    assert oracle.pack_codes([1, 0, 0, 0, 0, 0, 0, 3], 2) == g["kat_b"].tobytes() == b"\x01\xc0"
    with pytest.raises(oracle.OracleError):
        oracle.pack_codes([4], 2)


def test_pool_streams_match_reference():
    """OutlierPool.update streams replayed through the oracle cache: a key row
    [s, 0, 0, 0] has L1 score s, exactly as the golden generator built them."""
    g = load("pool_streams.npz")
    n = int(g["n"])
    i = 0
    while i < n:
        cap, aux_cap = int(g[f"{i}_cap"]), int(g[f"{i}_aux_cap"])
        gsize = g[f"{i}_scores"].size
        c = oracle.OracleCache(bits=2, group_size=gsize, residual=0, capacity=cap, aux_capacity=aux_cap, head_dim=4)
        while i < n and int(g[f"{i}_cap"]) == cap and int(g[f"{i}_aux_cap"]) == aux_cap \
                and g[f"{i}_scores"].size == gsize and (int(g[f"{i}_base"]) == c.total_tokens):
            before = set(c.substituted_positions.tolist())
            for s in g[f"{i}_scores"]:
                c.append(np.array([s, 0, 0, 0], np.float32), np.zeros(4, np.float32))
            pe = c.pool_entries()
            np.testing.assert_array_equal(pe["position"], g[f"{i}_entries"])
            np.testing.assert_array_equal(c.aux_entries()["position"], g[f"{i}_aux"])
            assert c.frozen == bool(g[f"{i}_frozen"])
            sel = sorted(set(c.substituted_positions.tolist()) - before)
            assert sel == g[f"{i}_selected"].tolist()
            i += 1


@pytest.mark.parametrize("name", ["cache_c0_n32.npz", "cache_c0_n3.npz", "cache_default.npz", "cache_freeze.npz"])
def test_cache_stream_matches_reference(name):
    g = load(name)
    bits, G, R, N, A, d = (int(x) for x in g["cfg"])
    c = oracle.OracleCache(bits, G, R, N, A, d)
    hist = []
    for k, v in zip(g["k"], g["v"]):
        nb = c.n_blocks
        c.append(k, v)
        if c.n_blocks != nb:
            pos = c.pool_entries()["position"].tolist()
            hist.append(pos + [-1] * (max(N, 1) - len(pos)))
    assert c.n_blocks == g["k_codes"].shape[0]
    for b in range(c.n_blocks):
        blk = c.block(b)
        assert blk["k_codes"] == g["k_codes"][b].tobytes()
        assert blk["v_codes"] == g["v_codes"][b].tobytes()
        np.testing.assert_array_equal(blk["k_xmin"], g["k_xmin"][b])
        np.testing.assert_array_equal(blk["k_step"], g["k_step"][b])
        np.testing.assert_array_equal(blk["v_xmin"], g["v_xmin"][b])
        np.testing.assert_array_equal(blk["v_step"], g["v_step"][b])
    pe = c.pool_entries()
    np.testing.assert_array_equal(pe["position"], g["pool_pos"])
    np.testing.assert_array_equal(pe["score"], g["pool_score"])
    np.testing.assert_array_equal(c.aux_entries()["position"], g["aux_pos"])
    assert c.frozen == bool(g["frozen"])
    np.testing.assert_array_equal(c.substituted_positions, g["substituted"])
    np.testing.assert_array_equal(np.array(hist).reshape(g["hist_entries"].shape), g["hist_entries"])
    mu = c.memory_usage()
    assert [mu["quantized_bits"], mu["param_bits"], mu["pending_bits"], mu["pool_bits"]] == g["memory"].tolist()
    assert c.pending_rows == int(g["pending_rows"])
    for q, out_ref, w_ref in zip(g["q"], g["attn_out"], g["attn_w"]):
        out, w, _ = c.attend(q, with_weights=True)
        # reference uses float32 BLAS dot products; the oracle evaluates in float64
        np.testing.assert_allclose(out, out_ref, atol=2e-5, rtol=1e-5)
        np.testing.assert_allclose(w, w_ref, atol=1e-6, rtol=1e-4)
        assert abs(float(w.sum(dtype=np.float64)) - 1.0) <= 1e-6


def test_reference_unit_examples():
    """Cache / attention examples restated from the reference's unit tests."""
    # tests/test_cache.py:60-68 trigger timing
    rng = np.random.default_rng(32)
    c = oracle.OracleCache(bits=2, group_size=4, residual=2, capacity=3, aux_capacity=32, head_dim=3)
    for _ in range(6):
        c.append(rng.standard_normal(3), rng.standard_normal(3))
    assert c.n_blocks == 1 and c.pending_rows == 2 and c.quantized_tokens == 4
    # tests/test_attention.py:102-110 single pending token
    c = oracle.OracleCache(bits=2, group_size=128, residual=32, capacity=3, aux_capacity=32, head_dim=2)
    c.append([1.0, 2.0], [5.0, -1.0])
    out, w, _ = c.attend(np.array([0.1, 0.2], np.float32), with_weights=True)
    np.testing.assert_allclose(w, [1.0])
    np.testing.assert_allclose(out, [5.0, -1.0])
    with pytest.raises(oracle.OracleError):
        oracle.OracleCache(head_dim=2).attend(np.zeros(2, np.float32))
    # tests/test_cache.py:174-184 single block accounting
    c = oracle.OracleCache(bits=2, group_size=128, residual=0, capacity=0, aux_capacity=32, head_dim=64)
    for _ in range(128):
        c.append(rng.standard_normal(64), rng.standard_normal(64))
    mu = c.memory_usage()
    assert mu["quantized_bits"] == 2 * 128 * 64 * 2 and mu["param_bits"] == (64 + 128) * 2 * 16
