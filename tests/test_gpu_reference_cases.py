"""The reference's own cache and attention test scenarios, restated against the GPU
path through the drop-in TieredCache / attend_mixed adapter.

Each test cites the reference test it restates (pkg/tests/test_cache.py,
pkg/tests/test_attention.py). The shapes are the reference tests' own (d 2..16,
G 4..16, so the generic CUDA-core kernels run). Differences from the originals:
rows are drawn as fp16 values (the GPU stores fp16 rows), and independent checks use
the C oracle (oracle/) in place of the reference's helper functions.
"""

import math

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def fp16_rows(a):
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float32)


def random_rows(rng, n, d):
    return fp16_rows(rng.standard_normal((n, d)))


def uniform_rows(rng, lo, hi, n, d):
    return fp16_rows(rng.uniform(lo, hi, size=(n, d)))


def make(**kw):
    from paper_2505_10938_b200 import EngineConfig, TieredCache

    layer = kw.pop("layer", 0)
    kw.setdefault("skip_layers", ())
    return TieredCache(EngineConfig(**kw), layer=layer, max_tokens=1024)


def fill(cache, keys, values):
    for k, v in zip(keys, values):
        cache.append(k, v)


def full_precision(q, keys, values):
    """Scalar attention in float64 (the role of test_attention.py:19-36)."""
    d = keys.shape[1]
    s = keys.astype(np.float64) @ q.astype(np.float64) / math.sqrt(d)
    w = np.exp(s - s.max())
    w /= w.sum()
    return w @ values.astype(np.float64), w, s


# ---------------------------------------------------------------- test_cache.py


def test_single_append():  # test_cache.py:44-49
    c = make(group_size=4, residual=2, head_dim=3, layer=2)
    c.append([1.0, 2.0, 3.0], [4.0, 5.0, 6.0])
    assert c.pending_rows == 1 and c.quantized_k == [] and c.total_tokens == 1


def test_zero_residual_quantizes_at_group():  # test_cache.py:51-57
    rng = np.random.default_rng(31)
    c = make(group_size=4, residual=0, head_dim=3, layer=2)
    fill(c, random_rows(rng, 4, 3), random_rows(rng, 4, 3))
    assert len(c.quantized_k) == 1 and c.pending_rows == 0 and c.quantized_tokens == 4


def test_residual_window_defers_trigger():  # test_cache.py:59-67
    rng = np.random.default_rng(32)
    c = make(group_size=4, residual=2, head_dim=3, layer=2)
    fill(c, random_rows(rng, 6, 3), random_rows(rng, 6, 3))
    assert len(c.quantized_k) == 1 and c.quantized_k[0].n_tokens == 4
    assert c.pending_rows == 2 and c.quantized_tokens == 4


def test_dimension_mismatch_and_manual_quantize():  # test_cache.py:69-78
    from paper_2505_10938_b200 import ContractViolation

    c = make(head_dim=3, layer=2)
    with pytest.raises(ContractViolation):
        c.append([1.0, 2.0], [1.0, 2.0, 3.0])
    c = make(group_size=4, residual=0, head_dim=3, layer=2)
    c.append([1.0, 2.0, 3.0], [1.0, 2.0, 3.0])
    with pytest.raises(ContractViolation):
        c.quantize_oldest_group()


def test_conservation_and_bounds():  # test_cache.py:80-90
    rng = np.random.default_rng(33)
    G, R = 8, 3
    c = make(group_size=G, residual=R, head_dim=4, layer=2)
    for _ in range(100):
        c.append(*random_rows(rng, 2, 4))
        assert c.quantized_tokens + c.pending_rows == c.total_tokens
        assert c.pending_rows <= G + R
        assert c.pending_rows - R < G


def test_zero_outliers_matches_direct_group_quantization():  # test_cache.py:93-110
    rng = np.random.default_rng(34)
    c = make(group_size=8, residual=2, outlier_num=0, head_dim=4, bits=2)
    keys, values = random_rows(rng, 30, 4), random_rows(rng, 30, 4)
    fill(c, keys, values)
    assert len(c.quantized_k) == 3
    for g in range(3):
        kc, kmin, kstep = oracle.quantize_group(keys[g * 8:(g + 1) * 8], 2, per_channel=True)
        vc, _, _ = oracle.quantize_group(values[g * 8:(g + 1) * 8], 2, per_channel=False)
        assert c.quantized_k[g].codes == kc
        assert c.quantized_v[g].codes == vc
        assert [p.x_min for p in c.quantized_k[g].params] == kmin.tolist()
        assert [p.step for p in c.quantized_k[g].params] == kstep.tolist()


def test_skip_layer_equals_explicit_zero():  # test_cache.py:112-127
    rng = np.random.default_rng(35)
    keys, values = random_rows(rng, 40, 4), random_rows(rng, 40, 4)
    skipped = make(group_size=8, residual=0, outlier_num=3, skip_layers=(0,), head_dim=4, layer=0)
    disabled = make(group_size=8, residual=0, outlier_num=0, head_dim=4, layer=0)
    fill(skipped, keys, values)
    fill(disabled, keys, values)
    assert len(skipped.quantized_k) == 5
    for a, b in zip(skipped.quantized_k, disabled.quantized_k):
        assert a.codes == b.codes and a.params == b.params


def test_planted_token_is_pooled_and_substituted():  # test_cache.py:131-150
    rng = np.random.default_rng(36)
    g, d = 16, 4
    c = make(group_size=g, residual=0, outlier_num=1, head_dim=d, bits=2)
    keys = uniform_rows(rng, 4.5, 5.5, g, d)
    keys[5] = fp16_rows(0.01)
    values = random_rows(rng, g, d)
    fill(c, keys, values)
    assert c.pool.positions == {5}
    assert c.substituted_positions == {5}
    recon = c.quantized_k[0].to_matrix()[5]
    step = max(p.step for p in c.quantized_k[0].params)
    assert np.abs(recon - keys.mean(axis=0)).max() <= step + 1e-6
    np.testing.assert_array_equal(c.pool.entries[0].key, keys[5])
    np.testing.assert_array_equal(c.pool.entries[0].value, values[5])


def test_pool_swap_sends_loser_to_aux():  # test_cache.py:152-166
    rng = np.random.default_rng(37)
    g, d = 8, 4
    c = make(group_size=g, residual=0, outlier_num=1, head_dim=d)
    first = uniform_rows(rng, 4.5, 5.5, g, d)
    first[2] = 0.5
    second = uniform_rows(rng, 4.5, 5.5, g, d)
    second[6] = fp16_rows(0.01)
    fill(c, first, random_rows(rng, g, d))
    assert c.pool.positions == {2}
    fill(c, second, random_rows(rng, g, d))
    assert c.pool.positions == {g + 6}
    assert [e.position for e in c.pool.aux] == [2]
    assert c.substituted_positions == {2, g + 6}


def test_memory_usage():  # test_cache.py:169-209
    assert make(layer=2, skip_layers=(0, 1)).memory_usage().total_bits == 0
    rng = np.random.default_rng(38)
    c = make(group_size=128, residual=0, outlier_num=0, head_dim=64, bits=2, layer=2)
    fill(c, random_rows(rng, 128, 64), random_rows(rng, 128, 64))
    u = c.memory_usage()
    assert u.quantized_bits == 2 * 128 * 64 * 2 and u.param_bits == (64 + 128) * 2 * 16 and u.pending_bits == 0
    assert (2 * 128 * 64 * 16) / u.total_bits == pytest.approx(6.7368, abs=1e-3)

    rng = np.random.default_rng(39)
    g, d = 8, 4
    c = make(group_size=g, residual=2, outlier_num=1, head_dim=d)
    keys = uniform_rows(rng, 4.5, 5.5, g + 2, d)
    keys[1] = fp16_rows(0.01)
    fill(c, keys, random_rows(rng, g + 2, d))
    u = c.memory_usage()
    assert u.pending_bits == 2 * d * 16 * 2 and u.pool_bits == 1 * d * 16 * 2

    rng = np.random.default_rng(40)
    c = make(group_size=8, residual=2, outlier_num=0, head_dim=4, layer=2)
    totals = []
    for _ in range(200):
        c.append(*random_rows(rng, 2, 4))
        if c.pending_rows == 2:
            totals.append(c.memory_usage().total_bits)
    assert len(totals) > 5 and all(a < b for a, b in zip(totals, totals[1:]))


# ------------------------------------------------------------ test_attention.py


def test_single_pending_token_and_empty_cache():  # test_attention.py:102-115
    from paper_2505_10938_b200 import ContractViolation, attend_mixed

    c = make(head_dim=2)
    c.append([1.0, 2.0], [5.0, -1.0])
    res = attend_mixed(fp16_rows([0.1, 0.2]), c)
    np.testing.assert_allclose(res.weights, [1.0])
    np.testing.assert_allclose(res.output, [5.0, -1.0])
    with pytest.raises(ContractViolation):
        attend_mixed(np.zeros(2, np.float32), make(head_dim=2, layer=2))


def test_weights_cover_every_token():  # test_attention.py:132-139
    from paper_2505_10938_b200 import attend_mixed

    rng = np.random.default_rng(44)
    c = make(group_size=8, residual=2, outlier_num=2, head_dim=4)
    fill(c, random_rows(rng, 37, 4), random_rows(rng, 37, 4))
    res = attend_mixed(random_rows(rng, 1, 4)[0], c)
    assert res.weights.shape == (37,)
    assert abs(float(res.weights.sum(dtype=np.float64)) - 1.0) <= 1e-6


def test_mixed_attention_matches_oracle_on_reconstruction():  # test_attention.py:117-130 (quantized mode)
    """attend_mixed over the quantized cache equals full-precision attention over the
    oracle's reconstructed_kv (attention.py:62-76) within the fp16 tolerance."""
    from paper_2505_10938_b200 import attend_mixed

    rng = np.random.default_rng(43)
    keys, values = random_rows(rng, 100, 8), random_rows(rng, 100, 8)
    c = make(group_size=16, residual=4, outlier_num=2, head_dim=8)
    ref = oracle.OracleCache(2, 16, 4, 2, 32, 8)
    fill(c, keys, values)
    ref.extend(keys, values)
    q = random_rows(rng, 1, 8)[0]
    K, V = ref.reconstructed_kv()
    want, w, s = full_precision(q, K, V)
    res = attend_mixed(q, c)
    assert np.abs(res.output - want).max() <= 2e-3 + 1e-2 * np.abs(want).max()
    np.testing.assert_allclose(res.weights, w, atol=1e-5, rtol=1e-3)
    np.testing.assert_allclose(res.scores, s, atol=1e-4, rtol=1e-4)


def test_pool_logit_ignores_shadow_row():  # test_attention.py:141-166
    from paper_2505_10938_b200 import attend_mixed

    rng = np.random.default_rng(45)
    g, d = 16, 4
    keys = uniform_rows(rng, 4.5, 5.5, g, d)
    keys[3] = fp16_rows(0.01)
    values = random_rows(rng, g, d)
    c = make(group_size=g, residual=0, outlier_num=1, head_dim=d)
    fill(c, keys, values)
    assert c.pool.positions == {3}
    q = random_rows(rng, 1, d)[0]
    res_a = attend_mixed(q, c)
    # corrupt the mean-substituted shadow row 3 in device memory: K codes +1 mod 4, V codes 0
    gpu = c.gpu
    blk = gpu.blocks[0, 0]
    cb = ((g * d * 2 + 7) // 8 + 15) & ~15  # V codes start (padded K code field, ott_b200.h)
    row = slice(3 * d * 2 // 8, 4 * d * 2 // 8)  # token 3 = codes 12..15 = byte 3 at d = 4, 2 bits
    kb = blk[row].cpu().numpy()
    codes = np.unpackbits(kb, bitorder="little").reshape(-1, 2) @ np.array([1, 2])
    codes = (codes + 1) % 4
    packed = np.packbits(np.stack([codes & 1, codes >> 1], 1).reshape(-1).astype(np.uint8), bitorder="little")
    blk[row] = torch.from_numpy(packed).to(blk.device)
    blk[cb + row.start: cb + row.stop] = 0
    c._snap = None
    assert c.quantized_k[0].code_matrix()[3].tolist() != oracle.unpack_codes(kb.tobytes(), 2, d).tolist()
    res_b = attend_mixed(q, c)
    np.testing.assert_array_equal(res_a.scores, res_b.scores)
    np.testing.assert_array_equal(res_a.output, res_b.output)


def test_outlier_tracking_beats_baseline_on_planted_trace():  # test_attention.py:168-185
    """Planted low-norm tokens that stretch the key range of their group: tracking them in
    the pool (N = 3) gives a lower mean L1 error vs full-precision attention than N = 0.
    (The reference plants with its own synthetic generator; this trace is built here.)"""
    from paper_2505_10938_b200 import attend_mixed

    rng = np.random.default_rng(12)
    T, d = 256, 16
    k = rng.standard_normal((T, d))
    k[:, :4] += 10.0  # large-magnitude channels
    k[::37, :4] = 0.01  # planted tokens: low L1 norm, far outside the channels' range
    k, v, q = fp16_rows(k), random_rows(rng, T, d), random_rows(rng, T, d)
    errors = {}
    for name, n_out in (("baseline", 0), ("tracked", 3)):
        c = make(group_size=64, residual=16, outlier_num=n_out, head_dim=d)
        errs = []
        for t in range(T):
            c.append(k[t], v[t])
            out = attend_mixed(q[t], c, with_weights=False).output
            want, _, _ = full_precision(q[t], k[: t + 1], v[: t + 1])
            errs.append(float(np.abs(out - want).sum()))
        errors[name] = float(np.mean(errs))
    assert errors["tracked"] < errors["baseline"]


def test_wider_step_does_not_reduce_logit_error():  # test_attention.py:188-209
    from paper_2505_10938_b200 import attend_mixed

    rng = np.random.default_rng(46)
    g, d = 64, 8
    results = []
    for eps in (2.0, 0.01):
        keys = rng.uniform(9.0, 11.0, size=(g, d))
        keys[:, 0] = np.linspace(9.0, 11.0, g)
        keys[::21, 0] = eps
        keys = fp16_rows(keys)
        values = random_rows(rng, g, d)
        q = np.zeros(d, np.float32)
        q[0] = 8.0
        c = make(group_size=g, residual=0, outlier_num=0, head_dim=d)
        fill(c, keys, values)
        res = attend_mixed(q, c)
        _, _, s = full_precision(q, keys, values)
        results.append((c.quantized_k[0].params[0].step, float(np.abs(res.scores - s).mean())))
    (step_narrow, err_narrow), (step_wide, err_wide) = results
    assert step_wide > step_narrow and err_wide >= err_narrow
