"""The reference's standalone objects on the GPU kernels: OutlierPool / OutlierEntry.from_rows /
score_tokens (outlier.py:24-117) replayed against the reference's own pool streams
(tests/golden/pool_streams.npz, written by kvtrace), and attend_full_precision
(attention.py:35-59) against the C oracle and the reference's test cases."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_score_tokens_kat():
    from paper_2505_10938_b200 import ContractViolation, score_tokens

    assert score_tokens(np.array([[1.0, -2.0, 3.0]], np.float32)).tolist() == [6.0]  # tests/test_outlier.py:20-27
    rng = np.random.default_rng(3)
    k = rng.standard_normal((33, 128)).astype(np.float32)
    exact = [float(np.abs(r.astype(np.float64)).sum()) for r in k]
    assert score_tokens(k).tolist() == exact
    with pytest.raises(ContractViolation):
        score_tokens(np.zeros((0, 4), np.float32))


def test_outlier_pool_streams_match_reference():
    from paper_2505_10938_b200 import OutlierEntry, OutlierPool

    g = np.load(os.path.join(GOLDEN, "pool_streams.npz"))
    n = int(g["n"])
    pool, key = None, None
    for i in range(n):
        cap, aux_cap, base = int(g[f"{i}_cap"]), int(g[f"{i}_aux_cap"]), int(g[f"{i}_base"])
        if base == 0 or (cap, aux_cap) != key:
            pool, key = OutlierPool(capacity=cap, aux_capacity=aux_cap), (cap, aux_cap)
        cands = []
        for j, s in enumerate(g[f"{i}_scores"]):
            row = np.zeros(4, np.float32)
            row[0] = s
            cands.append(OutlierEntry.from_rows(base + j, row, np.zeros(4, np.float32)))
        assert [c.score for c in cands] == g[f"{i}_scores"].tolist()
        sel, ev = pool.update(cands)
        assert sorted(sel) == g[f"{i}_selected"].tolist()
        assert [e.position for e in ev] == g[f"{i}_evicted"].tolist()
        assert [e.position for e in pool.entries] == g[f"{i}_entries"].tolist()
        assert [e.position for e in pool.aux] == g[f"{i}_aux"].tolist()
        assert pool.frozen == bool(g[f"{i}_frozen"])


def test_outlier_pool_contract():
    from paper_2505_10938_b200 import ContractViolation, OutlierEntry, OutlierPool

    z = np.zeros(2, np.float32)
    pool = OutlierPool(capacity=2, aux_capacity=1)
    with pytest.raises(ContractViolation):
        pool.update([OutlierEntry.from_rows(1, z, z), OutlierEntry.from_rows(1, z, z)])  # duplicates
    with pytest.raises(ContractViolation):
        OutlierPool(capacity=-1)
    # tie breaks toward the smaller position (tests/test_outlier.py:65-68)
    p = OutlierPool(capacity=1, aux_capacity=4)
    p.update([OutlierEntry(7, z, z, 1.0), OutlierEntry(3, z, z, 1.0)])
    assert p.positions == {3}
    assert OutlierPool(capacity=0).update([OutlierEntry(1, z, z, 0.0)]) == (set(), [])


@pytest.mark.parametrize("n,d", [(1, 4), (37, 16), (300, 128), (2049, 128)])
def test_attend_full_precision_vs_oracle(n, d):
    from paper_2505_10938_b200 import attend_full_precision

    rng = np.random.default_rng(n + d)
    k = (rng.standard_normal((n, d)) * np.where(np.arange(d) < 4, 15.0, 1.0)).astype(np.float32)
    v = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal(d).astype(np.float32)
    res = attend_full_precision(q, k, v)
    # the oracle's exact path: an N = 0 cache whose rows all stay pending (R >= n)
    ref = oracle.OracleCache(bits=2, group_size=4, residual=n + 4, capacity=0, aux_capacity=0, head_dim=d)
    ref.extend(k, v)
    out, w, s = ref.attend(q, with_weights=True)
    np.testing.assert_allclose(res.scores, s, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(res.weights, w, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(res.output, out, rtol=1e-5, atol=1e-5)
    assert abs(float(res.weights.astype(np.float64).sum()) - 1.0) <= 1e-6  # tests/test_acceptance.py:220-234


def test_attend_full_precision_contract():
    from paper_2505_10938_b200 import ContractViolation, attend_full_precision

    z = np.zeros((3, 4), np.float32)
    with pytest.raises(ContractViolation):
        attend_full_precision(np.zeros(4, np.float32), np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32))
    with pytest.raises(ContractViolation):
        attend_full_precision(np.zeros(5, np.float32), z, z)
    with pytest.raises(ContractViolation):
        attend_full_precision(np.zeros((1, 4), np.float32), z, z)
    # single token: weight 1, output = its value row (tests/test_attention.py:102-110)
    r = attend_full_precision(np.ones(4, np.float32), np.ones((1, 4), np.float32), np.arange(4, dtype=np.float32)[None])
    assert r.weights.tolist() == [1.0] and r.output.tolist() == [0.0, 1.0, 2.0, 3.0]
