"""ratio_curve on the GPU cache vs the reference's report.ratio_curve loop
(report.py:159-216) run on the same fp16-valued rows (golden ratio.npz)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["paper", "c1"])
def test_ratio_curve_matches_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10938_b200 import EngineConfig
    from paper_2505_10938_b200.report import ratio_curve

    cfg = {"paper": EngineConfig(bits=2, group_size=128, residual=32, outlier_num=3, head_dim=64),
           "c1": EngineConfig(bits=2, group_size=32, residual=128, outlier_num=32, head_dim=128)}[name]
    g = np.load(os.path.join(GOLDEN, "ratio.npz"))[name]
    rows = ratio_curve(cfg, [int(x) for x in g[:, 0]])
    for row, ref in zip(rows, g):
        assert row.seq_len == ref[0] and row.total_bits == ref[5]
        assert row.ratio_vs_fp16 == 2 * ref[0] * cfg.head_dim * 16 / ref[5]
    assert rows[0].ratio_vs_fp16 == 1.0 and rows[0].mode == "ott"
