"""Config-1 decoder fidelity plumbing (bench.py --config c1): the reference's simulate metric
(per-step attention-output L1 vs exact attention, cli.py:208-218) measured inside the decoder.
A lossless cache (residual window longer than the run) reproduces exact attention; with the
outlier-channel / outlier-token key structure, outlier tracking (N = 32) beats N = 0."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(ott_cfg, steps=48, T=320):
    from paper_2505_10938_b200.model import Decoder, DecoderConfig

    cfg = DecoderConfig(n_layers=4, hidden=512, n_heads=4, n_kv_heads=4, head_dim=128, mlp=1024, vocab=1000)
    prompt = torch.randint(0, cfg.vocab, (2, T), generator=torch.Generator().manual_seed(3)).cuda()
    m = Decoder(cfg, 2, T + steps + 8, kv="ott", ott=ott_cfg, seed=1, k_outliers=4, track_exact=True)
    tok = m.prefill(prompt)
    for _ in range(steps):
        tok = m.decode(tok)
    return sum(m.attn_l1) / len(m.attn_l1)


def _cfg(R, N):
    from paper_2505_10938_b200 import EngineConfig

    return EngineConfig(bits=2, group_size=32, residual=R, outlier_num=N, aux_capacity=32, skip_layers=(),
                        n_layers=4, n_heads=4, head_dim=128)


def test_lossless_cache_matches_exact_attention():
    assert _run(_cfg(512, 0)) < 0.05  # fp16 rows: only output rounding (128 channels)


def test_outlier_tracking_beats_n0_in_the_decoder():
    ott, n0 = _run(_cfg(32, 32)), _run(_cfg(32, 0))
    assert ott < 0.95 * n0, (ott, n0)  # measured 36.6 vs 43.0


def test_flash_fp16_baseline_matches_sdpa_decoder():
    """The independent fp16 baseline (plain KV cache + flash_attn_with_kvcache, graph-captured)
    decodes like the SDPA fp16 decoder: same greedy tokens, logits within fp16 noise."""
    import torch

    from paper_2505_10938_b200.model import Decoder, DecoderConfig

    pytest.importorskip("flash_attn")
    cfg = DecoderConfig(n_layers=2, hidden=512, n_heads=4, n_kv_heads=2, head_dim=128, mlp=1024, vocab=1000)
    prompt = torch.randint(0, cfg.vocab, (2, 200), generator=torch.Generator().manual_seed(5)).cuda()
    a = Decoder(cfg, 2, 240, kv="fp16", seed=3)
    b = Decoder(cfg, 2, 240, kv="flash", seed=3)
    ta, tb = a.prefill(prompt), b.prefill(prompt)
    assert torch.equal(ta, tb)
    for _ in range(8):
        ta, tb = a.decode(ta), b.decode_graph(tb)
        torch.testing.assert_close(a.last_logits.float(), b.last_logits.float(), atol=2e-2, rtol=0)
        assert torch.equal(ta, tb)
