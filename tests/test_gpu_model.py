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


@pytest.mark.parametrize("rows,dim", [(8, 4096), (3, 512), (2, 11008), (1, 24576)])
def test_rmsnorm_kernel_vs_torch_fp32(rows, dim):
    """ott_model_rmsnorm (register-resident row, one block reduction) against a float32 torch
    RMSNorm; fp16 output within one fp16 rounding of the float32 result (plus the fp16 weight
    product)."""
    from paper_2505_10938_b200 import _native

    g = torch.Generator(device="cuda").manual_seed(rows * dim)
    x = (torch.randn((rows, dim), generator=g, device="cuda") * 3).half()
    w = (torch.rand(dim, generator=g, device="cuda") + 0.5).half()
    y = torch.empty_like(x)
    _native.check(_native.lib().ott_model_rmsnorm(x.data_ptr(), w.data_ptr(), y.data_ptr(), rows, dim, 1e-5,
                                                  torch.cuda.current_stream().cuda_stream))
    xf = x.float()
    ref = (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5)).half().float() * w.float()
    torch.testing.assert_close(y.float(), ref, rtol=2e-3, atol=2e-3)


def test_rope_and_silu_kernels_vs_torch_fp32():
    """ott_model_rope_qkv (rotate-half RoPE at a device position, q/k/v split) and
    ott_model_silu_mul against float32 torch; fp16 outputs within fp16 rounding."""
    from paper_2505_10938_b200 import _native

    B, H, Hkv, d, P, n = 3, 6, 2, 128, 50, 1000
    g = torch.Generator(device="cuda").manual_seed(7)
    qkv = torch.randn((B, (H + 2 * Hkv) * d), generator=g, device="cuda").half()
    inv = 1.0 / (10000 ** (torch.arange(0, d, 2, device="cuda").float() / d))
    ang = torch.arange(P, device="cuda").float()[:, None] * inv[None]
    cos = torch.cat([ang.cos(), ang.cos()], -1).contiguous()
    sin = torch.cat([ang.sin(), ang.sin()], -1).contiguous()
    pos = torch.tensor([37], dtype=torch.int64, device="cuda")
    q = torch.empty((B, H, d), dtype=torch.float16, device="cuda")
    k = torch.empty((B, Hkv, d), dtype=torch.float16, device="cuda")
    v = torch.empty_like(k)
    st = torch.cuda.current_stream().cuda_stream
    _native.check(_native.lib().ott_model_rope_qkv(qkv.data_ptr(), cos.data_ptr(), sin.data_ptr(), pos.data_ptr(), 0,
                                                   q.data_ptr(), k.data_ptr(), v.data_ptr(), B, H, Hkv, d, st))
    x = qkv.float().view(B, H + 2 * Hkv, d)

    def rope(t):
        rot = torch.cat([-t[..., d // 2:], t[..., :d // 2]], -1)
        return t * cos[37] + rot * sin[37]

    torch.testing.assert_close(q.float(), rope(x[:, :H]), rtol=2e-3, atol=2e-3)
    torch.testing.assert_close(k.float(), rope(x[:, H:H + Hkv]), rtol=2e-3, atol=2e-3)
    assert torch.equal(v, qkv.view(B, H + 2 * Hkv, d)[:, H + Hkv:])

    h = torch.randn((B, 2 * n), generator=g, device="cuda").half()
    out = torch.empty((B, n), dtype=torch.float16, device="cuda")
    _native.check(_native.lib().ott_model_silu_mul(h.data_ptr(), out.data_ptr(), B, n, st))
    a, b = h.float()[:, :n], h.float()[:, n:]
    torch.testing.assert_close(out.float(), torch.nn.functional.silu(a) * b, rtol=2e-3, atol=2e-3)
