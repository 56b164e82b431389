"""Out-of-bounds write detection on the GPU path (compute-sanitizer is not available
on the GPU pool): every buffer the kernels write -- the cache's device state, the
attention workspace and the output -- is re-homed inside a larger allocation whose
head and tail are filled with a sentinel byte, a mixed workload runs through every
kernel family (bulk prefill incl. the scan + per-group quantizer, ring writes, due
flushes, fused append+attend, device-counter decode steps, all decode kernels), and
the sentinels must be intact afterwards. The final state is also checked bit-exact
against the oracle for one unit so the workload is known to have done real work."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PAD = 4096
SENT = 0xA5
CACHE_BUFS = ("blocks", "pend_k", "pend_v", "pool_mask", "subst_mask", "pool_pos", "pool_score", "pool_k",
              "pool_v", "aux_pos", "aux_score", "aux_k", "aux_v", "pool_meta")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


class Guards:
    def __init__(self):
        self.raws = []

    def wrap(self, t, name):
        nbytes = t.numel() * t.element_size()
        raw = torch.full((PAD + nbytes + PAD,), SENT, dtype=torch.uint8, device=t.device)
        view = raw[PAD:PAD + nbytes].view(t.dtype).view(t.shape)
        view.copy_(t)
        self.raws.append((name, raw, nbytes))
        return view

    def empty(self, shape, dtype, name):
        return self.wrap(torch.zeros(shape, dtype=dtype, device="cuda"), name)

    def check(self):
        torch.cuda.synchronize()
        bad = []
        for name, raw, nbytes in self.raws:
            head, tail = raw[:PAD], raw[PAD + nbytes:]
            if not bool((head == SENT).all()) or not bool((tail == SENT).all()):
                hb = int((head != SENT).sum())
                tb = int((tail != SENT).sum())
                bad.append(f"{name}: {hb} head / {tb} tail bytes overwritten")
        assert not bad, bad


def guarded_cache(cfg, B, Hkv, T, g):
    from paper_2505_10938_b200 import OTTCache
    from paper_2505_10938_b200 import _native

    cache = OTTCache(cfg, B, Hkv, max_tokens=T, keep_f64_params=True)
    for name in CACHE_BUFS:
        view = g.wrap(getattr(cache, name), name)
        setattr(cache, name, view)
        setattr(cache._c, name, view.data_ptr())
    cache.params64 = g.wrap(cache.params64, "params64")
    cache._c.params64 = cache.params64.data_ptr()
    cache.counters = g.wrap(cache.counters, "counters")
    L = _native.lib()

    def workspace(n_rep, n_splits):
        n = int(L.ott_attend_workspace_floats(cache._cref, n_rep, n_splits))
        return g.empty((n,), torch.float32, f"workspace({n_rep},{n_splits})")

    cache.workspace = workspace
    return cache


# (bits, G, R, N, A, d, n_rep, B, Hkv): one row per kernel family
CASES = [
    (2, 32, 32, 8, 16, 128, 8, 4, 4),      # K2 tensor path + K1 scan/prescore/frozen prefill
    (2, 32, 32, 24, 16, 128, 8, 2, 2),     # N > A: scan without prescore
    (2, 32, 32, 8, 16, 128, 8, 16, 8),     # many units: two-CTA fp tier
    (4, 32, 32, 8, 16, 128, 8, 4, 4),      # K2-4 tensor path + 4-bit per-group quantizer
    (8, 32, 32, 8, 16, 128, 8, 4, 4),      # K2-8 tensor path, generic flush
    (3, 32, 32, 8, 16, 128, 4, 4, 4),      # SIMT split-K path, other width
    (1, 32, 16, 4, 4, 128, 2, 2, 2),       # 1-bit
    (2, 16, 8, 4, 8, 64, 4, 2, 3),         # generic shapes
    (4, 7, 3, 3, 0, 40, 1, 2, 2),          # ragged generic shape, aux capacity 0 (frozen at start)
]


@pytest.mark.parametrize("bits,G,R,N,A,d,n_rep,B,Hkv", CASES)
def test_no_out_of_bounds_writes(bits, G, R, N, A, d, n_rep, B, Hkv):
    from paper_2505_10938_b200 import EngineConfig

    cfg = EngineConfig(bits=bits, group_size=G, residual=R, outlier_num=N, aux_capacity=A, skip_layers=(),
                       head_dim=d)
    n_pre, n_app, n_dec = 5 * G + R + 3, G + 2, G + 1
    T = n_pre + n_app + n_dec
    rng = np.random.default_rng(bits * 7919 + G * 31 + d + B)
    k = rng.standard_normal((B, Hkv, T, d)).astype(np.float16)
    k[..., : max(1, d // 8)] *= 12
    k[..., 3 * G, :] *= 40  # a spike row that must win a pool slot
    v = rng.standard_normal((B, Hkv, T, d)).astype(np.float16)
    q = rng.standard_normal((T, B, Hkv * n_rep, d)).astype(np.float16)
    g = Guards()
    cache = guarded_cache(cfg, B, Hkv, T, g)
    kt, vt, qt = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(q).cuda()
    kin = g.wrap(kt[:, :, :n_pre].contiguous(), "prefill k")
    vin = g.wrap(vt[:, :, :n_pre].contiguous(), "prefill v")
    cache.update(kin, vin)
    out = g.empty((B, Hkv * n_rep, d), torch.float16, "out")
    cache.attend(g.wrap(qt[0], "q"), out=out)
    for t in range(n_pre, n_pre + n_app):
        cache.append_attend(kt[:, :, t].contiguous(), vt[:, :, t].contiguous(), qt[t], out=out)
    cache.sync_counters()
    s = cache.splits(n_rep)
    for t in range(n_pre + n_app, T):
        cache.decode_step(kt[:, :, t].contiguous(), vt[:, :, t].contiguous(), qt[t].contiguous(), out, s)
    res = cache.attend(qt[T - 1].contiguous(), out=out).float().cpu().numpy()
    g.check()
    assert np.isfinite(res).all()
    assert cache.total_tokens == T

    ref = oracle.OracleCache(bits, G, R, N, A, d)
    ref.extend(k[B - 1, Hkv - 1].astype(np.float32), v[B - 1, Hkv - 1].astype(np.float32))
    u = cache.unit(B - 1, Hkv - 1)
    assert u.quantized_tokens == ref.quantized_tokens
    for b in range(ref.n_blocks):
        assert u.quantized_k[b].codes == ref.block(b)["k_codes"], b
        assert u.quantized_v[b].codes == ref.block(b)["v_codes"], b
    qi = q[T - 1, B - 1, (Hkv - 1) * n_rep].astype(np.float32)
    o_ref = ref.attend(qi, with_weights=True)[0]
    err = np.abs(res[B - 1, (Hkv - 1) * n_rep] - o_ref)
    assert (err <= 2e-3 + 1e-2 * np.abs(o_ref)).all(), err.max()
