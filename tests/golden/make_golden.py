"""Generate golden fixtures by running the REFERENCE package (kvtrace) itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/kvtrace read-only and writes small .npz
fixtures next to this file. Those fixtures pin (1) the CPU oracle in
``oracle/`` (tests/test_oracle_golden.py, CPU) and (2) the CUDA product
(tests/test_gpu_parity.py, GPU) without needing the reference at run time.

Inputs are fp16-representable float32 values (the product consumes fp16), plus
a few float32 streams that mirror the reference's own unit tests.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _kv():
    sys.path.insert(0, REF)
    import kvtrace  # noqa: E402

    return kvtrace


def fp16(a):
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float32)


def config0_stream(seed: int, T: int, d: int = 128, n_out_ch: int = 4, n_out_tok: int = 8):
    """BASELINE config 0 recipe: K ~ N(0,1), 4 seeded channels x15, 8 seeded tokens
    with those channels x0.05; V ~ N(0,1); q ~ N(0,1). fp16 values."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(0, 0, 0)))
    k = rng.standard_normal((T, d))
    ch = rng.choice(d, n_out_ch, replace=False)
    k[:, ch] *= 15.0
    tok = rng.choice(T, n_out_tok, replace=False)
    k[np.ix_(tok, ch)] *= 0.05
    v = rng.standard_normal((T, d))
    q = rng.standard_normal((4, d))
    return fp16(k), fp16(v), fp16(q)


def gen_quant_lines(kv):
    rng = np.random.default_rng(1234)
    lines, bits_l, codes_l, xmin_l, step_l = [], [], [], [], []

    def add(x, bits):
        c, p = kv.quantize_uniform(x, bits)
        lines.append(np.asarray(x, dtype=np.float64))
        bits_l.append(bits)
        codes_l.append(c.astype(np.int64))
        xmin_l.append(p.x_min)
        step_l.append(p.step)

    # KATs from the reference tests (tests/test_quant.py:35-80)
    add([0.0, 1.0, 2.0, 3.0], 2)
    add([5.0, 5.0, 5.0], 4)
    add([0.0, 0.5, 1.0], 1)
    add([7.5, 7.5], 2)
    for bits in (1, 2, 3, 4, 7, 8):
        for n in (1, 2, 5, 32, 128, 257):
            add(rng.uniform(-10, 10, size=n), bits)
            add(fp16(rng.standard_normal(n) * 15.0).astype(np.float64), bits)
            add((rng.standard_normal(n) * 1e-42).astype(np.float32).astype(np.float64), bits)
    for bits in (1, 2, 4, 8):  # lattice-aligned, tests/test_acceptance.py:85-90
        levels = (1 << bits) - 1
        lat = -10.0 + 0.5 * np.arange(levels + 1)
        rng.shuffle(lat)
        add(lat, bits)
    for _ in range(300):  # 2-bit fp16 lines, the product's domain
        n = int(rng.choice([32, 128]))
        add(fp16(rng.standard_normal(n) * rng.uniform(0.01, 40)).astype(np.float64), 2)
    offs = np.cumsum([0] + [len(x) for x in lines])
    np.savez_compressed(
        os.path.join(HERE, "quant_lines.npz"),
        x=np.concatenate(lines), offsets=offs, bits=np.array(bits_l), codes=np.concatenate(codes_l),
        x_min=np.array(xmin_l), step=np.array(step_l),
    )


def gen_pack(kv):
    rng = np.random.default_rng(99)
    out = {}
    for bits in range(1, 9):
        codes = rng.integers(0, 1 << bits, size=997)
        out[f"codes_{bits}"] = codes
        out[f"packed_{bits}"] = np.frombuffer(kv.pack_codes(codes, bits), dtype=np.uint8)
    out["kat_a"] = np.frombuffer(kv.pack_codes([0, 1, 2, 3], 2), dtype=np.uint8)
    out["kat_b"] = np.frombuffer(kv.pack_codes([1, 0, 0, 0, 0, 0, 0, 3], 2), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "pack.npz"), **out)


def gen_pool_streams(kv):
    """OutlierPool.update streams (outlier.py:84-117) with explicit scores."""
    rng = np.random.default_rng(7)
    recs = []
    for cap, aux_cap, g, n_groups, tie in [(3, 4, 8, 6, False), (2, 2, 4, 10, True), (1, 8, 8, 5, False),
                                            (5, 32, 32, 12, True), (32, 32, 32, 6, False), (0, 8, 4, 3, False),
                                            (2, 0, 4, 3, False)]:
        pool = kv.OutlierPool(capacity=cap, aux_capacity=aux_cap)
        pos = 0
        for _ in range(n_groups):
            if tie:
                scores = rng.integers(0, 6, size=g).astype(np.float64)
            else:
                scores = rng.uniform(0, 100, size=g)
            cands = []
            for i in range(g):
                key = np.zeros(4, dtype=np.float32)
                key[0] = scores[i]
                cands.append(kv.OutlierEntry.from_rows(pos + i, key, np.zeros(4, dtype=np.float32)))
            scores = np.array([c.score for c in cands])  # float32-rounded by from_rows
            sel, ev = pool.update(cands)
            recs.append(dict(cap=cap, aux_cap=aux_cap, base=pos, scores=scores,
                             selected=np.array(sorted(sel), dtype=np.int64),
                             evicted=np.array([e.position for e in ev], dtype=np.int64),
                             entries=np.array([e.position for e in pool.entries], dtype=np.int64),
                             aux=np.array([e.position for e in pool.aux], dtype=np.int64),
                             frozen=pool.frozen))
            pos += g
    flat = {}
    for i, r in enumerate(recs):
        for key, val in r.items():
            flat[f"{i}_{key}"] = np.asarray(val)
    flat["n"] = np.array(len(recs))
    np.savez_compressed(os.path.join(HERE, "pool_streams.npz"), **flat)


def run_cache(kv, k, v, qs, bits, G, R, N, A, d):
    cfg = kv.EngineConfig(bits=bits, group_size=G, residual=R, outlier_num=N, aux_capacity=A, skip_layers=(),
                          head_dim=d)
    c = kv.TieredCache(cfg, layer=0)
    hist_entries, hist_aux, hist_frozen = [], [], []
    for i in range(k.shape[0]):
        nb = len(c.quantized_k)
        c.append(k[i], v[i])
        if len(c.quantized_k) != nb:
            e = [x.position for x in c.pool.entries]
            hist_entries.append(e + [-1] * (max(N, 1) - len(e)))
            hist_aux.append(len(c.pool.aux))
            hist_frozen.append(c.pool.frozen)
    res = dict(k=k, v=v, q=qs, cfg=np.array([bits, G, R, N, A, d]))
    nb = len(c.quantized_k)
    res["k_codes"] = np.array([np.frombuffer(b.codes, np.uint8) for b in c.quantized_k]).reshape(nb, -1)
    res["v_codes"] = np.array([np.frombuffer(b.codes, np.uint8) for b in c.quantized_v]).reshape(nb, -1)
    res["k_xmin"] = np.array([[p.x_min for p in b.params] for b in c.quantized_k]).reshape(nb, d)
    res["k_step"] = np.array([[p.step for p in b.params] for b in c.quantized_k]).reshape(nb, d)
    res["v_xmin"] = np.array([[p.x_min for p in b.params] for b in c.quantized_v]).reshape(nb, G)
    res["v_step"] = np.array([[p.step for p in b.params] for b in c.quantized_v]).reshape(nb, G)
    res["pool_pos"] = np.array([e.position for e in c.pool.entries], dtype=np.int64)
    res["pool_score"] = np.array([e.score for e in c.pool.entries], dtype=np.float64)
    res["aux_pos"] = np.array([e.position for e in c.pool.aux], dtype=np.int64)
    res["frozen"] = np.array(c.pool.frozen)
    res["substituted"] = np.array(sorted(c.substituted_positions), dtype=np.int64)
    res["hist_entries"] = np.array(hist_entries, dtype=np.int64).reshape(len(hist_entries), max(N, 1))
    res["hist_aux"] = np.array(hist_aux, dtype=np.int64)
    res["hist_frozen"] = np.array(hist_frozen)
    mu = c.memory_usage()
    res["memory"] = np.array([mu.quantized_bits, mu.param_bits, mu.pending_bits, mu.pool_bits], dtype=np.int64)
    res["pending_rows"] = np.array(c.pending_rows)
    outs, ws = [], []
    for q in qs:
        r = kv.attend_mixed(q, c)
        outs.append(r.output)
        ws.append(r.weights)
    res["attn_out"] = np.array(outs)
    res["attn_w"] = np.array(ws)
    return res


def gen_caches(kv):
    # config 0 shape (d=128, G=32, R=128, A=32), both pool readings
    k, v, q = config0_stream(0, 1024)
    for N in (32, 3):
        np.savez_compressed(os.path.join(HERE, f"cache_c0_n{N}.npz"), **run_cache(kv, k, v, q, 2, 32, 128, N, 32, 128))
    # reference defaults (G=128, R=32, N=3, A=32, d=64) with planted low-L1 tokens
    rng = np.random.default_rng(5)
    T, d = 1400, 64
    k = rng.standard_normal((T, d))
    k[:, :3] = rng.uniform(4.0, 6.0, size=(T, 3))
    low = rng.choice(T, 40, replace=False)
    k[low] *= 0.02
    k, v = fp16(k), fp16(rng.standard_normal((T, d)))
    q = fp16(rng.standard_normal((3, d)))
    np.savez_compressed(os.path.join(HERE, "cache_default.npz"), **run_cache(kv, k, v, q, 2, 128, 32, 3, 32, 64))
    # fast-freezing pool: small aux so freezing happens mid-stream; G=32, d=64, R=0
    rng = np.random.default_rng(6)
    T, d = 800, 64
    k = rng.standard_normal((T, d)) * 3
    low = rng.choice(T, 60, replace=False)
    k[low] *= 0.01
    k, v = fp16(k), fp16(rng.standard_normal((T, d)))
    q = fp16(rng.standard_normal((2, d)))
    np.savez_compressed(os.path.join(HERE, "cache_freeze.npz"), **run_cache(kv, k, v, q, 2, 32, 0, 4, 5, 64))


def gen_trace(kv):
    """KVTRACE1 fixtures: (1) a tiny file written by the reference's write_trace (bytes +
    arrays) for the reader/writer round trip; (2) the reference's `simulate` replay
    (cli.py:189-236 restated: TieredCache.append + attend_mixed vs attend_full_precision,
    l1_error, memory_usage) on an fp16-valued synthetic trace from its own generator."""
    import io
    import tempfile

    from kvtrace.trace import SyntheticSpec, Trace, TraceHeader, generate_synthetic, write_trace
    from kvtrace.attention import attend_full_precision, l1_error

    rng = np.random.default_rng(77)
    tiny = Trace(TraceHeader(1, 2, 4, 3), *(fp16(rng.standard_normal((1, 2, 3, 4))) for _ in range(3)))
    with tempfile.NamedTemporaryFile(suffix=".kvt") as f:
        write_trace(f.name, tiny)
        raw = open(f.name, "rb").read()

    L, H, d, T = 2, 2, 128, 256
    tr = generate_synthetic(SyntheticSpec(seed=5), L, H, d, T)
    q, k, v = fp16(tr.q), fp16(tr.k), fp16(tr.v)
    G, R, N, A = 32, 64, 3, 32
    cfg = kv.EngineConfig(bits=2, group_size=G, residual=R, outlier_num=N, skip_layers=(), aux_capacity=A,
                          n_layers=L, n_heads=H, head_dim=d)
    caches = {(l, h): kv.TieredCache(cfg, layer=l) for l in range(L) for h in range(H)}
    errs = np.zeros(T)
    for t in range(T):
        tot = 0.0
        for (l, h), c in caches.items():
            c.append(k[l, h, t], v[l, h, t])
            mixed = kv.attend_mixed(q[l, h, t], c)
            ref = attend_full_precision(q[l, h, t], k[l, h, : t + 1], v[l, h, : t + 1])
            tot += l1_error(mixed.output, ref.output)
        errs[t] = tot / len(caches)
    mus = [c.memory_usage() for c in caches.values()]
    usage = np.array([sum(m.quantized_bits for m in mus), sum(m.param_bits for m in mus),
                      sum(m.pending_bits for m in mus), sum(m.pool_bits for m in mus)], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "trace.npz"), tiny_bytes=np.frombuffer(raw, np.uint8),
                        tiny_q=tiny.q, tiny_k=tiny.k, tiny_v=tiny.v,
                        q=q.astype(np.float16), k=k.astype(np.float16), v=v.astype(np.float16),
                        cfg=np.array([G, R, N, A]), step_errors=errs, usage=usage)


def gen_ratio(kv):
    """report.ratio_curve (report.py:159-216) restated with fp16-valued rows (the
    reference draws float32 N(0,1) rows; the product consumes fp16): memory bits and
    ratio vs fp16 at ascending lengths, for the paper setting and the config-1 cache."""
    from kvtrace.cache import TieredCache

    out = {}
    for name, cfg in (("paper", kv.EngineConfig(bits=2, group_size=128, residual=32, outlier_num=3, head_dim=64)),
                      ("c1", kv.EngineConfig(bits=2, group_size=32, residual=128, outlier_num=32, head_dim=128))):
        layer = 0
        while layer in cfg.skip_layers:
            layer += 1
        cache = TieredCache(cfg, layer=layer)
        rng = np.random.default_rng(0)
        d = cfg.head_dim
        seq = [128, 1024, 4096]
        rows, tok = [], 0
        for target in seq:
            while tok < target:
                cache.append(fp16(rng.standard_normal(d)), fp16(rng.standard_normal(d)))
                tok += 1
            u = cache.memory_usage()
            rows.append([target, u.quantized_bits, u.param_bits, u.pending_bits, u.pool_bits, u.total_bits])
        out[name] = np.array(rows, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "ratio.npz"), **out)


def main():
    kv = _kv()
    gen_quant_lines(kv)
    gen_pack(kv)
    gen_pool_streams(kv)
    gen_caches(kv)
    gen_trace(kv)
    gen_ratio(kv)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
