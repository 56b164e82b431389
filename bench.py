"""bench.py — OTT 2-bit quantized-KV decode on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE configs[4], the Llama-3-70B-shaped KV cache —
80 layers, B=128, H_q=64, H_kv=8, d=128, 16,384-token context, 2-bit G=32,
R=128, outlier pool 32 (aux 32, paper skip_layers (0, 1)). A decode step =
for every layer: append one token per (batch, kv head) unit (flush the
residual window when due) + mixed-tier attention for all 64 query heads.
Under torchrun (N>1) the B x H_kv units are partitioned across ranks (contiguous
unit ranges, GQA groups whole) and head outputs are all-gathered every layer (P2P
stores fused into the attention epilogue, or NCCL with OTT_GATHER=nccl).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c3|c3s|c2|c0|c1]
  python bench.py --impl reference ...   # CPU oracle port of the reference path

Prints one JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quantized-KV decode attention HBM GB/s (% of peak); decode tokens/sec at 1/2/4/8 GPU"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def unit_bytes(wl, Tq, Tp, pool_rows, ref_accounting=False):
    """Algorithmic HBM bytes one attend launch reads/writes per (batch, kv-head)
    unit: codes + params + full-precision tiers + q/out."""
    d, G = wl.head_dim, wl.group_size
    codes = 2 * Tq * d * wl.bits // 8
    if ref_accounting:  # reference cache.py:188-203 accounting: params at 16 bits
        params = (Tq // G) * d * 2 * 2 + Tq * 2 * 2
        mask = 0
    else:  # this build's layout: float32 (step, x_min) per line + 1 mask bit per token
        params = (Tq // G) * d * 2 * 4 + Tq * 2 * 4
        mask = Tq // 8
    fp = (Tp + pool_rows) * d * 2 * 2
    qo = 2 * wl.n_rep * d * 2
    return codes + params + mask + fp + qo


class Clocks:
    """Sample nvidia-smi SM clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            return None
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU arm


def cpu_sample(wl, n_units, steps, threads, seed=0):
    """Time the reference path restated in C (oracle/, OpenMP over units) on a
    bounded sample: n_units (layer, b, kv-head) units prefilled to the workload's
    context, then `steps` decode steps (append + n_rep attend_mixed calls each).
    Returns seconds per unit-step measured with all `threads` busy."""
    import numpy as np

    import oracle

    rng = np.random.default_rng(seed)
    d, T = wl.head_dim, wl.context
    scale = np.ones((n_units, 1, d), np.float32)
    for u in range(n_units):
        scale[u, 0, rng.choice(d, 4, replace=False)] = 15.0
    k = (rng.standard_normal((n_units, T, d), dtype=np.float32) * scale).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((n_units, T, d), dtype=np.float32).astype(np.float16).astype(np.float32)
    N = wl.outlier_num
    caches = [oracle.OracleCache(2, wl.group_size, wl.residual, N, wl.aux_capacity, d) for _ in range(n_units)]
    oracle.prefill(caches, k, v, threads)
    del k, v
    times = []
    for _ in range(steps):
        kr = (rng.standard_normal((n_units, d), dtype=np.float32) * scale[:, 0]).astype(np.float16).astype(np.float32)
        vr = rng.standard_normal((n_units, d), dtype=np.float32).astype(np.float16).astype(np.float32)
        q = rng.standard_normal((n_units, wl.n_rep, d), dtype=np.float32).astype(np.float16).astype(np.float32)
        t0 = time.perf_counter()
        oracle.decode_step(caches, kr, vr, q, wl.n_rep, threads)
        times.append(time.perf_counter() - t0)
    return statistics.median(times) / n_units


def workload_config(wl, world):
    """The `config` dict both arms print (workload only; measurements go elsewhere)."""
    U = wl.batch * wl.n_kv_heads
    cache_gb = wl.n_layers * U * (
        (max(0, (wl.context - wl.residual)) // wl.group_size) * (wl.group_size * wl.head_dim * wl.bits // 4
                                                                 + 8 * wl.head_dim + 8 * wl.group_size)
        + (wl.group_size + wl.residual + 2 * wl.outlier_num) * wl.head_dim * 4) / 1e9
    return {"workload": wl.name, "bits": wl.bits, "layers": wl.n_layers, "batch": wl.batch,
            "n_q_heads": wl.n_q_heads, "n_kv_heads": wl.n_kv_heads, "head_dim": wl.head_dim, "context": wl.context,
            "group_size": wl.group_size, "residual": wl.residual, "outlier_pool": wl.outlier_num,
            "aux_capacity": wl.aux_capacity, "skip_layers": list(wl.skip_layers),
            "partition": f"{U} (batch x kv-head) units / {world} rank(s), contiguous, GQA groups whole",
            "l2": ("working set > L2 (126 MB): ~%.0f GB of cache" % cache_gb if cache_gb > 0.126 else
                   "working set %.0f MB fits the 126 MB L2 (no flush between steps)" % (cache_gb * 1e3))}


def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    n_units = max(threads, 1)
    units_per_step = wl.n_layers * wl.batch * wl.n_kv_heads
    per_unit = cpu_sample(wl, n_units, args.warmup + args.steps, threads)
    step_s = per_unit * units_per_step
    tok_s = wl.batch / step_s
    sample = (f"{n_units} (layer,b,kv-head) units prefilled to T={wl.context}, {args.warmup + args.steps} decode "
              f"steps each (append + {wl.n_rep} attend_mixed), extrapolated x{units_per_step / n_units:.0f} to the "
              f"full step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 params / f32 attention", "data": "synthetic",
        "config": workload_config(wl, world),
        "extrapolated": True, "sample_units": n_units, "units_per_step": units_per_step,
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- GPU arm


def expected_k_halves(step64, d):
    """The record's fp16 K step halves (sh, sl) in pair order from exact float64 steps."""
    import numpy as np

    from paper_2505_10938_b200.cache import kpair_index

    step64 = np.asarray(step64, np.float64)
    sh = step64.astype(np.float16)
    sl = (step64 - sh.astype(np.float64)).astype(np.float16)
    idx = kpair_index(np.arange(d), d)
    sh_p, sl_p = np.empty(d, np.float16), np.empty(d, np.float16)
    sh_p[idx], sl_p[idx] = sh, sl
    return sh_p, sl_p


def check_unit(view, ref):
    """Bit-exact quantization state of one bench unit vs the oracle: codes, the record's K
    step halves, V params (float32 of the exact values), pool entries (positions, scores),
    aux positions, frozen flag."""
    import numpy as np

    d = view.config.head_dim
    if len(view.quantized_k) != ref.n_blocks:
        return False
    for b in range(ref.n_blocks):
        blk = ref.block(b)
        if view.quantized_k[b].codes != blk["k_codes"] or view.quantized_v[b].codes != blk["v_codes"]:
            return False
        sh, sl = expected_k_halves(blk["k_step"], d)
        if not (np.array_equal(view.k_sh16[b].view(np.uint16), sh.view(np.uint16))
                and np.array_equal(view.k_sl16[b].view(np.uint16), sl.view(np.uint16))
                and np.array_equal(view.v_step32[b], blk["v_step"].astype(np.float32))
                and np.array_equal(view.v_xmin32[b], blk["v_xmin"].astype(np.float32))):
            return False
    pe, ae = ref.pool_entries(), ref.aux_entries()
    return ([e.position for e in view.pool.entries] == pe["position"].tolist()
            and [e.score for e in view.pool.entries] == pe["score"].tolist()
            and [e.position for e in view.pool.aux] == ae["position"].tolist()
            and view.pool.frozen == ref.frozen)


def run_ours(args, wl, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_10938_b200 import EngineConfig, OTTCache
    from paper_2505_10938_b200.parallel import PeerGather, all_gather_heads, unit_bounds
    from paper_2505_10938_b200.workloads import decode_rows, fill_prefill

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    # scalars of the rank collectives live where the backend reduces them (gloo: host)
    coll_dev = dev if world == 1 or dist.get_backend() == "nccl" else torch.device("cpu")
    H, Hq, d, L, nrep = wl.n_kv_heads, wl.n_q_heads, wl.head_dim, wl.n_layers, wl.n_rep
    U = wl.batch * H
    u_lo, u_hi = unit_bounds(U, world, rank)
    Ul = u_hi - u_lo  # this rank's (batch x kv-head) units: one OTTCache "batch row" each
    cfg = EngineConfig(bits=wl.bits, group_size=wl.group_size, residual=wl.residual, outlier_num=wl.outlier_num,
                       aux_capacity=wl.aux_capacity, skip_layers=wl.skip_layers, n_layers=L, n_heads=H, head_dim=d)
    total_steps = 2 * (args.warmup + args.steps) + wl.group_size + 8
    max_tokens = wl.context + total_steps
    caches = [OTTCache(cfg, Ul, 1, max_tokens, layer=l, device=dev) for l in range(L)]
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    # parity sample (rank 0): units of the first layer (a paper skip layer: N = 0), the third
    # and the last layer; their fp16 input streams are kept on the host for the oracle
    check = rank == 0 and not args.no_parity
    samp_layers = sorted({0, min(2, L - 1), L - 1})
    samp = {l: sorted({(3 * l) % Ul, (Ul - 1 - 5 * l) % Ul}) for l in samp_layers} if check else {}
    host_pre = {}
    t0 = time.time()
    kbuf = torch.empty((Ul, 1, wl.context, d), dtype=torch.float16, device=dev)
    vbuf = torch.empty_like(kbuf)
    scales = []
    pev = []  # device time of each layer's bulk prefill (OTTCache.update = K1 over all groups)
    for l in range(L):
        scales.append(fill_prefill(gen, kbuf, vbuf))
        for u in samp.get(l, []):
            host_pre[(l, u)] = (kbuf[u, 0].cpu().numpy(), vbuf[u, 0].cpu().numpy())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        caches[l].update(kbuf, vbuf)
        e1.record()
        pev.append((e0, e1))
    torch.cuda.synchronize()
    prefill_ms = sum(a.elapsed_time(b) for a, b in pev)
    # algorithmic bytes of one layer's prefill: K/V rows in, block records + pending rows out
    n_grp = (wl.context - wl.residual) // wl.group_size
    prefill_bytes = Ul * (wl.context * d * 2 * 2 + n_grp * caches[0].record_bytes
                          + (wl.context - n_grp * wl.group_size) * d * 2 * 2)
    del kbuf, vbuf
    torch.cuda.empty_cache()
    prefill_s = time.time() - t0

    n_sets = 2
    kin = torch.empty((n_sets, L, Ul, 1, d), dtype=torch.float16, device=dev)
    vin = torch.empty_like(kin)
    for s in range(n_sets):
        for l in range(L):
            kin[s, l], vin[s, l] = decode_rows(gen, scales[l], Ul, 1)
    qin = torch.randn((n_sets, L, Ul, nrep, d), generator=gen, device=dev).half()
    outs = torch.empty((L, Ul, nrep, d), dtype=torch.float16, device=dev)
    # multi-GPU head-output all-gather: P2P stores fused into the attention's combine kernel
    # (parallel.PeerGather, default) or a separate NCCL all_gather per layer (OTT_GATHER=nccl)
    gather_mode = (os.environ.get("OTT_GATHER", "p2p") if world > 1 else "none")
    pg, gather_note = None, ""
    if gather_mode == "p2p":
        try:
            pg = PeerGather(caches, nrep)
        except Exception as exc:  # no P2P mapping between these GPUs: keep the NCCL collective
            gather_mode, gather_note = "nccl", f" (P2P unavailable: {type(exc).__name__}: {str(exc)[:120]})"
        ok = torch.tensor([1 if pg is not None else 0], device=coll_dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank must take the same path
        if not int(ok.item()) and pg is not None:
            pg.close()
            pg, gather_mode, gather_note = None, "nccl", " (P2P unavailable on another rank)"
    gathered = (torch.empty((L, U, nrep, d), dtype=torch.float16, device=dev) if gather_mode == "nccl" else None)
    splits = [c.splits(nrep) for c in caches]

    launches = {"n": 0}
    appended = []  # decode-row set of every step, in order (oracle replay)

    def step(i, ev=None, fev=None):
        s = i % n_sets
        appended.append(s)
        if pg is not None:
            pg.next_step()
        for l in range(L):
            c = caches[l]
            # the flush this token makes due (cache.py:138) never needs the token itself
            # (R >= 1): launched first, timed on its own
            if c.total_tokens + 1 - c.quantized_tokens - c.config.residual >= c.config.group_size:
                if fev is not None:
                    fe = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    fe[0].record()
                c.quantize_oldest_group()
                if fev is not None:
                    fe[1].record()
                    fev.append(fe)
                launches["n"] += 1
            if ev is not None:
                ev[l][0].record()
            # append + attend: the attention kernel writes the new K/V row into the ring
            c.append_attend(kin[s, l], vin[s, l], qin[s, l], out=outs[l] if pg is None else pg.out(l),
                            n_splits=splits[l])
            if ev is not None:
                ev[l][1].record()
            launches["n"] += 2
            if pg is not None:
                pg.wait(l)
            elif gathered is not None:
                all_gather_heads(outs[l], out=gathered[l])

    for i in range(args.warmup):
        step(i)
    # start the timed window at a step that flushes every layer: any K timed steps then hold
    # ceil(K / G) decode flushes per layer (cache.py:138), at least the proportional share
    pre = 0
    c0 = caches[0]
    while c0.total_tokens + 1 - c0.quantized_tokens - c0.config.residual < c0.config.group_size:
        step(args.warmup + pre)
        pre += 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local_rank)
    clocks.start()
    time.sleep(0.3)
    launches["n"] = 0
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(L)] for _ in range(args.steps)]
    fevs = []
    tok_before = [(c.quantized_tokens, c.total_tokens) for c in caches]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    for i in range(args.steps):
        step(args.warmup + pre + i, evs[i], fevs)
    end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = start.elapsed_time(end)
    ms_t = torch.tensor([ms], device=coll_dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ms_per_step = ms / args.steps
    value = wl.batch * args.steps / (ms / 1e3)  # whole-job decode tokens/s (all ranks)
    last_set = appended[-1]

    # roofline of the dominant kernel (attention): SURVEY 8(d) algorithmic bytes per launch
    # (16-bit param accounting, cache.py:188-203); this build's layout bytes beside it
    att_ms, att_bytes, att_bytes_ref = 0.0, 0, 0
    for i in range(args.steps):
        for l in range(L):
            att_ms += evs[i][l][0].elapsed_time(evs[i][l][1])
    n_att = args.steps * L
    for l, c in enumerate(caches):
        q0, t0_ = tok_before[l]
        for i in range(args.steps):
            T = t0_ + i + 1
            Tq = ((T - wl.residual) // wl.group_size) * wl.group_size if T >= wl.residual + wl.group_size else 0
            Tq = max(Tq, q0)
            pool_rows = min(c.N, Tq)
            att_bytes += Ul * unit_bytes(wl, Tq, T - Tq, pool_rows)
            att_bytes_ref += Ul * unit_bytes(wl, Tq, T - Tq, pool_rows, ref_accounting=True)
    avg_att_s = att_ms / n_att / 1e3
    achieved_ref = att_bytes_ref / n_att / avg_att_s / 1e9
    achieved_layout = att_bytes / n_att / avg_att_s / 1e9
    flush_ms = sum(a.elapsed_time(b) for a, b in fevs)
    peak, peak_kind = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_attention_summary.json")) as f:
            prof = json.load(f)
        if prof.get("workload") == wl.name:
            traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    gpu_launches = launches["n"]

    # parity of the bench's own caches (rank 0, after timing): sampled units vs the oracle fed
    # the same fp16 rows (prefill + every appended decode row), state bit-exact and the last
    # timed step's attention within tolerance
    parity = None
    if check:
        import oracle

        kin_h, vin_h, q_h = kin.cpu().numpy(), vin.cpu().numpy(), qin[last_set].cpu().numpy()
        out_h = (outs if pg is None else torch.stack([pg.out(l).view(Ul, nrep, d) for l in range(L)])).cpu().numpy()
        keys = [(l, u) for l in samp_layers for u in samp[l]]
        refs = [oracle.OracleCache(wl.bits, wl.group_size, wl.residual, cfg.outlier_capacity(l), wl.aux_capacity, d)
                for (l, u) in keys]
        threads = len(os.sched_getaffinity(0))
        oracle.prefill(refs, np.stack([host_pre[key][0] for key in keys]).astype(np.float32),
                       np.stack([host_pre[key][1] for key in keys]).astype(np.float32), threads)
        exact, worst = True, 0.0
        for ref, (l, u) in zip(refs, keys):
            for s in appended:
                ref.append(kin_h[s, l, u, 0].astype(np.float32), vin_h[s, l, u, 0].astype(np.float32))
            exact &= check_unit(caches[l].unit(u, 0), ref)
            for r in range(nrep):
                o_ref = ref.attend(q_h[l, u, r].astype(np.float32))
                err = np.abs(out_h[l, u, r].astype(np.float32) - o_ref)
                worst = max(worst, float((err / (2e-3 + 1e-2 * np.abs(o_ref))).max()))
        parity = {"units": [f"layer{l}/unit{u_lo + u}" for (l, u) in keys], "bit_exact": bool(exact),
                  "max_err_over_tol": worst, "tol": "2e-3 + 1e-2 |ref| (fp16 output vs oracle f32)",
                  "checked": "K/V codes, K step halves, V params, pool entries/scores, aux, frozen; "
                             "attention of the last timed step (all n_rep heads)"}

    # e2e: through the public API with HOST buffers (pinned), copies inside the timed region;
    # with N > 1 every rank reads back the gathered [B, H_q, d] of every layer
    e2e = None
    if not args.no_e2e:
        from paper_2505_10938_b200.pipeline import HostDecodePipeline

        k_h = kin[0].cpu().pin_memory()
        v_h = vin[0].cpu().pin_memory()
        qh = qin[0].cpu().pin_memory()
        o_h = torch.empty((L, U if world > 1 else Ul, nrep, d), dtype=torch.float16).pin_memory()
        gather = None
        if gathered is not None:
            def gather(o_local, l):
                all_gather_heads(o_local, out=gathered[l])
                return gathered[l]
        pipe = HostDecodePipeline(caches, nrep, gather=gather, peer_gather=pg, world=world)
        pipe.step(k_h, v_h, qh, o_h)  # warm-up (streams, events)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            pipe.step(k_h, v_h, qh, o_h)
        e1.record()
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], device=coll_dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        h2d = L * (k_h[0].numel() + v_h[0].numel() + qh[0].numel()) * 2
        d2h = L * o_h[0].numel() * 2
        e2e = {"value": wl.batch * args.steps / (float(e_ms.item()) / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
        if world > 1:  # the host copy of the last layer = an NCCL all-gather of the local rows
            last = L - 1
            local = pg.out(last).view(Ul, nrep, d) if pg is not None else pipe.o_d[last % 2].view(Ul, nrep, d)
            ref = all_gather_heads(local.contiguous())
            e2e["gathered_output_verified"] = bool(torch.equal(ref.cpu(), o_h[last]))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        n_units = threads
        per_unit = cpu_sample(wl, n_units, 2, threads)
        cpu_step = per_unit * L * U
        cpu = {"value": wl.batch / cpu_step, "unit": "tokens/s", "cores": threads, "kind": "port",
               "sample": f"{n_units} units prefilled to T={wl.context}, 2 decode steps (append + {nrep} "
                         f"attend_mixed each), extrapolated to {L * U} units per step"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": f"u{wl.bits} codes / fp16 K-param halves + f32 V params / f16 rows, "
                                          f"f32 accumulate", "data": "synthetic",
            "config": workload_config(wl, world),
            "gather": {"none": "none (1 GPU)", "nccl": "NCCL all_gather_into_tensor per layer",
                       "p2p": "P2P stores fused into the combine kernel + signal-pad barrier per layer"}[
                gather_mode] + gather_note,
            "roofline": {"bound": "hbm", "achieved": achieved_ref, "peak": peak, "unit": "GB/s",
                         "frac": achieved_ref / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes": "SURVEY 8(d) algorithmic bytes (16-bit params, cache.py:188-203)",
                         "kernel": "ott attend (split-K decode with fused ring write + combine)",
                         "avg_launch_us": avg_att_s * 1e6, "bytes_per_launch": att_bytes_ref / n_att,
                         "layout_bytes_per_launch": att_bytes / n_att, "achieved_layout_GBs": achieved_layout,
                         "frac_layout": achieved_layout / peak},
            "decode_flush": {"flushes_in_window": len(fevs),
                             "us_per_layer_flush": flush_ms * 1e3 / len(fevs) if fevs else None,
                             "ms_per_step_amortized": flush_ms / args.steps,
                             "untimed_steps_before_window": args.warmup + pre},
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            # bulk prefill (OTTCache.update, K1 over all groups), device-timed per layer
            "prefill": {"ms_per_layer": prefill_ms / L, "tokens_per_s": Ul * wl.context * L / (prefill_ms / 1e3),
                        "achieved_GBs": prefill_bytes * L / (prefill_ms / 1e3) / 1e9,
                        "frac": prefill_bytes * L / (prefill_ms / 1e3) / 1e9 / peak,
                        "bytes_per_layer": prefill_bytes, "tokens": "per (b, kv-head) unit",
                        "wall_s": round(prefill_s, 2)},
            "gpu_launches": gpu_launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)



# ----------------------------------------------------------------------------- config 1 (model decode)


def c1_fidelity(dev, prompt, steps, k_outliers):
    """Config-1 fidelity, teacher-forced on the fp16 decoder's greedy tokens: the reference's
    simulate metric (per-step attention-output L1 vs exact attention, mean over layers x
    batch x heads, cli.py:208-218) and the next-token distribution vs the fp16-KV decoder
    (KL(p_fp16 || p), mean |logit diff|, top-1 agreement), for OTT (N = 32) and N = 0 (the
    same quantizer without outlier tracking, KIVI-like)."""
    import torch

    from paper_2505_10938_b200 import EngineConfig
    from paper_2505_10938_b200.model import LLAMA2_7B, Decoder

    B, T = prompt.shape
    ref = Decoder(LLAMA2_7B, B, T + steps + 8, kv="fp16", device=dev, seed=0, k_outliers=k_outliers)
    toks = [ref.prefill(prompt)]
    ref_logits = []
    for t in range(steps):
        toks.append(ref.decode(toks[-1]))
        ref_logits.append(ref.last_logits.float())
    del ref
    torch.cuda.empty_cache()
    res = {}
    for name, n_out in (("ott_n32", 32), ("n0", 0)):
        cfg = EngineConfig(bits=2, group_size=32, residual=128, outlier_num=n_out, aux_capacity=32,
                           n_layers=LLAMA2_7B.n_layers, n_heads=LLAMA2_7B.n_kv_heads, head_dim=LLAMA2_7B.head_dim)
        m = Decoder(LLAMA2_7B, B, T + steps + 8, kv="ott", ott=cfg, device=dev, seed=0, k_outliers=k_outliers,
                    track_exact=True)
        m.prefill(prompt)
        kl, l1, agree = 0.0, 0.0, 0.0
        for t in range(steps):
            m.decode(toks[t])  # teacher forcing: the fp16 decoder's token stream
            lo, lr = m.last_logits.float(), ref_logits[t]
            lp, lq = torch.log_softmax(lr, -1), torch.log_softmax(lo, -1)
            kl += float((lp.exp() * (lp - lq)).sum(-1).mean())
            l1 += float((lo - lr).abs().mean())
            agree += float((lo.argmax(-1) == lr.argmax(-1)).float().mean())
        res[name] = {"attn_l1_per_step": sum(m.attn_l1) / len(m.attn_l1), "logit_kl_vs_fp16": kl / steps,
                     "logit_mean_abs_diff_vs_fp16": l1 / steps, "top1_agreement_vs_fp16": agree / steps}
        del m
        torch.cuda.empty_cache()
    return res


def run_c1(args, rank, world, local_rank):
    """BASELINE configs[1]: Llama-2-7B-shaped random-init decoder, B=8, 2048-token
    random prompt, 256 greedy decode steps with the OTT cache (2-bit, G=32, R=128,
    pool 32, paper skip_layers (0, 1)); the fp16-KV-cache decoder with the same
    weights is timed beside it. Replicas only under torchrun (each rank its own batch).
    The throughput runs use the plain random-init model; the fidelity runs (c1_fidelity) add
    the outlier-channel / outlier-token key structure (isotropic random-init keys would make
    every 2-bit scheme look alike)."""
    import torch

    from paper_2505_10938_b200.model import LLAMA2_7B, Decoder

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B, T, steps = 8, 2048, args.steps if args.steps != 32 else 256
    k_out = 4
    prompt = torch.randint(0, LLAMA2_7B.vocab, (B, T), generator=torch.Generator().manual_seed(rank)).to(dev)
    from paper_2505_10938_b200 import EngineConfig

    res = {}
    for kv in ("ott", "fp16", "flash"):
        # fp16 baselines: the same engine and CUDA graph with a residual window longer than the
        # run, so every K/V row stays in the fp16 tier; and an independent plain fp16 KV cache
        # attended by FlashAttention-2's decode kernel in the same graph step
        lossless = EngineConfig(bits=2, group_size=32, residual=T + steps + 64, outlier_num=0,
                                n_layers=LLAMA2_7B.n_layers, n_heads=LLAMA2_7B.n_kv_heads, head_dim=LLAMA2_7B.head_dim)
        if kv == "flash":
            m = Decoder(LLAMA2_7B, B, T + steps + 8, kv="flash", device=dev, seed=0)
        else:
            m = Decoder(LLAMA2_7B, B, T + steps + 8, kv="ott", ott=None if kv == "ott" else lossless, device=dev,
                        seed=0)
        torch.cuda.synchronize()
        t0 = time.time()
        tok = m.prefill(prompt)
        torch.cuda.synchronize()
        prefill_s = time.time() - t0
        # the whole decode step (32 layers) is one captured CUDA graph with the cache's
        # token counts in device memory
        dec = m.decode_graph
        for _ in range(args.warmup):  # warm-up decode steps (graph capture, cuBLAS heuristics)
            tok = dec(tok)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            tok = dec(tok)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[kv] = {"tok_s": B * steps / (ms / 1e3), "ms_per_step": ms / steps, "prefill_s": prefill_s}
        del m
        torch.cuda.empty_cache()
    fid = c1_fidelity(dev, prompt, 64, k_out) if not args.no_fidelity else None
    if rank == 0:
        print(json.dumps({
            "metric": "decode tokens/s (config 1: Llama-2-7B-shaped decoder, OTT cache)", "value": res["ott"]["tok_s"] * world,
            "unit": "tokens/s", "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": res["ott"]["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16 weights/activations, u2 KV codes",
            "data": "synthetic (random ids, random-init N(0, 0.02) weights; fidelity runs: + outlier-channel / "
                    "outlier-token key structure, model.Decoder(k_outliers=4))",
            "config": {"workload": "config1-llama2-7b-B8-prompt2048-decode%d" % steps, "batch": B, "prompt": T,
                       "layers": LLAMA2_7B.n_layers, "parallelism": f"replicas x{world}", "decode": "CUDA graph per step"},
            "fp16_kv_baseline": {"value": res["fp16"]["tok_s"] * world, "ms_per_step": res["fp16"]["ms_per_step"],
                                 "how": "same engine + CUDA graph, residual window > run: all K/V rows fp16"},
            "fp16_kv_flash_baseline": {"value": res["flash"]["tok_s"] * world,
                                       "ms_per_step": res["flash"]["ms_per_step"],
                                       "how": "plain fp16 KV cache + flash_attn_with_kvcache (FlashAttention-2 "
                                              "library decode kernel), same CUDA-graph step"},
            "prefill_s": {k_: round(r_["prefill_s"], 3) for k_, r_ in res.items()},
            "fidelity": fid and {"steps": 64, "teacher_forced": "fp16-KV decoder's greedy tokens", **fid},
        }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of sampled bench units")
    ap.add_argument("--no-fidelity", action="store_true", help="config 1: skip the teacher-forced fidelity runs")
    ap.add_argument("--bits", type=int, default=2, help="code width of the cache (BASELINE: 2)")
    ap.add_argument("--layers", type=int, default=0, help="override the workload's layer count (variants)")
    args = ap.parse_args()
    from paper_2505_10938_b200.workloads import WORKLOADS

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook (tests/test_gpu_bench_multirank.py): every rank on GPU 0 with a gloo process group
    # and the NCCL-style gather path, so the N > 1 branch runs on a one-GPU box; no rank's kernels
    # wait on another's (the gather is a host-side collective)
    one_gpu_test = os.environ.get("OTT_BENCH_ONE_GPU_TEST") == "1"
    if one_gpu_test:
        local_rank = 0
        os.environ["OTT_GATHER"] = "nccl"
    if args.config == "c1":
        if args.impl == "reference":
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "config 1 is a model decode; the reference "
                                  "has no model (bench.py --impl reference times the default config-4 path)"}))
            return
        run_c1(args, rank, world, local_rank)
        return
    wl = WORKLOADS[args.config]
    if args.bits != 2:  # a non-BASELINE variant, named as such
        import dataclasses

        wl = dataclasses.replace(wl, bits=args.bits, name=f"{wl.name}-{args.bits}bit")
    if args.layers:
        import dataclasses

        wl = dataclasses.replace(wl, n_layers=args.layers, name=f"{wl.name}-{args.layers}L")
    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if one_gpu_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, wl, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
