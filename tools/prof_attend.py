"""Standalone attention timing / ncu target: one layer of a BASELINE-shaped cache,
prefilled on the GPU, then `iters` attend calls (CUDA-event timed).

  python tools/prof_attend.py [--batch 64] [--kv 8] [--rep 4] [--ctx 8192] [--iters 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2505_10938_b200 import EngineConfig, OTTCache  # noqa: E402
from paper_2505_10938_b200.workloads import fill_prefill  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--kv", type=int, default=8)
ap.add_argument("--rep", type=int, default=4)
ap.add_argument("--ctx", type=int, default=8192)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--pool", type=int, default=32)
ap.add_argument("--bits", type=int, default=2)
ap.add_argument("--group", type=int, default=32)
ap.add_argument("--splits", type=int, default=0)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--append", action="store_true", help="time append_attend (fused ring write) steps")
ap.add_argument("--graph", action="store_true", help="capture the iters attend launches in one CUDA graph (no host gaps)")
args = ap.parse_args()

torch.cuda.set_device(0)
cfg = EngineConfig(bits=args.bits, group_size=args.group, residual=128, outlier_num=args.pool, aux_capacity=32, skip_layers=(),
                   head_dim=args.dim)
cache = OTTCache(cfg, args.batch, args.kv, args.ctx + 64 + args.iters)
gen = torch.Generator(device="cuda").manual_seed(0)
k = torch.empty((args.batch, args.kv, args.ctx, args.dim), dtype=torch.float16, device="cuda")
v = torch.empty_like(k)
fill_prefill(gen, k, v)
cache.update(k, v)
del k, v
q = torch.randn((args.batch, args.kv * args.rep, args.dim), generator=gen, device="cuda").half()
out = torch.empty_like(q)
splits = args.splits or cache.splits(args.rep)
for _ in range(3):
    cache.attend(q, out=out, n_splits=splits)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
kn = torch.randn((args.batch, args.kv, args.dim), generator=gen, device="cuda").half()
vn = torch.randn((args.batch, args.kv, args.dim), generator=gen, device="cuda").half()
if args.graph:  # same launches, replayed from one graph so small shapes are not host bound
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(args.iters):
            cache.attend(q, out=out, n_splits=splits)
    g.replay()
    torch.cuda.synchronize()
e0.record()
if args.graph:
    g.replay()
else:
    for _ in range(args.iters):
        if args.append:
            cache.append_attend(kn, vn, q, out=out, n_splits=splits)
        else:
            cache.attend(q, out=out, n_splits=splits)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.iters
Tq = cache.quantized_tokens
Tp = cache.total_tokens - Tq
U = args.batch * args.kv
per_unit = Tq * 64 * args.bits // 2 + (Tq // 32) * 1024 + Tq * 8 + Tq // 8 + (Tp + min(args.pool, Tq)) * 512 + 2 * args.rep * 256
gbs = U * per_unit / (ms * 1e-3) / 1e9
print(f"attend B={args.batch} Hkv={args.kv} rep={args.rep} T={args.ctx} splits={splits}: {ms * 1e3:.1f} us, "
      f"{gbs:.0f} GB/s algorithmic ({U * per_unit / 1e6:.1f} MB)")
