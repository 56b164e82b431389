"""Bulk-prefill (K1 flush) timing: OTTCache.update of a seeded config-0-style prompt.
  python tools/prof_flush.py [--batch 16] [--kv 8] [--ctx 4096] [--pool 32]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_10938_b200 import EngineConfig, OTTCache  # noqa: E402
from paper_2505_10938_b200.workloads import fill_prefill  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--kv", type=int, default=8)
ap.add_argument("--ctx", type=int, default=4096)
ap.add_argument("--pool", type=int, default=32)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--bits", type=int, default=2)
ap.add_argument("--group", type=int, default=32)
args = ap.parse_args()
torch.cuda.set_device(0)
cfg = EngineConfig(bits=args.bits, group_size=args.group, residual=128, outlier_num=args.pool, aux_capacity=32, skip_layers=(),
                   head_dim=128)
gen = torch.Generator(device="cuda").manual_seed(0)
k = torch.empty((args.batch, args.kv, args.ctx, 128), dtype=torch.float16, device="cuda")
v = torch.empty_like(k)
fill_prefill(gen, k, v)
ts = []
for _ in range(args.reps + 1):
    c = OTTCache(cfg, args.batch, args.kv, args.ctx + 64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c.update(k, v)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
groups = (args.ctx - 128) // 32
print(f"prefill B={args.batch} Hkv={args.kv} T={args.ctx} N={args.pool}: {min(ts[1:]):.3f} ms "
      f"({groups} groups/unit, {min(ts[1:]) * 1e3 / groups:.2f} us/group)")
