"""Per-CTA timeline of one K2 launch (variant build with -DOTT_EXP_TIMELINE, loaded through
OTT_LIB_PATH): start/end globaltimer, SM and CTA kind (quantized split vs full-precision tier).
  OTT_LIB_PATH=tools/variants/tl.so python tools/prof_timeline.py --batch 16 --rep 4 --ctx 4096"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_10938_b200 import EngineConfig, OTTCache, _native  # noqa: E402
from paper_2505_10938_b200.workloads import fill_prefill  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--kv", type=int, default=8)
ap.add_argument("--rep", type=int, default=4)
ap.add_argument("--ctx", type=int, default=4096)
ap.add_argument("--splits", type=int, default=0)
args = ap.parse_args()
torch.cuda.set_device(0)
cfg = EngineConfig(bits=2, group_size=32, residual=128, outlier_num=32, aux_capacity=32, skip_layers=(), head_dim=128)
cache = OTTCache(cfg, args.batch, args.kv, args.ctx + 64)
gen = torch.Generator(device="cuda").manual_seed(0)
k = torch.empty((args.batch, args.kv, args.ctx, 128), dtype=torch.float16, device="cuda")
v = torch.empty_like(k)
fill_prefill(gen, k, v)
cache.update(k, v)
q = torch.randn((args.batch, args.kv * args.rep, 128), generator=gen, device="cuda").half()
out = torch.empty_like(q)
splits = args.splits or cache.splits(args.rep)
lib = _native.lib()
lib.ott_exp_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
for _ in range(3):
    cache.attend(q, out=out, n_splits=splits)
torch.cuda.synchronize()
lib.ott_exp_timeline_clear()
cache.attend(q, out=out, n_splits=splits)
torch.cuda.synchronize()
U = args.batch * args.kv
n = min(16384, U * (splits + 2))
buf = np.zeros((n, 4), dtype=np.uint64)
assert lib.ott_exp_timeline(buf.ctypes.data, n) == 0
buf = buf[buf[:, 1] > 0]
t0 = buf[:, 0].min()
s, e = (buf[:, 0] - t0) / 1e3, (buf[:, 1] - t0) / 1e3
role = buf[:, 3].astype(np.int64)
y, nparts = role & 0xFFFF, role >> 40
kind = y >= splits
print(f"shape B={args.batch} Hkv={args.kv} rep={args.rep} T={args.ctx} splits={splits}: {len(buf)} CTAs, span {e.max():.1f} us")
for name, m in (("q whole", (~kind) & (nparts == 1)), ("q piece", (~kind) & (nparts > 1)), ("fp-tier", kind)):
    if m.any():
        d = e[m] - s[m]
        print(f"  {name:8s} n={m.sum():5d} start {s[m].min():6.1f}..{s[m].max():6.1f}  end {e[m].min():6.1f}..{e[m].max():6.1f}"
              f"  dur mean {d.mean():6.1f} max {d.max():6.1f} us")
sm = buf[:, 2].astype(int)
per_sm = np.bincount(sm, minlength=148)
last = np.array([e[sm == i].max() if (sm == i).any() else 0 for i in range(148)])
busy = np.array([(e[sm == i] - s[sm == i]).sum() for i in range(148)])
print(f"  CTAs per SM: min {per_sm.min()} max {per_sm.max()} mean {per_sm.mean():.2f}; last end per SM {last.min():.1f}..{last.max():.1f} us;"
      f" CTA-us per SM {busy.min():.0f}..{busy.max():.0f}")
hist = np.histogram(e, bins=10)[0]
print("  CTA end-time histogram (10 bins over the span):", hist.tolist())
U = args.batch * args.kv
# first-wave quantized CTAs: per-SM duration spread (same work per CTA)
w1 = (~kind) & (s < 1.0)
if w1.sum() > 0:
    d = e[w1] - s[w1]
    sms = sm[w1]
    per = {}
    for x, dd in zip(sms, d):
        per.setdefault(int(x), []).append(dd)
    cnt = np.array([len(per.get(i, [])) for i in range(148)])
    mean_by_sm = np.array([np.mean(per[i]) if i in per else np.nan for i in range(148)])
    print(f"  wave-1 quantized CTAs: {w1.sum()}, per SM {cnt.min()}..{cnt.max()}; duration {d.min():.1f}..{d.max():.1f} us;"
          f" per-SM mean duration {np.nanmin(mean_by_sm):.1f}..{np.nanmax(mean_by_sm):.1f}")
    order = np.argsort(mean_by_sm)
    print("  fastest SMs", [(int(i), round(float(mean_by_sm[i]), 1), int(cnt[i])) for i in order[:6]])
    print("  slowest SMs", [(int(i), round(float(mean_by_sm[i]), 1), int(cnt[i])) for i in order[-8:] if not np.isnan(mean_by_sm[i])])
    # unit index of wave-1 CTAs vs duration (data placement)
    units = ((role >> 16) & 0xFFFFFF)[w1]
    du = d
    print("  duration by unit quartile:", [round(float(du[(units >= U * k // 4) & (units < U * (k + 1) // 4)].mean()), 1)
                                          for k in range(4) if ((units >= U * k // 4) & (units < U * (k + 1) // 4)).any()])

# duration by dispatch rank (linear CTA index // SM count) of the quantized CTAs
lin = np.arange(len(buf))  # buffer rows are in linear blockIdx order (x fastest, then y)
rank = lin // 148
for rk in range(int(rank.max()) + 1):
    m = (~kind) & (rank == rk)
    if m.any():
        d = e[m] - s[m]
        print(f"  rank {rk}: {m.sum()} quantized CTAs, duration mean {d.mean():.1f} min {d.min():.1f} max {d.max():.1f} us, start {s[m].mean():.1f}")
