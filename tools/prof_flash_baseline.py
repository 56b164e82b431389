"""One decode-attention launch over an fp16 KV cache with FlashAttention-2's library kernel
(flash_attn_with_kvcache), for comparison with K2 on the same shape (graph-replayed, CUDA events).
  python tools/prof_flash_baseline.py [--batch 128] [--kv 8] [--rep 8] [--ctx 16384]"""
import argparse

import torch
from flash_attn import flash_attn_with_kvcache

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--kv", type=int, default=8)
ap.add_argument("--rep", type=int, default=8)
ap.add_argument("--ctx", type=int, default=16384)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
torch.cuda.set_device(0)
B, Hkv, H, T, d = args.batch, args.kv, args.kv * args.rep, args.ctx, 128
kc = torch.randn((B, T + 1, Hkv, d), device="cuda", dtype=torch.float16)
vc = torch.randn_like(kc)
q = torch.randn((B, 1, H, d), device="cuda", dtype=torch.float16)
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
for _ in range(3):
    flash_attn_with_kvcache(q, kc, vc, cache_seqlens=lens)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(args.iters):
        flash_attn_with_kvcache(q, kc, vc, cache_seqlens=lens)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / args.iters
nbytes = 2 * B * T * Hkv * d * 2
print(f"flash_attn_with_kvcache fp16 B={B} Hkv={Hkv} H={H} T={T}: {us:.1f} us, {nbytes / 1e6:.1f} MB, "
      f"{nbytes / (us * 1e-6) / 1e9:.0f} GB/s")
