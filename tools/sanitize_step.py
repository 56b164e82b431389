"""Small decode workload for compute-sanitizer (racecheck / synccheck / memcheck): bulk prefill
(scan + per-group flush kernels), host-count append_attend steps crossing a decode flush
(fused ring write, attention, PDL combine), device-counter decode steps, a 4-bit cache.

  compute-sanitizer --tool racecheck python tools/sanitize_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_10938_b200 import EngineConfig, OTTCache  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
for bits in (2, 4):
    cfg = EngineConfig(bits=bits, group_size=32, residual=32, outlier_num=8, aux_capacity=16, skip_layers=(),
                       head_dim=128)
    B, H, rep, T = 1, 2, 8, 200
    c = OTTCache(cfg, B, H, max_tokens=T + 80)
    k = torch.from_numpy((rng.standard_normal((B, H, T + 70, 128)) * np.where(np.arange(128) < 4, 15, 1))
                         .astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((B, H, T + 70, 128)).astype(np.float16)).cuda()
    q = torch.from_numpy(rng.standard_normal((B, H * rep, 128)).astype(np.float16)).cuda()
    c.update(k[:, :, :T].contiguous(), v[:, :, :T].contiguous())
    out = torch.empty_like(q)
    for t in range(T, T + 40):
        c.append_attend(k[:, :, t].contiguous(), v[:, :, t].contiguous(), q, out=out)
    c.sync_counters()
    s = c.splits(rep)
    for t in range(T + 40, T + 70):
        c.decode_step(k[:, :, t].contiguous(), v[:, :, t].contiguous(), q, out, s)
    torch.cuda.synchronize()
    print("bits", bits, "ok", float(out.float().abs().sum()))
