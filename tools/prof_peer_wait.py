"""Device time of PeerGather.wait (the per-layer symmetric-memory signal-pad barrier of the fused
head-output all-gather) at world size 1: 80 layers x 20 steps of wait() only, CUDA-event timed.

  python tools/prof_peer_wait.py
"""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2505_10938_b200 import EngineConfig, OTTCache  # noqa: E402
from paper_2505_10938_b200.parallel import PeerGather  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
L, steps = 80, 20
cfg = EngineConfig(bits=2, group_size=32, residual=128, outlier_num=32, aux_capacity=32, skip_layers=(), head_dim=128)
caches = [OTTCache(cfg, 128, 8, max_tokens=256) for _ in range(L)]
pg = PeerGather(caches, 8)
for _ in range(3):
    for l in range(L):
        pg.wait(l)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    pg.next_step()
    for l in range(L):
        pg.wait(l)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (steps * L)
print(f"PeerGather.wait at world 1: {us:.2f} us per layer ({us * L / 1e3:.3f} ms per 80-layer step)")
pg.close()
dist.destroy_process_group()
