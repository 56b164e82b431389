import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2505_10938_b200 import EngineConfig, OTTCache
from paper_2505_10938_b200.workloads import fill_prefill
cfg = EngineConfig(bits=2, group_size=32, residual=128, outlier_num=32, aux_capacity=32, skip_layers=(), head_dim=128)
B, H, T = 16, 8, 16384
gen = torch.Generator(device="cuda").manual_seed(0)
k = torch.empty((B, H, T, 128), dtype=torch.float16, device="cuda"); v = torch.empty_like(k)
fill_prefill(gen, k, v)
c = OTTCache(cfg, B, H, T + 64)
c.update(k, v)
sm = c.subst_mask.cpu().numpy().view(np.uint32)
grp_with_sel = (sm != 0).sum(1)
print("groups with substitutions per unit: mean", grp_with_sel.mean(), "max", grp_with_sel.max())
print("substituted positions per unit: mean", np.array([bin(int(x)).count('1') for x in sm.ravel()]).reshape(sm.shape).sum(1).mean())
meta = c.pool_meta.cpu().numpy(); print("frozen frac", meta[:,2].mean(), "aux", meta[:,1].mean())
ap = c.aux_pos.cpu().numpy(); print("last aux position (freeze point) mean", ap.max(1).mean(), "max", ap.max())
