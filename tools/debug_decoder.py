"""Debug: compare OTT vs fp16-cache attention inside the small decoder."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
from paper_2505_10938_b200.model import Decoder, DecoderConfig, apply_rope

torch.cuda.set_device(0)
cfg = DecoderConfig(n_layers=3, hidden=512, n_heads=4, n_kv_heads=4, head_dim=128, mlp=1024, vocab=1000)
B, T = 2, 400
prompt = torch.randint(0, cfg.vocab, (B, T), generator=torch.Generator().manual_seed(3)).cuda()
ott = Decoder(cfg, B, T + 16, kv="ott", seed=7)
ref = Decoder(cfg, B, T + 16, kv="fp16", seed=7)
t1, t2 = ott.prefill(prompt), ref.prefill(prompt)
print("prefill tokens equal", torch.equal(t1, t2))
for l in range(3):
    print("layer", l, "N", ott.caches[l].N, "Tq", ott.caches[l].quantized_tokens, "tot", ott.caches[l].total_tokens)
    kref = ref.k_cache[l, :, :, :T].float()
    vref = ref.v_cache[l, :, :, :T].float()
    print("  k std %.4f v std %.4f" % (kref.std().item(), vref.std().item()))
    q = torch.randn(B, 4, 128, device="cuda").half()
    o_ott = ott.caches[l].attend(q).float()
    o_ref = F.scaled_dot_product_attention(q.float()[:, :, None], kref, vref)[:, :, 0]
    err = (o_ott - o_ref).abs().max().item()
    print("  attend max err %.4g  |o| max %.4g" % (err, o_ref.abs().max().item()))
    # dequantized reconstruction error of K
    u = ott.caches[l].unit(0, 0)
    import numpy as np
    kq = np.concatenate([blk.to_matrix() if hasattr(blk, "to_matrix") else blk.dequantize() for blk in u.quantized_k]) if u.quantized_k else None
    if kq is not None:
        print("  K dequant max err (unit 0,0):", float(np.abs(kq - kref[0, 0, :kq.shape[0]].cpu().numpy()).max()))
