"""Config-1 decode timing / ncu target: Llama-2-7B-shaped decoder, B=8, 2048-token
prompt, N graph-replayed OTT decode steps.  python tools/prof_c1.py [--steps 4]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_10938_b200.model import LLAMA2_7B, Decoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--eager", action="store_true")
args = ap.parse_args()
torch.cuda.set_device(0)
B, T = 8, 2048
m = Decoder(LLAMA2_7B, B, T + args.steps + 16, kv="ott", seed=0)
prompt = torch.randint(0, LLAMA2_7B.vocab, (B, T), generator=torch.Generator().manual_seed(0)).cuda()
tok = m.prefill(prompt)
dec = m.decode if args.eager else m.decode_graph
tok = dec(tok)  # capture
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off: only the decode steps below
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.steps):
    tok = dec(tok)
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"decode {'eager' if args.eager else 'graph'}: {e0.elapsed_time(e1) / args.steps:.3f} ms/step")
