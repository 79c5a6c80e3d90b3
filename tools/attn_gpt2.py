"""Times the fused causal attention kernels at the GPT-2 1.5B bench shape
(micro-batch 1 x 1024 tokens, 25 heads, H = 1600) and, under ncu, gives one
launch of each to profile (`--iters 1 --warm 1`)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--warm", type=int, default=5)
args = ap.parse_args()


def bench(fn):
    for _ in range(args.warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / args.iters * 1e3  # us


dev = torch.device("cuda:0")
B, S, nh = 1, 1024, 25
H = nh * 64
R = B * S
qkv = torch.randn(3, nh, B, S, 64, device=dev).to(torch.bfloat16)
dout = torch.randn(nh, B, S, 64, device=dev).to(torch.bfloat16)
ctx = torch.zeros(R, H, dtype=torch.bfloat16, device=dev)
lse = torch.zeros(nh * B, S, device=dev)
dqkv = torch.zeros(R, 3 * H, dtype=torch.bfloat16, device=dev)
dsum = torch.zeros(nh * B, S, device=dev)
dq = torch.zeros(nh * B, S, 64, device=dev)
f = 4.0 * nh * B * S * S * 64 / 2  # causal QK^T + PV
t = bench(lambda: K.attention_fwd(qkv, ctx, lse, B, S, nh, H, True))
tb = bench(lambda: K.attention_bwd(qkv, ctx, lse, dout, dqkv, dsum, dq, B, S, nh, H, True))
print(f"gpt2 causal attention: fwd {t:.1f} us ({f / t * 1e-6:.0f} TF/s), "
      f"bwd {tb:.1f} us ({2.5 * f / tb * 1e-6:.0f} TF/s incl. S recompute)")
