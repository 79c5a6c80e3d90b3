"""Per-CTA phase breakdown of one attention forward launch from the kernel's
%globaltimer marks (AttentionDesc::trace).  Slots: 0 entry, 1 after setup,
2-5 S_j ready (softmax warp 2), 6-9 P_j written, 10 last O accumulated, 11 exit,
12 MMA warp saw Q, 15 smid.  python tools/attn_trace.py [B S heads causal] [--bwd]
(--bwd: the backward's main kernel, one CTA per key tile: 2-5 S/dP of query
tile i ready, 6-9 P/dS written, 10 last dQ drained, 11 exit)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402

bwd = "--bwd" in sys.argv
argv = [a for a in sys.argv[1:] if a != "--bwd"]
B, S, nh, causal = (int(a) for a in (argv + ["8", "512", "16", "0"][len(argv):])[:4])
dev = torch.device("cuda:0")
H = nh * 64
qkv = torch.randn(3, nh, B, S, 64, device=dev).to(torch.bfloat16)
ctx = torch.zeros(B * S, H, dtype=torch.bfloat16, device=dev)
lse = torch.zeros(nh * B, S, device=dev)
n_cta = nh * B * (S // 128) * (2 if causal and not bwd else 1)
trace = torch.zeros(n_cta * 16 + 16, dtype=torch.int64, device=dev)
if bwd:
    dout = torch.randn(nh, B, S, 64, device=dev).to(torch.bfloat16)
    dqkv = torch.zeros(B * S, 3 * H, dtype=torch.bfloat16, device=dev)
    dsum = torch.zeros(nh * B, S, device=dev)
    dq = torch.zeros(nh * B, S, 64, device=dev)
    K.attention_fwd(qkv, ctx, lse, B, S, nh, H, bool(causal))
for _ in range(5):
    if bwd:
        K.attention_bwd_traced(qkv, ctx, lse, dout, dqkv, dsum, dq, B, S, nh, H, trace, bool(causal))
    else:
        K.attention_fwd_traced(qkv, ctx, lse, B, S, nh, H, trace, bool(causal))
torch.cuda.synchronize()
t = trace.cpu().numpy()[: n_cta * 16].reshape(n_cta, 16).astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t[:, :12] - t0) / 1000.0  # us
rel[t[:, :12] == 0] = np.nan
print(f"{len(t)} CTAs, launch span {np.nanmax(rel[:, 11]):.2f} us")
names = ["entry", "setup", "S0", "S1", "S2", "S3", "P0", "P1", "P2", "P3", "O done", "exit"]
d = np.diff(rel, axis=1)
for i in range(11):
    print(f"  {names[i]:>6s} -> {names[i + 1]:<6s} median {np.nanmedian(d[:, i]):7.3f} us  p90 {np.nanpercentile(d[:, i], 90):7.3f}")
print(f"  CTA lifetime median {np.nanmedian(rel[:, 11] - rel[:, 0]):.2f} us")
ent = np.sort(rel[:, 0])
print("  entry-time quantiles (us):", np.round(np.nanpercentile(ent, [0, 25, 50, 57, 60, 75, 100]), 2))
sm = t[:, 15].astype(int)
per_sm = np.bincount(sm, minlength=148)
print("  CTAs per SM: min", per_sm.min(), "max", per_sm.max())
