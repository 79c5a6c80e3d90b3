"""Times the fused attention kernels and the stage's other non-GEMM kernels at
the bench shape (slice of 8 samples x 512 tokens, 16 heads, H = 1024)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402


def bench(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


dev = torch.device("cuda:0")
B, S, nh = 8, 512, 16
H = nh * 64
R = B * S
qkv = torch.randn(3, nh, B, S, 64, device=dev).to(torch.bfloat16)
dout = torch.randn(nh, B, S, 64, device=dev).to(torch.bfloat16)
ctx = torch.zeros(R, H, dtype=torch.bfloat16, device=dev)
lse = torch.zeros(nh * B, S, device=dev)
dqkv = torch.zeros(R, 3 * H, dtype=torch.bfloat16, device=dev)
dsum = torch.zeros(nh * B, S, device=dev)
dq = torch.zeros(nh * B, S, 64, device=dev)
fl = 4.0 * nh * B * S * S * 64  # QK^T + PV
for causal in (False, True):
    t = bench(lambda: K.attention_fwd(qkv, ctx, lse, B, S, nh, H, causal))
    tb = bench(lambda: K.attention_bwd(qkv, ctx, lse, dout, dqkv, dsum, dq, B, S, nh, H, causal))
    f = fl / (2 if causal else 1)
    print(f"causal={causal}: fwd {t:.1f} us ({f / t * 1e-6:.0f} TF), bwd {tb:.1f} us ({2.5 * f / tb * 1e-6:.0f} TF incl. recompute)")
x = torch.randn(R, H, device=dev).to(torch.bfloat16)
g = torch.ones(H, device=dev)
y = torch.empty_like(x)
mean = torch.empty(R, device=dev)
rstd = torch.empty(R, device=dev)
print(f"layernorm fwd {bench(lambda: K.layernorm_fwd(x, g, g, y, mean, rstd, R, H)):.1f} us "
      f"(HBM floor {(R * H * 4) / 6.5e12 * 1e6:.1f} us)")
dg = torch.zeros(H, device=dev)
print(f"layernorm bwd {bench(lambda: K.layernorm_bwd(x, x, mean, rstd, g, x, y, dg, dg, R, H)):.1f} us "
      f"(HBM floor {(R * H * 8) / 6.5e12 * 1e6:.1f} us)")
for cols in (1024, 3072, 4096):
    t = torch.randn(R, cols, device=dev).to(torch.bfloat16)
    db = torch.zeros(cols, device=dev)
    print(f"colsum {cols}: {bench(lambda: K.colsum_acc(t, db, R, cols)):.1f} us "
          f"(HBM floor {R * cols * 2 / 6.5e12 * 1e6:.1f} us)")
