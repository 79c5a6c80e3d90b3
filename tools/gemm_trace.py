"""Phase breakdown of one GEMM launch from the kernel's %globaltimer trace
(GemmDesc::trace): per CTA entry / prologue / first TMA / first MMA / last
commit / epilogue start / epilogue end / exit, in us relative to the
earliest entry.  python tools/gemm_trace.py o|ffn1|wgrad_gpt [--1sm]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
bf = torch.bfloat16
which = sys.argv[1]
one = "--1sm" in sys.argv
shapes = {"o": (4096, 1024, 1024, "fwd", K.EPI_BIAS | K.EPI_RESID), "ffn1": (4096, 4096, 1024, "fwd", K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT),
          "qkv": (4096, 3072, 1024, "fwd", K.EPI_BIAS), "ffn2": (4096, 1024, 4096, "fwd", K.EPI_BIAS | K.EPI_RESID),
          "plain": (4096, 1024, 1024, "fwd", 0), "wgrad_gpt": (1600, 6400, 1024, "wgrad", 0),
          "wgrad_o": (1024, 1024, 4096, "wgrad", 0), "big": (8192, 8192, 8192, "fwd", 0),
          "gpt_ffn2": (1024, 1600, 6400, "fwd", K.EPI_BIAS | K.EPI_RESID), "gpt_ffn2_plain": (1024, 1600, 6400, "fwd", 0)}
M, N, Kd, kind, epi = shapes[which]
tr = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
if kind == "fwd":
    A = torch.randn(M, Kd, device=dev).to(bf); B = torch.randn(N, Kd, device=dev).to(bf)
    C = torch.empty(M, N, device=dev, dtype=bf); X = torch.empty(M, N, device=dev, dtype=bf)
    R = torch.randn(M, N, device=dev).to(bf); bias = torch.zeros(N, device=dev)
    f = lambda t: K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=epi, bias=bias, resid=R if epi & K.EPI_RESID else None,
                         aux_out=X if epi & K.EPI_AUX_OUT else None, force_1sm=one, trace=t)
else:
    A = torch.randn(Kd, M, device=dev).to(bf); B = torch.randn(Kd, N, device=dev).to(bf)
    C = torch.zeros(M, N, device=dev)
    f = lambda t: K.gemm(A, B, C, M, N, Kd, lda=M, ldb=N, ldc=N, a_mn_major=True, b_mn_major=True,
                         epi=K.EPI_OUT_F32_ACC, force_1sm=one, trace=t)
for _ in range(5):
    f(None)
for _ in range(3):
    f(tr)
torch.cuda.synchronize()
t = tr.view(148, 16).cpu().numpy().astype("float64")
used = t[:, 0] > 0
t = t[used]
r = t - t[:, :1]  # cycles since this CTA's entry
names = ["entry", "prologue", "first_tma", "first_mma", "last_commit", "epi_start", "epi_end", "exit",
         "c0_tmem", "c0_epi_done", "c0_before_xwait", "c0_after_xwait", "c1_tmem", "c1_epi_done", "c1_before_xwait", "c1_after_xwait"]
import numpy as np  # noqa: E402
print(f"{which} {M}x{N}x{Kd} ctas={used.sum()} 1sm={one} (cycles since CTA entry)")
for i, n in enumerate(names):
    sel = t[:, i] > 0
    if not sel.any():
        continue
    nz = r[sel, i]
    print(f"  {n:12s} min {nz.min():8.0f}  median {np.median(nz):8.0f}  max {nz.max():8.0f}  (n={len(nz)})")
