"""Runs one GEMM shape a few times (for ncu): python tools/gemm_one.py o|ffn1|ffn2|wgrad_gpt [--cublas]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
bf = torch.bfloat16
which = sys.argv[1]
cub = "--cublas" in sys.argv
if which == "o":
    M, N, Kd = 4096, 1024, 1024
    A = torch.randn(M, Kd, device=dev).to(bf); B = torch.randn(N, Kd, device=dev).to(bf)
    C = torch.empty(M, N, device=dev, dtype=bf); R = torch.randn(M, N, device=dev).to(bf)
    bias = torch.zeros(N, device=dev)
    f = (lambda: torch.matmul(A, B.T, out=C)) if cub else \
        (lambda: K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=K.EPI_BIAS | K.EPI_RESID, bias=bias, resid=R))
elif which == "ffn2":
    M, N, Kd = 4096, 1024, 4096
    A = torch.randn(M, Kd, device=dev).to(bf); B = torch.randn(N, Kd, device=dev).to(bf)
    C = torch.empty(M, N, device=dev, dtype=bf); R = torch.randn(M, N, device=dev).to(bf)
    bias = torch.zeros(N, device=dev)
    f = (lambda: torch.matmul(A, B.T, out=C)) if cub else \
        (lambda: K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=K.EPI_BIAS | K.EPI_RESID, bias=bias, resid=R))
elif which == "ffn1":
    M, N, Kd = 4096, 4096, 1024
    A = torch.randn(M, Kd, device=dev).to(bf); B = torch.randn(N, Kd, device=dev).to(bf)
    C = torch.empty(M, N, device=dev, dtype=bf); X = torch.empty(M, N, device=dev, dtype=bf)
    bias = torch.zeros(N, device=dev)
    f = (lambda: torch.matmul(A, B.T, out=C)) if cub else \
        (lambda: K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT,
                        bias=bias, aux_out=X))
else:  # GPT-2 ffn2 wgrad: dW[1600, 6400] += dY[1024,1600]^T X[1024, 6400]
    M, N, Kd = 1600, 6400, 1024
    A = torch.randn(Kd, M, device=dev).to(bf); B = torch.randn(Kd, N, device=dev).to(bf)
    C = torch.zeros(M, N, device=dev); C16 = torch.empty(M, N, device=dev, dtype=bf)
    f = (lambda: torch.matmul(A.T, B, out=C16)) if cub else \
        (lambda: K.gemm(A, B, C, M, N, Kd, lda=M, ldb=N, ldc=N, a_mn_major=True, b_mn_major=True,
                        epi=K.EPI_OUT_F32_ACC))
for _ in range(6):
    f()
torch.cuda.synchronize()
print("ok")
