"""The step's dominant GEMMs at the bench shapes (BERT-48 replica slice of
4096 tokens), each launched a few times -- a short program for
`ncu --set full -k regex:gemm`.  Launch order: ffn1 (gelu+aux epilogue),
ffn2 (bias+residual), qkv, wgrad (fp32 accumulate)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
T, H, F = 4096, 1024, 4096
x = torch.randn(T, H, device=dev).to(torch.bfloat16)
w1 = (torch.randn(F, H, device=dev) * 0.03).to(torch.bfloat16)
w2 = (torch.randn(H, F, device=dev) * 0.03).to(torch.bfloat16)
wqkv = (torch.randn(3 * H, H, device=dev) * 0.03).to(torch.bfloat16)
b1 = torch.zeros(F, device=dev)
b2 = torch.zeros(H, device=dev)
g = torch.empty(T, F, device=dev, dtype=torch.bfloat16)
z = torch.empty(T, F, device=dev, dtype=torch.bfloat16)
y = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
qkv = torch.empty(T, 3 * H, device=dev, dtype=torch.bfloat16)
dw = torch.zeros(F, H, device=dev)
for rep in range(3):
    K.gemm(x, w1, g, T, F, H, lda=H, ldb=H, ldc=F, epi=K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT, bias=b1, aux_out=z)
    K.gemm(g, w2, y, T, H, F, lda=F, ldb=F, ldc=H, epi=K.EPI_BIAS | K.EPI_RESID, bias=b2, resid=x)
    K.gemm(x, wqkv, qkv, T, 3 * H, H, lda=H, ldb=H, ldc=3 * H, epi=K.EPI_BIAS, bias=b2.repeat(3))
    K.gemm(g, x, dw, F, H, T, lda=F, ldb=H, ldc=H, a_mn_major=True, b_mn_major=True, epi=K.EPI_OUT_F32_ACC)
torch.cuda.synchronize()
print("ok")
