"""Times the tcgen05 GEMM at the transformer-stage shapes (CUDA events)."""
import json
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
    return s.elapsed_time(e) / iters * 1e-3


def main():
    dev = torch.device("cuda:0")
    H = 1024
    out = []
    for T in (2048, 4096, 8192):
        for name, N, Kd in (("qkv", 3 * H, H), ("o", H, H), ("ffn1", 4 * H, H), ("ffn2", H, 4 * H)):
            A = torch.randn(T, Kd, device=dev).to(torch.bfloat16)
            W = torch.randn(N, Kd, device=dev).to(torch.bfloat16)
            C = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
            bias = torch.zeros(N, device=dev)
            fl = 2.0 * T * N * Kd
            row = {"T": T, "gemm": name}
            for bn in (0, 128, 256):
                t = bench(lambda: K.gemm(A, W, C, T, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=K.EPI_BIAS, bias=bias,
                                         force_bn=bn))
                row[f"fwd_bn{bn}_tflops"] = round(fl / t / 1e12, 1)
            # wgrad: dW[N,K] += dY^T X  (both MN-major), fp32 accumulate
            dY = torch.randn(T, N, device=dev).to(torch.bfloat16)
            dW = torch.zeros(N, Kd, device=dev)
            t = bench(lambda: K.gemm(dY, A, dW, N, Kd, T, lda=N, ldb=Kd, ldc=Kd, a_mn_major=True, b_mn_major=True,
                                     epi=K.EPI_OUT_F32_ACC))
            row["wgrad_tflops"] = round(fl / t / 1e12, 1)
            # dgrad: dX[T,K] = dY W  (B MN-major)
            dX = torch.empty(T, Kd, device=dev, dtype=torch.bfloat16)
            t = bench(lambda: K.gemm(dY, W, dX, T, Kd, N, lda=N, ldb=Kd, ldc=Kd, b_mn_major=True))
            row["dgrad_tflops"] = round(fl / t / 1e12, 1)
            t = bench(lambda: torch.matmul(A, W.T, out=C))
            row["cublas_tflops"] = round(fl / t / 1e12, 1)
            out.append(row)
            print(json.dumps(row), flush=True)
    A = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    B = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    C = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    t = bench(lambda: K.gemm(A, B, C, 8192, 8192, 8192, lda=8192, ldb=8192, ldc=8192), iters=10)
    t2 = bench(lambda: torch.matmul(A, B.T, out=C), iters=10)
    print(json.dumps({"square8192_tflops": round(2 * 8192**3 / t / 1e12, 1),
                      "cublas_8192_tflops": round(2 * 8192**3 / t2 / 1e12, 1)}))


if __name__ == "__main__":
    main()
