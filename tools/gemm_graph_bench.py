"""Per-shape tcgen05 GEMM vs cuBLAS at the BERT-48 stage shapes, each timed as
a CUDA graph of `reps` back-to-back launches (no host overhead), with the
epilogues the layers actually use.  Inputs rotate over `nbuf` buffer sets so
operands are not all L2-resident.

    python tools/gemm_graph_bench.py [--T 4096] [--variants default,1sm,bn128]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            fn(i)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 5 / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, nargs="+", default=[4096])
    ap.add_argument("--H", type=int, default=1024)
    ap.add_argument("--F", type=int, default=4096)
    ap.add_argument("--nbuf", type=int, default=4)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    H, F, nb = args.H, args.F, args.nbuf
    bf = torch.bfloat16
    total = {}
    for T in args.T:
        # (name, M, N, K, kind, epi): kind fwd = X W^T, dgrad = dY W, wgrad = dY^T X (fp32 +=)
        shapes = [("qkv", T, 3 * H, H, "fwd", K.EPI_BIAS), ("o", T, H, H, "fwd", K.EPI_BIAS | K.EPI_RESID),
                  ("ffn1", T, F, H, "fwd", K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT),
                  ("ffn2", T, H, F, "fwd", K.EPI_BIAS | K.EPI_RESID),
                  ("ffn2_dgrad", T, F, H, "dgrad", K.EPI_DGELU), ("ffn1_dgrad", T, H, F, "dgrad", 0),
                  ("o_dgrad", T, H, H, "dgrad", 0), ("qkv_dgrad", T, H, 3 * H, "dgrad", 0),
                  ("ffn2_wgrad", H, F, T, "wgrad", 0), ("ffn1_wgrad", F, H, T, "wgrad", 0),
                  ("o_wgrad", H, H, T, "wgrad", 0), ("qkv_wgrad", 3 * H, H, T, "wgrad", 0)]
        for name, M, N, Kd, kind, epi in shapes:
            fl = 2.0 * M * N * Kd
            if kind == "fwd":
                A = [torch.randn(M, Kd, device=dev).to(bf) for _ in range(nb)]
                B = [torch.randn(N, Kd, device=dev).to(bf) for _ in range(nb)]
                C = [torch.empty(M, N, device=dev, dtype=bf) for _ in range(nb)]
                aux = [torch.empty(M, N, device=dev, dtype=bf) for _ in range(nb)]
                res = [torch.randn(M, N, device=dev).to(bf) for _ in range(nb)]
                bias = torch.zeros(N, device=dev)

                def ours(i, v):
                    j = i % nb
                    K.gemm(A[j], B[j], C[j], M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=epi, bias=bias,
                           aux_out=aux[j] if epi & K.EPI_AUX_OUT else None,
                           resid=res[j] if epi & K.EPI_RESID else None, **v)

                def cub(i):
                    j = i % nb
                    torch.matmul(A[j], B[j].T, out=C[j])
            elif kind == "dgrad":  # dX[M=T, N] = dY[T, K] W[K, N]
                A = [torch.randn(M, Kd, device=dev).to(bf) for _ in range(nb)]
                B = [torch.randn(Kd, N, device=dev).to(bf) for _ in range(nb)]
                C = [torch.empty(M, N, device=dev, dtype=bf) for _ in range(nb)]
                aux = [torch.randn(M, N, device=dev).to(bf) for _ in range(nb)]

                def ours(i, v):
                    j = i % nb
                    K.gemm(A[j], B[j], C[j], M, N, Kd, lda=Kd, ldb=N, ldc=N, b_mn_major=True, epi=epi,
                           aux_in=aux[j] if epi & K.EPI_DGELU else None, **v)

                def cub(i):
                    j = i % nb
                    torch.matmul(A[j], B[j], out=C[j])
            else:  # dW[M, N] += dY[T, M]^T X[T, N]
                A = [torch.randn(Kd, M, device=dev).to(bf) for _ in range(nb)]
                B = [torch.randn(Kd, N, device=dev).to(bf) for _ in range(nb)]
                C = [torch.zeros(M, N, device=dev) for _ in range(nb)]
                C16 = [torch.empty(M, N, device=dev, dtype=bf) for _ in range(nb)]

                def ours(i, v):
                    j = i % nb
                    K.gemm(A[j], B[j], C[j], M, N, Kd, lda=M, ldb=N, ldc=N, a_mn_major=True, b_mn_major=True,
                           epi=K.EPI_OUT_F32_ACC, **v)

                def cub(i):
                    j = i % nb
                    torch.matmul(A[j].T, B[j], out=C16[j])
            row = {"T": T, "gemm": name, "M": M, "N": N, "K": Kd}
            for vname, v in (("ours", {}), ("1sm", {"force_1sm": True}), ("bn128", {"force_bn": 128, "force_1sm": True}),
                             ("pair256", {"force_bn": 256}), ("pair128", {"force_bn": 128})):
                try:
                    t = graph_time(lambda i: ours(i, v))
                    row[vname] = round(fl / t / 1e12, 1)
                    row[vname + "_us"] = round(t * 1e6, 2)
                except Exception as e:  # noqa: BLE001
                    row[vname] = str(e)[:60]
            t = graph_time(cub)
            row["cublas"] = round(fl / t / 1e12, 1)
            row["cublas_us"] = round(t * 1e6, 2)
            for k in ("ours", "cublas"):
                if isinstance(row.get(k), float):
                    total[k] = total.get(k, 0.0) + fl / (row[k] * 1e12)
            print(json.dumps(row), flush=True)
    print(json.dumps({"sum_us": {k: round(v * 1e6, 1) for k, v in total.items()}}))


if __name__ == "__main__":
    main()
