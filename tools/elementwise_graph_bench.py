"""Device time of the HBM-bound stage kernels (LayerNorm fwd/bwd, bias-grad
column sums) at the BERT-48 slice shape, each as a CUDA graph of `reps`
launches over rotating buffers (no host overhead), against the HBM floor
(algorithmic bytes / measured HBM bandwidth).

    python tools/elementwise_graph_bench.py [--rows 4096] [--h 1024]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_01045_b200 import kernels as K  # noqa: E402


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            fn(i)
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
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--h", type=int, default=1024)
    ap.add_argument("--nbuf", type=int, default=4)
    args = ap.parse_args()
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f).get("hbm_gbs", 6556.0)) * 1e9
    except Exception:  # noqa: BLE001
        hbm = 6556e9
    dev = torch.device("cuda:0")
    R, H, nb = args.rows, args.h, args.nbuf
    bf = torch.bfloat16
    x = [torch.randn(R, H, device=dev).to(bf) for _ in range(nb)]
    y = [torch.empty(R, H, device=dev, dtype=bf) for _ in range(nb)]
    dy = [torch.randn(R, H, device=dev).to(bf) for _ in range(nb)]
    dres = [torch.randn(R, H, device=dev).to(bf) for _ in range(nb)]
    dx = [torch.empty(R, H, device=dev, dtype=bf) for _ in range(nb)]
    mean = [torch.empty(R, device=dev) for _ in range(nb)]
    rstd = [torch.empty(R, device=dev) for _ in range(nb)]
    g = torch.ones(H, device=dev)
    bta = torch.zeros(H, device=dev)
    dg = torch.zeros(H, device=dev)
    db = torch.zeros(H, device=dev)
    out = []
    t = graph_time(lambda i: K.layernorm_fwd(x[i % nb], g, bta, y[i % nb], mean[i % nb], rstd[i % nb], R, H))
    out.append(("layernorm_fwd", t, R * H * 4 + R * 8))
    t = graph_time(lambda i: K.layernorm_bwd(dy[i % nb], x[i % nb], mean[i % nb], rstd[i % nb], g, dres[i % nb],
                                             dx[i % nb], dg, db, R, H))
    out.append(("layernorm_bwd (+dresid)", t, R * H * 8 + R * 8))
    for cols in (1024, 3072, 4096):
        tt = [torch.randn(R, cols, device=dev).to(bf) for _ in range(nb)]
        acc = torch.zeros(cols, device=dev)
        t = graph_time(lambda i: K.colsum_acc(tt[i % nb], acc, R, cols))
        out.append((f"colsum_acc {cols}", t, R * cols * 2))
    for name, t, byts in out:
        floor = byts / hbm
        print(json.dumps({"kernel": name, "us": round(t * 1e6, 2), "floor_us": round(floor * 1e6, 2),
                          "gbs": round(byts / t / 1e9), "frac": round(floor / t, 3)}))


if __name__ == "__main__":
    main()
