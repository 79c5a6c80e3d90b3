"""Peer-copy bandwidth of one 8 MiB activation send (BERT-48's Split-Concat
hand-off at 8 samples) as 1 copy vs k concurrent chunk copies on k streams,
GPU 0 -> GPU 1, device-timed with events, each variant captured as a CUDA
graph (as the executor's step is).

    python tools/p2p_chunks.py [--mib 8]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=float, nargs="+", default=[2, 4, 8, 16])
    args = ap.parse_args()
    assert torch.cuda.device_count() >= 2
    d0, d1 = torch.device("cuda:0"), torch.device("cuda:1")
    torch.cuda.set_device(0)
    for mib in args.mib:
        n = int(mib * (1 << 20)) // 2
        src = torch.randn(n, device=d0).to(torch.bfloat16)
        dst = torch.empty(n, dtype=torch.bfloat16, device=d1)
        for k in (1, 2, 4, 8):
            main_s = torch.cuda.Stream(d0)
            side = [torch.cuda.Stream(d0) for _ in range(k)]
            chunks = [(i * n // k, (i + 1) * n // k) for i in range(k)]

            def step():
                for s, (a, b) in zip(side, chunks):
                    s.wait_stream(main_s)
                    with torch.cuda.stream(s):
                        dst[a:b].copy_(src[a:b], non_blocking=True)
                for s in side:
                    main_s.wait_stream(s)

            with torch.cuda.stream(main_s):
                for _ in range(3):
                    step()
            torch.cuda.synchronize()
            mode = "graph"
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=main_s):
                    for _ in range(10):
                        step()
                torch.cuda.synchronize()
                run = g.replay
            except Exception:  # noqa: BLE001 -- eager fallback
                torch.cuda.synchronize()
                mode = "eager"

                def run():
                    for _ in range(10):
                        step()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(main_s):
                run()
                e0.record()
                for _ in range(5):
                    run()
                e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 50
            assert torch.equal(dst.cpu(), src.cpu())
            print(json.dumps({"mib": mib, "chunks": k, "mode": mode, "us": round(us, 2), "gbps": round(n * 2 / us / 1e3, 1)}))


if __name__ == "__main__":
    main()
