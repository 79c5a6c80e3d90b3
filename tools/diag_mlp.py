"""Diagnostic: per-tensor gradient error of the device step vs the fp64 oracle
and vs a bf16-rounding-emulating oracle (MLP)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.executor_ref import Model, batch_data, full_batch_step, init_layer  # noqa: E402
from paper_2007_01045_b200.runtime import Executor  # noqa: E402
from parity_util import rel_fro  # noqa: E402


def bf16(a):
    a = np.asarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def emulated(L, H, gbs, M):
    m = Model(kind="mlp", layers=L, hidden=H)
    ps = [init_layer(m, l, 1234) for l in range(L)]
    x, t = batch_data(m, 1234, 0, gbs)
    x, t = bf16(x), bf16(t)
    W = [bf16(p["W"]) for p in ps]
    b = [p["b"].astype(np.float64) for p in ps]
    B = gbs // M
    grads = {(l, k): 0 for l in range(L) for k in "Wb"}
    numel = gbs * H
    for i in range(M):
        xs = [x[i * B:(i + 1) * B]]
        for l in range(L):
            z = xs[-1] @ W[l].T + b[l]
            xs.append(bf16(np.maximum(z, 0) if l < L - 1 else z))
        dz = bf16(2 * (xs[-1] - t[i * B:(i + 1) * B]) / numel)
        for l in reversed(range(L)):
            grads[(l, "W")] = grads[(l, "W")] + dz.T @ xs[l]
            grads[(l, "b")] = grads[(l, "b")] + dz.sum(0)
            if l > 0:
                dz = bf16((dz @ W[l]) * (xs[l] > 0))
    return grads


for L, H, gbs, M in [(4, 256, 32, 4), (16, 1024, 64, 8)]:
    model = dict(kind="mlp", layers=L, hidden=H)
    plan = {"stages": [{"layers": [0, L], "gpus": [0]}]}
    ref = full_batch_step(model, gbs)
    em = emulated(L, H, gbs, M)
    ex = Executor(model, plan, M, gbs, apply=False)
    loss = ex.step()
    print(f"L={L} H={H}: loss gpu {loss:.6f} ref {ref.loss:.6f}")
    for l in range(L):
        for k in "Wb":
            g = ex.read(l, k, ref.grads[(l, k)].size, grad=True)
            print(f"  layer {l} {k}: vs fp64 {rel_fro(g, ref.grads[(l, k)]):.4f}  vs bf16-emulated "
                  f"{rel_fro(g, em[(l, k)]):.4f}  emulated-vs-fp64 {rel_fro(em[(l, k)], ref.grads[(l, k)]):.4f}")
    ex.close()
