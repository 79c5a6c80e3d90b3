"""Shared helpers for the GPU parity tests (device step vs the CPU oracle).

Stated tolerances.  The device runs every GEMM on bf16 operands with fp32
accumulation, stores activations / activation-gradients in bf16 and keeps
fp32 master weights and fp32 gradient accumulators.  Two oracles:

* ``bf16=True`` oracle (oracle/executor_ref.py) rounds to bf16 exactly where
  the device stores bf16 and does the arithmetic in fp64.  This is the parity
  check proper: every gradient tensor within EMU_GRAD_RTOL relative Frobenius
  error, the loss within EMU_LOSS_RTOL, the SGD update within EMU_GRAD_RTOL.
  What remains is fp32-vs-fp64 accumulation order and the occasional bf16
  rounding flip.
* exact fp64 oracle: the loss within LOSS_RTOL; gradients within
  FP64_GRAD_RTOL -- bf16 storage error compounds through depth (the exact
  bf16 emulation itself differs from fp64 by up to ~15% on the first layer of
  MLP16), so this is a sanity bound, not the parity criterion.
"""
import numpy as np

EMU_GRAD_RTOL = 0.02
# ReLU chains amplify any rounding difference geometrically toward the input
# (MLP16 on the device: 0.1% on layer 15 growing to ~5% on layer 0 vs the
# bf16 oracle), so the bound grows with the number of layers above.
EMU_DEPTH_RTOL = 0.004
EMU_LOSS_RTOL = 2e-3
LOSS_RTOL = 1e-2
FP64_GRAD_RTOL = 0.25
# VGG at test size (8-channel convs, 19 ReLU layers): bf16 storage error of
# the exact-emulation oracle itself reaches ~30% on the first conv
FP64_GRAD_RTOL_DEEP = 0.5


def rel_fro(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


def tensor_names(kind):
    if kind in ("mlp", "vgg"):
        return ["W", "b"]
    return ["ln1_g", "ln1_b", "Wqkv", "bqkv", "Wo", "bo", "ln2_g", "ln2_b", "W1", "b1", "W2", "b2"]


def check_loss(loss, emu, exact):
    assert abs(loss - emu.loss) <= EMU_LOSS_RTOL * abs(emu.loss), (loss, emu.loss)
    assert abs(loss - exact.loss) <= LOSS_RTOL * abs(exact.loss), (loss, exact.loss)


def check_grads(ex, emu, exact, layers, kind, n_layers=None, depth_rtol=EMU_DEPTH_RTOL, base_rtol=EMU_GRAD_RTOL):
    worst = 0.0
    n_layers = max(layers) + 1 if n_layers is None else n_layers
    for l in layers:
        tol = base_rtol + (depth_rtol * (n_layers - 1 - l) if kind in ("mlp", "vgg") else 0.0)
        for name in tensor_names(kind):
            got = ex.read(l, name, emu.grads[(l, name)].size, grad=True)
            e = rel_fro(got, emu.grads[(l, name)])
            assert e < tol, f"layer {l} {name}: grad rel err vs bf16 oracle {e:.4g} (tol {tol:.3g})"
            e64 = rel_fro(got, exact.grads[(l, name)])
            b64 = FP64_GRAD_RTOL_DEEP if kind == "vgg" else FP64_GRAD_RTOL
            assert e64 < b64, f"layer {l} {name}: grad rel err vs fp64 oracle {e64:.4g}"
            worst = max(worst, e)
    return worst


def check_update(ex, emu, layers, kind, model, lr, seed=1234, n_layers=None):
    """fp32 master weights after SGD must equal w_init - lr * grad (bf16
    oracle) up to fp32 rounding of w and EMU_GRAD_RTOL of the update."""
    from oracle.executor_ref import Model, init_layer
    m = Model.from_dict(model)
    worst = 0.0
    n_layers = m.layers if n_layers is None else n_layers
    for l in layers:
        ltol = EMU_GRAD_RTOL + (EMU_DEPTH_RTOL * (n_layers - 1 - l) if kind in ("mlp", "vgg") else 0.0)
        init = init_layer(m, l, seed)
        for name in tensor_names(kind):
            g = emu.grads[(l, name)].ravel()
            w0 = init[name].ravel().astype(np.float64)
            want = w0 - lr * g
            got = ex.read(l, name, g.size, grad=False).astype(np.float64)
            tol = 4 * 2.0 ** -24 * np.abs(w0) + 2 * ltol * np.abs(lr * g).max() + 1e-30
            bad = np.abs(got - want) > tol
            assert not bad.any(), f"layer {l} {name}: {int(bad.sum())} weights off, max err {np.abs(got - want).max():.3g}"
            worst = max(worst, float((np.abs(got - want) / tol).max()))
    return worst
