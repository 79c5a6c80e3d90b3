"""CPU numerical oracle for the DAPPLE training step (TEST INFRASTRUCTURE ONLY).

The reference has no numerical executor (loss/gradient
parity is *unpinned* by any reference test).  This module restates the
step's semantics from the paper's runtime section:

* forward graphs per stage in order, backward graphs in reverse order
  (PAPER.md:1192-1201);
* a micro-batch is split into even row slices over a stage's replicas, with
  split/concat at stage boundaries;
* every device accumulates gradients over all its micro-batches, then an
  AllReduce over the replicas, then Apply;
* so the step equals full-batch training at fixed GBS.

It is pinned internally: ``scheduled_step`` (which walks the exact per-stage
1F1B chain of the plan, slices micro-batches per replica and accumulates
per replica) must equal ``full_batch_step`` (one sequential fp64 pass) to
rounding -- tests/test_oracle_executor.py.  The GPU executor is then checked
against ``full_batch_step`` in fp32 within the bf16 tolerance stated in the
tests.

Synthetic data and weights come from ``hash_uniform`` -- the same splitmix64
keyed generator the device uses (csrc/kernels/elementwise.cu), so the oracle
and the GPU see identical inputs without shipping tensors.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_K_TENSOR = np.uint64(0xD1B54A32D192ED03)
_K_INDEX = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D649BB133111EB)


def mix64(seed: int, tensor: int, idx) -> np.ndarray:
    """splitmix64 finaliser of seed + tensor*K_T + idx*K_I (uint64)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.uint64(tensor) * _K_TENSOR + idx * _K_INDEX
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def hash_uniform(seed: int, tensor: int, idx) -> np.ndarray:
    """U(-1, 1) float32 keyed by (seed, tensor id, element index)."""
    z = mix64(seed, tensor, idx)
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return u * np.float32(2.0) - np.float32(1.0)


# ---------------------------------------------------------------- helpers
def _tid(layer: int, t: int) -> int:
    return 1000 + layer * 16 + t


def _u(seed, tensor, n, scale) -> np.ndarray:
    return np.float32(scale) * hash_uniform(seed, tensor, np.arange(n, dtype=np.uint64))


def _erf(x):
    from scipy.special import erf
    return erf(x)


# GELU in its tanh form, as the device computes it (gemm_tcgen05.cu gelu_f):
#   gelu(x) = 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
_K0 = math.sqrt(2.0 / math.pi)
_K1 = 0.044715


def gelu(x):
    return 0.5 * x * (1.0 + np.tanh(_K0 * (x + _K1 * x * x * x)))


def dgelu(x):
    t = np.tanh(_K0 * (x + _K1 * x * x * x))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * _K0 * (1.0 + 3.0 * _K1 * x * x)


@dataclass
class Model:
    kind: str = "mlp"  # mlp | bert | gpt
    layers: int = 16
    hidden: int = 1024
    heads: int = 16
    ffn: int = 4096
    seq: int = 1
    causal: bool = False
    eps: float = 1e-5
    vocab: int = 0  # > 0: GPT language model (token ids in, causal-LM cross-entropy out)
    # VGG-19 (kind "vgg"): image x image x 3 NHWC, conv widths width x {1,2,4,8,8}, FC fc, fc, classes
    image: int = 224
    width: int = 64
    fc: int = 4096
    classes: int = 1000
    # conv-net family (layers.h ModelSpec): convs per pool group, width multipliers, 3 FCs or the classifier only
    convs: tuple = (2, 2, 4, 4, 4)
    mults: tuple = (1, 2, 4, 8, 8)
    fcs: int = 3

    @staticmethod
    def from_dict(d: dict) -> "Model":
        m = Model(kind=d["kind"], layers=d["layers"], hidden=d.get("hidden", 8), heads=d.get("heads", 16),
                  ffn=d.get("ffn", 4 * d.get("hidden", 8)), seq=d.get("seq", 1), causal=d.get("causal", False),
                  vocab=d.get("vocab", 0), image=d.get("image", 224), width=d.get("width", 64),
                  fc=d.get("fc", 4096), classes=d.get("classes", 1000),
                  convs=tuple(d.get("convs", (2, 2, 4, 4, 4))), mults=tuple(d.get("mults", (1, 2, 4, 8, 8))),
                  fcs=d.get("fcs", 3))
        if m.kind == "mlp":
            m.seq = 1
        if m.kind == "gpt":
            m.causal = True
        if m.kind == "vgg":
            m.seq, m.hidden = 1, m.classes
        return m


def vgg_layer(model: Model, l: int) -> dict:
    """Shape of VGG profile layer l (csrc/runtime/layers.cu vgg_layer)."""
    hw, cin, idx = model.image, 3, 0
    for g, (convs, mult) in enumerate(zip(model.convs, model.mults)):
        for c in range(convs):
            cout = model.width * mult
            if idx == l:
                return dict(conv=True, h=hw, w=hw, cin=cin, cout=cout, kp=(9 * cin + 7) // 8 * 8, pool=c == convs - 1)
            cin, idx = cout, idx + 1
        hw //= 2
    f = l - sum(model.convs)  # FC index
    if not 0 <= f < model.fcs:
        raise IndexError("vgg_layer: layer index")
    return dict(conv=False, fin=hw * hw * cin if f == 0 else model.fc,
                fout=model.classes if f == model.fcs - 1 else model.fc, relu=f != model.fcs - 1)


def elems_per_sample(model: Model, l: int) -> int:
    if model.kind != "vgg":
        return model.seq * model.hidden
    if l >= model.layers:
        return model.classes
    v = vgg_layer(model, l)
    return v["h"] * v["w"] * v["cin"] if v["conv"] else v["fin"]


def init_layer(model: Model, layer: int, seed: int) -> dict:
    """Parameters of one layer exactly as the device initialises them
    (csrc/runtime/layers.cu bind())."""
    if model.kind == "vgg":
        v = vgg_layer(model, layer)
        if v["conv"]:
            n = v["cout"] * v["kp"]
            return {"W": _u(seed, _tid(layer, 0), n, np.sqrt(np.float32(6.0) / np.float32(9 * v["cin"]))).reshape(
                        v["cout"], v["kp"]), "b": _u(seed, _tid(layer, 1), v["cout"], 0.05)}
        n = v["fout"] * v["fin"]
        return {"W": _u(seed, _tid(layer, 0), n, np.sqrt(np.float32(6.0) / np.float32(v["fin"]))).reshape(
                    v["fout"], v["fin"]), "b": _u(seed, _tid(layer, 1), v["fout"], 0.05)}
    H, F = model.hidden, model.ffn
    if model.kind == "mlp":
        return {"W": _u(seed, _tid(layer, 0), H * H, np.sqrt(np.float32(6.0) / np.float32(H))).reshape(H, H),
                "b": _u(seed, _tid(layer, 1), H, 0.05)}
    sh = np.float32(1.0) / np.sqrt(np.float32(H))
    sf = np.float32(1.0) / np.sqrt(np.float32(F))
    return {"ln1_g": np.ones(H, np.float32), "ln1_b": np.zeros(H, np.float32),
            "Wqkv": _u(seed, _tid(layer, 2), 3 * H * H, sh).reshape(3 * H, H),
            "bqkv": _u(seed, _tid(layer, 3), 3 * H, 0.02),
            "Wo": _u(seed, _tid(layer, 4), H * H, sh).reshape(H, H), "bo": _u(seed, _tid(layer, 5), H, 0.02),
            "ln2_g": np.ones(H, np.float32), "ln2_b": np.zeros(H, np.float32),
            "W1": _u(seed, _tid(layer, 8), F * H, sh).reshape(F, H), "b1": _u(seed, _tid(layer, 9), F, 0.02),
            "W2": _u(seed, _tid(layer, 10), H * F, sf).reshape(H, F), "b2": _u(seed, _tid(layer, 11), H, 0.02)}


def vgg_batch(model: Model, seed: int, sample0: int, samples: int):
    """Images (NHWC, flattened per sample, U(-1,1) keyed by the element index)
    and class labels (splitmix64 of the sample index mod classes)."""
    e = elems_per_sample(model, 0)
    idx = np.arange(samples * e, dtype=np.uint64) + np.uint64(sample0 * e)
    x = hash_uniform(seed, 1, idx).reshape(samples, e)
    lab = (mix64(seed, 2, np.arange(samples, dtype=np.uint64) + np.uint64(sample0)) >> np.uint64(32)) % np.uint64(
        model.classes)
    return x, lab.astype(np.int64)


def _im2col(x, n, h, w, c, kp):
    xp = np.zeros((n, h + 2, w + 2, c), x.dtype)
    xp[:, 1:-1, 1:-1, :] = x.reshape(n, h, w, c)
    col = np.zeros((n, h, w, kp), x.dtype)
    for kh in range(3):
        for kw in range(3):
            col[..., (kh * 3 + kw) * c:(kh * 3 + kw + 1) * c] = xp[:, kh:kh + h, kw:kw + w, :]
    return col.reshape(n * h * w, kp)


def _col2im(dcol, n, h, w, c):
    d = dcol.reshape(n, h, w, -1)
    dxp = np.zeros((n, h + 2, w + 2, c), dcol.dtype)
    for kh in range(3):
        for kw in range(3):
            dxp[:, kh:kh + h, kw:kw + w, :] += d[..., (kh * 3 + kw) * c:(kh * 3 + kw + 1) * c]
    return dxp[:, 1:-1, 1:-1, :].reshape(n, h * w * c)


def _pool_argmax(yr, n, h, w, c):
    """First maximum of each 2x2 window in row-major window order."""
    win = yr.reshape(n, h // 2, 2, w // 2, 2, c).transpose(0, 1, 3, 5, 2, 4).reshape(n, h // 2, w // 2, c, 4)
    return win.max(-1), win.argmax(-1)


def vgg_forward(model: Model, l: int, p: dict, x, n: int, q):
    v = vgg_layer(model, l)
    if v["conv"]:
        col = _im2col(x, n, v["h"], v["w"], v["cin"], v["kp"])
        yr = q(np.maximum(col @ q(p["W"]).T + p["b"], 0))
        if not v["pool"]:
            return yr.reshape(n, -1), (x, yr)
        y, _ = _pool_argmax(yr, n, v["h"], v["w"], v["cout"])
        return y.reshape(n, -1), (x, yr)
    z = x @ q(p["W"]).T + p["b"]
    y = q(np.maximum(z, 0) if v["relu"] else z)
    return y, (x, y)


def vgg_backward(model: Model, l: int, p: dict, cache, dy, n: int, need_dx: bool, q):
    v = vgg_layer(model, l)
    x, y = cache
    if v["conv"]:
        h, w, c, co = v["h"], v["w"], v["cin"], v["cout"]
        if v["pool"]:
            _, arg = _pool_argmax(y, n, h, w, co)
            g = dy.reshape(n, h // 2, w // 2, co)
            win = y.reshape(n, h // 2, 2, w // 2, 2, co).transpose(0, 1, 3, 5, 2, 4).reshape(n, h // 2, w // 2, co, 4)
            mask = (np.arange(4) == arg[..., None]) & (win > 0)
            dzw = mask * g[..., None]
            dz = dzw.reshape(n, h // 2, w // 2, co, 2, 2).transpose(0, 1, 4, 2, 5, 3).reshape(n * h * w, co)
        else:
            dz = dy.reshape(n * h * w, co) * (y > 0)
        col = _im2col(x, n, h, w, c, v["kp"])
        g = {"W": dz.T @ col, "b": dz.sum(0)}
        dx = q(_col2im(q(dz @ q(p["W"])), n, h, w, c)) if need_dx else None
        return dx, g
    dz = dy * (y > 0) if v["relu"] else dy
    g = {"W": dz.T @ x, "b": dz.sum(0)}
    return (q(dz @ q(p["W"])) if need_dx else None), g


def class_ce(logits, labels, scale, q):
    """sum over rows of CE and q((softmax - onehot) * scale), as lm.cu computes it."""
    m = logits.max(-1, keepdims=True)
    e = np.exp(logits - m)
    ssum = e.sum(-1, keepdims=True)
    rows = np.arange(logits.shape[0])
    loss = float((np.log(ssum[:, 0]) + m[:, 0] - logits[rows, labels]).sum())
    d = e / ssum
    d[rows, labels] -= 1.0
    return loss, q(d * scale)


def batch_data(model: Model, seed: int, sample0: int, samples: int):
    """Input and target rows of samples [sample0, sample0 + samples):
    element (g, pos, h) is keyed by index (g * seq + pos) * H + h."""
    n = samples * model.seq * model.hidden
    idx = np.arange(n, dtype=np.uint64) + np.uint64(sample0 * model.seq * model.hidden)
    shape = (samples * model.seq, model.hidden)
    return hash_uniform(seed, 1, idx).reshape(shape), hash_uniform(seed, 2, idx).reshape(shape)


# ---------------------------------------------------------------- GPT LM ends
# Token ids and the LM parameters exactly as the device makes them
# (csrc/kernels/lm.cu fill_tokens, csrc/runtime/layers.cu TokenEmbedding /
# LmHead bind): inputs use tensor id 1, targets id 2, element index = global
# token index; wte / wpe ~ U(+-0.1) (ids 100, 101), Wout ~ U(+-1/sqrt(H))
# (id 112), LN_f gamma = 1, beta = 0.
def lm_tokens(model: Model, seed: int, sample0: int, samples: int):
    idx = np.arange(samples * model.seq, dtype=np.uint64) + np.uint64(sample0 * model.seq)
    tok = (mix64(seed, 1, idx) >> np.uint64(32)) % np.uint64(model.vocab)
    tgt = (mix64(seed, 2, idx) >> np.uint64(32)) % np.uint64(model.vocab)
    return tok.astype(np.int64), tgt.astype(np.int64)


def init_lm(model: Model, seed: int) -> dict:
    H, V, S = model.hidden, model.vocab, model.seq
    return {"wte": _u(seed, 100, V * H, 0.1).reshape(V, H), "wpe": _u(seed, 101, S * H, 0.1).reshape(S, H),
            "lnf_g": np.ones(H, np.float32), "lnf_b": np.zeros(H, np.float32),
            "Wout": _u(seed, 112, V * H, np.float32(1.0) / np.sqrt(np.float32(H))).reshape(V, H)}


def embed_forward(model: Model, p: dict, tok: np.ndarray, q=None):
    q = q or _ident
    pos = np.arange(tok.size) % model.seq
    return q(q(p["wte"])[tok] + q(p["wpe"])[pos])


def embed_backward(model: Model, tok: np.ndarray, dx: np.ndarray) -> dict:
    gwte = np.zeros((model.vocab, model.hidden), dx.dtype)
    np.add.at(gwte, tok, dx)
    gwpe = dx.reshape(-1, model.seq, model.hidden).sum(0)
    return {"wte": gwte, "wpe": gwpe}


def head_forward(model: Model, p: dict, y: np.ndarray, tgt: np.ndarray, ntok_global: int, q=None):
    """Returns (sum of token CE, cache).  The logits are stored in bf16 and the
    gradient (softmax - onehot) / ntok_global replaces them (lm.cu)."""
    q = q or _ident
    xn, c = _ln_fwd(y, p["lnf_g"], p["lnf_b"], model.eps)
    xn = q(xn)
    logits = q(xn @ q(p["Wout"]).T)
    m = logits.max(-1, keepdims=True)
    e = np.exp(logits - m)
    ssum = e.sum(-1, keepdims=True)
    rows = np.arange(logits.shape[0])
    loss = float((np.log(ssum[:, 0]) + m[:, 0] - logits[rows, tgt]).sum())
    d = e / ssum
    d[rows, tgt] -= 1.0
    return loss, (xn, c, q(d / ntok_global))


def head_backward(model: Model, p: dict, cache, q=None):
    q = q or _ident
    xn, c, dlog = cache
    g = {"Wout": dlog.T @ xn}
    dy, g["lnf_g"], g["lnf_b"] = _ln_bwd(q(dlog @ q(p["Wout"])), p["lnf_g"], c)
    return q(dy), g


def bf16_round(a) -> np.ndarray:
    """Round-to-nearest-even to bfloat16 (as __float2bfloat16_rn), returned
    as float64.  Used by the oracle's bf16 mode at exactly the points where
    the device stores a bf16 tensor."""
    a32 = np.asarray(a, dtype=np.float32)
    u = a32.view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def _ident(a):
    return a


MATRICES = {"W", "Wqkv", "Wo", "W1", "W2"}


def _gemm_weights(p, q):
    return {k: (q(v) if k in MATRICES else v) for k, v in p.items()}


# ---------------------------------------------------------------- layers
def _ln_fwd(x, g, b, eps):
    mean = x.mean(-1, keepdims=True)
    var = ((x - mean) ** 2).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + float(eps))
    xh = (x - mean) * rstd
    return xh * g + b, (xh, rstd)


def _ln_bwd(dy, g, cache):
    xh, rstd = cache
    gd = dy * g
    dx = rstd * (gd - gd.mean(-1, keepdims=True) - xh * (gd * xh).mean(-1, keepdims=True))
    return dx, (dy * xh).sum(0), dy.sum(0)


def layer_forward(model: Model, layer: int, p: dict, x: np.ndarray, samples: int, q=_ident):
    """Returns (y, cache).  x: [samples * seq, H] rows.  q rounds the tensors
    the device stores in bf16 (identity in the exact mode)."""
    if model.kind == "vgg":
        return vgg_forward(model, layer, p, x, samples, q)
    p = _gemm_weights(p, q)
    if model.kind == "mlp":
        z = x @ p["W"].T + p["b"]
        y = q(np.maximum(z, 0) if layer != model.layers - 1 else z)
        return y, (x,)
    H, nh, s = model.hidden, model.heads, model.seq
    d = H // nh
    ln1, c1 = _ln_fwd(x, p["ln1_g"], p["ln1_b"], model.eps)
    ln1 = q(ln1)
    qkv = q(ln1 @ p["Wqkv"].T + p["bqkv"])
    qh, k, v = (qkv[:, i * H:(i + 1) * H].reshape(samples, s, nh, d).transpose(0, 2, 1, 3) for i in range(3))
    sc = (qh @ k.transpose(0, 1, 3, 2)) * (1.0 / math.sqrt(d))
    if model.causal:
        sc = np.where(np.triu(np.ones((s, s), bool), 1), -np.inf, sc)
    # flash-attention numerics (csrc/kernels/attention.cu): unnormalised
    # exp(s - rowmax) is what gets rounded to bf16 for the PV product, the
    # row sum l stays fp32, the context is divided by l at the end
    e = np.exp(sc - sc.max(-1, keepdims=True))
    l = e.sum(-1, keepdims=True)
    P = e / l
    ctx = q(((q(e) @ v) / l).transpose(0, 2, 1, 3).reshape(samples * s, H))
    h = q(x + ctx @ p["Wo"].T + p["bo"])
    ln2, c2 = _ln_fwd(h, p["ln2_g"], p["ln2_b"], model.eps)
    ln2 = q(ln2)
    z1f = ln2 @ p["W1"].T + p["b1"]
    g = q(gelu(z1f))
    y = q(h + g @ p["W2"].T + p["b2"])
    return y, (x, ln1, c1, qh, k, v, P, ctx, h, ln2, c2, q(z1f), g)


def layer_backward(model: Model, layer: int, p: dict, cache, dy: np.ndarray, samples: int, need_dx=True,
                   q=_ident):
    """MLP layers take / return the gradient w.r.t. the pre-activation
    (layers.h gradient contract); transformer blocks w.r.t. the block
    output / input."""
    if model.kind == "vgg":
        return vgg_backward(model, layer, p, cache, dy, samples, need_dx, q)
    p = _gemm_weights(p, q)
    if model.kind == "mlp":
        (x,) = cache
        grads = {"W": dy.T @ x, "b": dy.sum(0)}
        dx = None
        if need_dx:
            dx = dy @ p["W"]
            if layer > 0:
                dx = dx * (x > 0)
            dx = q(dx)
        return dx, grads
    H, nh, s = model.hidden, model.heads, model.seq
    d = H // nh
    x, ln1, c1, qh, k, v, P, ctx, h, ln2, c2, z1, g = cache
    gr = {}
    gr["W2"], gr["b2"] = dy.T @ g, dy.sum(0)
    dz1 = q((dy @ p["W2"]) * dgelu(z1))
    gr["W1"], gr["b1"] = dz1.T @ ln2, dz1.sum(0)
    dh, gr["ln2_g"], gr["ln2_b"] = _ln_bwd(q(dz1 @ p["W1"]), p["ln2_g"], c2)
    dh = q(dh + dy)
    gr["Wo"], gr["bo"] = dh.T @ ctx, dh.sum(0)
    dctx = q(dh @ p["Wo"]).reshape(samples, s, nh, d).transpose(0, 2, 1, 3)
    # flash-attention backward: D = rowsum(dO * O) from the stored context,
    # dS from the fp32 probabilities, P and dS rounded to bf16 as MMA operands
    ctx_h = ctx.reshape(samples, s, nh, d).transpose(0, 2, 1, 3)
    D = (dctx * ctx_h).sum(-1, keepdims=True)
    dP = dctx @ v.transpose(0, 1, 3, 2)
    dS = P * (dP - D)
    scale = 1.0 / math.sqrt(d)
    dq = q(scale * (q(dS) @ k))
    dk = q(scale * (q(dS).transpose(0, 1, 3, 2) @ qh))
    dv = q(q(P).transpose(0, 1, 3, 2) @ dctx)
    dqkv = np.concatenate([t.transpose(0, 2, 1, 3).reshape(samples * s, H) for t in (dq, dk, dv)], axis=1)
    gr["Wqkv"], gr["bqkv"] = dqkv.T @ ln1, dqkv.sum(0)
    dx, gr["ln1_g"], gr["ln1_b"] = _ln_bwd(q(dqkv @ p["Wqkv"]), p["ln1_g"], c1)
    return q(dx + dh), gr


# ---------------------------------------------------------------- steps
@dataclass
class StepResult:
    loss: float
    grads: dict = field(default_factory=dict)   # (layer, name) -> summed gradient
    params: dict = field(default_factory=dict)  # (layer, name) -> parameter after SGD


def full_batch_step(model, gbs: int, seed: int = 1234, lr: float = 1e-3, dtype=np.float64,
                    layers=None, bf16: bool = False) -> StepResult:
    """One sequential pass over the whole global batch (the known answer the
    pipelined step must reproduce).  With bf16=True every
    tensor the device stores in bf16 (inputs, targets, GEMM weights,
    activations, activation gradients) is rounded to bf16 at the same point;
    arithmetic stays fp64."""
    model = Model.from_dict(model) if isinstance(model, dict) else model
    layers = range(model.layers) if layers is None else layers
    q = bf16_round if bf16 else _ident
    params = {l: {k: v.astype(dtype) for k, v in init_layer(model, l, seed).items()} for l in layers}
    lm = model.vocab > 0
    if lm:
        lmp = {k: v.astype(dtype) for k, v in init_lm(model, seed).items()}
        tok, tgt = lm_tokens(model, seed, 0, gbs)
        x = embed_forward(model, lmp, tok, q)
    elif model.kind == "vgg":
        x, labels = vgg_batch(model, seed, 0, gbs)
        x = q(x.astype(dtype))
    else:
        x, t = batch_data(model, seed, 0, gbs)
        x, t = q(x.astype(dtype)), q(t.astype(dtype))
    caches = []
    for l in layers:
        x, c = layer_forward(model, l, params[l], x, gbs, q=q)
        caches.append(c)
    res = StepResult(0.0)

    def record(owner, g, p):
        for k, v in g.items():
            res.grads[(owner, k)] = v
            res.params[(owner, k)] = p[k].astype(np.float32) - np.float32(lr) * v.astype(np.float32)

    if lm:
        ntok = gbs * model.seq
        lsum, hc = head_forward(model, lmp, x, tgt, ntok, q)
        res.loss = lsum / ntok
        dy, g = head_backward(model, lmp, hc, q)
        record("head", g, lmp)
    elif model.kind == "vgg":
        lsum, dy = class_ce(x, labels, 1.0 / gbs, q)
        res.loss = lsum / gbs
    else:
        numel = gbs * model.seq * model.hidden
        diff = x - t
        res.loss = float((diff * diff).sum() / numel)
        dy = q(2.0 * diff / numel)
    for li in reversed(range(len(caches))):
        l = list(layers)[li]
        dy, g = layer_backward(model, l, params[l], caches[li], dy, gbs, need_dx=li > 0 or lm, q=q)
        record(l, g, params[l])
    if lm:
        record("emb", embed_backward(model, tok, dy), lmp)
    return res


def scheduled_step(model, plan: dict, micro_batches: int, gbs: int, seed: int = 1234, lr: float = 1e-3,
                   dtype=np.float64) -> StepResult:
    """The DAPPLE step as the plan executes it: replica j of a stage with r
    replicas owns samples [B*j/r, B*(j+1)/r) of each micro-batch (an even
    split when r divides B), activations and gradients cross stage
    boundaries by interval overlap (Split-Concat), each replica accumulates
    its gradients over the micro-batches in chain order B_0..B_{M-1}, and the
    replica group sums them (AllReduce) before the update."""
    model = Model.from_dict(model) if isinstance(model, dict) else model
    stages = plan["stages"]
    B = gbs // micro_batches
    params = {l: {k: v.astype(dtype) for k, v in init_layer(model, l, seed).items()} for l in range(model.layers)}
    lm = model.vocab > 0
    vgg = model.kind == "vgg"
    if lm:
        params["emb"] = params["head"] = {k: v.astype(dtype) for k, v in init_lm(model, seed).items()}
        numel = gbs * model.seq  # CE is a mean over the global batch's tokens
    elif vgg:
        numel = gbs  # CE is a mean over the samples
    else:
        numel = gbs * model.seq * model.hidden
    acc = {}  # (stage, replica, layer | "emb" | "head", name) -> grad

    def add(key, v):
        acc[key] = acc[key] + v if key in acc else v

    loss = 0.0
    for i in range(micro_batches):
        xs = None  # per-replica input slices of the current stage
        caches = []
        for k, st in enumerate(stages):
            r = len(st["gpus"])
            lo, hi = st["layers"]
            cut = [B * j // r for j in range(r + 1)]  # sample boundaries of the replica slices
            if k == 0 and lm:
                toks = [lm_tokens(model, seed, i * B + cut[j], cut[j + 1] - cut[j])[0] for j in range(r)]
                xs = [embed_forward(model, params["emb"], t) for t in toks]
            elif k == 0 and vgg:
                xs = [vgg_batch(model, seed, i * B + cut[j], cut[j + 1] - cut[j])[0].astype(dtype) for j in range(r)]
            elif k == 0:
                xs = [batch_data(model, seed, i * B + cut[j], cut[j + 1] - cut[j])[0].astype(dtype)
                      for j in range(r)]
            else:
                whole = np.concatenate(xs, axis=0)  # split-concat: rows are batch-major
                xs = [whole[cut[j] * model.seq:cut[j + 1] * model.seq] for j in range(r)]
            stage_caches = []
            for j in range(r):
                x = xs[j]
                cs = []
                for l in range(lo, hi):
                    x, c = layer_forward(model, l, params[l], x, cut[j + 1] - cut[j])
                    cs.append(c)
                xs[j] = x
                stage_caches.append(cs)
            caches.append(stage_caches)
        # loss on the last stage
        last = stages[-1]
        r = len(last["gpus"])
        cut = [B * j // r for j in range(r + 1)]
        dys = []
        for j in range(r):
            if lm:
                tgt = lm_tokens(model, seed, i * B + cut[j], cut[j + 1] - cut[j])[1]
                lsum, hc = head_forward(model, params["head"], xs[j], tgt, numel)
                loss += lsum
                dy, g = head_backward(model, params["head"], hc)
                for name in ("Wout", "lnf_g", "lnf_b"):
                    add((len(stages) - 1, j, "head", name), g[name])
                dys.append(dy)
                continue
            if vgg:
                lab = vgg_batch(model, seed, i * B + cut[j], cut[j + 1] - cut[j])[1]
                lsum, dy = class_ce(xs[j], lab, 1.0 / numel, _ident)
                loss += lsum
                dys.append(dy)
                continue
            t = batch_data(model, seed, i * B + cut[j], cut[j + 1] - cut[j])[1].astype(dtype)
            diff = xs[j] - t
            loss += float((diff * diff).sum())
            dys.append(2.0 * diff / numel)
        for k in reversed(range(len(stages))):
            st = stages[k]
            r = len(st["gpus"])
            lo, hi = st["layers"]
            cut = [B * j // r for j in range(r + 1)]
            if k != len(stages) - 1:
                whole = np.concatenate(dys, axis=0)
                dys = [whole[cut[j] * model.seq:cut[j + 1] * model.seq] for j in range(r)]
            for j in range(r):
                dy = dys[j]
                for li, l in reversed(list(enumerate(range(lo, hi)))):
                    dy, g = layer_backward(model, l, params[l], caches[k][j][li], dy, cut[j + 1] - cut[j],
                                           need_dx=(l > 0 or lm))
                    for name, v in g.items():
                        add((k, j, l, name), v)
                if k == 0 and lm:
                    for name, v in embed_backward(model, toks[j], dy).items():
                        add((0, j, "emb", name), v)
                dys[j] = dy
    res = StepResult(loss / numel)
    for k, st in enumerate(stages):
        lo, hi = st["layers"]
        for l in range(lo, hi):
            for name in params[l]:
                g = sum(acc[(k, j, l, name)] for j in range(len(st["gpus"])))  # AllReduce
                res.grads[(l, name)] = g
                res.params[(l, name)] = params[l][name].astype(np.float32) - np.float32(lr) * g.astype(np.float32)
    if lm:
        for k, owner, names in ((0, "emb", ("wte", "wpe")), (len(stages) - 1, "head", ("Wout", "lnf_g", "lnf_b"))):
            for name in names:
                g = sum(acc[(k, j, owner, name)] for j in range(len(stages[k]["gpus"])))
                res.grads[(owner, name)] = g
                res.params[(owner, name)] = (params[owner][name].astype(np.float32) -
                                             np.float32(lr) * g.astype(np.float32))
    return res


class CpuTrainer:
    """The oracle's training step as a reusable CPU trainer (parameters kept
    across steps, in-place SGD) -- the CPU path bench.py times beside the GPU
    (cpu_baseline, and the `--impl reference` arm).  numpy dispatches the
    matrix products to its multithreaded BLAS, so it uses all host cores."""

    def __init__(self, model, seed: int = 1234, dtype=np.float32):
        self.model = Model.from_dict(model) if isinstance(model, dict) else model
        self.seed, self.dtype = seed, dtype
        self.params = {l: {k: v.astype(dtype) for k, v in init_layer(self.model, l, seed).items()}
                       for l in range(self.model.layers)}
        if self.model.vocab > 0:
            self.lm = {k: v.astype(dtype) for k, v in init_lm(self.model, seed).items()}

    def step(self, sample0: int, samples: int, lr: float = 1e-3) -> float:
        m = self.model
        lm = m.vocab > 0
        vgg = m.kind == "vgg"
        if lm:
            tok, tgt = lm_tokens(m, self.seed, sample0, samples)
            x = embed_forward(m, self.lm, tok)
        elif vgg:
            x, labels = vgg_batch(m, self.seed, sample0, samples)
            x = x.astype(self.dtype)
        else:
            x, t = batch_data(m, self.seed, sample0, samples)
            x, t = x.astype(self.dtype), t.astype(self.dtype)
        caches = []
        for l in range(m.layers):
            x, c = layer_forward(m, l, self.params[l], x, samples)
            caches.append(c)
        if lm:
            ntok = samples * m.seq
            lsum, hc = head_forward(m, self.lm, x, tgt, ntok)
            loss = lsum / ntok
            dy, g_head = head_backward(m, self.lm, hc)
        elif vgg:
            lsum, dy = class_ce(x, labels, 1.0 / samples, _ident)
            loss = lsum / samples
        else:
            numel = samples * m.seq * m.hidden
            diff = x - t
            loss = float((diff * diff).sum() / numel)
            dy = (2.0 / numel) * diff
        for l in reversed(range(m.layers)):
            dy, g = layer_backward(m, l, self.params[l], caches[l], dy, samples, need_dx=l > 0 or lm)
            for k, v in g.items():
                self.params[l][k] -= self.dtype(lr) * v.astype(self.dtype)
        if lm:
            for k, v in list(g_head.items()) + list(embed_backward(m, tok, dy).items()):
                self.lm[k] -= self.dtype(lr) * v.astype(self.dtype)
        return loss
