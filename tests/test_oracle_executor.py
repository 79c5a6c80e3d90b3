"""CPU oracle self-checks: the plan-scheduled step (replica slices,
Split-Concat, per-replica accumulation, AllReduce) equals the sequential
full-batch step, and the oracle's manual backward equals autograd."""
import numpy as np
import pytest

from oracle.executor_ref import Model, batch_data, full_batch_step, hash_uniform, init_layer, layer_forward, scheduled_step

PLANS = [
    {"stages": [{"layers": [0, 4], "gpus": [0]}]},
    {"stages": [{"layers": [0, 4], "gpus": [0, 1, 2, 3]}]},
    {"stages": [{"layers": [0, 2], "gpus": [0]}, {"layers": [2, 4], "gpus": [1]}]},
    {"stages": [{"layers": [0, 1], "gpus": [0, 1]}, {"layers": [1, 4], "gpus": [2, 3]}]},
    {"stages": [{"layers": [0, 3], "gpus": [0, 1, 2]}, {"layers": [3, 4], "gpus": [3]}]},
    {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 2], "gpus": [1, 2, 3]}, {"layers": [2, 4], "gpus": [4, 5]}]},
    # replica counts that do not divide the 12-sample micro-batch (uneven slices)
    {"stages": [{"layers": [0, 1], "gpus": [0]}, {"layers": [1, 4], "gpus": [1, 2, 3, 4, 5, 6, 7]}]},
    {"stages": [{"layers": [0, 2], "gpus": [0, 1, 2, 3, 4]}, {"layers": [2, 4], "gpus": [5, 6]}]},
]


@pytest.mark.parametrize("plan", PLANS)
@pytest.mark.parametrize("kind", ["mlp", "bert", "gpt"])
def test_scheduled_equals_full_batch(plan, kind):
    m = dict(kind=kind, layers=4, hidden=32, heads=2, ffn=64, seq=8)
    gbs, M = 24, 2  # 12 samples per micro-batch split over 1, 2, 3, 4 replicas
    a = full_batch_step(m, gbs)
    b = scheduled_step(m, plan, M, gbs)
    assert abs(a.loss - b.loss) <= 1e-12 * abs(a.loss)
    for key, g in a.grads.items():
        assert np.allclose(b.grads[key], g, rtol=1e-10, atol=1e-14), key


def test_hash_uniform_golden():
    # frozen values of the shared device/host generator
    v = hash_uniform(1234, 1, np.arange(4, dtype=np.uint64))
    assert v.dtype == np.float32 and np.all(np.abs(v) < 1)
    again = hash_uniform(1234, 1, np.arange(4, dtype=np.uint64))
    assert np.array_equal(v, again)
    assert not np.array_equal(v, hash_uniform(1235, 1, np.arange(4, dtype=np.uint64)))
    u = hash_uniform(7, 3, np.arange(200000, dtype=np.uint64))
    assert abs(float(u.mean())) < 0.01 and 0.32 < float(u.var()) < 0.35


@pytest.mark.parametrize("kind", ["mlp", "bert", "gpt"])
def test_manual_backward_matches_autograd(kind):
    torch = pytest.importorskip("torch")
    m = Model.from_dict(dict(kind=kind, layers=3, hidden=16, heads=2, ffn=32, seq=4))
    gbs = 3
    res = full_batch_step(m, gbs)
    params = {l: {k: torch.tensor(v, dtype=torch.float64, requires_grad=True)
                  for k, v in init_layer(m, l, 1234).items()} for l in range(m.layers)}
    x, t = (torch.tensor(a, dtype=torch.float64) for a in batch_data(m, 1234, 0, gbs))
    H, nh, s = m.hidden, m.heads, m.seq
    d = H // nh
    for l in range(m.layers):
        p = params[l]
        if kind == "mlp":
            z = x @ p["W"].T + p["b"]
            x = torch.relu(z) if l != m.layers - 1 else z
            continue
        ln1 = torch.nn.functional.layer_norm(x, (H,), p["ln1_g"], p["ln1_b"], m.eps)
        qkv = ln1 @ p["Wqkv"].T + p["bqkv"]
        q, k, v = (qkv[:, i * H:(i + 1) * H].reshape(gbs, s, nh, d).transpose(1, 2) for i in range(3))
        sc = q @ k.transpose(-1, -2) / d ** 0.5
        if m.causal:
            sc = sc.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool), 1), float("-inf"))
        ctx = (torch.softmax(sc, -1) @ v).transpose(1, 2).reshape(gbs * s, H)
        h = x + ctx @ p["Wo"].T + p["bo"]
        ln2 = torch.nn.functional.layer_norm(h, (H,), p["ln2_g"], p["ln2_b"], m.eps)
        x = h + torch.nn.functional.gelu(ln2 @ p["W1"].T + p["b1"], approximate="tanh") @ p["W2"].T + p["b2"]
    loss = ((x - t) ** 2).sum() / (gbs * s * H)
    loss.backward()
    assert abs(loss.item() - res.loss) < 1e-12
    for l in range(m.layers):
        for k, v in params[l].items():
            assert np.allclose(v.grad.numpy(), res.grads[(l, k)], rtol=1e-9, atol=1e-13), (l, k)


@pytest.mark.parametrize("plan", [PLANS[0], PLANS[3], PLANS[6]])
def test_scheduled_equals_full_batch_lm(plan):
    """GPT language model (token embedding + LN_f/vocab projection/CE head)."""
    m = dict(kind="gpt", layers=4, hidden=32, heads=2, ffn=64, seq=8, vocab=40)
    gbs, M = 24, 2
    a = full_batch_step(m, gbs)
    b = scheduled_step(m, plan, M, gbs)
    assert abs(a.loss - b.loss) <= 1e-12 * abs(a.loss)
    assert ("emb", "wte") in a.grads and ("head", "Wout") in a.grads
    for key, g in a.grads.items():
        assert np.allclose(b.grads[key], g, rtol=1e-10, atol=1e-14), key


def test_lm_head_and_embedding_match_autograd():
    """The oracle's manual LM-end gradients equal torch autograd in fp64."""
    import torch
    from oracle.executor_ref import embed_backward, embed_forward, head_backward, head_forward, init_lm, lm_tokens
    m = Model.from_dict(dict(kind="gpt", layers=1, hidden=16, heads=2, ffn=32, seq=4, vocab=24))
    p = {k: v.astype(np.float64) for k, v in init_lm(m, 7).items()}
    tok, tgt = lm_tokens(m, 7, 0, 3)
    assert tok.min() >= 0 and tok.max() < 24 and len(set(tok.tolist())) > 4
    x = embed_forward(m, p, tok)
    lsum, cache = head_forward(m, p, x, tgt, tok.size)
    dx, g = head_backward(m, p, cache)
    ge = embed_backward(m, tok, dx)
    tp = {k: torch.tensor(v, requires_grad=True) for k, v in p.items()}
    pos = torch.arange(tok.size) % m.seq
    tx = tp["wte"][torch.tensor(tok)] + tp["wpe"][pos]
    xn = torch.nn.functional.layer_norm(tx, (m.hidden,), tp["lnf_g"], tp["lnf_b"], eps=m.eps)
    loss = torch.nn.functional.cross_entropy(xn @ tp["Wout"].T, torch.tensor(tgt), reduction="mean")
    loss.backward()
    assert abs(loss.item() - lsum / tok.size) < 1e-12
    for k, v in [("Wout", g["Wout"]), ("lnf_g", g["lnf_g"]), ("lnf_b", g["lnf_b"]), ("wte", ge["wte"]),
                 ("wpe", ge["wpe"])]:
        assert np.allclose(tp[k].grad.numpy(), v, rtol=1e-9, atol=1e-12), k


VGG = dict(kind="vgg", layers=19, image=32, width=8, fc=32, classes=16)


@pytest.mark.parametrize("plan", [{"stages": [{"layers": [0, 19], "gpus": [0]}]},
                                  {"stages": [{"layers": [0, 16], "gpus": [0, 1, 2]},
                                                       {"layers": [16, 19], "gpus": [3]}]},
                                  {"stages": [{"layers": [0, 10], "gpus": [0]}, {"layers": [10, 19], "gpus": [1, 2]}]}])
def test_scheduled_equals_full_batch_vgg(plan):
    """VGG-19 (convs, pools, FCs, class CE) with uneven conv/FC replication."""
    gbs, M = 12, 2
    a = full_batch_step(VGG, gbs)
    b = scheduled_step(VGG, plan, M, gbs)
    assert abs(a.loss - b.loss) <= 1e-12 * abs(a.loss)
    for key, g in a.grads.items():
        assert np.allclose(b.grads[key], g, rtol=1e-9, atol=1e-13), key


# the conv-net family with other groups (C5's AmoebaNet-36 stand-in shape, small)
CONV36 = dict(kind="vgg", layers=8, image=16, width=8, fc=32, classes=16, convs=[3, 2, 2], mults=[1, 2, 4], fcs=1)


def test_scheduled_equals_full_batch_conv_family():
    plan = {"stages": [{"layers": [0, 4], "gpus": [0, 1]}, {"layers": [4, 8], "gpus": [2]}]}
    a = full_batch_step(CONV36, 8)
    b = scheduled_step(CONV36, plan, 2, 8)
    assert abs(a.loss - b.loss) <= 1e-12 * abs(a.loss)
    for key, g in a.grads.items():
        assert np.allclose(b.grads[key], g, rtol=1e-9, atol=1e-13), key


@pytest.mark.parametrize("cfg", [VGG, CONV36], ids=["vgg19", "conv-family"])
def test_vgg_manual_backward_matches_autograd(cfg):
    """The oracle's conv (im2col, (kh, kw, c) order, zero-padded K), pool
    (first max), ReLU and FC backward equal torch autograd in fp64."""
    import torch
    import torch.nn.functional as F
    from oracle.executor_ref import class_ce, layer_backward, vgg_batch, vgg_layer
    m = Model.from_dict(cfg)
    n = 2
    L = m.layers
    x0, lab = vgg_batch(m, 5, 0, n)
    params = {l: {k: v.astype(np.float64) for k, v in init_layer(m, l, 5).items()} for l in range(L)}
    x = x0.astype(np.float64)
    caches = []
    for l in range(L):
        x, c = layer_forward(m, l, params[l], x, n)
        caches.append(c)
    lsum, dy = class_ce(x, lab, 1.0 / n, lambda a: a)
    grads = {}
    for l in reversed(range(L)):
        dy, g = layer_backward(m, l, params[l], caches[l], dy, n, need_dx=l > 0)
        grads[l] = g
    # torch reference in NCHW
    tp = {l: {k: torch.tensor(v, requires_grad=True) for k, v in params[l].items()} for l in range(L)}
    t = torch.tensor(x0, dtype=torch.float64).view(n, m.image, m.image, 3).permute(0, 3, 1, 2)
    for l in range(L):
        v = vgg_layer(m, l)
        if v["conv"]:
            w = tp[l]["W"][:, :9 * v["cin"]].view(v["cout"], 3, 3, v["cin"]).permute(0, 3, 1, 2)
            t = torch.relu(F.conv2d(t, w, tp[l]["b"], padding=1))
            if v["pool"]:
                t = F.max_pool2d(t, 2)
        else:
            if t.dim() == 4:
                t = t.permute(0, 2, 3, 1).reshape(n, -1)
            t = t @ tp[l]["W"].T + tp[l]["b"]
            if v["relu"]:
                t = torch.relu(t)
    loss = F.cross_entropy(t, torch.tensor(lab), reduction="mean")
    loss.backward()
    assert abs(loss.item() - lsum / n) < 1e-10
    for l in range(L):
        for k in ("W", "b"):
            got = grads[l][k]
            want = tp[l][k].grad.numpy()
            if k == "W" and vgg_layer(m, l)["conv"]:
                v = vgg_layer(m, l)
                want = want[:, :9 * v["cin"]]
                got = got[:, :9 * v["cin"]]
            assert np.allclose(got, want, rtol=1e-8, atol=1e-12), (l, k)
