"""Elementwise stage kernels vs plain torch fp32 references."""
import pytest
import torch

from paper_2007_01045_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _rand(*shape, dev, scale=1.0, dtype=torch.bfloat16, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(*shape, generator=g) * 2 - 1) * scale).to(dtype).to(dev)


@pytest.mark.parametrize("rows,h", [(64, 1024), (300, 256), (17, 2048), (128, 1600)])
def test_layernorm_fwd_bwd(cuda, rows, h):
    x = _rand(rows, h, dev=cuda, seed=1, scale=3.0)
    gamma = 1 + _rand(h, dev=cuda, seed=2, dtype=torch.float32, scale=0.5)
    beta = _rand(h, dev=cuda, seed=3, dtype=torch.float32, scale=0.5)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=cuda)
    rstd = torch.empty(rows, device=cuda)
    K.layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, h, 1e-5)
    xr = x.float().requires_grad_(True)
    g_, b_ = gamma.clone().requires_grad_(True), beta.clone().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (h,), g_, b_, 1e-5)
    torch.cuda.synchronize()
    assert (y.float() - yr).abs().max().item() < 0.05
    dy = _rand(rows, h, dev=cuda, seed=4)
    dres = _rand(rows, h, dev=cuda, seed=5)
    dx = torch.empty_like(x)
    dgamma = torch.zeros(h, device=cuda)
    dbeta = torch.zeros(h, device=cuda)
    K.layernorm_bwd(dy, x, mean, rstd, gamma, dres, dx, dgamma, dbeta, rows, h)
    gx, gg, gb = torch.autograd.grad(yr, (xr, g_, b_), dy.float())
    torch.cuda.synchronize()
    ref_dx = gx + dres.float()
    assert (dx.float() - ref_dx).abs().max().item() < 0.02 * ref_dx.abs().max().item() + 0.02
    assert torch.allclose(dgamma, gg, rtol=1e-3, atol=1e-2)
    assert torch.allclose(dbeta, gb, rtol=1e-3, atol=1e-2)


@pytest.mark.parametrize("rows,h,with_dx", [(4096, 1024, True), (4096, 1024, False), (1024, 1600, True),
                                            (333, 2048, True), (70, 256, False), (5, 512, True)])
def test_layernorm_bwd_column_sums(cuda, rows, h, with_dx):
    """LayerNorm backward with the neighbouring layers' bias gradients folded in
    (sum dresid, sum dx) against torch fp32, at the BERT / GPT-2 slice shapes
    and ragged row counts (partial row groups, idle blocks)."""
    x = _rand(rows, h, dev=cuda, seed=11, scale=3.0)
    gamma = 1 + _rand(h, dev=cuda, seed=12, dtype=torch.float32, scale=0.5)
    beta = _rand(h, dev=cuda, seed=13, dtype=torch.float32, scale=0.5)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=cuda)
    rstd = torch.empty(rows, device=cuda)
    K.layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, h, 1e-5)
    dy = _rand(rows, h, dev=cuda, seed=14)
    dres = _rand(rows, h, dev=cuda, seed=15)
    dx = torch.empty_like(x)
    dgamma = torch.full((h,), 0.25, device=cuda)  # accumulates into existing gradients
    dbeta = torch.full((h,), -0.5, device=cuda)
    drs = torch.full((h,), 1.0, device=cuda)
    dxs = torch.full((h,), 2.0, device=cuda) if with_dx else None
    K.layernorm_bwd_colsum(dy, x, mean, rstd, gamma, dres, dx, dgamma, dbeta, drs, dxs, rows, h)
    xr = x.float().requires_grad_(True)
    g_, b_ = gamma.clone().requires_grad_(True), beta.clone().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (h,), g_, b_, 1e-5)
    gx, gg, gb = torch.autograd.grad(yr, (xr, g_, b_), dy.float())
    torch.cuda.synchronize()
    ref_dx = gx + dres.float()
    assert (dx.float() - ref_dx).abs().max().item() < 0.02 * ref_dx.abs().max().item() + 0.02
    tol = dict(rtol=1e-3, atol=1e-2 * max(1.0, rows / 512))
    assert torch.allclose(dgamma, gg + 0.25, **tol)
    assert torch.allclose(dbeta, gb - 0.5, **tol)
    assert torch.allclose(drs, dres.float().sum(0) + 1.0, **tol)
    if with_dx:
        assert torch.allclose(dxs, dx.float().sum(0) + 2.0, **tol)


@pytest.mark.parametrize("causal", [False, True])
def test_softmax(cuda, causal):
    z, L = 8, 512
    s = _rand(z * L, L, dev=cuda, seed=6, dtype=torch.float32, scale=4.0)
    p = torch.empty(z * L, L, dtype=torch.bfloat16, device=cuda)
    K.softmax_fwd(s, p, z * L, L, L, causal)
    sr = s.view(z, L, L).clone()
    if causal:
        sr = sr.masked_fill(torch.triu(torch.ones(L, L, dtype=torch.bool, device=cuda), 1), float("-inf"))
    sr.requires_grad_(True)
    pr = torch.softmax(sr, -1)
    torch.cuda.synchronize()
    assert (p.float().view(z, L, L) - pr).abs().max().item() < 4e-3
    dp = _rand(z * L, L, dev=cuda, seed=7, dtype=torch.float32)
    ds = torch.empty_like(p)
    K.softmax_bwd(p, dp, ds, z * L, L)
    ref = torch.autograd.grad(pr, sr, dp.view(z, L, L))[0]
    torch.cuda.synchronize()
    assert (ds.float().view(z, L, L) - ref).abs().max().item() < 2e-2 * ref.abs().max().item() + 1e-4


def test_colsum_mse_sgd(cuda):
    rows, cols = 3000, 1024
    dy = _rand(rows, cols, dev=cuda, seed=8)
    db = torch.ones(cols, device=cuda)
    K.colsum_acc(dy, db, rows, cols)
    torch.cuda.synchronize()
    assert torch.allclose(db, 1 + dy.float().sum(0), rtol=1e-4, atol=1e-2)

    y = _rand(rows, cols, dev=cuda, seed=9)
    t = _rand(rows, cols, dev=cuda, seed=10)
    g = torch.empty_like(y)
    loss = torch.zeros(1, device=cuda)
    n = rows * cols
    K.mse_loss(y, t, g, loss, n, 2.0 / n)
    torch.cuda.synchronize()
    d = y.float() - t.float()
    assert abs(loss.item() - (d * d).sum().item()) < 1e-3 * (d * d).sum().item()
    assert (g.float() - d * (2.0 / n)).abs().max().item() < 1e-2 * (2.0 / n) * 2

    w32 = _rand(10001, dev=cuda, seed=11, dtype=torch.float32)
    gr = _rand(10001, dev=cuda, seed=12, dtype=torch.float32)
    w16 = torch.empty(10001, dtype=torch.bfloat16, device=cuda)
    ref = w32 - 0.1 * gr
    K.sgd_apply(w32, gr, w16, 10001, 0.1)
    torch.cuda.synchronize()
    assert torch.allclose(w32, ref, atol=1e-6)
    assert torch.count_nonzero(gr).item() == 0
    assert torch.allclose(w16.float(), ref, atol=1e-2)


def test_fill_uniform_matches_numpy_hash(cuda):
    import numpy as np
    from oracle.executor_ref import hash_uniform
    x = torch.empty(4099, dtype=torch.float32, device=cuda)
    K.fill_uniform_f32(x, 4099, 1234, 7, 100, 0.5)
    torch.cuda.synchronize()
    ref = 0.5 * hash_uniform(1234, 7, np.arange(100, 100 + 4099, dtype=np.uint64))
    assert np.array_equal(x.cpu().numpy(), ref.astype(np.float32))
