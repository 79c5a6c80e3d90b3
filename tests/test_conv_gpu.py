"""VGG convolution support kernels (conv.cu) vs plain torch fp32 references,
and a conv forward / backward through im2col + the tcgen05 GEMM + col2im vs
torch.nn.functional.conv2d autograd."""
import pytest
import torch
import torch.nn.functional as F

from paper_2007_01045_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _rand(*shape, dev, scale=1.0, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(*shape, generator=g) * 2 - 1) * scale).to(torch.bfloat16).to(dev)


def _kp(c):
    return (9 * c + 7) // 8 * 8


@pytest.mark.parametrize("n,h,w,c", [(2, 8, 8, 8), (1, 14, 10, 16), (2, 6, 6, 3)])
def test_im2col_matches_unfold(cuda, n, h, w, c):
    x = _rand(n, h, w, c, dev=cuda, seed=1)
    kp = _kp(c)
    col = torch.full((n * h * w, kp), 7.0, dtype=torch.bfloat16, device=cuda)
    K.im2col3x3(x, col, n, h, w, c, kp)
    # torch unfold gives [n][c*9][h*w] with (c, kh, kw) ordering; ours is (kh, kw, c)
    u = F.unfold(x.permute(0, 3, 1, 2).float(), 3, padding=1).view(n, c, 9, h * w)
    ref = u.permute(0, 3, 2, 1).reshape(n * h * w, 9 * c)
    torch.cuda.synchronize()
    assert torch.equal(col[:, :9 * c].float(), ref)
    assert (col[:, 9 * c:] == 0).all()


@pytest.mark.parametrize("n,h,w,c", [(2, 8, 8, 8), (1, 14, 10, 16)])
def test_col2im_is_the_adjoint_of_im2col(cuda, n, h, w, c):
    kp = _kp(c)
    dcol = _rand(n * h * w, kp, dev=cuda, seed=2)
    dx = torch.empty(n, h, w, c, dtype=torch.bfloat16, device=cuda)
    K.col2im3x3(dcol, dx, n, h, w, c, kp)
    d = dcol[:, :9 * c].float().view(n, h * w, 9, c).permute(0, 3, 2, 1).reshape(n, c * 9, h * w)
    ref = F.fold(d, (h, w), 3, padding=1).permute(0, 2, 3, 1)
    torch.cuda.synchronize()
    assert (dx.float() - ref).abs().max().item() <= 0.02 * ref.abs().max().item()


@pytest.mark.parametrize("n,h,w,c", [(2, 8, 8, 8), (3, 14, 6, 64)])
def test_maxpool_fwd_and_relu_bwd(cuda, n, h, w, c):
    x = torch.relu(_rand(n, h, w, c, dev=cuda, seed=3).float()).to(torch.bfloat16)
    y = torch.empty(n, h // 2, w // 2, c, dtype=torch.bfloat16, device=cuda)
    K.maxpool2_fwd(x, y, n, h, w, c)
    xr = x.float().permute(0, 3, 1, 2).requires_grad_(True)
    yr = F.max_pool2d(xr, 2)
    torch.cuda.synchronize()
    assert torch.equal(y.float(), yr.permute(0, 2, 3, 1))
    dy = _rand(n, h // 2, w // 2, c, dev=cuda, seed=4)
    dz = torch.empty_like(x)
    K.maxpool2_relu_bwd(x, dy, dz, n, h, w, c)
    (g,) = torch.autograd.grad(yr, xr, dy.float().permute(0, 3, 1, 2))
    ref = (g * (xr > 0)).permute(0, 2, 3, 1)
    torch.cuda.synchronize()
    assert torch.equal(dz.float(), ref)


def test_relu_bwd(cuda):
    y = torch.relu(_rand(4096, dev=cuda, seed=5).float()).to(torch.bfloat16)
    dy = _rand(4096, dev=cuda, seed=6)
    dz = torch.empty_like(dy)
    K.relu_bwd(y, dy, dz, 4096)
    torch.cuda.synchronize()
    assert torch.equal(dz.float(), dy.float() * (y.float() > 0))


@pytest.mark.parametrize("n,h,w,c,co", [(2, 16, 16, 64, 128), (2, 12, 12, 3, 64)])
def test_conv_via_columns_matches_conv2d(cuda, n, h, w, c, co):
    """y = im2col(x) W^T (+b, ReLU) ; dW = dz^T col ; dx = col2im(dz W)."""
    kp = _kp(c)
    x = _rand(n, h, w, c, dev=cuda, seed=7)
    wt = _rand(co, 3, 3, c, dev=cuda, seed=8, scale=0.2)  # [co][kh][kw][c]
    wk = torch.zeros(co, kp, dtype=torch.bfloat16, device=cuda)
    wk[:, :9 * c] = wt.reshape(co, 9 * c)
    bias = torch.zeros(co, device=cuda)
    col = torch.empty(n * h * w, kp, dtype=torch.bfloat16, device=cuda)
    K.im2col3x3(x, col, n, h, w, c, kp)
    y = torch.empty(n * h * w, co, dtype=torch.bfloat16, device=cuda)
    K.gemm(col, wk, y, n * h * w, co, kp, lda=kp, ldb=kp, ldc=co, epi=K.EPI_BIAS, bias=bias)
    xr = x.float().permute(0, 3, 1, 2).requires_grad_(True)
    wr = wt.float().permute(0, 3, 1, 2).requires_grad_(True)
    yr = F.conv2d(xr, wr, padding=1)
    torch.cuda.synchronize()
    ref = yr.permute(0, 2, 3, 1).reshape(n * h * w, co)
    assert (y.float() - ref).abs().max().item() <= 0.02 * ref.abs().max().item()
    dz = _rand(n * h * w, co, dev=cuda, seed=9)
    dw = torch.zeros(co, kp, device=cuda)
    K.gemm(dz, col, dw, co, kp, n * h * w, lda=co, ldb=kp, ldc=kp, a_mn_major=True, b_mn_major=True,
           epi=K.EPI_OUT_F32_ACC)
    gx, gw = torch.autograd.grad(yr, (xr, wr), dz.float().view(n, h, w, co).permute(0, 3, 1, 2))
    gw_ref = gw.permute(0, 2, 3, 1).reshape(co, 9 * c)
    torch.cuda.synchronize()
    assert (dw[:, :9 * c] - gw_ref).abs().max().item() <= 0.02 * gw_ref.abs().max().item()
    if kp > 9 * c:
        assert dw[:, 9 * c:].abs().max().item() == 0.0
    if c % 8 == 0:
        dcol = torch.empty(n * h * w, kp, dtype=torch.bfloat16, device=cuda)
        K.gemm(dz, wk, dcol, n * h * w, kp, co, lda=co, ldb=kp, ldc=kp, b_mn_major=True)
        dx = torch.empty(n, h, w, c, dtype=torch.bfloat16, device=cuda)
        K.col2im3x3(dcol, dx, n, h, w, c, kp)
        gx_ref = gx.permute(0, 2, 3, 1)
        torch.cuda.synchronize()
        assert (dx.float() - gx_ref).abs().max().item() <= 0.03 * gx_ref.abs().max().item()


@pytest.mark.parametrize("n,h,w,c,co,one_sm", [(2, 16, 16, 64, 128, False), (3, 14, 14, 128, 256, False),
                                              (2, 8, 8, 64, 64, True)])
def test_implicit_gemm_conv_matches_explicit_columns(cuda, n, h, w, c, co, one_sm):
    """TMA im2col-mode operands (no column matrix) give bit-identical results
    to im2col + the same GEMM: forward (A operand) and weight gradient (B)."""
    kp = 9 * c
    x = _rand(n, h, w, c, dev=cuda, seed=21)
    wk = _rand(co, kp, dev=cuda, seed=22, scale=0.1)
    bias = _rand(co, dev=cuda, seed=23, scale=0.1).float()
    rows = n * h * w
    col = torch.empty(rows, kp, dtype=torch.bfloat16, device=cuda)
    K.im2col3x3(x, col, n, h, w, c, kp)
    y_ref = torch.empty(rows, co, dtype=torch.bfloat16, device=cuda)
    K.gemm(col, wk, y_ref, rows, co, kp, lda=kp, ldb=kp, ldc=co, epi=K.EPI_BIAS | K.EPI_RELU, bias=bias,
           force_1sm=one_sm)
    y = torch.empty_like(y_ref)
    K.gemm(x, wk, y, rows, co, kp, lda=kp, ldb=kp, ldc=co, epi=K.EPI_BIAS | K.EPI_RELU, bias=bias,
           force_1sm=one_sm, conv=(1, x, n, h, w, c))
    dz = _rand(rows, co, dev=cuda, seed=24)
    dw_ref = torch.zeros(co, kp, device=cuda)
    K.gemm(dz, col, dw_ref, co, kp, rows, lda=co, ldb=kp, ldc=kp, a_mn_major=True, b_mn_major=True,
           epi=K.EPI_OUT_F32_ACC, force_1sm=one_sm)
    dw = torch.zeros(co, kp, device=cuda)
    K.gemm(dz, x, dw, co, kp, rows, lda=co, ldb=kp, ldc=kp, a_mn_major=True, b_mn_major=True,
           epi=K.EPI_OUT_F32_ACC, force_1sm=one_sm, conv=(2, x, n, h, w, c))
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    assert torch.allclose(dw, dw_ref, rtol=1e-5, atol=1e-4)  # split-K partial sums meet in a different order
