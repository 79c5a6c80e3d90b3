"""tcgen05 GEMM vs a plain torch fp32 reference on the same bf16 operands."""
import pytest
import torch

from paper_2007_01045_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _rand(*shape, dev, scale=1.0, dtype=torch.bfloat16, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(*shape, generator=g) * 2 - 1) * scale).to(dtype).to(dev)


def _close(out, ref, tol):
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    assert err <= tol * scale, f"max err {err:.4g} vs scale {scale:.4g}"


@pytest.mark.parametrize("M,N,Kd", [(128, 256, 64), (256, 512, 1024), (300, 200, 136), (1024, 3072, 1024),
                                    (64, 64, 16), (513, 1000, 520), (4096, 1024, 1024)])
@pytest.mark.parametrize("bn", [0, 64, 128, 256])
@pytest.mark.parametrize("one_sm", [False, True])
def test_gemm_kk(cuda, M, N, Kd, bn, one_sm):
    A = _rand(M, Kd, dev=cuda, seed=1)
    B = _rand(N, Kd, dev=cuda, seed=2)
    C = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, force_bn=bn, force_1sm=one_sm)
    torch.cuda.synchronize()
    _close(C, A.float() @ B.float().T, 2e-2)


@pytest.mark.parametrize("a_mn,b_mn", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,Kd", [(256, 256, 128), (384, 640, 1024), (200, 136, 72), (1000, 520, 264)])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_gemm_mn_major(cuda, a_mn, b_mn, M, N, Kd, bn):
    At = _rand(Kd, M, dev=cuda, seed=3) if a_mn else _rand(M, Kd, dev=cuda, seed=3)
    Bt = _rand(Kd, N, dev=cuda, seed=4) if b_mn else _rand(N, Kd, dev=cuda, seed=4)
    A = At.T if a_mn else At
    B = Bt.T if b_mn else Bt
    C = torch.zeros(M, N, dtype=torch.float32, device=cuda)
    K.gemm(At, Bt, C, M, N, Kd, lda=(M if a_mn else Kd), ldb=(N if b_mn else Kd), ldc=N, a_mn_major=a_mn,
           b_mn_major=b_mn, epi=K.EPI_OUT_F32, force_bn=bn)
    torch.cuda.synchronize()
    _close(C, A.float() @ B.float().T, 1e-3)


@pytest.mark.parametrize("T,n_out,k_in", [(1024, 768, 512), (4096, 1024, 1024), (4096, 1000, 520), (4096, 3072, 1024),
                                          (4096, 2816, 1024)])
def test_gemm_wgrad_accumulates(cuda, T, n_out, k_in):
    # dW[N_out, K_in] += dY^T X over two micro-batches (both operands MN-major;
    # few output tiles -> split-K with atomic fp32 accumulation)
    dW = torch.zeros(n_out, k_in, dtype=torch.float32, device=cuda)
    ref = torch.zeros_like(dW)
    for mb in range(2):
        dY = _rand(T, n_out, dev=cuda, seed=10 + mb)
        X = _rand(T, k_in, dev=cuda, seed=20 + mb)
        K.gemm(dY, X, dW, n_out, k_in, T, lda=n_out, ldb=k_in, ldc=k_in, a_mn_major=True, b_mn_major=True,
               epi=K.EPI_OUT_F32_ACC)
        ref += dY.float().T @ X.float()
    torch.cuda.synchronize()
    _close(dW, ref, 1e-3)


def test_gemm_bias_gelu_aux(cuda):
    M, N, Kd = 512, 1024, 256
    A = _rand(M, Kd, dev=cuda, seed=5)
    B = _rand(N, Kd, dev=cuda, seed=6, scale=0.1)
    bias = _rand(N, dev=cuda, seed=7, dtype=torch.float32)
    C = torch.empty(M, N, dtype=torch.bfloat16, device=cuda)
    Z = torch.empty(M, N, dtype=torch.bfloat16, device=cuda)
    K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT, bias=bias,
           aux_out=Z)
    torch.cuda.synchronize()
    z = A.float() @ B.float().T + bias
    _close(Z, z, 2e-2)
    _close(C, torch.nn.functional.gelu(z, approximate="tanh"), 2e-2)


def test_gemm_dgelu_and_resid(cuda):
    M, N, Kd = 256, 512, 384
    A = _rand(M, Kd, dev=cuda, seed=8)
    B = _rand(N, Kd, dev=cuda, seed=9, scale=0.1)
    Z = _rand(M, N, dev=cuda, seed=11, scale=2.0)
    R = _rand(M, N, dev=cuda, seed=12)
    C = torch.empty(M, N, dtype=torch.bfloat16, device=cuda)
    K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=K.EPI_DGELU, aux_in=Z)
    torch.cuda.synchronize()
    z = Z.float().requires_grad_(True)
    g = torch.autograd.grad(torch.nn.functional.gelu(z, approximate="tanh").sum(), z)[0]
    _close(C, (A.float() @ B.float().T) * g, 2e-2)
    K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=K.EPI_RESID, resid=R, alpha=0.5)
    torch.cuda.synchronize()
    _close(C, 0.5 * (A.float() @ B.float().T) + R.float(), 2e-2)


def test_gemm_attention_head_split_merge(cuda):
    # QKV projection with head-split store, then batched S = Q K^T and
    # ctx = P V with head-merge store, as the transformer stage uses them.
    B_, S, H, nh = 2, 256, 256, 4
    d = H // nh
    T = B_ * S
    X = _rand(T, H, dev=cuda, seed=13)
    W = _rand(3 * H, H, dev=cuda, seed=14, scale=0.1)
    qkv = torch.empty(3, nh, B_, S, d, dtype=torch.bfloat16, device=cuda)
    K.gemm(X, W, qkv, T, 3 * H, H, lda=H, ldb=H, ldc=d, ndiv=d, s_no=T * d)
    ref = (X.float() @ W.float().T).view(B_, S, 3, nh, d).permute(2, 3, 0, 1, 4)
    torch.cuda.synchronize()
    _close(qkv, ref, 2e-2)
    q, k, v = qkv[0].reshape(nh * B_, S, d), qkv[1].reshape(nh * B_, S, d), qkv[2].reshape(nh * B_, S, d)
    Sc = torch.empty(nh * B_, S, S, dtype=torch.float32, device=cuda)
    K.gemm(q, k, Sc, S, S, d, lda=d, ldb=d, ldc=S, batch=nh * B_, a_batch_stride=S * d, b_batch_stride=S * d,
           epi=K.EPI_OUT_F32, alpha=0.125)
    torch.cuda.synchronize()
    _close(Sc, 0.125 * q.float() @ k.float().transpose(1, 2), 1e-3)
    P = torch.softmax(Sc, -1).to(torch.bfloat16)
    ctx = torch.empty(T, H, dtype=torch.bfloat16, device=cuda)
    # z = h*B + b ; row = b*S + s ; col = h*d + j
    K.gemm(P, v, ctx, S, d, S, lda=S, ldb=d, ldc=H, batch=nh * B_, a_batch_stride=S * S, b_batch_stride=S * d,
           b_mn_major=True, zdiv=B_, s_zo=d, s_zi=S * H)
    torch.cuda.synchronize()
    ref_ctx = (P.float() @ v.float()).view(nh, B_, S, d).permute(1, 2, 0, 3).reshape(T, H)
    _close(ctx, ref_ctx, 2e-2)


@pytest.mark.parametrize("m,n,k,one_sm", [(4096, 4096, 1024, False), (300, 200, 128, True), (1024, 1600, 6400, False)])
def test_gemm_colsum_epilogue(cuda, m, n, k, one_sm):
    """DPL_EPI_COLSUM: colsum[n] += sum over rows of the stored bf16 output
    (the FFN bias gradient fused into the dgrad GEMM)."""
    import torch
    from paper_2007_01045_b200 import kernels as K
    g = torch.Generator(device="cpu").manual_seed(11)
    a = (torch.rand(m, k, generator=g) - 0.5).to(torch.bfloat16).to(cuda)
    b = (torch.rand(n, k, generator=g) - 0.5).to(torch.bfloat16).to(cuda)
    c = torch.empty(m, n, dtype=torch.bfloat16, device=cuda)
    cs = torch.full((n,), 0.5, device=cuda)
    K.gemm(a, b, c, m, n, k, lda=k, ldb=k, ldc=n, epi=K.EPI_OUT_BF16 | K.EPI_COLSUM, colsum=cs, force_1sm=one_sm)
    torch.cuda.synchronize()
    ref = c.float().sum(0) + 0.5
    assert torch.allclose(c.float(), a.float() @ b.float().T, rtol=2e-2, atol=2e-2)
    assert torch.allclose(cs, ref, rtol=1e-4, atol=1e-2 * m ** 0.5 * 0.01)


@pytest.mark.parametrize("M,N,Kd,epi", [
    (1024, 1600, 6400, "bias+resid"),   # GPT-2 ffn2 at one sample per micro-batch (28 pair tiles)
    (2048, 1024, 4096, "plain"),        # BERT dgrad at a 4-sample replica slice (32 pair tiles)
    (1024, 1024, 1024, "dgelu"),        # 16 pair tiles, act' epilogue
    (1000, 1600, 1600, "bias"),         # ragged M
])
def test_gemm_split_k_bf16(cuda, M, N, Kd, epi):
    """bf16-output GEMMs that would leave most CTA pairs idle run as split-K
    fp32 reduce-add into a zeroed scratch + a bf16 epilogue pass; the result
    matches the unsplit GEMM and torch, and the scratch is left zero."""
    A = _rand(M, Kd, dev=cuda, seed=11)
    B = _rand(N, Kd, dev=cuda, seed=12)
    bias = _rand(N, dev=cuda, seed=13, dtype=torch.float32)
    res = _rand(M, N, dev=cuda, seed=14)
    z = _rand(M, N, dev=cuda, seed=15, scale=3.0)
    flags = {"plain": 0, "bias": K.EPI_BIAS, "bias+resid": K.EPI_BIAS | K.EPI_RESID, "dgelu": K.EPI_DGELU}[epi]
    kw = dict(lda=Kd, ldb=Kd, ldc=N, epi=flags, bias=bias if flags & K.EPI_BIAS else None,
              resid=res if flags & K.EPI_RESID else None, aux_in=z if flags & K.EPI_DGELU else None)
    ws = torch.zeros(M * N, dtype=torch.float32, device=cuda)
    C1 = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    C2 = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    K.gemm(A, B, C1, M, N, Kd, **kw)
    for _ in range(2):  # twice: the scratch must come back zeroed
        K.gemm(A, B, C2, M, N, Kd, split_ws=ws, **kw)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    if flags & K.EPI_BIAS:
        ref = ref + bias
    if flags & K.EPI_RESID:
        ref = ref + res.float()
    if flags & K.EPI_DGELU:
        zf = z.float()
        t = torch.tanh(0.7978845608028654 * (zf + 0.044715 * zf ** 3))
        ref = ref * (0.5 * (1 + t) + 0.5 * zf * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * zf * zf))
    _close(C2, ref, 2e-2)
    _close(C2, C1.float(), 2e-2)
    assert int((ws != 0).sum()) == 0


@pytest.mark.parametrize("M,N,Kd,epi,mn", [
    (4096, 4096, 1024, "bias+gelu+aux", False),  # BERT ffn1: 256 pair tiles = 3 waves + 34 -> 68 halves
    (4096, 4096, 1024, "dgelu", False),          # BERT ffn2 dgrad
    (4096, 4096, 1024, "resid", False),
    (2048, 6400, 1600, "bias+gelu+aux", False),  # 200 tiles -> 2 waves + 52 -> 104 halves (no split: > 74)
    (3072, 4096, 1600, "bias", False),           # 192 tiles -> 148 whole + 44 -> 88 halves (no split)
    (4096, 4608, 520, "bias+gelu+aux", False),   # 288 tiles -> 3 waves + 66 (no split: 132 > 74)
    (4096, 4352, 520, "resid", False),           # 272 tiles -> 3 waves + 50 (no split) ; sanity of the rule
    (6144, 4096, 1024, "bias+gelu+aux", False),  # 384 tiles -> 5 waves + 14 -> 28 halves
    (4096, 4096, 1024, "f32acc", True),          # weight-gradient form: MN-major operands, fp32 reduce-add
    (4000, 4000, 520, "bias", False),            # ragged edges in the split tail
])
def test_gemm_split_tail_halves(cuda, M, N, Kd, epi, mn):
    """Pair-kernel GEMMs whose last wave fills at most half the CTA pairs run
    that wave's tiles as two 256 x 128 halves each (GemmParams.split_tail);
    every output element, bias / activation / aux / residual / fp32
    accumulation included, matches torch fp32."""
    A = _rand(M, Kd, dev=cuda, seed=31)
    B = _rand(N, Kd, dev=cuda, seed=32, scale=0.2)
    bias = _rand(N, dev=cuda, seed=33, dtype=torch.float32)
    z = _rand(M, N, dev=cuda, seed=34, scale=2.0)
    res = _rand(M, N, dev=cuda, seed=35)
    ref = A.float() @ B.float().T
    if epi == "f32acc":
        At, Bt = A.T.contiguous(), B.T.contiguous()
        C = torch.full((M, N), 0.5, dtype=torch.float32, device=cuda)
        K.gemm(At, Bt, C, M, N, Kd, lda=M, ldb=N, ldc=N, a_mn_major=True, b_mn_major=True, epi=K.EPI_OUT_F32_ACC)
        torch.cuda.synchronize()
        _close(C, ref + 0.5, 1e-3)
        return
    flags = {"bias": K.EPI_BIAS, "bias+gelu+aux": K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT, "dgelu": K.EPI_DGELU,
             "resid": K.EPI_RESID}[epi]
    C = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    Z = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=flags, bias=bias if flags & K.EPI_BIAS else None,
           aux_in=z if flags & K.EPI_DGELU else None, resid=res if flags & K.EPI_RESID else None,
           aux_out=Z if flags & K.EPI_AUX_OUT else None)
    torch.cuda.synchronize()
    if flags & K.EPI_BIAS:
        ref = ref + bias
    if flags & K.EPI_AUX_OUT:
        _close(Z, ref, 2e-2)
    if flags & K.EPI_GELU:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    if flags & K.EPI_RESID:
        ref = ref + res.float()
    if flags & K.EPI_DGELU:
        zf = z.float().requires_grad_(True)
        ref = ref * torch.autograd.grad(torch.nn.functional.gelu(zf, approximate="tanh").sum(), zf)[0]
    _close(C, ref, 2e-2)


@pytest.mark.parametrize("M,N,Kd,epi", [
    (1024, 4800, 1600, "bias"),            # GPT-2 qkv (default choice: 256 x 192 pairs)
    (1024, 6400, 1600, "bias+gelu+aux"),   # GPT-2 ffn1: ragged last n-block (6400 = 33 x 192 + 64)
    (2048, 3072, 1024, "bias"),            # BERT qkv at a 4-sample replica slice
    (300, 1000, 520, "resid"),             # ragged M and N
    (512, 192, 64, "plain"),               # one n-block
])
@pytest.mark.parametrize("forced", [True, False])
def test_gemm_pair_bn192(cuda, M, N, Kd, epi, forced):
    """256 x 192 CTA-pair tiles (K-major B): every epilogue against torch fp32,
    forced and as the default tile choice."""
    A = _rand(M, Kd, dev=cuda, seed=41)
    B = _rand(N, Kd, dev=cuda, seed=42, scale=0.2)
    bias = _rand(N, dev=cuda, seed=43, dtype=torch.float32)
    res = _rand(M, N, dev=cuda, seed=44)
    flags = {"plain": 0, "bias": K.EPI_BIAS, "bias+gelu+aux": K.EPI_BIAS | K.EPI_GELU | K.EPI_AUX_OUT,
             "resid": K.EPI_RESID}[epi]
    C = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    Z = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    K.gemm(A, B, C, M, N, Kd, lda=Kd, ldb=Kd, ldc=N, epi=flags, bias=bias if flags & K.EPI_BIAS else None,
           resid=res if flags & K.EPI_RESID else None, aux_out=Z if flags & K.EPI_AUX_OUT else None,
           force_bn=192 if forced else 0)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    if flags & K.EPI_BIAS:
        ref = ref + bias
    if flags & K.EPI_AUX_OUT:
        _close(Z, ref, 2e-2)
    if flags & K.EPI_GELU:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    if flags & K.EPI_RESID:
        ref = ref + res.float()
    _close(C, ref, 2e-2)
