"""Python front for the individual sm_100a stage kernels (dpl_k_* in
include/dapple.h).  torch tensors are used only as device allocations; every
call goes straight to libdapple.so on the tensor's current CUDA stream."""
from __future__ import annotations

import ctypes

from ._lib import (EPI_AUX_OUT, EPI_BIAS, EPI_DGELU, EPI_DRELU, EPI_GELU, EPI_OUT_BF16, EPI_OUT_F32,  # noqa: F401
                   EPI_OUT_F32_ACC, EPI_RELU, EPI_RESID, EPI_COLSUM, GemmDesc, check, lib)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def gemm(A, B, C, M, N, K, *, lda, ldb, ldc, a_mn_major=False, b_mn_major=False, batch=1, a_batch_stride=0,
         b_batch_stride=0, epi=EPI_OUT_BF16, alpha=1.0, bias=None, aux_in=None, resid=None, aux_out=None, zdiv=1,
         s_zo=None, s_zi=0, ndiv=1 << 30, s_no=0, force_bn=0, force_1sm=False, trace=None, colsum=None, conv=None,
         split_ws=None):
    """C[z,m,n] = epi(alpha * sum_k A[z,m,k] * B[z,n,k]) (see csrc/kernels/gemm.h)."""
    d = GemmDesc()
    d.M, d.N, d.K, d.batch = M, N, K, batch
    d.A, d.lda, d.a_batch_stride, d.a_mn_major = A.data_ptr(), lda, a_batch_stride, int(a_mn_major)
    d.B, d.ldb, d.b_batch_stride, d.b_mn_major = B.data_ptr(), ldb, b_batch_stride, int(b_mn_major)
    d.C, d.ldc, d.zdiv = C.data_ptr(), ldc, zdiv
    d.s_zo = M * ldc if s_zo is None else s_zo
    d.s_zi, d.ndiv, d.s_no = s_zi, ndiv, s_no
    d.epi, d.alpha = epi, alpha
    d.bias = None if bias is None else bias.data_ptr()
    d.aux_in = None if aux_in is None else aux_in.data_ptr()
    d.resid = None if resid is None else resid.data_ptr()
    d.aux_out = None if aux_out is None else aux_out.data_ptr()
    d.force_bn = force_bn
    d.force_1sm = int(force_1sm)
    d.trace = None if trace is None else trace.data_ptr()
    d.colsum = None if colsum is None else colsum.data_ptr()
    if split_ws is not None:  # zeroed fp32 scratch: split-K for bf16 outputs with few tiles
        d.split_ws, d.split_ws_bytes = split_ws.data_ptr(), split_ws.numel() * split_ws.element_size()
    if conv is not None:  # (operand 1|2, x NHWC tensor, n, h, w, c): implicit-GEMM convolution
        d.conv_operand, x, d.conv_n, d.conv_h, d.conv_w, d.conv_c = conv
        d.conv_x = x.data_ptr()
    check(lib().dpl_k_gemm(ctypes.byref(d), _stream()))


def layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, h, eps=1e-5):
    check(lib().dpl_k_layernorm_fwd(_ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), _ptr(mean), _ptr(rstd), rows, h, eps,
                                    _stream()))


def layernorm_bwd(dy, x, mean, rstd, gamma, dresid, dx, dgamma, dbeta, rows, h):
    check(lib().dpl_k_layernorm_bwd(_ptr(dy), _ptr(x), _ptr(mean), _ptr(rstd), _ptr(gamma), _ptr(dresid), _ptr(dx),
                                    _ptr(dgamma), _ptr(dbeta), rows, h, _stream()))


def layernorm_bwd_colsum(dy, x, mean, rstd, gamma, dresid, dx, dgamma, dbeta, dresid_colsum, dx_colsum, rows, h):
    check(lib().dpl_k_layernorm_bwd_colsum(_ptr(dy), _ptr(x), _ptr(mean), _ptr(rstd), _ptr(gamma), _ptr(dresid),
                                           _ptr(dx), _ptr(dgamma), _ptr(dbeta), _ptr(dresid_colsum), _ptr(dx_colsum),
                                           rows, h, _stream()))


def softmax_fwd(s, p, rows, length, q_len, causal=False):
    check(lib().dpl_k_softmax_fwd(_ptr(s), _ptr(p), rows, length, q_len, int(causal), _stream()))


def softmax_bwd(p, dp, ds, rows, length):
    check(lib().dpl_k_softmax_bwd(_ptr(p), _ptr(dp), _ptr(ds), rows, length, _stream()))


def colsum_acc(dy, db, rows, cols):
    check(lib().dpl_k_colsum_acc(_ptr(dy), _ptr(db), rows, cols, _stream()))


def mse_loss(y, t, dy, loss_acc, n, grad_scale):
    check(lib().dpl_k_mse_loss(_ptr(y), _ptr(t), _ptr(dy), _ptr(loss_acc), n, grad_scale, _stream()))


def fill_tokens(dst, n, seed, tensor, idx0, vocab):
    check(lib().dpl_k_fill_tokens(_ptr(dst), n, seed, tensor, idx0, vocab, _stream()))


def embed_fwd(tok, wte, wpe, x, rows, seq, h):
    check(lib().dpl_k_embed_fwd(_ptr(tok), _ptr(wte), _ptr(wpe), _ptr(x), rows, seq, h, _stream()))


def embed_bwd(tok, dx, gwte, gwpe, rows, seq, h):
    check(lib().dpl_k_embed_bwd(_ptr(tok), _ptr(dx), _ptr(gwte), _ptr(gwpe), rows, seq, h, _stream()))


def cross_entropy_padded(logits, tgt, loss_acc, rows, vocab, ld, grad_scale):
    check(lib().dpl_k_cross_entropy_padded(_ptr(logits), _ptr(tgt), _ptr(loss_acc), rows, vocab, ld, grad_scale,
                                           _stream()))


def cross_entropy(logits, tgt, loss_acc, rows, vocab, grad_scale):
    """In place: logits rows -> (softmax - onehot(tgt)) * grad_scale; loss_acc += sum CE."""
    check(lib().dpl_k_cross_entropy(_ptr(logits), _ptr(tgt), _ptr(loss_acc), rows, vocab, grad_scale, _stream()))


def im2col3x3(x, col, n, h, w, c, kp):
    check(lib().dpl_k_im2col3x3(_ptr(x), _ptr(col), n, h, w, c, kp, _stream()))


def col2im3x3(dcol, dx, n, h, w, c, kp):
    check(lib().dpl_k_col2im3x3(_ptr(dcol), _ptr(dx), n, h, w, c, kp, _stream()))


def maxpool2_fwd(x, y, n, h, w, c):
    check(lib().dpl_k_maxpool2_fwd(_ptr(x), _ptr(y), n, h, w, c, _stream()))


def maxpool2_relu_bwd(x, dy, dz, n, h, w, c):
    check(lib().dpl_k_maxpool2_relu_bwd(_ptr(x), _ptr(dy), _ptr(dz), n, h, w, c, _stream()))


def relu_bwd(y, dy, dz, n):
    check(lib().dpl_k_relu_bwd(_ptr(y), _ptr(dy), _ptr(dz), n, _stream()))


def sgd_apply(w32, g, w16, n, lr):
    check(lib().dpl_k_sgd_apply(_ptr(w32), _ptr(g), _ptr(w16), n, lr, _stream()))


def fill_uniform_bf16(dst, n, seed, tensor, idx0=0, scale=1.0):
    check(lib().dpl_k_fill_uniform_bf16(_ptr(dst), n, seed, tensor, idx0, scale, _stream()))


def fill_uniform_f32(dst, n, seed, tensor, idx0=0, scale=1.0):
    check(lib().dpl_k_fill_uniform_f32(_ptr(dst), n, seed, tensor, idx0, scale, _stream()))


def attention_fwd(qkv, ctx, lse, samples, seq, heads, ldc, causal=False):
    """Fused flash attention forward (head dim 64): qkv [3][heads][B][S][64],
    ctx [B*S][ldc] head-merged, lse [heads*B][S]."""
    check(lib().dpl_k_attention_fwd(_ptr(qkv), _ptr(ctx), ldc, _ptr(lse), samples, seq, heads, int(causal), _stream()))


def attention_fwd_traced(qkv, ctx, lse, samples, seq, heads, ldc, trace, causal=False):
    """attention_fwd with per-CTA %globaltimer marks in trace (int64, 16 per CTA)."""
    check(lib().dpl_k_attention_fwd_traced(_ptr(qkv), _ptr(ctx), ldc, _ptr(lse), samples, seq, heads, int(causal),
                                           _ptr(trace), _stream()))


def attention_bwd(qkv, ctx, lse, dout, dqkv, dsum, dq_acc, samples, seq, heads, ldc, causal=False):
    """Fused flash attention backward (head dim 64)."""
    check(lib().dpl_k_attention_bwd(_ptr(qkv), _ptr(ctx), ldc, _ptr(lse), _ptr(dout), _ptr(dqkv), _ptr(dsum),
                                    _ptr(dq_acc), samples, seq, heads, int(causal), _stream()))


def attention_bwd_traced(qkv, ctx, lse, dout, dqkv, dsum, dq_acc, samples, seq, heads, ldc, trace, causal=False):
    """attention_bwd with per-CTA %globaltimer marks of the main kernel in trace (int64, 16 per CTA)."""
    check(lib().dpl_k_attention_bwd_traced(_ptr(qkv), _ptr(ctx), ldc, _ptr(lse), _ptr(dout), _ptr(dqkv), _ptr(dsum),
                                           _ptr(dq_acc), samples, seq, heads, int(causal), _ptr(trace), _stream()))
