// Host launchers for the HBM-bound stage kernels (elementwise.cu).
// All tensors are row-major; bf16 tensors are passed as void*.  Row lengths
// must be multiples of 8 elements (16-byte vectors).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dpl {

void layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y, float* mean, float* rstd, int rows,
                   int h, float eps, cudaStream_t s);
// ws: kLnBwdBlocks * 4 * h floats of scratch.  Optionally also accumulates
// the column sums of dresid and of dx (bias gradients of the neighbouring
// layers) so they need no separate pass.
constexpr int kLnBwdBlocks = 148 * 4;
void layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gamma,
                   const void* dresid, void* dx, float* dgamma, float* dbeta, int rows, int h, cudaStream_t s,
                   float* ws, float* dresid_colsum = nullptr, float* dx_colsum = nullptr);
void softmax_fwd(const float* s, void* p, int rows, int len, int q_len, int causal, cudaStream_t st);
void softmax_bwd(const void* p, const float* dp, void* ds, int rows, int len, cudaStream_t st);
void colsum_acc(const void* dy, float* db, int rows, int cols, cudaStream_t s);
// Epilogue of a split-K bf16 GEMM: C[m][n] = bf16((acc[m][n] * alpha + bias[n]
// + resid[m][n]) * gelu'(aux_in[m][n])) with the optional terms selected by
// epi (gemm.h kBias / kResid / kDGelu), acc [M][N] fp32 dense; acc is zeroed.
void split_epilogue(float* acc, void* c, long long ldc, int m, int n, float alpha, const float* bias,
                    const void* resid, const void* aux_in, uint32_t epi, cudaStream_t s);
void mse_loss(const void* y, const void* t, void* dy, float* loss_acc, long long n, float grad_scale, cudaStream_t s);
void sgd_apply(float* w32, float* g, void* w16, long long n, float lr, cudaStream_t s);
void fill_uniform_bf16(void* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                       cudaStream_t s);
void fill_uniform_f32(float* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                      cudaStream_t s);
void fill_const_f32(float* dst, long long n, float v, cudaStream_t s);
void cast_f32_bf16(const float* src, void* dst, long long n, cudaStream_t s);

}  // namespace dpl
