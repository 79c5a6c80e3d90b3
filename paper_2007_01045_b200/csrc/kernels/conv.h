// Host launchers for the VGG convolution support kernels (conv.cu).  A 3x3,
// stride-1, pad-1 convolution over NHWC bf16 activations runs on the tcgen05
// GEMM through explicit columns:
//   col[(n*H + h)*W + w][(kh*3 + kw)*C + c] = x[n][h+kh-1][w+kw-1][c]   (0 outside)
// (row length kp >= 9C, zero padded to a multiple of 8), y = col W^T.
// All HBM-bound.
#pragma once

#include <cuda_runtime.h>

namespace dpl {

void im2col3x3(const void* x, void* col, int n, int h, int w, int c, int kp, cudaStream_t s);
// dx[n][h][w][c] = sum_{kh,kw} dcol[(n*H + h+1-kh)*W + w+1-kw][(kh*3+kw)*C + c]   (C % 8 == 0)
void col2im3x3(const void* dcol, void* dx, int n, int h, int w, int c, int kp, cudaStream_t s);
// y[n][h/2][w/2][c] = max of the 2x2 window of x   (C % 8 == 0, h and w even)
void maxpool2_fwd(const void* x, void* y, int n, int h, int w, int c, cudaStream_t s);
// Unpool + ReLU': dz[n][h][w][c] = dy[n][h/2][w/2][c] at the first maximum of
// its window (row-major window order) if that x > 0, else 0.  x = post-ReLU.
void maxpool2_relu_bwd(const void* x, const void* dy, void* dz, int n, int h, int w, int c, cudaStream_t s);
// dz = dy * (y > 0)
void relu_bwd(const void* y, const void* dy, void* dz, long long n, cudaStream_t s);
// Weights of the transposed conv (backward data): wt[c][t*cout + co] =
// w[co][(8 - t)*cin + c] (t = kh*3 + kw), so dx = conv3x3(dz, wt)
void conv_weight_flip(const void* w, void* wt, int cin, int cout, int kp, cudaStream_t s);

}  // namespace dpl
