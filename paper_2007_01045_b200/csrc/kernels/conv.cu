// VGG convolution support kernels (see conv.h).  Work per launch:
//   im2col3x3       reads x (9x from L2), writes N*H*W*kp*2 bytes
//   col2im3x3       reads 9 column taps per output vector, writes N*H*W*C*2 bytes
//   maxpool2_fwd    reads 4 vectors, writes 1 per output vector
//   maxpool2_relu_bwd  reads 4 x vectors + 1 dy vector, writes 4 dz vectors
// One thread per 16-byte vector (8 channels) wherever C % 8 == 0.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>

#include "conv.h"
#include "gemm.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace dpl {

namespace {

using bf16 = __nv_bfloat16;

int grid_for(long long n, int block) {
  const long long g = (n + block - 1) / block;
  return static_cast<int>(std::min<long long>(std::max<long long>(g, 1), 148LL * 32));
}

__device__ __forceinline__ void unpack(const uint4& r, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = __bfloat1622float2(h[e]);
    f[2 * e] = x.x;
    f[2 * e + 1] = x.y;
  }
}

__device__ __forceinline__ uint4 pack(const float (&f)[8]) {
  uint4 r;
  uint32_t* w = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    w[e] = *reinterpret_cast<uint32_t*>(&h);
  }
  return r;
}

// C % 8 == 0: thread per (pixel, tap, 8-channel vector); zero tail columns 9C..kp
__global__ void im2col_vec_kernel(const bf16* __restrict__ x, bf16* __restrict__ col, int n, int h, int w, int c,
                                  int kp) {
  ptx::pdl_wait();
  const int cv = c / 8;
  const int per_px = kp / 8;  // vectors per column row (9 * cv taps, then zero tail)
  const long long total = static_cast<long long>(n) * h * w * per_px;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long px = i / per_px;
    const int v = static_cast<int>(i % per_px);
    uint4 out = make_uint4(0u, 0u, 0u, 0u);
    if (v < 9 * cv) {
      const int tap = v / cv, ci = v % cv;
      const int kh = tap / 3, kw = tap % 3;
      const int ww = static_cast<int>(px % w);
      const long long t = px / w;
      const int hh = static_cast<int>(t % h);
      const long long nn = t / h;
      const int hs = hh + kh - 1, ws = ww + kw - 1;
      if (hs >= 0 && hs < h && ws >= 0 && ws < w)
        out = *reinterpret_cast<const uint4*>(x + ((nn * h + hs) * w + ws) * c + ci * 8);
    }
    *reinterpret_cast<uint4*>(col + px * kp + v * 8) = out;
  }
}

// any C (the RGB input): thread per column element
__global__ void im2col_scalar_kernel(const bf16* __restrict__ x, bf16* __restrict__ col, int n, int h, int w, int c,
                                     int kp) {
  ptx::pdl_wait();
  const long long total = static_cast<long long>(n) * h * w * kp;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long px = i / kp;
    const int k = static_cast<int>(i % kp);
    bf16 out = __float2bfloat16_rn(0.f);
    if (k < 9 * c) {
      const int tap = k / c, ci = k % c;
      const int kh = tap / 3, kw = tap % 3;
      const int ww = static_cast<int>(px % w);
      const long long t = px / w;
      const int hh = static_cast<int>(t % h);
      const long long nn = t / h;
      const int hs = hh + kh - 1, ws = ww + kw - 1;
      if (hs >= 0 && hs < h && ws >= 0 && ws < w) out = x[((nn * h + hs) * w + ws) * c + ci];
    }
    col[i] = out;
  }
}

__global__ void col2im_kernel(const bf16* __restrict__ dcol, bf16* __restrict__ dx, int n, int h, int w, int c,
                              int kp) {
  ptx::pdl_wait();
  const int cv = c / 8;
  const long long total = static_cast<long long>(n) * h * w * cv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ci = static_cast<int>(i % cv);
    const long long px = i / cv;
    const int ww = static_cast<int>(px % w);
    const long long t = px / w;
    const int hh = static_cast<int>(t % h);
    const long long nn = t / h;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int ho = hh + 1 - kh;  // output pixel whose tap (kh, kw) reads (hh, ww)
      if (ho < 0 || ho >= h) continue;
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const int wo = ww + 1 - kw;
        if (wo < 0 || wo >= w) continue;
        float f[8];
        unpack(*reinterpret_cast<const uint4*>(dcol + ((nn * h + ho) * w + wo) * kp + (kh * 3 + kw) * c + ci * 8), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += f[e];
      }
    }
    *reinterpret_cast<uint4*>(dx + px * c + ci * 8) = pack(acc);
  }
}

__global__ void maxpool_fwd_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, int n, int h, int w, int c) {
  ptx::pdl_wait();
  const int cv = c / 8, ho = h / 2, wo = w / 2;
  const long long total = static_cast<long long>(n) * ho * wo * cv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ci = static_cast<int>(i % cv);
    const long long po = i / cv;
    const int pw = static_cast<int>(po % wo);
    const long long t = po / wo;
    const int ph = static_cast<int>(t % ho);
    const long long nn = t / ho;
    float m[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float f[8];
      unpack(*reinterpret_cast<const uint4*>(x + ((nn * h + 2 * ph + (q >> 1)) * w + 2 * pw + (q & 1)) * c + ci * 8), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) m[e] = q == 0 ? f[e] : fmaxf(m[e], f[e]);
    }
    *reinterpret_cast<uint4*>(y + po * c + ci * 8) = pack(m);
  }
}

__global__ void maxpool_relu_bwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ dy, bf16* __restrict__ dz,
                                        int n, int h, int w, int c) {
  ptx::pdl_wait();
  const int cv = c / 8, ho = h / 2, wo = w / 2;
  const long long total = static_cast<long long>(n) * ho * wo * cv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ci = static_cast<int>(i % cv);
    const long long po = i / cv;
    const int pw = static_cast<int>(po % wo);
    const long long t = po / wo;
    const int ph = static_cast<int>(t % ho);
    const long long nn = t / ho;
    float v[4][8], g[8];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      unpack(*reinterpret_cast<const uint4*>(x + ((nn * h + 2 * ph + (q >> 1)) * w + 2 * pw + (q & 1)) * c + ci * 8),
             v[q]);
    unpack(*reinterpret_cast<const uint4*>(dy + po * c + ci * 8), g);
    int arg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int a = 0;
      float m = v[0][e];
#pragma unroll
      for (int q = 1; q < 4; ++q)
        if (v[q][e] > m) {
          m = v[q][e];
          a = q;
        }
      arg[e] = m > 0.f ? a : -1;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = arg[e] == q ? g[e] : 0.f;
      *reinterpret_cast<uint4*>(dz + ((nn * h + 2 * ph + (q >> 1)) * w + 2 * pw + (q & 1)) * c + ci * 8) = pack(o);
    }
  }
}

__global__ void relu_bwd_kernel(const bf16* __restrict__ y, const bf16* __restrict__ dy, bf16* __restrict__ dz,
                                long long nvec) {
  ptx::pdl_wait();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nvec;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8], g[8];
    unpack(reinterpret_cast<const uint4*>(y)[i], a);
    unpack(reinterpret_cast<const uint4*>(dy)[i], g);
#pragma unroll
    for (int e = 0; e < 8; ++e) g[e] = a[e] > 0.f ? g[e] : 0.f;
    reinterpret_cast<uint4*>(dz)[i] = pack(g);
  }
}

__global__ void conv_weight_flip_kernel(const bf16* __restrict__ w, bf16* __restrict__ wt, int cin, int cout,
                                        int kp) {
  ptx::pdl_wait();
  const long long total = static_cast<long long>(cin) * 9 * cout;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i / (9LL * cout));
    const int r = static_cast<int>(i % (9LL * cout));
    const int t = r / cout, co = r % cout;
    wt[i] = w[static_cast<long long>(co) * kp + (8 - t) * cin + c];
  }
}

}  // namespace

void conv_weight_flip(const void* w, void* wt, int cin, int cout, int kp, cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("conv_weight_flip", s);
  launch_pdl(conv_weight_flip_kernel, dim3(grid_for(static_cast<long long>(cin) * 9 * cout, 256)), dim3(256), 0, s,
             static_cast<const bf16*>(w), static_cast<bf16*>(wt), cin, cout, kp);
}

void im2col3x3(const void* x, void* col, int n, int h, int w, int c, int kp, cudaStream_t s) {
  if (kp < 9 * c || kp % 8) throw std::invalid_argument("im2col3x3: kp must be >= 9C and a multiple of 8");
  count_launch();
  TimedLaunch timed_("im2col", s);
  const auto* px = static_cast<const bf16*>(x);
  auto* pc = static_cast<bf16*>(col);
  if (c % 8 == 0)
    launch_pdl(im2col_vec_kernel, dim3(grid_for(static_cast<long long>(n) * h * w * (kp / 8), 256)), dim3(256), 0, s,
               px, pc, n, h, w, c, kp);
  else
    launch_pdl(im2col_scalar_kernel, dim3(grid_for(static_cast<long long>(n) * h * w * kp, 256)), dim3(256), 0, s, px,
               pc, n, h, w, c, kp);
}

void col2im3x3(const void* dcol, void* dx, int n, int h, int w, int c, int kp, cudaStream_t s) {
  if (c % 8 || kp < 9 * c || kp % 8) throw std::invalid_argument("col2im3x3: C % 8 == 0 and kp >= 9C required");
  count_launch();
  TimedLaunch timed_("col2im", s);
  launch_pdl(col2im_kernel, dim3(grid_for(static_cast<long long>(n) * h * w * (c / 8), 256)), dim3(256), 0, s,
             static_cast<const bf16*>(dcol), static_cast<bf16*>(dx), n, h, w, c, kp);
}

void maxpool2_fwd(const void* x, void* y, int n, int h, int w, int c, cudaStream_t s) {
  if (c % 8 || h % 2 || w % 2) throw std::invalid_argument("maxpool2_fwd: C % 8 == 0 and even H, W required");
  count_launch();
  TimedLaunch timed_("maxpool_fwd", s);
  launch_pdl(maxpool_fwd_kernel, dim3(grid_for(static_cast<long long>(n) * (h / 2) * (w / 2) * (c / 8), 256)),
             dim3(256), 0, s, static_cast<const bf16*>(x), static_cast<bf16*>(y), n, h, w, c);
}

void maxpool2_relu_bwd(const void* x, const void* dy, void* dz, int n, int h, int w, int c, cudaStream_t s) {
  if (c % 8 || h % 2 || w % 2) throw std::invalid_argument("maxpool2_relu_bwd: C % 8 == 0 and even H, W required");
  count_launch();
  TimedLaunch timed_("maxpool_relu_bwd", s);
  launch_pdl(maxpool_relu_bwd_kernel, dim3(grid_for(static_cast<long long>(n) * (h / 2) * (w / 2) * (c / 8), 256)),
             dim3(256), 0, s, static_cast<const bf16*>(x), static_cast<const bf16*>(dy), static_cast<bf16*>(dz), n, h,
             w, c);
}

void relu_bwd(const void* y, const void* dy, void* dz, long long n, cudaStream_t s) {
  if (n % 8) throw std::invalid_argument("relu_bwd: n % 8 == 0 required");
  count_launch();
  TimedLaunch timed_("relu_bwd", s);
  launch_pdl(relu_bwd_kernel, dim3(grid_for(n / 8, 256)), dim3(256), 0, s, static_cast<const bf16*>(y),
             static_cast<const bf16*>(dy), static_cast<bf16*>(dz), n / 8);
}

}  // namespace dpl
