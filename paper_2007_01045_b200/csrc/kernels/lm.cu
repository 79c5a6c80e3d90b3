// Language-model ends of a GPT pipeline (config C4): the
// token + position embedding on the first stage and the softmax
// cross-entropy over the vocabulary on the last.  All HBM-bound:
//   embed_fwd   reads one wte row + one wpe row per token row, writes x
//               (6 B/elem: 2+2 read, 2 write);
//   embed_bwd   reads dx, red.add's into the fp32 wte / wpe gradients
//               (2 B read + 2 x 4 B red per element);
//   cross_entropy_fwd_bwd  one CTA per token row: pass 1 streams the bf16
//               logits row once (online max / sum-exp), pass 2 re-reads it
//               (the 100 KB row is still in L2) and writes the gradient
//               (softmax - onehot) * scale in place -- 2 B read + 2 B write
//               per logit from HBM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <stdexcept>

#include "gemm.h"
#include "launch.cuh"
#include "lm.h"
#include "ptx.cuh"

namespace dpl {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t tensor, uint64_t idx) {
  uint64_t z = seed + tensor * 0xD1B54A32D192ED03ull + idx * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D649BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void unpack8(const uint4& r, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = __bfloat1622float2(h[e]);
    f[2 * e] = x.x;
    f[2 * e + 1] = x.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 r;
  uint32_t* w = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    w[e] = *reinterpret_cast<uint32_t*>(&h);
  }
  return r;
}

int grid_for(long long n, int block) {
  const long long g = (n + block - 1) / block;
  return static_cast<int>(std::min<long long>(std::max<long long>(g, 1), 148LL * 16));
}

__global__ void fill_tokens_kernel(int* __restrict__ dst, long long n, uint64_t seed, uint64_t tensor, long long idx0,
                                   int vocab) {
  ptx::pdl_wait();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<int>((mix64(seed, tensor, static_cast<uint64_t>(idx0 + i)) >> 32) %
                              static_cast<uint64_t>(vocab));
}

__global__ void embed_fwd_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ wte,
                                 const __nv_bfloat16* __restrict__ wpe, __nv_bfloat16* __restrict__ x, int rows,
                                 int seq, int h) {
  ptx::pdl_wait();
  const int vpr = h / 8;
  const long long nvec = static_cast<long long>(rows) * vpr;
  for (long long vi = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; vi < nvec;
       vi += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(vi / vpr), c = static_cast<int>(vi % vpr) * 8;
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(wte + static_cast<size_t>(tok[r]) * h + c), a);
    unpack8(*reinterpret_cast<const uint4*>(wpe + static_cast<size_t>(r % seq) * h + c), b);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] += b[e];
    *reinterpret_cast<uint4*>(x + static_cast<size_t>(r) * h + c) = pack8(a);
  }
}

__global__ void embed_bwd_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ dx,
                                 float* __restrict__ gwte, float* __restrict__ gwpe, int rows, int seq, int h) {
  ptx::pdl_wait();
  const int vpr = h / 8;
  const long long nvec = static_cast<long long>(rows) * vpr;
  for (long long vi = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; vi < nvec;
       vi += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(vi / vpr), c = static_cast<int>(vi % vpr) * 8;
    float g[8];
    unpack8(*reinterpret_cast<const uint4*>(dx + static_cast<size_t>(r) * h + c), g);
    float4* t = reinterpret_cast<float4*>(gwte + static_cast<size_t>(tok[r]) * h + c);
    float4* p = reinterpret_cast<float4*>(gwpe + static_cast<size_t>(r % seq) * h + c);
    atomicAdd(t, make_float4(g[0], g[1], g[2], g[3]));
    atomicAdd(t + 1, make_float4(g[4], g[5], g[6], g[7]));
    atomicAdd(p, make_float4(g[0], g[1], g[2], g[3]));
    atomicAdd(p + 1, make_float4(g[4], g[5], g[6], g[7]));
  }
}

constexpr int kCeThreads = 512;

// combine two (max, sum-exp) pairs
__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  s = (m == -FLT_MAX ? 0.f : s * __expf(m - mn)) + (m2 == -FLT_MAX ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}

// Row stride `ld` (a multiple of 8) may exceed the vocabulary: columns
// [vocab, ld) are padding (e.g. GPT-2's 50257 stored as 50264) -- excluded
// from the softmax and given a zero gradient.
__global__ void __launch_bounds__(kCeThreads) ce_kernel(__nv_bfloat16* __restrict__ logits,
                                                        const int* __restrict__ tgt, float* __restrict__ loss_acc,
                                                        int vocab, int ld, float grad_scale) {
  ptx::pdl_wait();
  const int r = blockIdx.x;
  __nv_bfloat16* row = logits + static_cast<size_t>(r) * ld;
  const uint4* rv = reinterpret_cast<const uint4*>(row);
  const int nvec = ld / 8;
  float m = -FLT_MAX, s = 0.f;
  for (int v = threadIdx.x; v < nvec; v += kCeThreads) {
    float f[8];
    unpack8(rv[v], f);
    if (v * 8 + 8 > vocab) {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (v * 8 + e >= vocab) f[e] = -FLT_MAX;
    }
    float lm = f[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) lm = fmaxf(lm, f[e]);
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) ls += f[e] == -FLT_MAX ? 0.f : __expf(f[e] - lm);
    ms_merge(m, s, lm, ls);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    ms_merge(m, s, m2, s2);
  }
  __shared__ float pm[kCeThreads / 32], ps[kCeThreads / 32];
  __shared__ float row_m, row_inv_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    pm[warp] = m;
    ps[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < kCeThreads / 32 ? pm[lane] : -FLT_MAX;
    s = lane < kCeThreads / 32 ? ps[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
      ms_merge(m, s, m2, s2);
    }
    if (lane == 0) {
      row_m = m;
      row_inv_s = 1.f / s;
      const int t = tgt[r];
      atomicAdd(loss_acc, m + __logf(s) - __bfloat162float(row[t]));
    }
  }
  __syncthreads();
  const float mm = row_m, inv = row_inv_s;
  const int t = tgt[r];
  uint4* wv = reinterpret_cast<uint4*>(row);
  for (int v = threadIdx.x; v < nvec; v += kCeThreads) {
    float f[8];
    unpack8(wv[v], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float p = __expf(f[e] - mm) * inv;
      f[e] = v * 8 + e < vocab ? (p - (v * 8 + e == t ? 1.f : 0.f)) * grad_scale : 0.f;
    }
    wv[v] = pack8(f);
  }
}

}  // namespace

void fill_tokens(int* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, int vocab, cudaStream_t s) {
  if (vocab < 1) throw std::invalid_argument("fill_tokens: vocab must be >= 1");
  count_launch();
  TimedLaunch timed_("fill_tokens", s);
  launch_pdl(fill_tokens_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, dst, n, seed, tensor, idx0, vocab);
}

void embed_fwd(const int* tok, const void* wte, const void* wpe, void* x, int rows, int seq, int h, cudaStream_t s) {
  if (h % 8) throw std::invalid_argument("embed_fwd: hidden must be a multiple of 8");
  count_launch();
  TimedLaunch timed_("embed_fwd", s);
  launch_pdl(embed_fwd_kernel, dim3(grid_for(static_cast<long long>(rows) * h / 8, 256)), dim3(256), 0, s, tok,
             static_cast<const __nv_bfloat16*>(wte), static_cast<const __nv_bfloat16*>(wpe),
             static_cast<__nv_bfloat16*>(x), rows, seq, h);
}

void embed_bwd(const int* tok, const void* dx, float* gwte, float* gwpe, int rows, int seq, int h, cudaStream_t s) {
  if (h % 8) throw std::invalid_argument("embed_bwd: hidden must be a multiple of 8");
  count_launch();
  TimedLaunch timed_("embed_bwd", s);
  launch_pdl(embed_bwd_kernel, dim3(grid_for(static_cast<long long>(rows) * h / 8, 256)), dim3(256), 0, s, tok,
             static_cast<const __nv_bfloat16*>(dx), gwte, gwpe, rows, seq, h);
}

void cross_entropy_fwd_bwd(void* logits, const int* tgt, float* loss_acc, int rows, int vocab, float grad_scale,
                           cudaStream_t s, int ld) {
  if (ld == 0) ld = vocab;
  if (ld % 8 || vocab < 1 || vocab > ld)
    throw std::invalid_argument("cross_entropy: row stride must be a multiple of 8 and >= vocab");
  count_launch();
  TimedLaunch timed_("cross_entropy", s);
  launch_pdl(ce_kernel, dim3(rows), dim3(kCeThreads), 0, s, static_cast<__nv_bfloat16*>(logits), tgt, loss_acc, vocab,
             ld, grad_scale);
}

}  // namespace dpl
