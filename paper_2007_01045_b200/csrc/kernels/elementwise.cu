// HBM-bound stage kernels (N1/N2/N6): LayerNorm fwd/bwd, attention softmax
// fwd/bwd, bias-gradient column sums, MSE loss, SGD apply, and the seeded
// synthetic-data generator.  One warp per row, 16-byte vector accesses,
// warp-shuffle reductions; per-column gradient partials are reduced in
// shared memory and folded into fp32 gradient buffers with one atomic per
// column per block.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <cstdint>
#include <type_traits>

#include "elementwise.h"
#include "gemm.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace dpl {

namespace {

// Rows are processed one per warp with kMaxVec 8-element vectors per lane
// held in registers (kMaxVec in {1,2,4,8}: rows up to 2048 elements).
template <typename F>
void dispatch_vec(int len, F&& f) {
  const int v = (len / 8 + 31) / 32;
  if (v <= 1) f(std::integral_constant<int, 1>{});
  else if (v <= 2) f(std::integral_constant<int, 2>{});
  else if (v <= 4) f(std::integral_constant<int, 4>{});
  else f(std::integral_constant<int, 8>{});
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 r = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = __bfloat1622float2(h[e]);
    f[2 * e] = x.x;
    f[2 * e + 1] = x.y;
  }
}
__device__ __forceinline__ void load8(const float* p, float (&f)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 r;
  uint32_t* w = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    w[e] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = r;
}

// ------------------------------------------------------------ LayerNorm
__device__ __forceinline__ void unpack8(const uint4& r, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = __bfloat1622float2(h[e]);
    f[2 * e] = x.x;
    f[2 * e + 1] = x.y;
  }
}
__device__ __forceinline__ void lds8(const float* p, float (&f)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
__device__ __forceinline__ void ldg8(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// Packed fp32x2 helpers (FADD2 / FMUL2 / FFMA2: one FMA-pipe instruction per
// two values) and bf16x2 <-> fp32x2 conversions.  The LayerNorm kernels issue
// ~3x fewer instructions per element this way; at one row per warp they were
// issue-bound (ncu: 45% issue-active, 0.9 TB/s), not HBM-bound.
__device__ __forceinline__ float2 bf2f(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ uint32_t f2bf(float2 v) {
  __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 ff2(float a) { return make_float2(a, a); }

// One warp per row; the row stays in registers as packed bf16 (4 registers
// per 8 values), so the kernel fits 64 registers and keeps 32 warps per SM in
// flight.  gamma / beta (parameters, not written by the preceding kernel) are
// staged in shared memory before the programmatic-dependency wait, so their
// load overlaps the producer's tail instead of following the row load.
// Two-pass statistics (mean, then the centred sum of squares) as before, all
// math on fp32x2 pairs.
template <int kMaxVec>
__global__ void __launch_bounds__(256, 4)
    layernorm_fwd_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ gamma,
                         const float* __restrict__ beta, __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                         float* __restrict__ rstd_out, int rows, int h, float eps) {
  extern __shared__ float4 ln_par[];  // gamma [h], beta [h]
  float* sg = reinterpret_cast<float*>(ln_par);
  float* sb = sg + h;
  for (int i = threadIdx.x; i < h / 4; i += blockDim.x) {
    reinterpret_cast<float4*>(sg)[i] = __ldg(reinterpret_cast<const float4*>(gamma) + i);
    reinterpret_cast<float4*>(sb)[i] = __ldg(reinterpret_cast<const float4*>(beta) + i);
  }
  __syncthreads();
  ptx::pdl_wait();
  ptx::pdl_trigger();  // dependents (GEMMs) may start their prologue; they wait for our completion
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = h / 8;
  const float inv_h = 1.0f / h;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const __nv_bfloat16* xr = x + static_cast<long long>(row) * h;
    uint4 raw[kMaxVec];
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i)
      if (lane + 32 * i < nvec) raw[i] = *reinterpret_cast<const uint4*>(xr + (lane + 32 * i) * 8);
    float2 s2 = ff2(0.f);
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      if (lane + 32 * i < nvec) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&raw[i]);
#pragma unroll
        for (int e = 0; e < 4; ++e) s2 = __fadd2_rn(s2, bf2f(w[e]));
      }
    }
    const float mean = warp_sum(s2.x + s2.y) * inv_h;
    const float2 nm = ff2(-mean);
    float2 q2 = ff2(0.f);
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      if (lane + 32 * i < nvec) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&raw[i]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 d = __fadd2_rn(bf2f(w[e]), nm);
          q2 = __ffma2_rn(d, d, q2);
        }
      }
    }
    const float rstd = rsqrtf(warp_sum(q2.x + q2.y) * inv_h + eps);
    const float2 r2 = ff2(rstd);
    __nv_bfloat16* yr = y + static_cast<long long>(row) * h;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&raw[i]);
        const float4* g4 = reinterpret_cast<const float4*>(sg + vi * 8);
        const float4* b4 = reinterpret_cast<const float4*>(sb + vi * 8);
        const float4 ga = g4[0], gb = g4[1], ba = b4[0], bb = b4[1];
        const float2 g[4] = {make_float2(ga.x, ga.y), make_float2(ga.z, ga.w), make_float2(gb.x, gb.y),
                             make_float2(gb.z, gb.w)};
        const float2 b[4] = {make_float2(ba.x, ba.y), make_float2(ba.z, ba.w), make_float2(bb.x, bb.y),
                             make_float2(bb.z, bb.w)};
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          ow[e] = f2bf(__ffma2_rn(__fmul2_rn(__fadd2_rn(bf2f(w[e]), nm), r2), g[e], b[e]));
        *reinterpret_cast<uint4*>(yr + vi * 8) = o;
      }
    }
    if (lane == 0) {
      mean_out[row] = mean;
      rstd_out[row] = rstd;
    }
  }
}

// dx = rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat)) [+ dresid]
// Row kernel: one warp per row, pure streaming (no column reductions); x and
// dy stay packed in registers, xhat and g*dy are recomputed in pass 2 (fp32x2
// pairs throughout).
template <int kMaxVec>
__global__ void __launch_bounds__(256, kMaxVec > 4 ? 2 : 4)  // h > 1024 (GPT-2): registers for x, dy without spills
    layernorm_bwd_rows_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                              const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                              const float* __restrict__ gamma, const __nv_bfloat16* __restrict__ dresid,
                              __nv_bfloat16* __restrict__ dx, int rows, int h) {
  extern __shared__ float4 ln_par[];  // gamma [h] (staged before the dependency wait), then a bf16 row per warp
  float* sg = reinterpret_cast<float*>(ln_par);
  for (int i = threadIdx.x; i < h / 4; i += blockDim.x)
    reinterpret_cast<float4*>(sg)[i] = __ldg(reinterpret_cast<const float4*>(gamma) + i);
  __syncthreads();
  ptx::pdl_wait();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = h / 8;
  const float inv_h = 1.0f / h;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const long long base = static_cast<long long>(row) * h;
    const float mean = mean_in[row];
    const float rstd = rstd_in[row];
    uint4 rx[kMaxVec], rd[kMaxVec];
    // the residual gradient is fetched with x and dy -- asynchronously into
    // this warp's shared-memory row (cp.async: no registers held), so its
    // latency overlaps theirs instead of following the row reductions
    __nv_bfloat16* srow = reinterpret_cast<__nv_bfloat16*>(sg + h) + (threadIdx.x >> 5) * h;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        rx[i] = *reinterpret_cast<const uint4*>(x + base + vi * 8);
        rd[i] = *reinterpret_cast<const uint4*>(dy + base + vi * 8);
        if (dresid)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_addr(srow + vi * 8)),
                       "l"(dresid + base + vi * 8)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // xhat = x * rstd + (-mean * rstd)
    const float2 r2 = ff2(rstd), c2 = ff2(-mean * rstd);
    float2 s1 = ff2(0.f), s2 = ff2(0.f);
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        const uint32_t* wx = reinterpret_cast<const uint32_t*>(&rx[i]);
        const uint32_t* wd = reinterpret_cast<const uint32_t*>(&rd[i]);
        const float2* g = reinterpret_cast<const float2*>(sg + vi * 8);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 gd = __fmul2_rn(bf2f(wd[e]), g[e]);
          s1 = __fadd2_rn(s1, gd);
          s2 = __ffma2_rn(gd, __ffma2_rn(bf2f(wx[e]), r2, c2), s2);
        }
      }
    }
    const float m1 = warp_sum(s1.x + s1.y) * inv_h;
    const float m2 = warp_sum(s2.x + s2.y) * inv_h;
    const float2 nm1 = ff2(-m1), nm2 = ff2(-m2);
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // this thread's own residual chunks
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        const uint32_t* wx = reinterpret_cast<const uint32_t*>(&rx[i]);
        const uint32_t* wd = reinterpret_cast<const uint32_t*>(&rd[i]);
        const float2* g = reinterpret_cast<const float2*>(sg + vi * 8);
        uint4 rr = make_uint4(0u, 0u, 0u, 0u);
        if (dresid) rr = *reinterpret_cast<const uint4*>(srow + vi * 8);
        const uint32_t* wr = reinterpret_cast<const uint32_t*>(&rr);
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 xh = __ffma2_rn(bf2f(wx[e]), r2, c2);
          const float2 t = __fadd2_rn(__ffma2_rn(xh, nm2, __fmul2_rn(bf2f(wd[e]), g[e])), nm1);
          ow[e] = f2bf(__ffma2_rn(t, r2, bf2f(wr[e])));
        }
        *reinterpret_cast<uint4*>(dx + base + vi * 8) = o;
      }
    }
  }
}

// Fused LayerNorm backward: the dx rows AND the per-block column partials of
// dgamma = sum dy*xhat, dbeta = sum dy [, sum dresid [, sum dx]] in one pass
// over x / dy / dresid (the three-launch form re-read all of them, and dx, in
// a column kernel).  A row is spread over kTPR threads (one 8-column vector
// each, so every thread owns the same columns for the whole block and keeps
// their partials in registers); 512 / kTPR row groups per block take kR rows
// at a time, the row statistics meet in shared memory across the row group's
// warps (named barrier per group, double-buffered by iteration parity).  One
// block per SM; ws[block][k][h] partials are summed by ln_param_reduce_kernel
// in block order (deterministic).
constexpr int kLnFusedR = 4;
template <int kThreads, int kTPR, int kRed>
__global__ void __launch_bounds__(kThreads, 512 / kThreads)
    ln_bwd_fused_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                        const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                        const float* __restrict__ gamma, const __nv_bfloat16* __restrict__ dresid,
                        __nv_bfloat16* __restrict__ dx, float* __restrict__ ws, int rows, int h, int rows_per_block) {
  constexpr int kRG = kThreads / kTPR;
  constexpr int kWPR = kTPR / 32;
  constexpr int kR = kLnFusedR;
  extern __shared__ float4 ln_fused_smem[];
  float* sg = reinterpret_cast<float*>(ln_fused_smem);                 // gamma [h]
  float* red = sg + h;                                                  // [2][kRG][kWPR][kR][2]
  float* part = red + 2 * kRG * kWPR * kR * 2;                          // [kRG][kRed][h]
  __nv_bfloat16* sres = reinterpret_cast<__nv_bfloat16*>(part + kRG * kRed * h);  // [kRG][kR][h]
  for (int i = threadIdx.x; i < h / 4; i += blockDim.x)
    reinterpret_cast<float4*>(sg)[i] = __ldg(reinterpret_cast<const float4*>(gamma) + i);
  __syncthreads();
  ptx::pdl_wait();
  ptx::pdl_trigger();  // dependents (GEMMs) may start their prologue; they wait for our completion
  const int rg = threadIdx.x / kTPR;
  const int vi = threadIdx.x % kTPR;  // this thread's 8-column vector
  const int wr = vi >> 5, lane = threadIdx.x & 31;
  const int nvec = h / 8;
  const bool act = vi < nvec;
  const float inv_h = 1.0f / h;
  float2 g[4];
  if (act) {
    const float2* g2 = reinterpret_cast<const float2*>(sg + vi * 8);
#pragma unroll
    for (int e = 0; e < 4; ++e) g[e] = g2[e];
  }
  float2 acc[kRed][4];
#pragma unroll
  for (int k = 0; k < kRed; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[k][e] = ff2(0.f);
  __nv_bfloat16* my_res = sres + rg * kR * h;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  int par = 0;
  for (int rb = r0 + rg * kR; rb - rg * kR < r1; rb += kRG * kR, par ^= 1) {
    // every row group runs the same number of iterations (named barriers)
    uint4 rx[kR], rd[kR];
    float mean[kR], rstd[kR];
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int r = rb + j;
      mean[j] = 0.f;
      rstd[j] = 0.f;
      if (r < r1) {
        mean[j] = mean_in[r];
        rstd[j] = rstd_in[r];
        if (act) {
          const long long off = static_cast<long long>(r) * h + vi * 8;
          rx[j] = *reinterpret_cast<const uint4*>(x + off);
          rd[j] = *reinterpret_cast<const uint4*>(dy + off);
          if (dresid)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_addr(my_res + j * h + vi * 8)),
                         "l"(dresid + off)
                         : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    float st[kR][2];
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      float2 s1 = ff2(0.f), s2 = ff2(0.f);
      if (rb + j < r1 && act) {
        const float2 r2 = ff2(rstd[j]), c2 = ff2(-mean[j] * rstd[j]);
        const uint32_t* wx = reinterpret_cast<const uint32_t*>(&rx[j]);
        const uint32_t* wd = reinterpret_cast<const uint32_t*>(&rd[j]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 gd = __fmul2_rn(bf2f(wd[e]), g[e]);
          s1 = __fadd2_rn(s1, gd);
          s2 = __ffma2_rn(gd, __ffma2_rn(bf2f(wx[e]), r2, c2), s2);
        }
      }
      st[j][0] = warp_sum(s1.x + s1.y);
      st[j][1] = warp_sum(s2.x + s2.y);
    }
    if constexpr (kWPR > 1) {
      float* rr = red + ((par * kRG + rg) * kWPR) * kR * 2;
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < kR; ++j) {
          rr[(wr * kR + j) * 2] = st[j][0];
          rr[(wr * kR + j) * 2 + 1] = st[j][1];
        }
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + rg), "r"(kTPR) : "memory");
#pragma unroll
      for (int j = 0; j < kR; ++j) {
        float a = 0.f, b = 0.f;
#pragma unroll
        for (int w = 0; w < kWPR; ++w) {
          a += rr[(w * kR + j) * 2];
          b += rr[(w * kR + j) * 2 + 1];
        }
        st[j][0] = a;
        st[j][1] = b;
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // this thread's own residual chunks
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      if (rb + j < r1 && act) {
        const float2 r2 = ff2(rstd[j]), c2 = ff2(-mean[j] * rstd[j]);
        const float2 nm1 = ff2(-st[j][0] * inv_h), nm2 = ff2(-st[j][1] * inv_h);
        const uint32_t* wx = reinterpret_cast<const uint32_t*>(&rx[j]);
        const uint32_t* wd = reinterpret_cast<const uint32_t*>(&rd[j]);
        uint4 rr4 = make_uint4(0u, 0u, 0u, 0u);
        if (dresid) rr4 = *reinterpret_cast<const uint4*>(my_res + j * h + vi * 8);
        const uint32_t* wres = reinterpret_cast<const uint32_t*>(&rr4);
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 dv = bf2f(wd[e]);
          const float2 xh = __ffma2_rn(bf2f(wx[e]), r2, c2);
          const float2 t = __fadd2_rn(__ffma2_rn(xh, nm2, __fmul2_rn(dv, g[e])), nm1);
          const float2 rv = bf2f(wres[e]);
          ow[e] = f2bf(__ffma2_rn(t, r2, rv));
          acc[0][e] = __ffma2_rn(dv, xh, acc[0][e]);
          acc[1][e] = __fadd2_rn(acc[1][e], dv);
          if constexpr (kRed > 2) acc[2][e] = __fadd2_rn(acc[2][e], rv);
          if constexpr (kRed > 3) acc[3][e] = __fadd2_rn(acc[3][e], bf2f(ow[e]));  // the stored (bf16) dx
        }
        *reinterpret_cast<uint4*>(dx + static_cast<long long>(rb + j) * h + vi * 8) = o;
      }
    }
  }
  // row groups meet in shared memory; one ws row per reduction per block
  if (act) {
#pragma unroll
    for (int k = 0; k < kRed; ++k) {
      float4* d = reinterpret_cast<float4*>(part + (rg * kRed + k) * h + vi * 8);
      d[0] = make_float4(acc[k][0].x, acc[k][0].y, acc[k][1].x, acc[k][1].y);
      d[1] = make_float4(acc[k][2].x, acc[k][2].y, acc[k][3].x, acc[k][3].y);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kRed * h; i += blockDim.x) {
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < kRG; ++q) sum += part[q * kRed * h + i];
    ws[static_cast<long long>(blockIdx.x) * kRed * h + i] = sum;
  }
}

// Column reductions over a slab of 64 rows (block = 32 column vectors x 8
// row phases):
//   0: sum dy*xhat (dgamma)  1: sum dy (dbeta)  2: sum dresid  3: sum dx
// -> ws[blockIdx.y][nred][h]; ln_param_reduce_kernel sums the slabs.
template <int kRed>
__global__ void __launch_bounds__(256, 4)
    ln_bwd_cols_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                       const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                       const __nv_bfloat16* __restrict__ dresid, const __nv_bfloat16* __restrict__ dx,
                       float* __restrict__ ws, int rows, int h) {
  ptx::pdl_wait();
  ptx::pdl_trigger();  // dependents (GEMMs) may start their prologue; they wait for our completion
  __shared__ float part[8][kRed][257];
  const int vx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int vi = blockIdx.x * 32 + vx;
  const int nvec = h / 8;
  const int r0 = blockIdx.y * 64;
  float2 acc[kRed][4];
#pragma unroll
  for (int k = 0; k < kRed; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[k][e] = ff2(0.f);
  if (vi < nvec) {
#pragma unroll 4
    for (int t = 0; t < 8; ++t) {
      const int r = r0 + ry + 8 * t;
      if (r < rows) {
        const long long off = static_cast<long long>(r) * h + vi * 8;
        const uint4 rx = *reinterpret_cast<const uint4*>(x + off);
        const uint4 rd = *reinterpret_cast<const uint4*>(dy + off);
        uint4 ra, rb;
        if constexpr (kRed > 2) ra = *reinterpret_cast<const uint4*>(dresid + off);
        if constexpr (kRed > 3) rb = *reinterpret_cast<const uint4*>(dx + off);
        const float rstd = rstd_in[r];
        const float2 r2 = ff2(rstd), c2 = ff2(-mean_in[r] * rstd);
        const uint32_t* wx = reinterpret_cast<const uint32_t*>(&rx);
        const uint32_t* wd = reinterpret_cast<const uint32_t*>(&rd);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 dv = bf2f(wd[e]);
          acc[0][e] = __ffma2_rn(dv, __ffma2_rn(bf2f(wx[e]), r2, c2), acc[0][e]);
          acc[1][e] = __fadd2_rn(acc[1][e], dv);
        }
        if constexpr (kRed > 2) {
          const uint32_t* wa = reinterpret_cast<const uint32_t*>(&ra);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[2][e] = __fadd2_rn(acc[2][e], bf2f(wa[e]));
        }
        if constexpr (kRed > 3) {
          const uint32_t* wb = reinterpret_cast<const uint32_t*>(&rb);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[3][e] = __fadd2_rn(acc[3][e], bf2f(wb[e]));
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kRed; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      part[ry][k][vx * 8 + 2 * e] = acc[k][e].x;
      part[ry][k][vx * 8 + 2 * e + 1] = acc[k][e].y;
    }
  __syncthreads();
  const int c = threadIdx.x;  // 256 columns
  const int col = blockIdx.x * 256 + c;
  if (col < h) {
#pragma unroll
    for (int k = 0; k < kRed; ++k) {
      float sum = 0.f;
#pragma unroll
      for (int y = 0; y < 8; ++y) sum += part[y][k][c];
      ws[(static_cast<long long>(blockIdx.y) * kRed + k) * h + col] = sum;
    }
  }
}

// dst_k[c] += sum_b ws[b][k][c] for each of the nred column reductions.
// Block: 32 columns x 16 slab groups; each thread sums every 16th slab with
// eight loads in flight at a time (the partials are L2-resident: the sum is
// latency-bound, so the loads must overlap), then the 16 groups meet in smem.
__global__ void __launch_bounds__(512) ln_param_reduce_kernel(const float* __restrict__ ws, float* d0, float* d1,
                                                              float* d2, float* d3, int blocks, int nred, int h) {
  ptx::pdl_wait();
  ptx::pdl_trigger();  // dependents (GEMMs) may start their prologue; they wait for our completion
  __shared__ float part[16][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + tx;  // (k, c) flattened
  const long long stride = static_cast<long long>(nred) * h;
  float s = 0.f;
  if (i < nred * h) {
    for (int b0 = ty; b0 < blocks; b0 += 16 * 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + 16 * u;
        v[u] = b < blocks ? ws[b * stride + i] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
  }
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && i < nred * h) {
#pragma unroll
    for (int y = 1; y < 16; ++y) s += part[y][tx];
    const int k = i / h, c = i % h;
    float* d = k == 0 ? d0 : k == 1 ? d1 : k == 2 ? d2 : d3;
    d[c] += s;
  }
}

// ------------------------------------------------------------ softmax
// S fp32 [rows][L] (already scaled), P bf16.  Causal: row r is query
// (r % q_len) and keys k > q are masked.
template <int kMaxVec>
__global__ void softmax_fwd_kernel(const float* __restrict__ s, __nv_bfloat16* __restrict__ p, int rows, int len,
                                   int q_len, int causal) {
  ptx::pdl_wait();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = len / 8;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const float* sr = s + static_cast<long long>(row) * len;
    const int q = row % q_len;
    float v[kMaxVec][8];
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        load8(sr + vi * 8, v[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (causal && vi * 8 + e > q) v[i][e] = -INFINITY;
          mx = fmaxf(mx, v[i][e]);
        }
      }
    }
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      if (lane + 32 * i < nvec) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          v[i][e] = __expf(v[i][e] - mx);
          sum += v[i][e];
        }
      }
    }
    const float inv = 1.f / warp_sum(sum);
    __nv_bfloat16* pr = p + static_cast<long long>(row) * len;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = v[i][e] * inv;
        store8(pr + vi * 8, o);
      }
    }
  }
}

// dS = P * (dP - sum(P * dP))   (P bf16, dP fp32 -> dS bf16)
template <int kMaxVec>
__global__ void softmax_bwd_kernel(const __nv_bfloat16* __restrict__ p, const float* __restrict__ dp,
                                   __nv_bfloat16* __restrict__ ds, int rows, int len) {
  ptx::pdl_wait();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = len / 8;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const long long base = static_cast<long long>(row) * len;
    float pv[kMaxVec][8], gv[kMaxVec][8];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        load8(p + base + vi * 8, pv[i]);
        load8(dp + base + vi * 8, gv[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) dot += pv[i][e] * gv[i][e];
      }
    }
    dot = warp_sum(dot);
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nvec) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = pv[i][e] * (gv[i][e] - dot);
        store8(ds + base + vi * 8, o);
      }
    }
  }
}

// ------------------------------------------------------------ bias grads
// db[c] += sum_r dy[r][c].  Block = 32 column-vectors (256 columns) x 8 row
// phases; a warp reads 512 contiguous bytes of a row; the 8 row phases are
// reduced in shared memory, then one atomic per column per block.
__global__ void __launch_bounds__(256, 4) colsum_acc_kernel(const __nv_bfloat16* __restrict__ dy, float* __restrict__ db, int rows, int cols,
                                  int rows_per_block) {
  ptx::pdl_wait();
  ptx::pdl_trigger();  // dependents (GEMMs) may start their prologue; they wait for our completion
  __shared__ float part[8][256 + 1];
  const int vx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int vi = blockIdx.x * 32 + vx;
  const int nvec = cols / 8;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (vi < nvec) {
    for (int r = r0 + ry; r < r1; r += 32) {
      uint4 f[4];
#pragma unroll
      for (int t = 0; t < 4; ++t)  // 4 independent loads in flight
        if (r + 8 * t < r1) f[t] = *reinterpret_cast<const uint4*>(dy + static_cast<long long>(r + 8 * t) * cols + vi * 8);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (r + 8 * t < r1) {
          float v[8];
          unpack8(f[t], v);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += v[e];
        }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[ry][vx * 8 + e] = acc[e];
  __syncthreads();
  const int c = threadIdx.x;  // 256 threads, one column each
  const int col = blockIdx.x * 256 + c;
  if (col < cols) {
    float s = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) s += part[y][c];
    atomicAdd(db + col, s);
  }
}

// ------------------------------------------------------------ split-K epilogue
// The same GELU derivative as the GEMM epilogue (gemm_tcgen05.cu dgelu_f:
// tanh form, tanh on the SFU), so a split GEMM rounds like an unsplit one.
__device__ __forceinline__ float split_dgelu(float x) {
  constexpr float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(k0 * fmaf(k1 * x, x2, x)));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * k0 * fmaf(3.0f * k1, x2, 1.0f);
}

template <bool kBiasT, bool kResidT, bool kDGeluT>
__global__ void __launch_bounds__(256) split_epilogue_kernel(float* __restrict__ acc, __nv_bfloat16* __restrict__ c,
                                                             long long ldc, int m, int n, float alpha,
                                                             const float* __restrict__ bias,
                                                             const __nv_bfloat16* __restrict__ resid,
                                                             const __nv_bfloat16* __restrict__ aux_in) {
  ptx::pdl_wait();
  ptx::pdl_trigger();  // dependents (GEMMs) may start their prologue; they wait for our completion
  const int nv = n / 8;
  const long long total = static_cast<long long>(m) * nv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / nv), col = static_cast<int>(i % nv) * 8;
    float* a = acc + static_cast<long long>(row) * n + col;
    float v[8];
    load8(a, v);
    *reinterpret_cast<float4*>(a) = make_float4(0.f, 0.f, 0.f, 0.f);  // scratch left zero
    *reinterpret_cast<float4*>(a + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    const long long off = static_cast<long long>(row) * ldc + col;
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] *= alpha;
    if (kBiasT) {
      float b[8];
      ldg8(bias + col, b);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] += b[e];
    }
    if (kResidT) {
      float r[8];
      load8(resid + off, r);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] += r[e];
    }
    if (kDGeluT) {
      float z[8];
      load8(aux_in + off, z);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] *= split_dgelu(z[e]);
    }
    store8(c + off, v);
  }
}

// ------------------------------------------------------------ loss
// loss_acc += sum (y - t)^2 ; dy = (y - t) * grad_scale  (grad_scale = 2/numel)
__global__ void mse_kernel(const __nv_bfloat16* __restrict__ y, const __nv_bfloat16* __restrict__ t,
                           __nv_bfloat16* __restrict__ dy, float* __restrict__ loss_acc, long long n,
                           float grad_scale) {
  ptx::pdl_wait();
  float local = 0.f;
  const long long nvec = n / 8;
  for (long long vi = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; vi < nvec;
       vi += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8], b[8], o[8];
    load8(y + vi * 8, a);
    load8(t + vi * 8, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float d = a[e] - b[e];
      local += d * d;
      o[e] = d * grad_scale;
    }
    store8(dy + vi * 8, o);
  }
  local = warp_sum(local);
  __shared__ float part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) atomicAdd(loss_acc, v);
  }
}

// ------------------------------------------------------------ optimizer
// w32 -= lr * g ; w16 = bf16(w32) ; g = 0   (fp32 master weights)
__global__ void sgd_kernel(float* __restrict__ w32, float* __restrict__ g, __nv_bfloat16* __restrict__ w16,
                           long long n, float lr) {
  ptx::pdl_wait();
  const long long nvec = n / 4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nvec;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 w = reinterpret_cast<float4*>(w32)[i];
    const float4 gg = reinterpret_cast<float4*>(g)[i];
    w.x -= lr * gg.x;
    w.y -= lr * gg.y;
    w.z -= lr * gg.z;
    w.w -= lr * gg.w;
    reinterpret_cast<float4*>(w32)[i] = w;
    reinterpret_cast<float4*>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (w16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(w.x, w.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(w.z, w.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(w16)[i] = pk;
    }
  }
  // scalar tail
  for (long long i = nvec * 4 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    w32[i] -= lr * g[i];
    g[i] = 0.f;
    if (w16) w16[i] = __float2bfloat16_rn(w32[i]);
  }
}

// ------------------------------------------------------------ synthetic data
__device__ __forceinline__ float hash_uniform(uint64_t seed, uint64_t tensor, uint64_t idx) {
  uint64_t z = seed + tensor * 0xD1B54A32D192ED03ull + idx * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D649BB133111EBull;
  z ^= z >> 31;
  return static_cast<float>(z >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
}

// dst[r][c] = scale * U(-1,1) keyed by (seed, tensor, (row0 + r) * cols + c)
__global__ void fill_uniform_bf16_kernel(__nv_bfloat16* dst, long long n, uint64_t seed, uint64_t tensor,
                                         long long idx0, float scale) {
  ptx::pdl_wait();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = __float2bfloat16_rn(scale * hash_uniform(seed, tensor, static_cast<uint64_t>(idx0 + i)));
}
__global__ void fill_uniform_f32_kernel(float* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0,
                                        float scale) {
  ptx::pdl_wait();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = scale * hash_uniform(seed, tensor, static_cast<uint64_t>(idx0 + i));
}
__global__ void fill_const_f32_kernel(float* dst, long long n, float v) {
  ptx::pdl_wait();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = v;
}
__global__ void cast_f32_bf16_kernel(const float* src, __nv_bfloat16* dst, long long n) {
  ptx::pdl_wait();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

int grid_for(long long work, int threads) {
  long long g = (work + threads - 1) / threads;
  const long long cap = 148LL * 16;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

void layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y, float* mean, float* rstd, int rows,
                   int h, float eps, cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("layernorm_fwd", s);
  const int warps = 8;
  const int grid = std::max(1, std::min((rows + warps - 1) / warps, 148 * 8));
  dispatch_vec(h, [&](auto v) {
    launch_pdl(layernorm_fwd_kernel<decltype(v)::value>, dim3(grid), dim3(warps * 32), 2 * h * sizeof(float), s, 
        static_cast<const __nv_bfloat16*>(x), gamma, beta, static_cast<__nv_bfloat16*>(y), mean, rstd, rows, h, eps);
  });
}

void layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gamma,
                   const void* dresid, void* dx, float* dgamma, float* dbeta, int rows, int h, cudaStream_t s,
                   float* ws, float* dresid_colsum, float* dx_colsum) {
  TimedLaunch timed_("layernorm_bwd", s);
  if (!ws) throw std::invalid_argument("layernorm_bwd: workspace required");
  if (dx_colsum && !dresid_colsum) throw std::invalid_argument("layernorm_bwd: dx_colsum needs dresid_colsum");
  if (dresid_colsum && !dresid) throw std::invalid_argument("layernorm_bwd: dresid_colsum needs dresid");
  const auto* pdy = static_cast<const __nv_bfloat16*>(dy);
  const auto* px = static_cast<const __nv_bfloat16*>(x);
  const auto* pr = static_cast<const __nv_bfloat16*>(dresid);
  auto* pdx = static_cast<__nv_bfloat16*>(dx);
  const int nred = dx_colsum ? 4 : (dresid_colsum ? 3 : 2);
  static const bool fused = [] {
    const char* e = std::getenv("DPL_LN_BWD_FUSED");
    return !(e && e[0] == '0');
  }();
  if (fused && h <= 2048) {
    count_launch(2);
    // blocks per SM (A/B knob): 1 x 512 threads (default; 13.1 vs 13.5 us at 4096 x 1024) or 2 x 256
    static const int bps = [] {
      const char* e = std::getenv("DPL_LN_FUSED_BPS");
      return e && e[0] == '2' ? 2 : 1;
    }();
    const int threads = 512 / bps;
    const int nvec = h / 8;
    const int tpr = std::min(threads, nvec <= 32 ? 32 : nvec <= 64 ? 64 : nvec <= 128 ? 128 : 256);
    const int rg = threads / tpr;
    const int grid = std::max(1, std::min(148 * bps, (rows + rg * kLnFusedR - 1) / (rg * kLnFusedR)));
    const int rpb = (rows + grid - 1) / grid;
    const size_t smem = h * sizeof(float) + 2 * (threads / 32) * kLnFusedR * 2 * sizeof(float) +
                        static_cast<size_t>(rg) * nred * h * sizeof(float) +
                        (pr ? static_cast<size_t>(rg) * kLnFusedR * h * sizeof(__nv_bfloat16) : 0);
    auto go = [&](auto thr_c, auto tpr_c, auto red_c) {
      constexpr int N = decltype(thr_c)::value, T = decltype(tpr_c)::value, R = decltype(red_c)::value;
      if constexpr (T <= N) {
        static std::once_flag once;  // one per instantiation
        std::call_once(once, [] {
          cudaFuncSetAttribute(ln_bwd_fused_kernel<N, T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
        });
        launch_pdl(ln_bwd_fused_kernel<N, T, R>, dim3(grid), dim3(N), smem, s, pdy, px, mean, rstd, gamma, pr, pdx, ws,
                   rows, h, rpb);
      }
    };
    auto by_red = [&](auto thr_c, auto tpr_c) {
      if (nred == 2) go(thr_c, tpr_c, std::integral_constant<int, 2>{});
      else if (nred == 3) go(thr_c, tpr_c, std::integral_constant<int, 3>{});
      else go(thr_c, tpr_c, std::integral_constant<int, 4>{});
    };
    auto by_tpr = [&](auto thr_c) {
      if (tpr == 32) by_red(thr_c, std::integral_constant<int, 32>{});
      else if (tpr == 64) by_red(thr_c, std::integral_constant<int, 64>{});
      else if (tpr == 128) by_red(thr_c, std::integral_constant<int, 128>{});
      else by_red(thr_c, std::integral_constant<int, 256>{});
    };
    if (threads == 512) by_tpr(std::integral_constant<int, 512>{});
    else by_tpr(std::integral_constant<int, 256>{});
    launch_pdl(ln_param_reduce_kernel, dim3((nred * h + 31) / 32), dim3(512), 0, s, ws, dgamma, dbeta, dresid_colsum,
               dx_colsum, grid, nred, h);
    return;
  }
  count_launch(3);
  const int warps = 8;
  const int grid = std::max(1, std::min((rows + warps - 1) / warps, 148 * 8));
  dispatch_vec(h, [&](auto v) {
    launch_pdl(layernorm_bwd_rows_kernel<decltype(v)::value>, dim3(grid), dim3(warps * 32),
               h * sizeof(float) + (pr ? warps * h * sizeof(__nv_bfloat16) : 0), s, pdy, px, mean, rstd, gamma, pr, pdx,
                                                                              rows, h);
  });
  const int slabs = (rows + 63) / 64;
  if (static_cast<long long>(slabs) * nred * h > static_cast<long long>(kLnBwdBlocks) * 4 * h)
    throw std::invalid_argument("layernorm_bwd: too many rows for the workspace");
  const dim3 cg((h / 8 + 31) / 32, slabs);
  if (nred == 2) launch_pdl(ln_bwd_cols_kernel<2>, dim3(cg), dim3(256), 0, s, pdy, px, mean, rstd, pr, pdx, ws, rows, h);
  else if (nred == 3) launch_pdl(ln_bwd_cols_kernel<3>, dim3(cg), dim3(256), 0, s, pdy, px, mean, rstd, pr, pdx, ws, rows, h);
  else launch_pdl(ln_bwd_cols_kernel<4>, dim3(cg), dim3(256), 0, s, pdy, px, mean, rstd, pr, pdx, ws, rows, h);
  launch_pdl(ln_param_reduce_kernel, dim3((nred * h + 31) / 32), dim3(512), 0, s, ws, dgamma, dbeta, dresid_colsum,
             dx_colsum, slabs, nred, h);
}

void softmax_fwd(const float* s, void* p, int rows, int len, int q_len, int causal, cudaStream_t st) {
  count_launch();
  TimedLaunch timed_("softmax_fwd", st);
  const int warps = 8;
  const int grid = std::max(1, std::min((rows + warps - 1) / warps, 148 * 16));
  dispatch_vec(len, [&](auto v) {
    launch_pdl(softmax_fwd_kernel<decltype(v)::value>, dim3(grid), dim3(warps * 32), 0, st, s, static_cast<__nv_bfloat16*>(p), rows, len,
                                                                        q_len, causal);
  });
}

void softmax_bwd(const void* p, const float* dp, void* ds, int rows, int len, cudaStream_t st) {
  count_launch();
  TimedLaunch timed_("softmax_bwd", st);
  const int warps = 8;
  const int grid = std::max(1, std::min((rows + warps - 1) / warps, 148 * 16));
  dispatch_vec(len, [&](auto v) {
    launch_pdl(softmax_bwd_kernel<decltype(v)::value>, dim3(grid), dim3(warps * 32), 0, st, static_cast<const __nv_bfloat16*>(p), dp,
                                                                        static_cast<__nv_bfloat16*>(ds), rows, len);
  });
}

void colsum_acc(const void* dy, float* db, int rows, int cols, cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("colsum_acc", s);
  const int gx = (cols + 255) / 256;
  // about four blocks per SM (the occupancy the kernel's launch bounds
  // allow: 32 warps x 64 bytes in flight per lane), at least 64 rows per block
  int gy = std::max(1, std::min((rows + 63) / 64, (148 * 4 + gx - 1) / gx));
  const int rpb = (rows + gy - 1) / gy;
  gy = (rows + rpb - 1) / rpb;
  launch_pdl(colsum_acc_kernel, dim3(gx, gy), dim3(256), 0, s, static_cast<const __nv_bfloat16*>(dy), db, rows, cols, rpb);
}

void split_epilogue(float* acc, void* c, long long ldc, int m, int n, float alpha, const float* bias,
                    const void* resid, const void* aux_in, uint32_t epi, cudaStream_t s) {
  constexpr uint32_t kB = 1u << 2, kR = 1u << 8, kDG = 1u << 6;  // gemm.h kBias / kResid / kDGelu
  if (n % 8 || ldc % 8) throw std::invalid_argument("split_epilogue: N and ldc must be multiples of 8");
  if (epi & ~(kB | kR | kDG)) throw std::invalid_argument("split_epilogue: unsupported epilogue flags");
  count_launch();
  TimedLaunch timed_("gemm_split_epilogue", s);
  const int grid = grid_for(static_cast<long long>(m) * n / 8, 256);
  auto* pc = static_cast<__nv_bfloat16*>(c);
  const auto* pr = static_cast<const __nv_bfloat16*>(resid);
  const auto* pa = static_cast<const __nv_bfloat16*>(aux_in);
  auto go = [&](auto kernel) { launch_pdl(kernel, dim3(grid), dim3(256), 0, s, acc, pc, ldc, m, n, alpha, bias, pr, pa); };
  const bool b = epi & kB, r = epi & kR, dg = epi & kDG;
  if (!b && !r && !dg) go(split_epilogue_kernel<false, false, false>);
  else if (b && !r && !dg) go(split_epilogue_kernel<true, false, false>);
  else if (b && r && !dg) go(split_epilogue_kernel<true, true, false>);
  else if (!b && r && !dg) go(split_epilogue_kernel<false, true, false>);
  else if (!b && !r && dg) go(split_epilogue_kernel<false, false, true>);
  else if (b && !r && dg) go(split_epilogue_kernel<true, false, true>);
  else if (!b && r && dg) go(split_epilogue_kernel<false, true, true>);
  else go(split_epilogue_kernel<true, true, true>);
}

void mse_loss(const void* y, const void* t, void* dy, float* loss_acc, long long n, float grad_scale, cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("mse_loss", s);
  launch_pdl(mse_kernel, dim3(grid_for(n / 8, 256)), dim3(256), 0, s, static_cast<const __nv_bfloat16*>(y),
                                                   static_cast<const __nv_bfloat16*>(t),
                                                   static_cast<__nv_bfloat16*>(dy), loss_acc, n, grad_scale);
}

void sgd_apply(float* w32, float* g, void* w16, long long n, float lr, cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("sgd_apply", s);
  launch_pdl(sgd_kernel, dim3(grid_for(n / 4, 256)), dim3(256), 0, s, w32, g, static_cast<__nv_bfloat16*>(w16), n, lr);
}

void fill_uniform_bf16(void* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                       cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("fill_uniform", s);
  launch_pdl(fill_uniform_bf16_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, static_cast<__nv_bfloat16*>(dst), n, seed, tensor, idx0,
                                                            scale);
}

void fill_uniform_f32(float* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                      cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("fill_uniform", s);
  launch_pdl(fill_uniform_f32_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, dst, n, seed, tensor, idx0, scale);
}

void fill_const_f32(float* dst, long long n, float v, cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("fill_const", s);
  launch_pdl(fill_const_f32_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, dst, n, v);
}

void cast_f32_bf16(const float* src, void* dst, long long n, cudaStream_t s) {
  count_launch();
  TimedLaunch timed_("cast_f32_bf16", s);
  launch_pdl(cast_f32_bf16_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, src, static_cast<__nv_bfloat16*>(dst), n);
}

}  // namespace dpl
