// Persistent warp-specialised bf16 GEMM for sm_100a (stage kernels N1/N2).
//
//   warp 0      TMA producer: A/B tiles -> smem ring (SWIZZLE_128B)
//   warp 1      MMA issuer: tcgen05.mma (M=128, N=BN, K=16) into TMEM
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-11  epilogue: tcgen05.ld -> bias / residual / activation /
//               activation-derivative / fp32 gradient accumulation -> global
//               (two warps per TMEM lane quadrant, alternating 32-column
//               chunks, TMEM loads double buffered)
//
// The accumulator is double buffered in TMEM so the epilogue of tile i
// overlaps the MMAs of tile i+1.  Operands may be K-major or MN-major (the
// backward GEMMs dX = dY W and dW += dY^T X read transposed operands straight
// from their forward layouts; no transpose kernels).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>

#include "elementwise.h"
#include "gemm.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace dpl {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kSmemBudget = 227 * 1024;  // dynamic smem of every GEMM CTA
constexpr int kMaxStages = 8;
constexpr int kMaxNx = 4;  // TMA epilogue extra-tensor buffers per warp
constexpr int kEpiBars = kMaxNx + 1;  // per epilogue warp: x buffers + bias slice

// smem: [1 KB align slack][stages x stage][epilogue carve-out][1 KB barriers];
// the split between ring depth and epilogue staging is per GEMM (host)
template <int BN>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int kSmem = kSmemBudget;
};

// GELU, tanh form (as GPT-2 / BERT implementations use):
//   gelu(x) = 0.5 x (1 + tanh(k0 (x + k1 x^3)))
// tanh via the SFU (tanh.approx.f32, one MUFU op).
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kGeluK0 = 0.7978845608028654f;  // sqrt(2/pi)
constexpr float kGeluK1 = 0.044715f;
__device__ __forceinline__ float gelu_f(float x) {
  const float t = tanh_fast(kGeluK0 * fmaf(kGeluK1 * x, x * x, x));
  return 0.5f * x * (1.0f + t);
}
__device__ __forceinline__ float dgelu_f(float x) {
  const float x2 = x * x;
  const float t = tanh_fast(kGeluK0 * fmaf(kGeluK1 * x, x2, x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * kGeluK0 * fmaf(3.0f * kGeluK1, x2, 1.0f);
}
// the same two functions on packed fp32x2 operands (FMUL2 / FFMA2 / FADD2:
// half the FMA-pipe instructions of the TMA epilogue's activation math)
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 gelu2(float2 x) {
  const float2 c = __ffma2_rn(__fmul2_rn(f2(kGeluK1), x), __fmul2_rn(x, x), x);
  const float2 g = __fmul2_rn(f2(kGeluK0), c);
  const float2 t = make_float2(tanh_fast(g.x), tanh_fast(g.y));
  return __fmul2_rn(__fmul2_rn(f2(0.5f), x), __fadd2_rn(f2(1.0f), t));
}
__device__ __forceinline__ float2 dgelu2(float2 x) {
  const float2 x2 = __fmul2_rn(x, x);
  const float2 g = __fmul2_rn(f2(kGeluK0), __ffma2_rn(__fmul2_rn(f2(kGeluK1), x), x2, x));
  const float2 t = make_float2(tanh_fast(g.x), tanh_fast(g.y));
  const float2 one_m_tt = __ffma2_rn(make_float2(-t.x, -t.y), t, f2(1.0f));
  const float2 a = __fmul2_rn(__fmul2_rn(__fmul2_rn(f2(0.5f), x), one_m_tt), f2(kGeluK0));
  return __ffma2_rn(a, __ffma2_rn(f2(3.0f * kGeluK1), x2, f2(1.0f)), __fmul2_rn(f2(0.5f), __fadd2_rn(f2(1.0f), t)));
}

// Implicit-GEMM convolution: load the im2col tile whose first pixel (output
// position, row-major n, h, w) is `pixel` and whose 64 channels start at
// K / N index `kidx` (= tap * C + c0, C % 64 == 0) into dst.
template <bool kPair>
__device__ __forceinline__ void conv_tile_load(const GemmParams& p, const CUtensorMap* map, void* dst, uint64_t* bar,
                                               int pixel, int kidx) {
  const int tap = kidx / p.conv_c, c0 = kidx % p.conv_c;
  const int hw = p.conv_h * p.conv_w;
  const int n = pixel / hw, rem = pixel % hw;
  const int ho = rem / p.conv_w, wo = rem % p.conv_w;
  const uint16_t kh = static_cast<uint16_t>(tap / 3), kw = static_cast<uint16_t>(tap % 3);
  if (kPair) ptx::tma_load_im2col_4d_2sm(dst, map, bar, c0, wo - 1, ho - 1, n, kw, kh);
  else ptx::tma_load_im2col_4d(dst, map, bar, c0, wo - 1, ho - 1, n, kw, kh);
}

// diagnostics: phase timestamps per CTA (GemmDesc::trace)
__device__ __forceinline__ void trace_mark(const GemmParams& p, int slot) {
  if (p.trace) {
    p.trace[blockIdx.x * 16 + slot] = clock64();  // SM cycles (compare within one CTA)
  }
}

__device__ __forceinline__ long long out_offset(const GemmParams& p, int z, int m, int n) {
  return static_cast<long long>(z / p.zdiv) * p.s_zo + static_cast<long long>(z % p.zdiv) * p.s_zi +
         static_cast<long long>(m) * p.ldc + static_cast<long long>(n / p.ndiv) * p.s_no + (n % p.ndiv);
}

// Global operands of one thread's 32-column epilogue chunk (bias, residual,
// activation input), loaded one chunk ahead so their latency overlaps the
// previous chunk's math.
// One prefetched bf16 operand: the residual if kResid, else the activation
// input of kDGelu / kDRelu (a GEMM that needs both loads aux_in directly).
struct EpiExtras {
  uint4 v[4];
};

__device__ __forceinline__ const __nv_bfloat16* prefetched_tensor(const GemmParams& p) {
  if (p.epi & kResid) return p.resid;
  if (p.epi & (kDGelu | kDRelu)) return p.aux_in;
  return nullptr;
}

__device__ __forceinline__ void epilogue_prefetch(const GemmParams& p, int z, int row, int n0, EpiExtras& x) {
  const __nv_bfloat16* src = prefetched_tensor(p);
  if (!src || row >= p.M || n0 >= p.N || !p.vec_ok || p.N - n0 < 32) return;
  const uint4* s4 = reinterpret_cast<const uint4*>(src + out_offset(p, z, row, n0));
#pragma unroll
  for (int q = 0; q < 4; ++q) x.v[q] = s4[q];
}

__device__ __forceinline__ void unpack_bf16x8(const uint4& r, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 v = __bfloat1622float2(h[e]);
    f[2 * e] = v.x;
    f[2 * e + 1] = v.y;
  }
}

// Apply the epilogue to one thread's 32 consecutive columns of one row.
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int z, int row, int n0, const uint32_t (&raw)[32],
                                               const EpiExtras& x) {
  if (row >= p.M || n0 >= p.N) return;
  const long long off = out_offset(p, z, row, n0);
  const int ncols = min(32, p.N - n0);
  const bool full = (ncols == 32) && p.vec_ok;
  const uint32_t epi = p.epi;

  float v[32];
  if (p.alpha != 1.0f) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]) * p.alpha;
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
  }

  if (epi & kBias) {
    if (full) {
      const float4* b4 = reinterpret_cast<const float4*>(p.bias + n0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = __ldg(b4 + q);
        v[4 * q] += b.x;
        v[4 * q + 1] += b.y;
        v[4 * q + 2] += b.z;
        v[4 * q + 3] += b.w;
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < ncols) v[j] += p.bias[n0 + j];
    }
  }
  if (epi & kResid) {
    if (full) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float f[8];
        unpack_bf16x8(x.v[q], f);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[8 * q + e] += f[e];
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < ncols) v[j] += __bfloat162float(p.resid[off + j]);
    }
  }
  if (epi & (kDGelu | kDRelu)) {
    const bool gelu = (epi & kDGelu) != 0;
    if (full) {
      const uint4* a4 = reinterpret_cast<const uint4*>(p.aux_in + off);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float zq[8];
        unpack_bf16x8((epi & kResid) ? a4[q] : x.v[q], zq);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[8 * q + e] *= gelu ? dgelu_f(zq[e]) : (zq[e] > 0.f ? 1.f : 0.f);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float zj = j < ncols ? __bfloat162float(p.aux_in[off + j]) : 0.f;
        v[j] *= gelu ? dgelu_f(zj) : (zj > 0.f ? 1.f : 0.f);
      }
    }
  }
  if (epi & kAuxOut) {
    if (full) {
      uint4* o4 = reinterpret_cast<uint4*>(p.aux_out + off);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
          wp[e] = *reinterpret_cast<uint32_t*>(&h);
        }
        o4[q] = w;
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < ncols) p.aux_out[off + j] = __float2bfloat16_rn(v[j]);
    }
  }
  if (epi & kGelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
  } else if (epi & kRelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }

  const uint32_t kind = epi & kOutMask;
  if (kind == kOutBf16) {
    __nv_bfloat16* c = static_cast<__nv_bfloat16*>(p.C) + off;
    if (full) {
      uint4* c4 = reinterpret_cast<uint4*>(c);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
          wp[e] = *reinterpret_cast<uint32_t*>(&h);
        }
        c4[q] = w;
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < ncols) c[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* c = static_cast<float*>(p.C) + off;
    const bool acc = kind == kOutF32Acc;
    if (acc && p.k_splits > 1) {
      // split-K partial sums meet in the fp32 accumulator
      if (full) {
        float4* c4 = reinterpret_cast<float4*>(c);
#pragma unroll
        for (int q = 0; q < 8; ++q) atomicAdd(c4 + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < ncols) atomicAdd(c + j, v[j]);
      }
    } else if (full) {
      float4* c4 = reinterpret_cast<float4*>(c);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 w = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (acc) {
          const float4 o = c4[q];
          w.x += o.x;
          w.y += o.y;
          w.z += o.z;
          w.w += o.w;
        }
        c4[q] = w;
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < ncols) c[j] = acc ? c[j] + v[j] : v[j];
    }
  }
}

// ---------------------------------------------------------------- TMA epilogue
// Per epilogue warp a smem region (p.epi_warp_bytes) holding two 32-row x
// 32-column output chunk buffers (chunk g is staged while chunk g-1's bulk
// store drains) and p.epi_nx chunk buffers of the extra tensor: the
// residual / activation input (bulk-loaded as soon as the warp starts the
// tile, so its DRAM latency hides under the mainloop) or the aux output
// (bulk-stored with the output).
//   bf16 chunk: 32 rows x 64 B, 64B-swizzled:  unit q of row r at r*64  + ((q ^ (r>>1 & 3)) << 4)
//   fp32 chunk: 32 rows x 128 B, 128B-swizzled: unit q of row r at r*128 + ((q ^ (r & 7)) << 4)
// so a warp's row-per-lane 16-byte accesses are bank-conflict free.  TMEM
// loads are double buffered: chunk j+1 streams out of TMEM while chunk j is
// processed.
constexpr int kXBytes = 32 * 32 * 2;

struct EpiTma {
  uint8_t* region;  // this warp's region
  uint64_t* xbar;   // this warp's input barriers (one per x buffer, then the bias slice's)
  uint32_t seq;     // chunks processed by this warp
  uint32_t xph;     // input barrier phase bits (bit kMaxNx: bias)
};

__device__ __forceinline__ bool epi_has_x_in(const GemmParams& p) { return (p.epi & (kResid | kDGelu | kDRelu)) != 0; }

__device__ __forceinline__ void epi_coords(const GemmParams& p, int z, int m, int n, int (&c)[5]) {
  c[0] = n % p.c_inner;
  c[1] = m;
  c[2] = n / p.c_inner;
  c[3] = z % p.zdiv;
  c[4] = z / p.zdiv;
}

__device__ __forceinline__ uint8_t* epi_xbuf(const GemmParams& p, const EpiTma& e, int b) {
  return e.region + 2 * p.epi_out_bytes + b * kXBytes;
}
// bias slice of the current tile: after the output and x buffers
__device__ __forceinline__ float* epi_bias(const GemmParams& p, const EpiTma& e) {
  return reinterpret_cast<float*>(e.region + p.epi_warp_bytes - p.epi_tile_cols * 4);
}

// whole warp (one elected lane issues): bulk-load the extra input of the
// chunk at (row0, n0) into x buffer b
__device__ __forceinline__ void epi_issue_x(const GemmParams& p, EpiTma& e, int b, int z, int row0, int n0) {
  int c[5];
  epi_coords(p, z, row0, n0, c);
  ptx::tma_load_5d_e(epi_xbuf(p, e, b), &p.tma_x, &e.xbar[b], kXBytes, c[0], c[1], c[2], c[3], c[4]);
}

// Before the tile's accumulator is ready: prefetch up to epi_nx input chunks
// of this warp (chunk j covers columns col0 + (half + 2 j) * 32).
template <int kPerWarp>
__device__ __forceinline__ void epi_tile_prefetch(const GemmParams& p, EpiTma& e, int z, int row0, int col0, int half) {
  const uint32_t lane = ptx::lane_id();
  const bool bias = (p.epi & kBias) != 0;
  if (!epi_has_x_in(p) && !bias) return;
  // the previous tile's generic reads of these buffers precede the new bulk loads
  ptx::fence_proxy_async_smem();
  __syncwarp();
  if (bias) {
    const int cols = min(p.epi_tile_cols, p.N - col0);
    const uint32_t bytes = static_cast<uint32_t>((cols * 4 + 15) & ~15);
    ptx::bulk_load_e(epi_bias(p, e), p.bias + col0, bytes, &e.xbar[kMaxNx]);
  }
  if (!epi_has_x_in(p)) return;
#pragma unroll
  for (int j = 0; j < kPerWarp; ++j) {
    const int n0 = col0 + (half + 2 * j) * 32;
    if (j < p.epi_nx && n0 < p.N) epi_issue_x(p, e, (e.seq + j) % p.epi_nx, z, row0, n0);
  }
}

#define EPI_MARK(J, K) \
  if (threadIdx.x == 128 && e.seq < 2 && (J) < 2) trace_mark(p, 8 + (J) * 4 + (K))

template <int kPerWarp>
__device__ __forceinline__ void epi_tile_tma(const GemmParams& p, EpiTma& e, uint32_t tbase, int z, int row0, int col0,
                                             int half) {
  const uint32_t lane = ptx::lane_id();
  const uint32_t epi = p.epi;
  const bool x_in = epi_has_x_in(p);
  const uint32_t kind = epi & kOutMask;
  const bool f32 = kind != kOutBf16;
  if (epi & kBias) {
    ptx::mbar_wait(&e.xbar[kMaxNx], (e.xph >> kMaxNx) & 1);
    e.xph ^= 1u << kMaxNx;
  }
  const float* bias_s = epi_bias(p, e) - col0;  // indexed by global column
#pragma unroll 1
  for (int j = 0; j < kPerWarp; ++j) {
    const int c = half + 2 * j;
    const int n0 = col0 + c * 32;
    uint32_t raw[32];
    ptx::tmem_ld_32x32b_x32(tbase + c * 32, raw);
    ptx::tmem_wait_ld();
    EPI_MARK(j, 0);
    if (n0 >= p.N) {  // chunk entirely right of the matrix (no load was issued for it)
      ++e.seq;
      continue;
    }
    const int ob = e.seq & 1;
    const int xb = e.seq % p.epi_nx;
    float v[32];
    {
      const float2 al = make_float2(p.alpha, p.alpha);
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        const float2 r = __fmul2_rn(make_float2(__uint_as_float(raw[k]), __uint_as_float(raw[k + 1])), al);
        v[k] = r.x;
        v[k + 1] = r.y;
      }
    }
    if (epi & kBias) {  // smem broadcast reads (columns past N hold junk; they are clipped on store)
      const float4* b4 = reinterpret_cast<const float4*>(bias_s + n0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 bb = b4[q];
        const float2 lo = __fadd2_rn(make_float2(v[4 * q], v[4 * q + 1]), make_float2(bb.x, bb.y));
        const float2 hi = __fadd2_rn(make_float2(v[4 * q + 2], v[4 * q + 3]), make_float2(bb.z, bb.w));
        v[4 * q] = lo.x;
        v[4 * q + 1] = lo.y;
        v[4 * q + 2] = hi.x;
        v[4 * q + 3] = hi.y;
      }
    }
    uint8_t* xbuf = epi_xbuf(p, e, xb);
    if (x_in) {
      EPI_MARK(j, 2);
      ptx::mbar_wait(&e.xbar[xb], (e.xph >> xb) & 1);
      e.xph ^= 1u << xb;
      EPI_MARK(j, 3);
      float xv[32];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 r = *reinterpret_cast<const uint4*>(xbuf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4));
        unpack_bf16x8(r, xv + 8 * q);
      }
      // buffers are refilled only when a warp has more chunks than buffers
      if (j + p.epi_nx < kPerWarp) {
        ptx::fence_proxy_async_smem();
        __syncwarp();
        const int n2 = col0 + (c + 2 * p.epi_nx) * 32;
        if (n2 < p.N) epi_issue_x(p, e, xb, z, row0, n2);
      }
      if (epi & kResid) {
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const float2 r = __fadd2_rn(make_float2(v[k], v[k + 1]), make_float2(xv[k], xv[k + 1]));
          v[k] = r.x;
          v[k + 1] = r.y;
        }
      } else if (epi & kDGelu) {
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const float2 r = __fmul2_rn(make_float2(v[k], v[k + 1]), dgelu2(make_float2(xv[k], xv[k + 1])));
          v[k] = r.x;
          v[k + 1] = r.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] *= xv[k] > 0.f ? 1.f : 0.f;
      }
    }
    EPI_MARK(j, 1);
    // output buffer ob (and the aux buffer) were last read by the bulk store two chunks ago
    ptx::bulk_wait_read<1>();
    __syncwarp();
    if (epi & kAuxOut) {
      uint8_t* abuf = epi_xbuf(p, e, ob);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q + 2 * k], v[8 * q + 2 * k + 1]);
          wp[k] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(abuf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = w;
      }
    }
    if (epi & kGelu) {
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        const float2 r = gelu2(make_float2(v[k], v[k + 1]));
        v[k] = r.x;
        v[k + 1] = r.y;
      }
    } else if (epi & kRelu) {
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = fmaxf(v[k], 0.f);
    }
    uint8_t* obuf = e.region + ob * p.epi_out_bytes;
    if (f32) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(obuf + lane * 128 + ((q ^ (lane & 7)) << 4)) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q + 2 * k], v[8 * q + 2 * k + 1]);
          wp[k] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(obuf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = w;
      }
    }
    if (epi & kColSum) {
      // column sums of the staged (bf16) chunk: lane j sums column j over the valid rows
      __syncwarp();
      if (!f32) {
        float cs = 0.f;
        const int q = lane >> 3, e = lane & 7;
        const int rows = min(32, p.M - row0);
        for (int r = 0; r < rows; ++r)
          cs += __bfloat162float(
              *reinterpret_cast<const __nv_bfloat16*>(obuf + r * 64 + ((q ^ ((r >> 1) & 3)) << 4) + e * 2));
        if (n0 + static_cast<int>(lane) < p.N) atomicAdd(p.colsum + n0 + lane, cs);
      }
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    {
      int cc[5];
      epi_coords(p, z, row0, n0, cc);
      ptx::tma_store_chunk_e(&p.tma_c, obuf, kind == kOutF32Acc, &p.tma_x,
                             (epi & kAuxOut) ? epi_xbuf(p, e, ob) : nullptr, cc);
    }
    ++e.seq;
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) gemm_bf16_tcgen05(const __grid_constant__ GemmParams p) {
  if (threadIdx.x == 0) trace_mark(p, 0);
  using C = Cfg<BN>;
  const int S = p.stages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * C::kABytes;
  uint8_t* smem_epi = smem + S * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + kEpiWarps * p.epi_warp_bytes);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* xbar = tmem_empty + 2;  // kMaxNx per epilogue warp (TMA epilogue inputs)
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(xbar + kEpiBars * kEpiWarps);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&p.tma_a);
    ptx::tma_prefetch_desc(&p.tma_b);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      ptx::mbar_init(&tmem_empty[a], 32 * kEpiWarps);
    }
    for (int i = 0; i < kEpiBars * kEpiWarps; ++i) ptx::mbar_init(&xbar[i], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_base_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  // prologue done: wait for the producer kernel's writes, let the next kernel launch
  ptx::pdl_wait();
  ptx::pdl_trigger();
  if (threadIdx.x == 0) trace_mark(p, 1);

  const int tiles_per_z = p.num_m_blocks * p.num_n_blocks;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int first_tile = blockIdx.x;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const int ks = t % p.k_splits;
        const int tt = t / p.k_splits;
        const int z = tt / tiles_per_z;
        const int r = tt % tiles_per_z;
        const int mb = r % p.num_m_blocks;
        const int nb = r / p.num_m_blocks;
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(p.num_k_blocks, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          uint8_t* sa = smem_a + stage * C::kABytes;
          uint8_t* sb = smem_b + stage * C::kBBytes;
          if (p.conv_operand == 1) {
            conv_tile_load<false>(p, &p.tma_a, sa, &full[stage], mb * kBM, kb * kBK);
          } else if (!p.a_mn_major) {
            ptx::tma_load_3d(sa, &p.tma_a, &full[stage], kb * kBK, mb * kBM, z);
          } else {
#pragma unroll
            for (int j = 0; j < kBM / 64; ++j)
              ptx::tma_load_3d(sa + j * 64 * kBK * 2, &p.tma_a, &full[stage], mb * kBM + j * 64, kb * kBK, z);
          }
          if (p.conv_operand == 2) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              conv_tile_load<false>(p, &p.tma_b, sb + j * 64 * kBK * 2, &full[stage], kb * kBK, nb * BN + j * 64);
          } else if (!p.b_mn_major) {
            ptx::tma_load_3d(sb, &p.tma_b, &full[stage], kb * kBK, nb * BN, z);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              ptx::tma_load_3d(sb + j * 64 * kBK * 2, &p.tma_b, &full[stage], nb * BN + j * 64, kb * kBK, z);
          }
          if (t == first_tile && kb == kb0) trace_mark(p, 2);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (the whole warp runs the loop; one elected lane issues each MMA)
    {
      const uint32_t idesc = ptx::idesc_bf16_f32(kBM, BN, p.a_mn_major != 0, p.b_mn_major != 0);
      // K-major: 8-row groups 1024 B apart, advance 32 B per K=16 step.
      // MN-major: 64-wide MN chunks 8 KB apart (LBO), 8-row K groups 1 KB
      // apart (SBO), advance 16 rows = 2 KB per K=16 step.
      const uint32_t a_lbo = p.a_mn_major ? 64 * kBK * 2 : 16;
      const uint32_t b_lbo = p.b_mn_major ? 64 * kBK * 2 : 16;
      const uint32_t a_step = p.a_mn_major ? 16 * 128 : 32;
      const uint32_t b_step = p.b_mn_major ? 16 * 128 : 32;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const int ks = t % p.k_splits;
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(p.num_k_blocks, kb0 + p.kb_per_split);
        ptx::mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (lane == 0 && t == static_cast<int>(blockIdx.x) && kb == kb0) trace_mark(p, 3);
          const uint32_t sa = ptx::smem_addr(smem_a + stage * C::kABytes);
          const uint32_t sb = ptx::smem_addr(smem_b + stage * C::kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = ptx::smem_desc_sw128(sa + k * a_step, a_lbo, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(sb + k * b_step, b_lbo, 1024);
            ptx::mma_bf16_e(tmem_d, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          ptx::mma_commit_e(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit_e(&tmem_full[acc]);
        if (lane == 0) trace_mark(p, 4);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4 && p.tma_epi) {
    // ------------------------------------------------------------ TMA epilogue
    const uint32_t quad = warp & 3;
    const int half = (warp - 4) >> 2;
    EpiTma e{smem_epi + (warp - 4) * p.epi_warp_bytes, xbar + kEpiBars * (warp - 4), 0, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      const int tt = t / p.k_splits;
      const int z = tt / tiles_per_z;
      const int r = tt % tiles_per_z;
      const int mb = r % p.num_m_blocks;
      const int nb = r / p.num_m_blocks;
      const int row0 = mb * kBM + quad * 32;
      epi_tile_prefetch<BN / 64>(p, e, z, row0, nb * BN, half);
      ptx::mbar_wait(&tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
      if (warp == 4 && ptx::lane_id() == 0 && t == static_cast<int>(blockIdx.x)) trace_mark(p, 5);
      epi_tile_tma<BN / 64>(p, e, tmem_base + ((quad * 32) << 16) + acc * BN, z, row0, nb * BN, half);
      ptx::tc_fence_before();
      if (warp == 4 && ptx::lane_id() == 0) trace_mark(p, 6);
      ptx::mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    ptx::bulk_wait<0>();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t quad = warp & 3;          // TMEM lane quadrant this warp may access
    const int half = (warp - 4) >> 2;        // which alternating column chunks
    constexpr int kChunks = BN / 32;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      const int tt = t / p.k_splits;
      const int z = tt / tiles_per_z;
      const int r = tt % tiles_per_z;
      const int mb = r % p.num_m_blocks;
      const int nb = r / p.num_m_blocks;
      ptx::mbar_wait(&tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
      if (warp == 4 && lane == 0 && t == static_cast<int>(blockIdx.x)) trace_mark(p, 5);
      const int row = mb * kBM + quad * 32 + lane;
      const uint32_t tbase = tmem_base + ((quad * 32) << 16) + acc * BN;
      if (half < kChunks) {
        // two register buffers, statically indexed: load chunk c+2 while
        // chunk c is processed
        uint32_t ra[32], rb[32];
        EpiExtras xa, xb;
        epilogue_prefetch(p, z, row, nb * BN + half * 32, xa);
        ptx::tmem_ld_32x32b_x32(tbase + half * 32, ra);
        ptx::tmem_wait_ld();
#pragma unroll 1
        for (int c = half; c < kChunks; c += 4) {
          const bool more = c + 2 < kChunks;
          if (more) {
            epilogue_prefetch(p, z, row, nb * BN + (c + 2) * 32, xb);
            ptx::tmem_ld_32x32b_x32(tbase + (c + 2) * 32, rb);
          }
          epilogue_chunk(p, z, row, nb * BN + c * 32, ra, xa);
          ptx::tmem_wait_ld();
          if (!more) break;
          if (c + 4 < kChunks) {
            epilogue_prefetch(p, z, row, nb * BN + (c + 4) * 32, xa);
            ptx::tmem_ld_32x32b_x32(tbase + (c + 4) * 32, ra);
          }
          epilogue_chunk(p, z, row, nb * BN + (c + 2) * 32, rb, xb);
          ptx::tmem_wait_ld();
        }
      }
      ptx::tc_fence_before();
      if (warp == 4 && lane == 0) trace_mark(p, 6);
      ptx::mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 0) trace_mark(p, 7);
}


// ---------------------------------------------------------------- CTA pair
// cta_group::2 variant: a cluster of two CTAs on one TPC computes a 256 x 256
// tile.  Each CTA stages its own 128 rows of A and its own 128-column half of
// B (32 KB per stage instead of 48 KB for the same MMA work per SM); the
// leader CTA issues M=256 MMAs that read both CTAs' smem and write each CTA's
// 128 accumulator rows into its own TMEM.  Both CTAs' TMA bytes land on the
// leader's full barrier; the leader's commits multicast to both CTAs' empty /
// tmem_full barriers; both CTAs' epilogue warps release the leader's
// tmem_empty barrier.
// Pair tile 256 x BN2 (BN2 = 256, or 128 for short-M / narrow shapes: half
// the B bytes per stage, so a deeper ring covers the TMA latency).
template <int BN2>
struct PairCfg {
  static constexpr int kBN = BN2;
  static constexpr int kABytes = kBM * kBK * 2;        // 16 KB: this CTA's 128 rows of A
  static constexpr int kBBytes = (kBN / 2) * kBK * 2;  // this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = kBN == 192 ? 512 : 2 * kBN;  // double-buffered accumulator (power of two)
};
namespace pair {
constexpr int kSmem = kSmemBudget;
}  // namespace pair

// Work units of the pair kernel: tiles [0, num_tiles - split_tail) whole,
// then each of the last split_tail tiles as two 256 x BN2/2 halves (hh 0 / 1),
// so a last wave that would leave most pairs idle finishes in half the time.
struct PairUnit {
  int t, hh;  // tile, half (-1: whole tile)
};
__device__ __forceinline__ PairUnit pair_unit(const GemmParams& p, int u) {
  const int whole = p.num_tiles - p.split_tail;
  if (u < whole) return {u, -1};
  return {whole + ((u - whole) >> 1), (u - whole) & 1};
}

template <int BN2>
__global__ void __launch_bounds__(kThreads, 1) gemm_bf16_tcgen05_2sm(const __grid_constant__ GemmParams p) {
  if (threadIdx.x == 0) trace_mark(p, 0);
  using Pc = PairCfg<BN2>;
  constexpr int kBN = Pc::kBN, kABytes = Pc::kABytes, kBBytes = Pc::kBBytes, kStageBytes = Pc::kStageBytes;
  const int S = p.stages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * kABytes;
  uint8_t* smem_epi = smem + S * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_epi + kEpiWarps * p.epi_warp_bytes);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* xbar = tmem_empty + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(xbar + kEpiBars * kEpiWarps);

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&p.tma_a);
    ptx::tma_prefetch_desc(&p.tma_b);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 2);   // leader's expect_tx + the peer's remote arrive
      ptx::mbar_init(&empty[s], 1);  // one multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      ptx::mbar_init(&tmem_empty[a], 2 * kEpiWarps);  // one arrive per epilogue warp of both CTAs
    }
    for (int i = 0; i < kEpiBars * kEpiWarps; ++i) ptx::mbar_init(&xbar[i], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm<Pc::kTmemCols>(tmem_base_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  ptx::pdl_wait();
  ptx::pdl_trigger();
  if (threadIdx.x == 0) trace_mark(p, 1);
  const int tiles_per_z = p.num_m_blocks * p.num_n_blocks;
  const int n_units = p.num_tiles + p.split_tail;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int first_tile = pair_id;
      for (int u = pair_id; u < n_units; u += n_pairs) {
        const PairUnit un = pair_unit(p, u);
        const int t = un.t;
        const int ks = t % p.k_splits;
        const int tt = t / p.k_splits;
        const int z = tt / tiles_per_z;
        const int r = tt % tiles_per_z;
        const int mb = r % p.num_m_blocks;
        const int nb = r / p.num_m_blocks;
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(p.num_k_blocks, kb0 + p.kb_per_split);
        const int m0 = mb * 256 + rank * 128;
        // a half unit loads the same boxes from its half's start (the second
        // 64 rows of each CTA's B box are not read by the N = BN2/2 MMA)
        const int n0 = nb * kBN + (un.hh < 0 ? rank * (kBN / 2) : un.hh * (kBN / 2) + rank * (kBN / 4));
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
          else ptx::mbar_arrive_cluster(&full[stage], 0);
          uint8_t* sa = smem_a + stage * kABytes;
          uint8_t* sb = smem_b + stage * kBBytes;
          if (p.conv_operand == 1) {
            conv_tile_load<true>(p, &p.tma_a, sa, &full[stage], m0, kb * kBK);
          } else if (!p.a_mn_major) {
            ptx::tma_load_3d_2sm(sa, &p.tma_a, &full[stage], kb * kBK, m0, z);
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j) ptx::tma_load_3d_2sm(sa + j * 64 * kBK * 2, &p.tma_a, &full[stage], m0 + j * 64, kb * kBK, z);
          }
          if (p.conv_operand == 2) {
#pragma unroll
            for (int j = 0; j < kBN / 128; ++j)
              conv_tile_load<true>(p, &p.tma_b, sb + j * 64 * kBK * 2, &full[stage], kb * kBK, n0 + j * 64);
          } else if (!p.b_mn_major) {
            ptx::tma_load_3d_2sm(sb, &p.tma_b, &full[stage], kb * kBK, n0, z);
          } else {
#pragma unroll
            for (int j = 0; j < kBN / 128; ++j)
              ptx::tma_load_3d_2sm(sb + j * 64 * kBK * 2, &p.tma_b, &full[stage], n0 + j * 64, kb * kBK, z);
          }
          if (u == first_tile && kb == kb0) trace_mark(p, 2);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // the whole warp runs the loop; one elected lane issues each MMA
      const uint32_t idesc_whole = ptx::idesc_bf16_f32(256, kBN, p.a_mn_major != 0, p.b_mn_major != 0);
      const uint32_t idesc_half = ptx::idesc_bf16_f32(256, kBN / 2, p.a_mn_major != 0, p.b_mn_major != 0);
      const uint32_t a_lbo = p.a_mn_major ? 64 * kBK * 2 : 16;
      const uint32_t b_lbo = p.b_mn_major ? 64 * kBK * 2 : 16;
      const uint32_t a_step = p.a_mn_major ? 16 * 128 : 32;
      const uint32_t b_step = p.b_mn_major ? 16 * 128 : 32;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair_id; u < n_units; u += n_pairs) {
        const PairUnit un = pair_unit(p, u);
        const uint32_t idesc = un.hh < 0 ? idesc_whole : idesc_half;
        const int ks = un.t % p.k_splits;
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(p.num_k_blocks, kb0 + p.kb_per_split);
        ptx::mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * kBN;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (lane == 0 && u == pair_id && kb == kb0) trace_mark(p, 3);
          const uint32_t sa = ptx::smem_addr(smem_a + stage * kABytes);
          const uint32_t sb = ptx::smem_addr(smem_b + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = ptx::smem_desc_sw128(sa + k * a_step, a_lbo, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(sb + k * b_step, b_lbo, 1024);
            ptx::mma_bf16_2sm_e(tmem_d, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          ptx::mma_commit_2sm_e(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit_2sm_e(&tmem_full[acc]);
        if (lane == 0) trace_mark(p, 4);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4 && p.tma_epi) {
    const uint32_t quad = warp & 3;
    const int half = (warp - 4) >> 2;
    EpiTma e{smem_epi + (warp - 4) * p.epi_warp_bytes, xbar + kEpiBars * (warp - 4), 0, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair_id; u < n_units; u += n_pairs) {
      const PairUnit un = pair_unit(p, u);
      const int tt = un.t / p.k_splits;
      const int z = tt / tiles_per_z;
      const int r = tt % tiles_per_z;
      const int mb = r % p.num_m_blocks;
      const int nb = r / p.num_m_blocks;
      const int row0 = mb * 256 + rank * 128 + quad * 32;
      const uint32_t taddr = tmem_base + ((quad * 32) << 16) + acc * kBN;
      if (un.hh < 0) {
        epi_tile_prefetch<kBN / 64>(p, e, z, row0, nb * kBN, half);
        ptx::mbar_wait(&tmem_full[acc], acc_phase);
        ptx::tc_fence_after();
        if (warp == 4 && lane == 0 && u == pair_id) trace_mark(p, 5);
        epi_tile_tma<kBN / 64>(p, e, taddr, z, row0, nb * kBN, half);
      } else if constexpr (kBN == 256) {
        const int col0 = nb * kBN + un.hh * (kBN / 2);
        epi_tile_prefetch<kBN / 128>(p, e, z, row0, col0, half);
        ptx::mbar_wait(&tmem_full[acc], acc_phase);
        ptx::tc_fence_after();
        epi_tile_tma<kBN / 128>(p, e, taddr, z, row0, col0, half);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (warp == 4 && lane == 0) trace_mark(p, 6);
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&tmem_empty[acc]);
        else ptx::mbar_arrive_cluster(&tmem_empty[acc], 0);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    ptx::bulk_wait<0>();
  } else if (warp >= 4) {
    const uint32_t quad = warp & 3;
    const int half = (warp - 4) >> 2;
    constexpr int kChunks = kBN / 32;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair_id; u < n_units; u += n_pairs) {  // whole tiles only (split_tail needs the TMA epilogue)
      const int t = pair_unit(p, u).t;
      const int tt = t / p.k_splits;
      const int z = tt / tiles_per_z;
      const int r = tt % tiles_per_z;
      const int mb = r % p.num_m_blocks;
      const int nb = r / p.num_m_blocks;
      ptx::mbar_wait(&tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
      if (warp == 4 && lane == 0 && t == pair_id) trace_mark(p, 5);
      const int row = mb * 256 + rank * 128 + quad * 32 + lane;
      const uint32_t tbase = tmem_base + ((quad * 32) << 16) + acc * kBN;
      uint32_t ra[32], rb[32];
      EpiExtras xa, xb;
      epilogue_prefetch(p, z, row, nb * kBN + half * 32, xa);
      ptx::tmem_ld_32x32b_x32(tbase + half * 32, ra);
      ptx::tmem_wait_ld();
#pragma unroll 1
      for (int c = half; c < kChunks; c += 4) {
        const bool more = c + 2 < kChunks;
        if (more) {
          epilogue_prefetch(p, z, row, nb * kBN + (c + 2) * 32, xb);
          ptx::tmem_ld_32x32b_x32(tbase + (c + 2) * 32, rb);
        }
        epilogue_chunk(p, z, row, nb * kBN + c * 32, ra, xa);
        ptx::tmem_wait_ld();
        if (!more) break;
        if (c + 4 < kChunks) {
          epilogue_prefetch(p, z, row, nb * kBN + (c + 4) * 32, xa);
          ptx::tmem_ld_32x32b_x32(tbase + (c + 4) * 32, ra);
        }
        epilogue_chunk(p, z, row, nb * kBN + (c + 2) * 32, rb, xb);
        ptx::tmem_wait_ld();
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (warp == 4 && lane == 0) trace_mark(p, 6);
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&tmem_empty[acc]);
        else ptx::mbar_arrive_cluster(&tmem_empty[acc], 0);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync_relaxed();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<Pc::kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 0) trace_mark(p, 7);
}

// ---------------------------------------------------------------- host side

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !ptr) {
      throw std::runtime_error("dpl: cuTensorMapEncodeTiled unavailable");
    }
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 3-D bf16 tensor map over [batch][outer][inner] with a (64 x box_outer)
// SWIZZLE_128B box.
CUtensorMap make_map(const void* base, long long inner, long long outer, long long ld, int batch,
                     long long batch_stride, int box_outer) {
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) throw std::invalid_argument("dpl gemm: operand not 16B aligned");
  if ((ld * 2) % 16 != 0) throw std::invalid_argument("dpl gemm: leading dimension must be a multiple of 8");
  if (batch > 1 && (batch_stride * 2) % 16 != 0) throw std::invalid_argument("dpl gemm: batch stride alignment");
  CUtensorMap map;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer),
                        static_cast<cuuint64_t>(batch)};
  const long long bs = batch > 1 ? batch_stride : ld * outer;
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 2), static_cast<cuuint64_t>(bs * 2)};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_outer), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult rc = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw std::runtime_error("dpl gemm: cuTensorMapEncodeTiled failed (" + std::to_string(rc) + ")");
  return map;
}

// 5-D map over the epilogue addressing of C (gemm.h):
//   [n % inner][m][n / inner][z % zdiv][z / zdiv], box 32 columns x 32 rows.
// Size-1 dimensions get a consistent non-zero stride.
CUtensorMap make_epi_map(const void* base, bool f32, const GemmDesc& d, int inner, int nhi) {
  const long long esz = f32 ? 4 : 2;
  const long long zhi = d.batch / d.zdiv;
  const long long s1 = d.ldc;
  const long long s2 = nhi > 1 ? d.s_no : s1 * d.M;
  const long long s3 = d.zdiv > 1 ? d.s_zi : s2 * nhi;
  const long long s4 = zhi > 1 ? d.s_zo : s3 * d.zdiv;
  CUtensorMap map;
  cuuint64_t dims[5] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(d.M), static_cast<cuuint64_t>(nhi),
                        static_cast<cuuint64_t>(d.zdiv), static_cast<cuuint64_t>(zhi)};
  cuuint64_t strides[4] = {static_cast<cuuint64_t>(s1 * esz), static_cast<cuuint64_t>(s2 * esz),
                           static_cast<cuuint64_t>(s3 * esz), static_cast<cuuint64_t>(s4 * esz)};
  cuuint32_t box[5] = {32, 32, 1, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult rc = encode_fn()(&map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw std::runtime_error("dpl gemm: epilogue tensor map failed (" + std::to_string(rc) + ")");
  return map;
}

// im2col map over NHWC x [n][h][w][c]: a 3x3 pad-1 filter origin per output
// pixel (pixel box corners {-1, -1}), 64 channels x `pixels` pixels per load,
// SWIZZLE_128B (the same smem image as a [pixels x 64] K-major / MN-major tile)
CUtensorMap make_im2col_map(const void* x, int n, int h, int w, int c, int pixels) {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !ptr)
      throw std::runtime_error("dpl: cuTensorMapEncodeIm2col unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(ptr);
  }();
  if (reinterpret_cast<uintptr_t>(x) % 16) throw std::invalid_argument("dpl gemm: conv input not 16B aligned");
  CUtensorMap map;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h),
                        static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2, static_cast<cuuint64_t>(w) * c * 2,
                           static_cast<cuuint64_t>(h) * w * c * 2};
  int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult rc = fn(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower, upper,
                         64, static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw std::runtime_error("dpl gemm: im2col tensor map failed (" + std::to_string(rc) + ")");
  return map;
}

template <int BN>
void configure_kernel() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(gemm_bf16_tcgen05<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::kSmem);
  });
}

int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Split-K for a bf16-output GEMM that leaves most CTA pairs idle (e.g. the
// N = 1024 / 1600 GEMMs of 1024- and 2048-row replica slices: 16-32 pair
// tiles for 74 pairs): the fp32 reduce-add GEMM (the wgrad path, split-K
// built in) accumulates into the cache's zeroed scratch, then
// split_epilogue applies bias / residual / act' and writes bf16.
static bool split_bf16_candidate(const GemmDesc& d) {
  static const bool enabled = [] {  // DPL_GEMM_SPLIT_BF16=0: never
    const char* e = std::getenv("DPL_GEMM_SPLIT_BF16");
    return !(e && e[0] == '0');
  }();
  if (!enabled || !d.split_ws || (d.epi & kOutMask) != kOutBf16 || d.batch != 1 || d.zdiv != 1 ||
      d.ndiv < d.N || d.conv_operand || d.trace || d.force_bn || d.force_1sm)
    return false;
  if (d.epi & ~static_cast<uint32_t>(kBias | kResid | kDGelu)) return false;
  if (d.N % 8 || d.ldc % 8 || static_cast<size_t>(d.M) * d.N * 4 > d.split_ws_bytes) return false;
  if (d.M < 256 || d.N <= 128) return false;  // the CTA-pair kernel's shapes only
  const long long pair_tiles = static_cast<long long>((d.M + 255) / 256) * ((d.N + 255) / 256);
  const int kblocks = (d.K + 63) / 64;
  const int pairs = num_sms() / 2;
  // at most half the pairs busy, and enough K for the split to pay for the
  // fp32 round trip of the separate epilogue pass: K >= 3072 (GPT-2 N=1
  // 55.2-55.5 samples/s at >= 48 K blocks, 54.7-55.0 at >= 16, 53.9 off;
  // DPL_GEMM_SPLIT_MIN_KB overrides)
  static const int min_kb = [] {
    const char* e = std::getenv("DPL_GEMM_SPLIT_MIN_KB");
    return e ? std::max(16, std::atoi(e)) : 48;
  }();
  return pair_tiles * 2 <= pairs && kblocks >= min_kb;
}

void GemmOp::prepare(const GemmDesc& d) {
  if (d.M <= 0 || d.N <= 0 || d.K <= 0 || d.batch <= 0) throw std::invalid_argument("dpl gemm: empty problem");
  if (split_bf16_candidate(d)) {
    GemmDesc inner = d;
    inner.C = d.split_ws;
    inner.ldc = d.N;
    inner.epi = kOutF32Acc;
    inner.alpha = 1.0f;
    inner.bias = nullptr;
    inner.resid = nullptr;
    inner.aux_in = nullptr;
    inner.aux_out = nullptr;
    inner.colsum = nullptr;
    inner.split_ws = nullptr;
    split_ = std::make_shared<GemmOp>();
    split_->prepare(inner);
    split_desc_ = d;
    params_ = split_->params_;
    bn_ = split_->bn_;
    grid_ = split_->grid_;
    smem_ = split_->smem_;
    return;
  }
  if (d.ndiv % 32 != 0) throw std::invalid_argument("dpl gemm: ndiv must be a multiple of 32");
  int bn = d.force_bn;
  if (bn == 0 && (d.epi & kOutMask) == kOutF32Acc && d.N > 128) bn = 256;  // split-K fills the machine
  if (bn == 0) {
    if (d.N <= 64) {
      bn = 64;
    } else {
      // minimise waves x tile width, charging the 128-wide tile ~40% more
      // per FLOP (half the operand reuse per byte fetched; measured on B200:
      // 4096x4096x1024 runs at 878 TF with BN=256 vs 713 TF with BN=128, and
      // at GPT-2's 1024-token shapes 1024x4800x1600 / 1024x6400x1600 the
      // 256x256 pair beats the 256x128 pair by 10-24% despite a ragged
      // second wave: tools/gemm_graph_bench.py --T 1024 --H 1600 --F 6400)
      const int sms = num_sms();
      static const double narrow_cost = [] {  // DPL_GEMM_BN128_COST: A/B knob
        const char* e = std::getenv("DPL_GEMM_BN128_COST");
        return e ? std::atof(e) : 1.4;
      }();
      // 256 x 192 pair tiles (K-major B only: an MN-major B tile is loaded in
      // 64-column boxes) for shapes whose 256-wide last wave is ragged, e.g.
      // GPT-2's 1024 x 1600 / 1024 x 4800 / 1024 x 6400 or BERT's 2048-row
      // replica slices (DPL_GEMM_BN192_COST: A/B knob, 0 disables)
      static const double mid_cost = [] {
        const char* e = std::getenv("DPL_GEMM_BN192_COST");
        return e ? std::atof(e) : 1.1;
      }();
      const bool allow192 = mid_cost > 0 && !d.b_mn_major && !d.conv_operand && d.M >= 256 && !d.force_1sm;
      double best = -1;
      for (int cand : {256, 192, 128}) {
        if (cand == 192 && !allow192) continue;
        const long long tiles = static_cast<long long>(ceil_div(d.M, kBM)) * ceil_div(d.N, cand) * d.batch;
        const double cost = static_cast<double>((tiles + sms - 1) / sms) * cand *
                            (cand == 128 ? narrow_cost : cand == 192 ? mid_cost : 1.0);
        if (best < 0 || cost < best) {
          best = cost;
          bn = cand;
        }
      }
    }
  }
  static const bool pair_enabled = [] {
    const char* e = std::getenv("DPL_GEMM_2SM");
    return !(e && e[0] == '0');
  }();
  static const bool pair128 = [] {
    const char* e = std::getenv("DPL_GEMM_PAIR128");
    return !(e && e[0] == '0');
  }();
  // 256x128 pairs help the 1024-row transformer GEMMs but not the implicit
  // convolutions (VGG-19 N=1: 3719 vs 3889 samples/s with them), which keep
  // the 1-SM 128x128 tile
  if (bn == 192 && (d.b_mn_major || d.conv_operand || d.M < 256 || d.force_1sm || !pair_enabled))
    throw std::invalid_argument("dpl gemm: BN 192 needs the pair kernel with a K-major B");
  const bool two_sm = pair_enabled && !d.force_1sm && d.M >= 256 &&
                      (bn == 256 || bn == 192 || (bn == 128 && pair128 && !d.conv_operand));
  const int bm = two_sm ? 256 : kBM;
  GemmParams& p = params_;
  p = GemmParams{};
  p.two_sm = two_sm;
  p.M = d.M;
  p.N = d.N;
  p.K = d.K;
  p.batch = d.batch;
  p.a_mn_major = d.a_mn_major;
  p.b_mn_major = d.b_mn_major;
  p.conv_operand = d.conv_operand;
  if (d.conv_operand) {
    if (d.conv_c % 64 || d.batch != 1 || !d.conv_x)
      throw std::invalid_argument("dpl gemm: implicit conv needs C % 64 == 0, batch 1 and an input");
    if (d.conv_operand == 1 && (d.a_mn_major || d.K != 9 * d.conv_c || d.M != d.conv_n * d.conv_h * d.conv_w))
      throw std::invalid_argument("dpl gemm: implicit conv A operand shape");
    if (d.conv_operand == 2 && (!d.b_mn_major || d.N != 9 * d.conv_c || d.K != d.conv_n * d.conv_h * d.conv_w))
      throw std::invalid_argument("dpl gemm: implicit conv B operand shape");
    p.conv_h = d.conv_h;
    p.conv_w = d.conv_w;
    p.conv_c = d.conv_c;
  }
  p.tma_a = d.conv_operand == 1 ? make_im2col_map(d.conv_x, d.conv_n, d.conv_h, d.conv_w, d.conv_c, kBM)
            : d.a_mn_major      ? make_map(d.A, d.M, d.K, d.lda, d.batch, d.a_batch_stride, kBK)
                                : make_map(d.A, d.K, d.M, d.lda, d.batch, d.a_batch_stride, kBM);
  p.tma_b = d.conv_operand == 2 ? make_im2col_map(d.conv_x, d.conv_n, d.conv_h, d.conv_w, d.conv_c, kBK)
            : d.b_mn_major      ? make_map(d.B, d.N, d.K, d.ldb, d.batch, d.b_batch_stride, kBK)
                                : make_map(d.B, d.K, d.N, d.ldb, d.batch, d.b_batch_stride, two_sm ? bn / 2 : bn);
  p.num_m_blocks = ceil_div(d.M, bm);
  p.num_n_blocks = ceil_div(d.N, bn);
  p.num_k_blocks = ceil_div(d.K, kBK);
  p.k_splits = 1;
  p.kb_per_split = p.num_k_blocks;
  if ((d.epi & kOutMask) == kOutF32Acc && d.epi != kOutF32Acc)
    throw std::invalid_argument("dpl gemm: fp32 accumulation takes no other epilogue flags");
  if (d.epi == kOutF32Acc) {
    // too few tiles for the SMs: split K (>= 8 k-blocks per split) and let
    // the fp32 accumulator absorb the partial sums atomically
    const int sms = two_sm ? num_sms() / 2 : num_sms();
    const int tiles = p.num_m_blocks * p.num_n_blocks * d.batch;
    int splits = 1;
    while (tiles * splits * 2 <= sms && p.num_k_blocks / (splits * 2) >= 8) splits *= 2;
    // a non-power-of-two split when it fills the waves much better: e.g. the
    // 3072 x 1024 QKV weight gradient (48 pair tiles, K = 4096) at 3 splits
    // runs 144 units in 2 waves = 2/3 of the unsplit mainloop per pair
    static const bool any_split = [] {  // DPL_GEMM_SPLIT_ANY=0: powers of two only (A/B)
      const char* e = std::getenv("DPL_GEMM_SPLIT_ANY");
      return !(e && e[0] == '0');
    }();
    if (any_split) {
      auto cost = [&](int sp) {  // mainloop waves per K, plus ~8% per extra fp32 reduce-add pass
        return static_cast<double>(ceil_div(tiles * sp, sms)) / sp * (1.0 + 0.08 * (sp - 1));
      };
      int best = splits;
      for (int sp = 2; sp <= 8; ++sp)
        if (p.num_k_blocks / sp >= 8 && cost(sp) < 0.8 * cost(best)) best = sp;
      splits = best;
    }
    p.kb_per_split = ceil_div(p.num_k_blocks, splits);
    p.k_splits = ceil_div(p.num_k_blocks, p.kb_per_split);
  }
  p.num_tiles = p.num_m_blocks * p.num_n_blocks * d.batch * p.k_splits;
  p.epi = d.epi;
  p.alpha = d.alpha;
  p.C = d.C;
  p.ldc = d.ldc;
  p.zdiv = d.zdiv;
  p.ndiv = d.ndiv;
  p.s_zo = d.s_zo;
  p.s_zi = d.s_zi;
  p.s_no = d.s_no;
  p.bias = d.bias;
  p.aux_in = static_cast<const __nv_bfloat16*>(d.aux_in);
  p.resid = static_cast<const __nv_bfloat16*>(d.resid);
  p.aux_out = static_cast<__nv_bfloat16*>(d.aux_out);
  // 16-byte vector epilogue needs every row/segment start 16B aligned
  const int esz = (d.epi & kOutMask) == kOutBf16 ? 2 : 4;
  const bool aligned = reinterpret_cast<uintptr_t>(d.C) % 16 == 0 && (d.ldc * esz) % 16 == 0 &&
                       (d.s_zo * esz) % 16 == 0 && (d.s_zi * esz) % 16 == 0 && (d.s_no * esz) % 16 == 0 &&
                       (!d.bias || reinterpret_cast<uintptr_t>(d.bias) % 16 == 0) &&
                       (!d.aux_in || reinterpret_cast<uintptr_t>(d.aux_in) % 16 == 0) &&
                       (!d.resid || reinterpret_cast<uintptr_t>(d.resid) % 16 == 0) &&
                       (!d.aux_out || reinterpret_cast<uintptr_t>(d.aux_out) % 16 == 0) &&
                       ((d.epi & kOutMask) == kOutBf16 || (d.ldc * 2) % 16 == 0);
  const bool aux_aligned = !(d.aux_in || d.resid || d.aux_out) || ((d.ldc * 2) % 16 == 0 && (d.s_zo * 2) % 16 == 0 &&
                                                                   (d.s_zi * 2) % 16 == 0 && (d.s_no * 2) % 16 == 0);
  p.vec_ok = aligned && aux_aligned;
  colsum_fallback_ = false;
  p.trace = d.trace;
  p.colsum = d.colsum;
  if ((d.epi & kColSum) && (!d.colsum || (d.epi & kOutMask) != kOutBf16 || d.batch != 1))
    throw std::invalid_argument("dpl gemm: kColSum needs a colsum target, a bf16 output and batch 1");
  // TMA epilogue: bulk tensor stores / fp32 reduce-adds from swizzled smem
  // chunks, extra input bulk-loaded ahead of use (see EpiTma)
  {
    static const bool tma_enabled = [] {
      const char* e = std::getenv("DPL_GEMM_TMA_EPI");
      return !(e && e[0] == '0');
    }();
    const uint32_t kind = d.epi & kOutMask;
    const bool x_in = (d.epi & (kResid | kDGelu | kDRelu)) != 0;
    const bool two_in = (d.epi & kResid) && (d.epi & (kDGelu | kDRelu));
    const bool aux = (d.epi & kAuxOut) != 0;
    bool ok = tma_enabled && p.vec_ok && d.N >= 32 && d.batch % d.zdiv == 0 && (d.ndiv >= d.N || d.N % d.ndiv == 0) &&
              !two_in && !(x_in && aux);
    if (kind != kOutBf16 && (x_in || aux)) ok = false;
    if ((d.epi & kBias) && (d.N % 4 != 0 || reinterpret_cast<uintptr_t>(d.bias) % 16 != 0)) ok = false;
    const int stage_bytes = two_sm ? (kBM + bn / 2) * kBK * 2 : (kBM + bn) * kBK * 2;
    const int ring = kSmemBudget - 2048;
    p.stages = std::min(kMaxStages, ring / stage_bytes);
    if (ok) {
      // carve the staging out of the ring, keeping >= 4 stages
      const int per_warp = bn / 64;  // chunks per epilogue warp per tile
      p.epi_out_bytes = kind == kOutBf16 ? 2048 : 4096;
      // prefetched residual / activation-input chunks per warp: one, so the
      // ring keeps a fifth stage -- the mainloop gains more from the deeper
      // ring than the epilogue loses to the exposed input loads (BERT-48
      // ffn2 34.8 -> 31.0 us, ffn2 dgrad 46.2 -> 43.5, o 15.9 -> 15.4;
      // DPL_GEMM_X_BUFS=2 restores the previous carve-out)
      static const int max_nx = [] {
        const char* e = std::getenv("DPL_GEMM_X_BUFS");
        return e ? std::max(1, std::min(kMaxNx, std::atoi(e))) : 1;
      }();
      p.epi_nx = x_in ? std::min(max_nx, per_warp) : (aux ? 2 : 1);
      p.epi_tile_cols = bn;
      const int bias_bytes = (d.epi & kBias) ? p.epi_tile_cols * 4 : 0;
      for (;;) {
        // 1 KB multiple: every warp's chunk buffers stay swizzle-atom aligned
        p.epi_warp_bytes = (2 * p.epi_out_bytes + (x_in || aux ? p.epi_nx * kXBytes : 0) + bias_bytes + 1023) & ~1023;
        p.stages = std::min(kMaxStages, (ring - kEpiWarps * p.epi_warp_bytes) / stage_bytes);
        if (p.stages >= 4 || !x_in || p.epi_nx <= std::min(2, max_nx)) break;
        p.epi_nx /= 2;
      }
      ok = p.stages >= 4;
    }
    if (!ok) {
      p.epi_warp_bytes = 0;
      p.stages = std::min(kMaxStages, ring / stage_bytes);
    }
    if (ok) {
      const int inner = d.ndiv >= d.N ? d.N : d.ndiv;
      const int nhi = d.N / inner;
      p.c_inner = inner;
      p.tma_c = make_epi_map(d.C, kind != kOutBf16, d, inner, nhi);
      const void* x = x_in ? ((d.epi & kResid) ? d.resid : d.aux_in) : (aux ? d.aux_out : nullptr);
      if (x) p.tma_x = make_epi_map(x, false, d, inner, nhi);
      p.tma_epi = 1;
    }
    // without the TMA epilogue the column sums run as a separate pass
    colsum_fallback_ = (d.epi & kColSum) && !p.tma_epi;
    if (colsum_fallback_) {
      if (d.ldc != d.N || d.zdiv != 1 || d.ndiv < d.N)
        throw std::invalid_argument("dpl gemm: kColSum fallback needs a plain [M][N] output");
      p.epi &= ~static_cast<uint32_t>(kColSum);
    }
  }
  bn_ = bn;
  static const int max_ctas = [] {  // DPL_GEMM_MAX_CTAS: diagnostic cap on the persistent grid
    const char* e = std::getenv("DPL_GEMM_MAX_CTAS");
    return e ? std::max(2, std::atoi(e)) : 1 << 30;
  }();
  const int sms = std::min(num_sms(), d.max_ctas > 1 ? std::min(max_ctas, d.max_ctas) : max_ctas);
  grid_ = two_sm ? 2 * std::min(p.num_tiles, sms / 2) : std::min(p.num_tiles, sms);
  // a last wave of at most half the pairs runs as 256 x 128 halves (two per
  // tile): e.g. 4096 x 4096 has 256 tiles on 74 pairs = 3 waves + 34 tiles.
  // Only for full-machine grids with >= 2 whole waves: GPT-2's 1.0-1.4-wave
  // 1024-row GEMMs and the capped side-stream grids measured slower with it
  // (GPT-2 N=1 54.8 vs 56.1 samples/s), the side stream already fills idle pairs
  static const bool split_tail = [] {  // DPL_GEMM_SPLIT_TAIL=0: whole last wave (A/B)
    const char* e = std::getenv("DPL_GEMM_SPLIT_TAIL");
    return !(e && e[0] == '0');
  }();
  p.split_tail = 0;
  if (split_tail && two_sm && bn == 256 && p.tma_epi && !p.conv_operand && p.k_splits == 1) {
    const int pairs = grid_ / 2;
    const int rem = p.num_tiles % pairs;
    if (pairs * 2 >= num_sms() - 1 && p.num_tiles >= 2 * pairs && rem > 0 && 2 * rem <= pairs) p.split_tail = rem;
  }
  if (two_sm) {
    smem_ = pair::kSmem;
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(gemm_bf16_tcgen05_2sm<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, pair::kSmem);
      cudaFuncSetAttribute(gemm_bf16_tcgen05_2sm<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, pair::kSmem);
      cudaFuncSetAttribute(gemm_bf16_tcgen05_2sm<192>, cudaFuncAttributeMaxDynamicSharedMemorySize, pair::kSmem);
    });
    return;
  }
  switch (bn) {
    case 64: smem_ = Cfg<64>::kSmem; configure_kernel<64>(); break;
    case 128: smem_ = Cfg<128>::kSmem; configure_kernel<128>(); break;
    case 256: smem_ = Cfg<256>::kSmem; configure_kernel<256>(); break;
    default: throw std::invalid_argument("dpl gemm: BN must be 64, 128 or 256");
  }
}

struct GemmCache::Impl {
  std::unordered_map<std::string, std::unique_ptr<GemmOp>> ops;
};

const GemmOp& GemmCache::get(const GemmDesc& dd) {
  if (!impl_) impl_ = std::make_shared<Impl>();
  GemmDesc d = dd;  // this cache's split-K scratch (not part of the key: one per cache)
  d.split_ws = split_ws;
  d.split_ws_bytes = split_ws_bytes;
  if (max_ctas_override) d.max_ctas = max_ctas_override;
  // explicit field-wise key: no padding bytes
  const long long f[] = {d.M, d.N, d.K, d.batch,
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.A)), d.lda, d.a_batch_stride,
                         d.a_mn_major,
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.B)), d.ldb, d.b_batch_stride,
                         d.b_mn_major,
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.C)), d.ldc, d.zdiv, d.s_zo, d.s_zi,
                         d.ndiv, d.s_no, static_cast<long long>(d.epi),
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.bias)),
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.aux_in)),
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.resid)),
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.aux_out)), d.force_bn, d.force_1sm,
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.trace)),
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.colsum)),
                         static_cast<long long>(reinterpret_cast<uintptr_t>(d.conv_x)), d.conv_operand, d.conv_n,
                         d.conv_h, d.conv_w, d.conv_c, d.max_ctas};
  std::string key(reinterpret_cast<const char*>(f), sizeof f);
  uint32_t a;
  std::memcpy(&a, &d.alpha, 4);
  key.append(reinterpret_cast<const char*>(&a), 4);
  auto it = impl_->ops.find(key);
  if (it == impl_->ops.end()) {
    auto op = std::make_unique<GemmOp>();
    op->prepare(d);
    it = impl_->ops.emplace(std::move(key), std::move(op)).first;
  }
  return *it->second;
}

size_t GemmCache::size() const { return impl_ ? impl_->ops.size() : 0; }

cudaEvent_t GemmProfile::take() {
  if (used == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return pool[used++];
}

void GemmCache::run(const GemmDesc& d, cudaStream_t s) {
  const GemmOp& op = get(d);
  if (!profile.enabled) {
    op.launch(s);
    return;
  }
  GemmProfile::Rec r;
  r.start = profile.take();
  r.end = profile.take();
  r.flops = op.flops();
  r.M = d.M;
  r.N = d.N;
  r.K = d.K;
  r.batch = d.batch;
  r.bn = op.bn();
  const bool ext = kernel_timer().capturing;
  if (ext) cudaEventRecordWithFlags(r.start, s, cudaEventRecordExternal);
  else cudaEventRecord(r.start, s);
  op.launch(s);
  if (ext) cudaEventRecordWithFlags(r.end, s, cudaEventRecordExternal);
  else cudaEventRecord(r.end, s);
  profile.recs.push_back(r);
}

void GemmOp::launch(cudaStream_t stream) const {
  if (split_) {
    split_->launch_kernel(stream);
    const GemmDesc& d = split_desc_;
    split_epilogue(d.split_ws, d.C, d.ldc, d.M, d.N, d.alpha, d.bias, d.resid, d.aux_in, d.epi, stream);
    return;
  }
  launch_kernel(stream);
  if (colsum_fallback_)  // kColSum without the TMA epilogue: a column-sum pass over C
    colsum_acc(params_.C, params_.colsum, params_.M, params_.N, stream);
}

void GemmOp::launch_kernel(cudaStream_t stream) const {
  count_launch();
  TimedLaunch timed_("gemm_bf16_tcgen05", stream, flops());
  if (params_.two_sm) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const cudaError_t e = bn_ == 256   ? cudaLaunchKernelEx(&cfg, gemm_bf16_tcgen05_2sm<256>, params_)
                          : bn_ == 192 ? cudaLaunchKernelEx(&cfg, gemm_bf16_tcgen05_2sm<192>, params_)
                                       : cudaLaunchKernelEx(&cfg, gemm_bf16_tcgen05_2sm<128>, params_);
    if (e != cudaSuccess) throw std::runtime_error(std::string("dpl gemm: pair launch failed: ") + cudaGetErrorString(e));
    return;
  }
  switch (bn_) {
    case 64: launch_pdl(gemm_bf16_tcgen05<64>, dim3(grid_), dim3(kThreads), smem_, stream, params_); break;
    case 128: launch_pdl(gemm_bf16_tcgen05<128>, dim3(grid_), dim3(kThreads), smem_, stream, params_); break;
    case 256: launch_pdl(gemm_bf16_tcgen05<256>, dim3(grid_), dim3(kThreads), smem_, stream, params_); break;
    default: throw std::logic_error("dpl gemm: launch before prepare");
  }
}

}  // namespace dpl
