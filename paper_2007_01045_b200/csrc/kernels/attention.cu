// Fused attention (flash style) for head dim 64 on sm_100a.
//
// Forward, one CTA per (z = head * B + sample, 128-query tile):
//   warp 0      TMA: Q tile once, K/V tiles (128 keys) through a 2-stage ring
//   warp 1      MMA: S_j = Q K_j^T  (M=128, N=128, K=64)   -> TMEM (2 buffers)
//                    O_j = P_j V_j   (M=128, N=64,  K=128)  -> TMEM (2 buffers)
//   warp 2      TMEM allocator
//   warps 4-7   softmax: one thread per query row reads its S row from TMEM
//               (no cross-thread reductions), keeps the running max / sum
//               (online softmax, exp2 on the SFU), writes P_j (bf16) into a
//               SWIZZLE_128B smem tile for the PV MMA, and accumulates
//               O = O * alpha + O_j in registers.
// Output: context head-merged into [R][H] (row = b*S + q, col = h*64 + j),
// and the per-row log-sum-exp (natural log of the scaled scores) for the
// backward pass.  S and P never touch HBM.
//
// Layout: qkv is head-split [3][heads][B][S][64] (written that way by the QKV
// GEMM epilogue), so one 3-D tensor map {64, S, 3*heads*B} serves Q, K and V.
// Because a [128 x 64] bf16 tile is exactly 128 rows of one 128-byte swizzle
// atom, the same smem bytes are a valid K-major operand (M/N = rows) and a
// valid MN-major operand (K = rows); P is written once in that layout.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "attention.h"
#include "gemm.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace dpl {

namespace {

constexpr int kT = 128;           // query / key tile
constexpr int kD = 64;            // head dim
constexpr int kTileBytes = kT * kD * 2;  // 16 KB
constexpr int kFwdThreads = 320;      // warp 0 TMA, warp 1 MMA, warps 2-9 softmax
constexpr int kSoftmaxThreads = 256;

struct AttnFwdParams {
  CUtensorMap qkv;  // {64, S, 3*heads*B}
  int S, B, heads, causal, z_count;
  float scale_log2;  // (1/sqrt(d)) * log2(e)
  __nv_bfloat16* ctx;
  long long ldc;  // H
  float* lse;     // [z][S]
  // Causal split schedule (n_items > 0): blockIdx = (z, item); item i covers
  // key tiles [lo, hi) of query tile qt, half = 0 (whole range) or 1 / 2.
  float* part;    // [z][S/128][2][66][128]: o[64], m, l per row, per half
  int* flags;     // [z][S/128] tickets
  int n_items;
  long long* trace;  // 16 %globaltimer slots per CTA (diagnostics), or null
  unsigned char it_qt[32], it_lo[32], it_hi[32], it_half[32];
};

__device__ __forceinline__ float exp2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// byte offset of 16-byte chunk `c` (0..7) of row `r` inside a SWIZZLE_128B
// [rows x 64] bf16 tile (1024-byte aligned)
__device__ __forceinline__ uint32_t sw128(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Two CTAs per SM (~66 KB smem, 256 TMEM columns each).  Ten warps: warp 0
// TMA (and the TMEM allocation), warp 1 MMA, warps 2-9 softmax -- two threads
// per query row, each owning 64 of the tile's 128 key columns and 32 of the
// 64 output columns, so four softmax warps per SM sub-partition hide each
// other's TMEM-load / SFU latency.
// TMEM: S [0,128) fp32, P [128,192) bf16 pairs, O [192,256) fp32.  P goes
// from the softmax registers to tensor memory (tcgen05.st) and the PV MMA
// reads its A operand from there, and O accumulates in tensor memory across
// key tiles: shared memory carries only the TMA tiles and the MMAs' Q / K / V
// operands (80 KB per CTA-tile instead of 144 KB with P staged in smem --
// the per-SM shared-memory bandwidth is what bounded the smem-P form).
// O is rescaled only when a row's max grows by more than 2^8 (the stale max
// keeps every P <= 256); l and the output use the same reference max.
// The row max of a tile is combined through shared memory (a 64-thread
// named barrier per lane quadrant); the row sums stay per thread until the
// end.  The MMA warp issues S_{j+1} ahead of PV_j and the softmax releases
// S_j at its last TMEM load.
__global__ void __launch_bounds__(kFwdThreads, 2) attn_fwd_kernel(const __grid_constant__ AttnFwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                // 16 KB
  uint8_t* sK = sQ + kTileBytes;     // 16 KB
  uint8_t* sV = sK + kTileBytes;     // 2 x 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = bars + 2;
  uint64_t* s_full = bars + 3;
  uint64_t* s_empty = bars + 4;
  uint64_t* p_full = bars + 5;
  uint64_t* p_empty = bars + 6;   // PV_j done: P free, O holds tiles 0..j
  uint64_t* v_full = bars + 7;    // [2]
  uint64_t* v_empty = bars + 9;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);
  int* ticket = reinterpret_cast<int*>(bars + 12);
  float* xch = reinterpret_cast<float*>(bars + 13);  // [2 tiles][2 halves][128 rows] row-max / row-sum exchange

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  long long* trace = p.trace ? p.trace + 16LL * (blockIdx.x + gridDim.x * blockIdx.y) : nullptr;
  auto mark = [&](int slot) {
    if (trace) trace[slot] = static_cast<long long>(ptx::globaltimer_ns());
  };
  if (warp == 2 && lane == 0) {
    mark(0);
    if (trace) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[15] = smid;
    }
  }
  int qt, z, kv_lo, half = 0, n_kv;
  if (p.n_items) {
    z = blockIdx.x;
    qt = p.it_qt[blockIdx.y];
    kv_lo = p.it_lo[blockIdx.y];
    n_kv = p.it_hi[blockIdx.y] - kv_lo;
    half = p.it_half[blockIdx.y];
  } else {
    qt = blockIdx.x;
    z = blockIdx.y;
    kv_lo = 0;
    n_kv = p.causal ? qt + 1 : p.S / kT;
  }
  const int q0 = qt * kT;
  const int zk = p.z_count + z, zv = 2 * p.z_count + z;
  constexpr uint32_t kColP = 128, kColO = 192;

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch_desc(&p.qkv);
      ptx::mbar_init(q_full, 1);
      ptx::mbar_init(k_full, 1);
      ptx::mbar_init(k_empty, 1);
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_init(&v_full[i], 1);
        ptx::mbar_init(&v_empty[i], 1);
      }
      ptx::mbar_init(s_full, 1);
      ptx::mbar_init(s_empty, kSoftmaxThreads);
      ptx::mbar_init(p_full, kSoftmaxThreads);
      ptx::mbar_init(p_empty, 1);
      ptx::fence_barrier_init();
    }
    __syncwarp();
    ptx::tmem_alloc<256>(tmem_slot);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();
  if (warp == 2 && lane == 0) mark(1);

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(q_full, kTileBytes);
      ptx::tma_load_3d(sQ, &p.qkv, q_full, 0, q0, z);
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        ptx::mbar_wait(k_empty, (j & 1) ^ 1);  // S_{j-1} done
        ptx::mbar_arrive_expect_tx(k_full, kTileBytes);
        ptx::tma_load_3d(sK, &p.qkv, k_full, 0, (kv_lo + j) * kT, zk);
        ptx::mbar_wait(&v_empty[b], ((j >> 1) & 1) ^ 1);  // PV_{j-2} done
        ptx::mbar_arrive_expect_tx(&v_full[b], kTileBytes);
        ptx::tma_load_3d(sV + b * kTileBytes, &p.qkv, &v_full[b], 0, (kv_lo + j) * kT, zv);
      }
    }
  } else if (warp == 1) {  // whole warp: descriptors uniform, one elected lane issues
    {
      const uint32_t idesc_s = ptx::idesc_bf16_f32(kT, kT, false, false);  // Q K-major, K K-major
      const uint32_t idesc_o = ptx::idesc_bf16_f32(kT, kD, false, true);   // P (TMEM) K-major, V MN-major
      const uint32_t aq = ptx::smem_addr(sQ), bk = ptx::smem_addr(sK);
      // S_j = Q K_j^T once K_j landed and the softmax read S_{j-1}
      auto issue_s = [&](int j) {
        const uint32_t ph = j & 1;
        ptx::mbar_wait(k_full, ph);
        ptx::mbar_wait(s_empty, ph ^ 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < kD / 16; ++k)
          ptx::mma_bf16_e(tmem, ptx::smem_desc_sw128(aq + k * 32, 16, 1024), ptx::smem_desc_sw128(bk + k * 32, 16, 1024),
                        idesc_s, k > 0);
        ptx::mma_commit_e(s_full);
        ptx::mma_commit_e(k_empty);
      };
      ptx::mbar_wait(q_full, 0);
      if (lane == 0) mark(12);
      if (n_kv > 0) issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        const uint32_t ph = j & 1;
        if (j + 1 < n_kv) issue_s(j + 1);
        // O (+)= P_j V_j, P_j from tensor memory (16 keys = 8 columns per step)
        const int vb = j & 1;
        const uint32_t bv = ptx::smem_addr(sV + vb * kTileBytes);
        ptx::mbar_wait(&v_full[vb], (j >> 1) & 1);
        ptx::mbar_wait(p_full, ph);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < kT / 16; ++k)
          ptx::mma_bf16_ts_e(tmem + kColO, tmem + kColP + k * 8, ptx::smem_desc_sw128(bv + k * 16 * 128, 16, 1024),
                           idesc_o, (j | k) != 0);
        ptx::mma_commit_e(&v_empty[vb]);
        ptx::mma_commit_e(p_empty);
      }
    }
  } else {
    const int quad = warp & 3;
    const int kh = (warp - 2) >> 2;  // key columns [64*kh, 64*kh+64), output columns [32*kh, 32*kh+32)
    const int r = quad * 32 + lane;  // query row within the tile
    const int q = q0 + r;
    const uint32_t trow = (quad * 32) << 16;
    const float c = p.scale_log2;
    // the two warps of a lane quadrant meet at a named barrier
    auto pair_sync = [&]() {
      switch (quad) {  // immediate barrier ids (a register id reserves all 16)
        case 0: asm volatile("bar.sync 1, 64;" ::: "memory"); break;
        case 1: asm volatile("bar.sync 2, 64;" ::: "memory"); break;
        case 2: asm volatile("bar.sync 3, 64;" ::: "memory"); break;
        default: asm volatile("bar.sync 4, 64;" ::: "memory"); break;
      }
    };
    constexpr float kRescale = 8.f;  // log2 headroom of the stale max
    float m = -INFINITY, l = 0.f;    // reference max (scaled, log2 units) and this half's row sum
    for (int j = 0; j < n_kv; ++j) {
      const uint32_t ph = j & 1;
      ptx::mbar_wait(s_full, ph);
      ptx::tc_fence_after();
      if (r == 0 && kh == 0 && j < 4) mark(2 + j);
      const bool diag = p.causal && kv_lo + j == qt;
      const int lim = diag ? r - 64 * kh : 63;  // last unmasked key column of this row, in this half
      // pass 1: row max of the raw scores over this half (scale > 0 commutes with max)
      float mx = -INFINITY;
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + trow + 64 * kh + cc * 32, v);
        ptx::tmem_wait_ld();
        if (!diag) {
#pragma unroll
          for (int e = 0; e < 32; ++e) mx = fmaxf(mx, __uint_as_float(v[e]));
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) mx = cc * 32 + e <= lim ? fmaxf(mx, __uint_as_float(v[e])) : mx;
        }
      }
      float* xm = xch + (j & 1) * 256;
      xm[kh * 128 + r] = mx;
      pair_sync();
      mx = fmaxf(mx, xm[(kh ^ 1) * 128 + r]) * c;
      ptx::mbar_wait(p_empty, ph ^ 1);  // PV_{j-1} done: P free, O current
      // new reference max where a row's max grew past the headroom (both
      // halves of a row decide alike); the TMEM rescale of O is warp-wide
      // (.sync.aligned), with alpha = 1 on the rows that keep theirs
      const bool need = mx > m + kRescale;
      const float alpha = need ? exp2_fast(m - mx) : 1.f;
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        ptx::tc_fence_after();
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + trow + kColO + 32 * kh, v);
        ptx::tmem_wait_ld();
        uint32_t w[16];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
          for (int e = 0; e < 16; ++e) w[e] = __float_as_uint(__uint_as_float(v[16 * h2 + e]) * alpha);
          ptx::tmem_st_32x32b_x16(tmem + trow + kColO + 32 * kh + 16 * h2, w);
        }
      }
      if (need) {
        l *= alpha;
        m = mx;
      }
      float2 rs2 = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + trow + 64 * kh + cc * 32, v);
        ptx::tmem_wait_ld();
        if (cc == 1) {  // S_j fully read: the MMA may write S_{j+1}
          ptx::tc_fence_before();
          ptx::mbar_arrive(s_empty);
        }
        uint32_t pk[16];
        if (!diag) {  // packed fp32x2 FMA / add: half the scale and row-sum instructions
          const float2 c2 = make_float2(c, c), nm2 = make_float2(-m, -m);
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), c2, nm2);
            const float p0 = exp2_fast(x.x), p1 = exp2_fast(x.y);
            rs2 = __fadd2_rn(rs2, make_float2(p0, p1));
            pk[e >> 1] = pack_bf16(p0, p1);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float p0 = cc * 32 + e <= lim ? exp2_fast(fmaf(__uint_as_float(v[e]), c, -m)) : 0.f;
            const float p1 = cc * 32 + e + 1 <= lim ? exp2_fast(fmaf(__uint_as_float(v[e + 1]), c, -m)) : 0.f;
            rs2.x += p0;
            rs2.x += p1;
            pk[e >> 1] = pack_bf16(p0, p1);
          }
        }
        ptx::tmem_st_32x32b_x16(tmem + trow + kColP + 32 * kh + 16 * cc, pk);
      }
      l += rs2.x + rs2.y;  // this half's share of the row sum
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full);
      if (r == 0 && kh == 0 && j < 4) mark(6 + j);
    }
    // O of this thread's 32 columns once the last PV finished
    float o[32];
    ptx::mbar_wait(p_empty, (n_kv - 1) & 1);
    ptx::tc_fence_after();
    {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + trow + kColO + 32 * kh, v);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __uint_as_float(v[e]);
    }
    // full row sum: the two halves' shares (same reference max)
    {
      float* xl = xch + (n_kv & 1) * 256;
      xl[kh * 128 + r] = l;
      pair_sync();
      l += xl[(kh ^ 1) * 128 + r];
    }
    if (r == 0 && kh == 0) mark(10);
    bool write_out = true;
    if (half) {
      // Publish this half's (o, m, l); the CTA that takes ticket 1 merges
      // the other half's partial and writes the output.
      const int nq = p.S / kT;
      const long long tile = static_cast<long long>(z) * nq + qt;
      float* mine = p.part + (tile * 2 + (half - 1)) * 66 * kT;
      const float* other = p.part + (tile * 2 + (2 - half)) * 66 * kT;
#pragma unroll
      for (int e = 0; e < 32; ++e) __stcg(mine + (32 * kh + e) * kT + r, o[e]);
      if (kh == 0) {
        __stcg(mine + 64 * kT + r, m);
        __stcg(mine + 65 * kT + r, l);
      }
      __threadfence();
      asm volatile("bar.sync 5, %0;" ::"n"(kSoftmaxThreads) : "memory");
      if (warp == 2 && lane == 0) {
        const int t = atomicAdd(p.flags + tile, 1);
        if (t == 1) p.flags[tile] = 0;  // both halves in: ready for the next call
        *ticket = t;
      }
      asm volatile("bar.sync 5, %0;" ::"n"(kSoftmaxThreads) : "memory");
      write_out = *ticket == 1;
      if (write_out) {  // merged in half order (1, 2) whichever CTA runs it: deterministic
        __threadfence();
        const bool first = half == 1;
        const float mo = __ldcg(other + 64 * kT + r), lo = __ldcg(other + 65 * kT + r);
        const float m1 = first ? m : mo, m2 = first ? mo : m;
        const float l1 = first ? l : lo, l2 = first ? lo : l;
        const float mm = fmaxf(m1, m2);
        const float s1 = exp2_fast(m1 - mm), s2 = exp2_fast(m2 - mm);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float ot = __ldcg(other + (32 * kh + e) * kT + r);
          o[e] = fmaf(first ? o[e] : ot, s1, (first ? ot : o[e]) * s2);
        }
        l = fmaf(l1, s1, l2 * s2);
        m = mm;
      }
    }
    if (write_out) {
      const float inv = 1.f / l;
      const int b = z % p.B, h = z / p.B;
      __nv_bfloat16* out = p.ctx + static_cast<long long>(b * p.S + q) * p.ldc + h * kD + 32 * kh;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4 w;
        w.x = pack_bf16(o[8 * u + 0] * inv, o[8 * u + 1] * inv);
        w.y = pack_bf16(o[8 * u + 2] * inv, o[8 * u + 3] * inv);
        w.z = pack_bf16(o[8 * u + 4] * inv, o[8 * u + 5] * inv);
        w.w = pack_bf16(o[8 * u + 6] * inv, o[8 * u + 7] * inv);
        reinterpret_cast<uint4*>(out)[u] = w;
      }
      if (kh == 0) p.lse[static_cast<long long>(z) * p.S + q] = (m + log2f(l)) * 0.69314718055994531f;
    }
  }

  ptx::pdl_trigger();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2 && lane == 0) mark(11);
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem);
  }
}

// ---------------------------------------------------------------- backward
// One CTA per (z, 128-key tile j), looping over query tiles i:
//   MMA1(i):  S = Q_i K_j^T,  dP = dO_i V_j^T                (TMEM, 128 x 128 each)
//   softmax:  P = exp(scale*S - lse),  dS = P * (dP - D)     (warps 4-11 -> smem bf16)
//   MMA2(i):  dV += P^T dO_i,  dK += dS^T Q_i                 (TMEM, accumulate over i)
//             dQ_i = dS K_j  -> fp32 atomics into dq_acc[z][S][64] (summed over the key tiles)
// Software pipeline: P/dS are double buffered in smem and the MMA warp
// issues MMA1(i+1) before MMA2(i), so the softmax of tile i+1 runs on the
// CUDA cores while the tensor core does tile i's gradient MMAs; the dQ_i
// drain follows softmax(i+1).
// D = rowsum(dO * O) comes from attn_bwd_prep_kernel; dq_acc is turned into
// bf16 by attn_bwd_dq_kernel.  dK, dV are written head-merged into dqkv.
constexpr int kBwdThreads = 384;  // warps 4-11: two per TMEM lane quadrant

struct AttnBwdParams {
  CUtensorMap qkv;   // {64, S, 3*heads*B}
  CUtensorMap dout;  // {64, S, heads*B}   dO head-split
  int S, B, heads, causal, z_count;
  float scale, scale_log2;
  const float* lse;  // [z][S]
  const float* dsum; // [z][S]  D
  float* dq_acc;     // [z][S][64]
  __nv_bfloat16* dqkv;  // [B*S][3H]
  long long ld;         // 3H
  int H;
  long long* trace;     // 16 %globaltimer slots per CTA (diagnostics), or null
};

__global__ void __launch_bounds__(kBwdThreads, 1) attn_bwd_kernel(const __grid_constant__ AttnBwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;                         // 16 KB
  uint8_t* sV = sK + kTileBytes;              // 16 KB
  uint8_t* sQ = sV + kTileBytes;              // 2 x 16 KB
  uint8_t* sO = sQ + 2 * kTileBytes;          // 2 x 16 KB (dO)
  uint8_t* sP = sO + 2 * kTileBytes;          // 2 buffers x 32 KB (two 64-key halves each)
  uint8_t* sS = sP + 4 * kTileBytes;          // 2 buffers x 32 KB (dS)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sS + 4 * kTileBytes);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;   // [2]
  uint64_t* qdo_empty = bars + 3;  // [2]
  uint64_t* sp_full = bars + 5;
  uint64_t* sp_empty = bars + 6;
  uint64_t* pds_full = bars + 7;   // [2]
  uint64_t* pds_empty = bars + 9;  // [2]
  uint64_t* dq_full = bars + 11;
  uint64_t* dq_empty = bars + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  long long* trace = p.trace ? p.trace + 16LL * (blockIdx.x + gridDim.x * blockIdx.y) : nullptr;
  auto mark = [&](int slot) {
    if (trace) trace[slot] = static_cast<long long>(ptx::globaltimer_ns());
  };
  if (warp == 4 && lane == 0) {
    mark(0);
    if (trace) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[15] = smid;
    }
  }
  // causal: blockIdx = (z, j) so the block scheduler hands out every head's
  // longest key tile (j = 0 walks all query tiles) first and the short ones
  // fill the tail of the >1-wave grid; non-causal: (j, z)
  const int j = p.causal ? blockIdx.y : blockIdx.x, z = p.causal ? blockIdx.x : blockIdx.y;
  const int k0 = j * kT;
  const int n_q = p.S / kT;
  const int i_first = p.causal ? j : 0;
  const int n_iter = n_q - i_first;
  const int zk = p.z_count + z, zv = 2 * p.z_count + z;
  // TMEM: S [0,128), dP [128,256), dV [256,320), dK [320,384), dQ [384,448)

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&p.qkv);
    ptx::tma_prefetch_desc(&p.dout);
    ptx::mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&qdo_full[i], 1);
      ptx::mbar_init(&qdo_empty[i], 1);
      ptx::mbar_init(&pds_full[i], 256);
      ptx::mbar_init(&pds_empty[i], 1);
    }
    ptx::mbar_init(sp_full, 1);
    ptx::mbar_init(sp_empty, 256);
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_empty, 256);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();
  if (warp == 4 && lane == 0) mark(1);

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(kv_full, 2 * kTileBytes);
      ptx::tma_load_3d(sK, &p.qkv, kv_full, 0, k0, zk);
      ptx::tma_load_3d(sV, &p.qkv, kv_full, 0, k0, zv);
      for (int it = 0; it < n_iter; ++it) {
        const int st = it & 1, q0 = (i_first + it) * kT;
        ptx::mbar_wait(&qdo_empty[st], ((it >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&qdo_full[st], 2 * kTileBytes);
        ptx::tma_load_3d(sQ + st * kTileBytes, &p.qkv, &qdo_full[st], 0, q0, z);
        ptx::tma_load_3d(sO + st * kTileBytes, &p.dout, &qdo_full[st], 0, q0, z);
      }
    }
  } else if (warp == 1) {  // whole warp: descriptors uniform, one elected lane issues
    {
      const uint32_t id_sq = ptx::idesc_bf16_f32(kT, kT, false, false);  // S, dP: K-major A and B
      const uint32_t id_tt = ptx::idesc_bf16_f32(kT, kD, true, true);    // dV, dK: A^T, B MN-major
      const uint32_t id_dq = ptx::idesc_bf16_f32(kT, kD, false, true);   // dQ: dS K-major, K MN-major
      const uint32_t ak = ptx::smem_addr(sK), av = ptx::smem_addr(sV);
      // MMA1(it): S / dP of query tile it into TMEM (single buffer, freed by the softmax warps)
      auto mma1 = [&](int it) {
        const int st = it & 1;
        const uint32_t aq = ptx::smem_addr(sQ + st * kTileBytes), ao = ptx::smem_addr(sO + st * kTileBytes);
        ptx::mbar_wait(&qdo_full[st], (it >> 1) & 1);
        ptx::mbar_wait(sp_empty, (it & 1) ^ 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          ptx::mma_bf16_e(tmem, ptx::smem_desc_sw128(aq + k * 32, 16, 1024), ptx::smem_desc_sw128(ak + k * 32, 16, 1024),
                        id_sq, k > 0);
          ptx::mma_bf16_e(tmem + 128, ptx::smem_desc_sw128(ao + k * 32, 16, 1024),
                        ptx::smem_desc_sw128(av + k * 32, 16, 1024), id_sq, k > 0);
        }
        ptx::mma_commit_e(sp_full);
      };
      ptx::mbar_wait(kv_full, 0);
      if (n_iter > 0) mma1(0);
      for (int it = 0; it < n_iter; ++it) {
        const int st = it & 1, b = it & 1;
        const uint32_t aq = ptx::smem_addr(sQ + st * kTileBytes), ao = ptx::smem_addr(sO + st * kTileBytes);
        const uint32_t ap = ptx::smem_addr(sP + b * 2 * kTileBytes), as = ptx::smem_addr(sS + b * 2 * kTileBytes);
        // next tile's scores as soon as softmax(it) has S / dP in registers:
        // they overlap the rest of softmax(it) and this tile's gradients
        if (it + 1 < n_iter) mma1(it + 1);
        ptx::mbar_wait(&pds_full[b], (it >> 1) & 1);  // softmax(it) wrote P / dS
        ptx::mbar_wait(dq_empty, (it & 1) ^ 1);       // dQ(it-1) drained
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < kT / 16; ++k) {
          // A^T views: 64-key halves 16 KB apart (LBO), 16 query rows per K step
          const uint32_t row_step = k * 16 * 128;
          ptx::mma_bf16_e(tmem + 256, ptx::smem_desc_sw128(ap + row_step, kTileBytes, 1024),
                        ptx::smem_desc_sw128(ao + row_step, 16, 1024), id_tt, (it | k) != 0);
          ptx::mma_bf16_e(tmem + 320, ptx::smem_desc_sw128(as + row_step, kTileBytes, 1024),
                        ptx::smem_desc_sw128(aq + row_step, 16, 1024), id_tt, (it | k) != 0);
          const uint32_t a_off = (k >> 2) * kTileBytes + (k & 3) * 32;
          ptx::mma_bf16_e(tmem + 384, ptx::smem_desc_sw128(as + a_off, 16, 1024),
                        ptx::smem_desc_sw128(ak + row_step, 16, 1024), id_dq, k > 0);
        }
        ptx::mma_commit_e(&qdo_empty[st]);
        ptx::mma_commit_e(&pds_empty[b]);
        ptx::mma_commit_e(dq_full);
      }
    }
  } else if (warp >= 4) {
    const int quad = warp & 3;
    const int half = (warp - 4) >> 2;  // key columns [64*half, 64*half + 64); dQ / dK-dV split likewise
    const int r = quad * 32 + lane;
    const uint32_t trow = (quad * 32) << 16;
    const int b = z % p.B, h = z / p.B;
    // dQ partial of query tile `it` (this key tile's share) -> fp32 atomics
    auto drain_dq = [&](int it) {
      const int q = (i_first + it) * kT + r;
      ptx::mbar_wait(dq_full, it & 1);
      ptx::tc_fence_after();
      float4* dst = reinterpret_cast<float4*>(p.dq_acc + (static_cast<long long>(z) * p.S + q) * kD);
      const int c = half;  // 32 of the 64 dQ columns
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + trow + 384 + c * 32, v);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      ptx::mbar_arrive(dq_empty);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        atomicAdd(dst + c * 8 + u, make_float4(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]),
                                               __uint_as_float(v[4 * u + 2]), __uint_as_float(v[4 * u + 3])));
    };
    // lse / D of the next query tile are loaded one iteration ahead
    float lse_n = 0.f, dsum_n = 0.f;
    if (n_iter > 0) {
      const long long idx = static_cast<long long>(z) * p.S + i_first * kT + r;
      lse_n = p.lse[idx];
      dsum_n = p.dsum[idx];
    }
    for (int it = 0; it < n_iter; ++it) {
      const int i = i_first + it, q = i * kT + r;
      const int pb = it & 1;
      const float lse2 = lse_n * 1.4426950408889634f;
      const float dsum = dsum_n;
      if (it + 1 < n_iter) {
        const long long idx = static_cast<long long>(z) * p.S + q + kT;
        lse_n = p.lse[idx];
        dsum_n = p.dsum[idx];
      }
      const bool diag = p.causal && i == j;
      ptx::mbar_wait(sp_full, it & 1);
      ptx::tc_fence_after();
      if (warp == 4 && lane == 0 && it < 4) mark(2 + it);
      uint32_t vs[2][32], vp[2][32];
      ptx::tmem_ld_32x32b_x32(tmem + trow + (2 * half) * 32, vs[0]);
      ptx::tmem_ld_32x32b_x32(tmem + trow + 128 + (2 * half) * 32, vp[0]);
      ptx::tmem_ld_32x32b_x32(tmem + trow + (2 * half + 1) * 32, vs[1]);
      ptx::tmem_ld_32x32b_x32(tmem + trow + 128 + (2 * half + 1) * 32, vp[1]);
      ptx::tmem_wait_ld();
      // S / dP are in registers: MMA1(it+1) may overwrite them
      ptx::tc_fence_before();
      ptx::mbar_arrive(sp_empty);
      ptx::mbar_wait(&pds_empty[pb], ((it >> 1) & 1) ^ 1);  // MMA2(it-2) done with this P / dS buffer
      uint8_t* hp0 = sP + pb * 2 * kTileBytes;
      uint8_t* hs0 = sS + pb * 2 * kTileBytes;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = 2 * half + cc;
        float pv[32], dv[32];
        if (!diag) {  // packed fp32x2 arithmetic: one FMA / add / mul per two scores
          const float2 sl2 = make_float2(p.scale_log2, p.scale_log2), nl2 = make_float2(-lse2, -lse2);
          const float2 nd2 = make_float2(-dsum, -dsum);
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float2 x =
                __ffma2_rn(make_float2(__uint_as_float(vs[cc][e]), __uint_as_float(vs[cc][e + 1])), sl2, nl2);
            pv[e] = exp2_fast(x.x);
            pv[e + 1] = exp2_fast(x.y);
            const float2 d = __fmul2_rn(make_float2(pv[e], pv[e + 1]),
                                        __fadd2_rn(make_float2(__uint_as_float(vp[cc][e]), __uint_as_float(vp[cc][e + 1])), nd2));
            dv[e] = d.x;
            dv[e + 1] = d.y;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const bool masked = k0 + c * 32 + e > q;
            const float pe = masked ? 0.f : exp2_fast(__uint_as_float(vs[cc][e]) * p.scale_log2 - lse2);
            pv[e] = pe;
            dv[e] = pe * (__uint_as_float(vp[cc][e]) - dsum);
          }
        }
        uint8_t* hp = hp0 + (c >> 1) * kTileBytes;
        uint8_t* hs = hs0 + (c >> 1) * kTileBytes;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int chunk = (c & 1) * 4 + u;
          uint4 w;
          w.x = pack_bf16(pv[8 * u + 0], pv[8 * u + 1]);
          w.y = pack_bf16(pv[8 * u + 2], pv[8 * u + 3]);
          w.z = pack_bf16(pv[8 * u + 4], pv[8 * u + 5]);
          w.w = pack_bf16(pv[8 * u + 6], pv[8 * u + 7]);
          *reinterpret_cast<uint4*>(hp + sw128(r, chunk)) = w;
          w.x = pack_bf16(dv[8 * u + 0], dv[8 * u + 1]);
          w.y = pack_bf16(dv[8 * u + 2], dv[8 * u + 3]);
          w.z = pack_bf16(dv[8 * u + 4], dv[8 * u + 5]);
          w.w = pack_bf16(dv[8 * u + 6], dv[8 * u + 7]);
          *reinterpret_cast<uint4*>(hs + sw128(r, chunk)) = w;
        }
      }
      fence_async_smem();
      ptx::mbar_arrive(&pds_full[pb]);
      if (warp == 4 && lane == 0 && it < 4) mark(6 + it);
      if (it > 0) drain_dq(it - 1);
    }
    if (n_iter > 0) drain_dq(n_iter - 1);
    if (warp == 4 && lane == 0) mark(10);
    // dV, dK of this key tile (all MMAs done once the last dQ arrived)
    const int key = k0 + r;
    __nv_bfloat16* row = p.dqkv + static_cast<long long>(b * p.S + key) * p.ld + h * kD;
    {
      const int which = half;  // 0: dV (cols 2H..), 1: dK (cols H.., scaled)
      const float f = which ? p.scale : 1.f;
      __nv_bfloat16* out = row + (which ? p.H : 2 * p.H);
#pragma unroll
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + trow + (which ? 320 : 256) + c * 32, v);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 w;
          w.x = pack_bf16(f * __uint_as_float(v[8 * u + 0]), f * __uint_as_float(v[8 * u + 1]));
          w.y = pack_bf16(f * __uint_as_float(v[8 * u + 2]), f * __uint_as_float(v[8 * u + 3]));
          w.z = pack_bf16(f * __uint_as_float(v[8 * u + 4]), f * __uint_as_float(v[8 * u + 5]));
          w.w = pack_bf16(f * __uint_as_float(v[8 * u + 6]), f * __uint_as_float(v[8 * u + 7]));
          reinterpret_cast<uint4*>(out + c * 32)[u] = w;
        }
      }
    }
  }

  ptx::pdl_trigger();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4 && lane == 0) mark(11);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// D[z][q] = sum_j dO[z][q][j] * O[b*S+q][h*64+j]; zeroes dq_acc.  Four rows
// per warp: 8 lanes x 8 elements (16-byte loads) per row, 16-byte zero stores.
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
                                     long long ldo, float* __restrict__ dsum, float* __restrict__ dq_acc, int S, int B,
                                     int rows) {
  ptx::pdl_wait();
  ptx::pdl_trigger();
  const int lane = threadIdx.x & 31, sub = lane >> 3, l8 = lane & 7;
  const int groups = (blockDim.x >> 5) * 4;
  for (int row = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4 + sub; row < rows;
       row += gridDim.x * groups) {
    const int z = row / S, q = row % S, b = z % B, h = z / B;
    const uint4 a = reinterpret_cast<const uint4*>(dout + static_cast<long long>(row) * kD)[l8];
    const uint4 c = reinterpret_cast<const uint4*>(out + static_cast<long long>(b * S + q) * ldo + h * kD)[l8];
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c);
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __bfloat1622float2(pa[e]), y = __bfloat1622float2(pc[e]);
      acc += x.x * y.x + x.y * y.y;
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (l8 == 0) dsum[row] = acc;
    float4* zq = reinterpret_cast<float4*>(dq_acc + static_cast<long long>(row) * kD);
    zq[2 * l8] = make_float4(0.f, 0.f, 0.f, 0.f);
    zq[2 * l8 + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// dqkv[b*S+q][h*64+j] = bf16(scale * dq_acc[z][q][j]); two rows per warp,
// 16 lanes x 4 floats per row
__global__ void attn_bwd_dq_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, long long ld,
                                   float scale, int S, int B, int rows) {
  ptx::pdl_wait();
  ptx::pdl_trigger();
  const int lane = threadIdx.x & 31, sub = lane >> 4, l16 = lane & 15;
  const int groups = (blockDim.x >> 5) * 2;
  for (int row = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 2 + sub; row < rows;
       row += gridDim.x * groups) {
    const int z = row / S, q = row % S, b = z % B, h = z / B;
    const float4 v = reinterpret_cast<const float4*>(dq_acc + static_cast<long long>(row) * kD)[l16];
    uint2 w;
    w.x = pack_bf16(scale * v.x, scale * v.y);
    w.y = pack_bf16(scale * v.z, scale * v.w);
    reinterpret_cast<uint2*>(dqkv + static_cast<long long>(b * S + q) * ld + h * kD)[l16] = w;
  }
}

constexpr int kBwdSmem = 1024 + 14 * kTileBytes + 256;

PFN_cuTensorMapEncodeTiled_v12000 encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      throw std::runtime_error("dpl: cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }();
  return fn;
}

CUtensorMap head_map(const void* base, int S, long long mats) {
  CUtensorMap map;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(mats)};
  cuuint64_t strides[2] = {kD * 2, static_cast<cuuint64_t>(S) * kD * 2};
  cuuint32_t box[3] = {kD, kT, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult rc = encode()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw std::runtime_error("dpl attention: tensor map encode failed");
  return map;
}

constexpr int kFwdSmem = 1024 + 4 * kTileBytes + 256 + 2 * 2 * 128 * 4;

}  // namespace

void AttentionOp::prepare(const AttentionDesc& d) {
  if (d.head_dim != kD) throw std::invalid_argument("dpl attention: head dim must be 64");
  if (d.seq % kT != 0) throw std::invalid_argument("dpl attention: sequence length must be a multiple of 128");
  desc_ = d;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
  });
  fwd_map_ = head_map(d.qkv, d.seq, 3LL * d.heads * d.samples);
  if (d.dout) dout_map_ = head_map(d.dout, d.seq, 1LL * d.heads * d.samples);
  ready_ = true;
}

void AttentionOp::forward(cudaStream_t s) const {
  if (!ready_) throw std::logic_error("dpl attention: forward before prepare");
  AttnFwdParams p;
  p.qkv = fwd_map_;
  p.S = desc_.seq;
  p.B = desc_.samples;
  p.heads = desc_.heads;
  p.causal = desc_.causal;
  p.z_count = desc_.heads * desc_.samples;
  p.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(kD));
  p.ctx = static_cast<__nv_bfloat16*>(desc_.ctx);
  p.ldc = desc_.ldc;
  p.lse = desc_.lse;
  p.part = desc_.fwd_part;
  p.flags = desc_.fwd_flags;
  p.n_items = 0;
  p.trace = desc_.trace;
  const int nq = desc_.seq / kT;
  static const bool split_on = [] {
    const char* e = std::getenv("DPL_ATTN_SPLIT");
    return !e || std::atoi(e) != 0;
  }();
  if (split_on && desc_.causal && p.part && p.flags && nq <= 16) {
    // Work items, longest first: query tiles with >= 4 key tiles split in two
    // (the grid is one wave at small batch and the step waits on the longest CTA).
    struct Item { int qt, lo, hi, half; };
    std::vector<Item> items;
    for (int qt = 0; qt < nq; ++qt) {
      const int n = qt + 1;
      if (n >= 4) {
        items.push_back({qt, 0, n / 2, 1});
        items.push_back({qt, n / 2, n, 2});
      } else {
        items.push_back({qt, 0, n, 0});
      }
    }
    std::stable_sort(items.begin(), items.end(),
                     [](const Item& x, const Item& y) { return x.hi - x.lo > y.hi - y.lo; });
    p.n_items = static_cast<int>(items.size());
    for (int i = 0; i < p.n_items; ++i) {
      p.it_qt[i] = static_cast<unsigned char>(items[i].qt);
      p.it_lo[i] = static_cast<unsigned char>(items[i].lo);
      p.it_hi[i] = static_cast<unsigned char>(items[i].hi);
      p.it_half[i] = static_cast<unsigned char>(items[i].half);
    }
  }
  count_launch();
  TimedLaunch timed_("attention_fwd", s, 4.0 * p.z_count * desc_.seq * desc_.seq * kD / (desc_.causal ? 2 : 1));
  const dim3 grid = p.n_items ? dim3(p.z_count, p.n_items) : dim3(nq, p.z_count);
  launch_pdl(attn_fwd_kernel, grid, dim3(kFwdThreads), kFwdSmem, s, p);
}

void AttentionOp::backward(cudaStream_t s) const {
  if (!ready_ || !desc_.dout || !desc_.dqkv || !desc_.dsum || !desc_.dq_acc)
    throw std::logic_error("dpl attention: backward needs dout, dqkv and workspaces");
  const int z_count = desc_.heads * desc_.samples;
  const int rows = z_count * desc_.seq;
  const float scale = 1.0f / std::sqrt(static_cast<float>(kD));
  count_launch(3);
  TimedLaunch timed_("attention_bwd", s, 10.0 * z_count * desc_.seq * desc_.seq * kD / (desc_.causal ? 2 : 1));
  // rows = z * S is a multiple of 4 (S % 128 == 0): a warp's four rows are all valid or all past the end
  launch_pdl(attn_bwd_prep_kernel, dim3(std::min((rows + 31) / 32, 148 * 16)), dim3(256), 0, s,
             static_cast<const __nv_bfloat16*>(desc_.dout), static_cast<const __nv_bfloat16*>(desc_.ctx), desc_.ldc,
             desc_.dsum, desc_.dq_acc, desc_.seq, desc_.samples, rows);
  AttnBwdParams p;
  p.qkv = fwd_map_;
  p.dout = dout_map_;
  p.S = desc_.seq;
  p.B = desc_.samples;
  p.heads = desc_.heads;
  p.causal = desc_.causal;
  p.z_count = z_count;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.lse = desc_.lse;
  p.dsum = desc_.dsum;
  p.dq_acc = desc_.dq_acc;
  p.dqkv = static_cast<__nv_bfloat16*>(desc_.dqkv);
  p.ld = 3LL * desc_.heads * kD;
  p.H = desc_.heads * kD;
  p.trace = desc_.trace;
  const dim3 bgrid = desc_.causal ? dim3(z_count, desc_.seq / kT) : dim3(desc_.seq / kT, z_count);
  launch_pdl(attn_bwd_kernel, bgrid, dim3(kBwdThreads), kBwdSmem, s, p);
  launch_pdl(attn_bwd_dq_kernel, dim3(std::min((rows + 15) / 16, 148 * 16)), dim3(256), 0, s,
             static_cast<const float*>(desc_.dq_acc), p.dqkv, p.ld, scale, desc_.seq, desc_.samples, rows);
}

}  // namespace dpl
