// In-stage replica gradient AllReduce over peer memory (N4; PAPER.md:1248-1252,
// cost model costmodel.cpp:41-50).  The flag rounds around it are stream
// memory operations issued by the executor (executor.cu signal / wait_flag).
//
// Replica j of an r-way stage owns chunk j of every parameter block.  When
// all r replicas have signalled that a block's gradients are final, replica j
// reads chunk j from the r fp32 gradient buffers (its own plus r-1 peer
// mappings over NVLink), sums them in replica order 0..r-1 and stores the sum
// back into all r buffers.  Every element is reduced by exactly one rank in a
// fixed order, so all replicas end bit-identical and the result does not
// depend on timing.  Per rank this moves (r-1)/r of the block in and
// (r-1)/r out over the links -- the ring AllReduce's 2(r-1)/r -- in one
// kernel and two flag rounds instead of a ring's 2(r-1) steps.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "collective.h"
#include "launch.cuh"

namespace dpl {

namespace {

__global__ void __launch_bounds__(256) replica_sum_kernel(ReplicaPtrs ptrs, int r, long long lo, long long hi) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // 16-byte body: lo / hi are multiples of 4 floats except possibly hi == n
  const long long lo4 = (lo + 3) / 4, hi4 = hi / 4;
  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  constexpr int kU = 4;  // independent 16-byte loads per replica in flight per thread
  for (long long base = lo4 + tid; base < hi4; base += stride * kU) {
    float4 acc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long i = base + u * stride;
      acc[u] = i < hi4 ? __ldcv(reinterpret_cast<const float4*>(ptrs.g[0]) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int q = 1; q < r; ++q) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const long long i = base + u * stride;
        if (i < hi4) {
          const float4 v = __ldcv(reinterpret_cast<const float4*>(ptrs.g[q]) + i);
          acc[u].x += v.x;
          acc[u].y += v.y;
          acc[u].z += v.z;
          acc[u].w += v.w;
        }
      }
    }
    for (int q = 0; q < r; ++q) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const long long i = base + u * stride;
        if (i < hi4) __stcg(reinterpret_cast<float4*>(ptrs.g[q]) + i, acc[u]);
      }
    }
  }
  // scalar tail (a block whose length is not a multiple of 4)
  for (long long i = hi4 * 4 + tid; i < hi; i += stride) {
    if (i < lo) continue;
    float acc = __ldcv(ptrs.g[0] + i);
    for (int q = 1; q < r; ++q) acc += __ldcv(ptrs.g[q] + i);
    for (int q = 0; q < r; ++q) __stcg(ptrs.g[q] + i, acc);
  }
}

}  // namespace

long long replica_chunk_lo(long long n, int j, int r) {
  if (j <= 0) return 0;
  if (j >= r) return n;
  return (n * j / r) / 64 * 64;  // 256-byte aligned chunk starts
}

void replica_allreduce_chunk(const ReplicaPtrs& ptrs, int r, long long n, int j, cudaStream_t s) {
  if (r < 1 || r > kMaxReplicas) throw std::invalid_argument("dpl: replica count out of range");
  const long long lo = replica_chunk_lo(n, j, r), hi = replica_chunk_lo(n, j + 1, r);
  if (hi <= lo) return;
  count_launch();
  TimedLaunch timed_("replica_allreduce", s);
  const long long vec = (hi - lo + 3) / 4;
  const int blocks = static_cast<int>(std::min<long long>(64, std::max<long long>(1, (vec + 1023) / 1024)));
  launch_pdl(replica_sum_kernel, dim3(blocks), dim3(256), 0, s, ptrs, r, lo, hi);
}

}  // namespace dpl
