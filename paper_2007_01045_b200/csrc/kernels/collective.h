// Peer-memory replica AllReduce (collective.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gemm.h"

namespace dpl {

constexpr int kMaxReplicas = 16;

// fp32 gradient buffers of the r replicas (replica order), each at the same
// parameter-block offset; peers' buffers are peer mappings (CUDA IPC, or plain
// pointers for ranks sharing this process)
struct ReplicaPtrs {
  float* g[kMaxReplicas];
};

// first element of replica j's chunk of an n-element block (256-byte aligned)
long long replica_chunk_lo(long long n, int j, int r);
// sum chunk j of the block over the r buffers (replica order) and store the
// sum into all of them
void replica_allreduce_chunk(const ReplicaPtrs& ptrs, int r, long long n, int j, cudaStream_t s);

}  // namespace dpl
