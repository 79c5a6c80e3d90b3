// Fused attention (attention.cu).  qkv is head-split [3][heads][B][S][64];
// ctx is written head-merged into [B*S][ldc] (col = head*64 + j); lse is
// [heads*B][S] fp32 (natural log-sum-exp of the scaled scores).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

namespace dpl {

struct AttentionDesc {
  const void* qkv = nullptr;
  void* ctx = nullptr;
  long long ldc = 0;
  float* lse = nullptr;
  int samples = 1, seq = 128, heads = 1, head_dim = 64;
  int causal = 0;
  // backward: dO head-split [heads][B][S][64]; dqkv [B*S][3H] (dQ, dK, dV
  // written head-merged); workspaces dsum [heads*B][S], dq_acc [heads*B][S][64]
  const void* dout = nullptr;
  void* dqkv = nullptr;
  float* dsum = nullptr;
  float* dq_acc = nullptr;
  // causal forward split (optional): query tiles with >= 4 key tiles run as
  // two CTAs over halves of the key range, the second to finish merges.
  // fwd_part [heads*B][S/128][2][66][128] fp32, fwd_flags [heads*B][S/128]
  // int (zero before the first call; the merging CTA re-zeroes its entry).
  float* fwd_part = nullptr;
  int* fwd_flags = nullptr;
  // diagnostics (tools/attn_trace.py): per-CTA %globaltimer marks of the
  // forward, 16 slots per CTA; null in the product path
  long long* trace = nullptr;
};

class AttentionOp {
 public:
  void prepare(const AttentionDesc& d);
  void forward(cudaStream_t s) const;
  void backward(cudaStream_t s) const;

 private:
  AttentionDesc desc_;
  CUtensorMap fwd_map_{};
  CUtensorMap dout_map_{};
  bool ready_ = false;
};

}  // namespace dpl
