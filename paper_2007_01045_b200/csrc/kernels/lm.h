// Host launchers for the language-model ends of a GPT stage pipeline
// (lm.cu): synthetic token ids, token + position embedding forward /
// backward, and the fused softmax cross-entropy over the vocabulary.
// All HBM-bound; rows are token rows, h and vocab multiples of 8.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dpl {

// dst[i] = (splitmix64(seed, tensor, idx0 + i) >> 32) % vocab   (oracle: lm_tokens)
void fill_tokens(int* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, int vocab, cudaStream_t s);
// x[r] = bf16(wte[tok[r]] + wpe[r % seq])
void embed_fwd(const int* tok, const void* wte, const void* wpe, void* x, int rows, int seq, int h, cudaStream_t s);
// gwte[tok[r]] += dx[r] ; gwpe[r % seq] += dx[r]   (fp32 vector atomics)
void embed_bwd(const int* tok, const void* dx, float* gwte, float* gwpe, int rows, int seq, int h, cudaStream_t s);
// Per row r of logits [rows][ld] (bf16; ld = vocab rounded up to 8, 0 = vocab):
// loss_acc += logsumexp(row[:vocab]) - row[tgt[r]] and, in place,
// row <- bf16((softmax(row[:vocab]) - onehot(tgt[r])) * grad_scale), padding 0.
void cross_entropy_fwd_bwd(void* logits, const int* tgt, float* loss_acc, int rows, int vocab, float grad_scale,
                           cudaStream_t s, int ld = 0);

}  // namespace dpl
