// extern "C" shims over the stage kernels (include/dapple.h, section 3).
#include <cuda_runtime.h>

#include <atomic>
#include <exception>
#include <stdexcept>
#include <string>

#include "dapple.h"
#include "kernels/attention.h"
#include "kernels/elementwise.h"
#include "kernels/lm.h"
#include "kernels/conv.h"
#include "kernels/gemm.h"

namespace dpl {
thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
void count_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

KernelTimer& kernel_timer() {
  static KernelTimer t;
  return t;
}
cudaEvent_t KernelTimer::take() {
  if (used == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return pool[used++];
}
TimedLaunch::TimedLaunch(const char* name, cudaStream_t s, double flops) : s_(s), on_(kernel_timer().enabled) {
  if (!on_) return;
  KernelTimer& t = kernel_timer();
  KernelTimer::Rec r{name, t.take(), t.take(), flops};
  if (t.capturing) cudaEventRecordWithFlags(r.start, s, cudaEventRecordExternal);
  else cudaEventRecord(r.start, s);
  t.recs.push_back(r);
}
TimedLaunch::~TimedLaunch() {
  if (!on_) return;
  KernelTimer& t = kernel_timer();
  if (t.capturing) cudaEventRecordWithFlags(t.recs.back().end, s_, cudaEventRecordExternal);
  else cudaEventRecord(t.recs.back().end, s_);
}

int fail(const std::string& what) {
  g_last_error = what;
  return 1;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(std::string("CUDA: ") + cudaGetErrorString(e));
    return 0;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}
}  // namespace dpl

using dpl::guarded;

extern "C" {

const char* dpl_last_error(void) { return dpl::g_last_error.c_str(); }
const char* dpl_version(void) { return "dapple-b200 0.1 (sm_100a)"; }
long long dpl_k_launch_count(void) { return dpl::g_launches.load(); }

int dpl_k_gemm(const dpl_gemm_desc* d, void* stream) {
  return guarded([&] {
    dpl::GemmDesc g;
    g.M = d->M; g.N = d->N; g.K = d->K; g.batch = d->batch;
    g.A = d->A; g.lda = d->lda; g.a_batch_stride = d->a_batch_stride; g.a_mn_major = d->a_mn_major;
    g.B = d->B; g.ldb = d->ldb; g.b_batch_stride = d->b_batch_stride; g.b_mn_major = d->b_mn_major;
    g.C = d->C; g.ldc = d->ldc; g.zdiv = d->zdiv; g.s_zo = d->s_zo; g.s_zi = d->s_zi;
    g.ndiv = d->ndiv; g.s_no = d->s_no; g.epi = d->epi; g.alpha = d->alpha; g.bias = d->bias;
    g.aux_in = d->aux_in; g.resid = d->resid; g.aux_out = d->aux_out; g.force_bn = d->force_bn; g.force_1sm = d->force_1sm;
    g.trace = d->trace;
    g.colsum = d->colsum;
    g.conv_x = d->conv_x;
    g.conv_operand = d->conv_operand;
    g.conv_n = d->conv_n;
    g.conv_h = d->conv_h;
    g.conv_w = d->conv_w;
    g.conv_c = d->conv_c;
    g.split_ws = d->split_ws;
    g.split_ws_bytes = d->split_ws_bytes;
    dpl::GemmOp op;
    op.prepare(g);
    op.launch(static_cast<cudaStream_t>(stream));
  });
}

int dpl_k_attention_fwd_traced(const void* qkv, void* ctx, long long ldc, float* lse, int samples, int seq, int heads,
                               int causal, long long* trace, void* stream);

int dpl_k_attention_fwd(const void* qkv, void* ctx, long long ldc, float* lse, int samples, int seq, int heads,
                        int causal, void* stream) {
  return dpl_k_attention_fwd_traced(qkv, ctx, ldc, lse, samples, seq, heads, causal, nullptr, stream);
}

int dpl_k_attention_fwd_traced(const void* qkv, void* ctx, long long ldc, float* lse, int samples, int seq, int heads,
                               int causal, long long* trace, void* stream) {
  return guarded([&] {
    dpl::AttentionDesc d;
    d.trace = trace;
    d.qkv = qkv;
    d.ctx = ctx;
    d.ldc = ldc;
    d.lse = lse;
    d.samples = samples;
    d.seq = seq;
    d.heads = heads;
    d.causal = causal;
    const auto st = static_cast<cudaStream_t>(stream);
    void* ws = nullptr;
    const size_t tiles = static_cast<size_t>(heads) * samples * (seq / 128);
    const size_t part_bytes = tiles * 2 * 66 * 128 * sizeof(float);
    if (causal) {  // split-schedule workspace, as the executor provides it
      if (cudaMallocAsync(&ws, part_bytes + tiles * sizeof(int), st) != cudaSuccess)
        throw std::runtime_error("attention_fwd: workspace allocation failed");
      cudaMemsetAsync(static_cast<char*>(ws) + part_bytes, 0, tiles * sizeof(int), st);
      d.fwd_part = static_cast<float*>(ws);
      d.fwd_flags = reinterpret_cast<int*>(static_cast<char*>(ws) + part_bytes);
    }
    dpl::AttentionOp op;
    op.prepare(d);
    op.forward(st);
    if (ws) cudaFreeAsync(ws, st);
  });
}

int dpl_k_attention_bwd_traced(const void* qkv, const void* ctx, long long ldc, const float* lse, const void* dout,
                               void* dqkv, float* dsum, float* dq_acc, int samples, int seq, int heads, int causal,
                               long long* trace, void* stream);

int dpl_k_attention_bwd(const void* qkv, const void* ctx, long long ldc, const float* lse, const void* dout,
                        void* dqkv, float* dsum, float* dq_acc, int samples, int seq, int heads, int causal,
                        void* stream) {
  return dpl_k_attention_bwd_traced(qkv, ctx, ldc, lse, dout, dqkv, dsum, dq_acc, samples, seq, heads, causal, nullptr,
                                    stream);
}

int dpl_k_attention_bwd_traced(const void* qkv, const void* ctx, long long ldc, const float* lse, const void* dout,
                               void* dqkv, float* dsum, float* dq_acc, int samples, int seq, int heads, int causal,
                               long long* trace, void* stream) {
  return guarded([&] {
    dpl::AttentionDesc d;
    d.trace = trace;
    d.qkv = qkv;
    d.ctx = const_cast<void*>(ctx);
    d.ldc = ldc;
    d.lse = const_cast<float*>(lse);
    d.dout = dout;
    d.dqkv = dqkv;
    d.dsum = dsum;
    d.dq_acc = dq_acc;
    d.samples = samples;
    d.seq = seq;
    d.heads = heads;
    d.causal = causal;
    dpl::AttentionOp op;
    op.prepare(d);
    op.backward(static_cast<cudaStream_t>(stream));
  });
}

int dpl_k_layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y, float* mean, float* rstd,
                        int rows, int h, float eps, void* stream) {
  return guarded([&] { dpl::layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, h, eps, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gamma,
                        const void* dresid, void* dx, float* dgamma, float* dbeta, int rows, int h, void* stream) {
  return guarded([&] {
    float* ws = nullptr;
    const size_t bytes = static_cast<size_t>(dpl::kLnBwdBlocks) * 4 * h * sizeof(float);
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, static_cast<cudaStream_t>(stream)) != cudaSuccess)
      throw std::runtime_error("layernorm_bwd: workspace allocation failed");
    dpl::layernorm_bwd(dy, x, mean, rstd, gamma, dresid, dx, dgamma, dbeta, rows, h, static_cast<cudaStream_t>(stream),
                       ws);
    cudaFreeAsync(ws, static_cast<cudaStream_t>(stream));
  });
}

int dpl_k_layernorm_bwd_colsum(const void* dy, const void* x, const float* mean, const float* rstd, const float* gamma,
                               const void* dresid, void* dx, float* dgamma, float* dbeta, float* dresid_colsum,
                               float* dx_colsum, int rows, int h, void* stream) {
  return guarded([&] {
    float* ws = nullptr;
    const size_t bytes = static_cast<size_t>(dpl::kLnBwdBlocks) * 4 * h * sizeof(float);
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, static_cast<cudaStream_t>(stream)) != cudaSuccess)
      throw std::runtime_error("layernorm_bwd: workspace allocation failed");
    dpl::layernorm_bwd(dy, x, mean, rstd, gamma, dresid, dx, dgamma, dbeta, rows, h, static_cast<cudaStream_t>(stream),
                       ws, dresid_colsum, dx_colsum);
    cudaFreeAsync(ws, static_cast<cudaStream_t>(stream));
  });
}

int dpl_k_softmax_fwd(const float* s, void* p, int rows, int len, int q_len, int causal, void* stream) {
  return guarded([&] { dpl::softmax_fwd(s, p, rows, len, q_len, causal, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_softmax_bwd(const void* p, const float* dp, void* ds, int rows, int len, void* stream) {
  return guarded([&] { dpl::softmax_bwd(p, dp, ds, rows, len, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_colsum_acc(const void* dy, float* db, int rows, int cols, void* stream) {
  return guarded([&] { dpl::colsum_acc(dy, db, rows, cols, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_mse_loss(const void* y, const void* t, void* dy, float* loss_acc, long long n, float grad_scale,
                   void* stream) {
  return guarded([&] { dpl::mse_loss(y, t, dy, loss_acc, n, grad_scale, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_fill_tokens(int* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, int vocab, void* stream) {
  return guarded([&] { dpl::fill_tokens(dst, n, seed, tensor, idx0, vocab, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_embed_fwd(const int* tok, const void* wte, const void* wpe, void* x, int rows, int seq, int h, void* stream) {
  return guarded([&] { dpl::embed_fwd(tok, wte, wpe, x, rows, seq, h, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_embed_bwd(const int* tok, const void* dx, float* gwte, float* gwpe, int rows, int seq, int h, void* stream) {
  return guarded([&] { dpl::embed_bwd(tok, dx, gwte, gwpe, rows, seq, h, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_cross_entropy_padded(void* logits, const int* tgt, float* loss_acc, int rows, int vocab, int ld,
                               float grad_scale, void* stream) {
  return guarded([&] {
    dpl::cross_entropy_fwd_bwd(logits, tgt, loss_acc, rows, vocab, grad_scale, static_cast<cudaStream_t>(stream), ld);
  });
}

int dpl_k_cross_entropy(void* logits, const int* tgt, float* loss_acc, int rows, int vocab, float grad_scale,
                        void* stream) {
  return guarded(
      [&] { dpl::cross_entropy_fwd_bwd(logits, tgt, loss_acc, rows, vocab, grad_scale, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_im2col3x3(const void* x, void* col, int n, int h, int w, int c, int kp, void* stream) {
  return guarded([&] { dpl::im2col3x3(x, col, n, h, w, c, kp, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_col2im3x3(const void* dcol, void* dx, int n, int h, int w, int c, int kp, void* stream) {
  return guarded([&] { dpl::col2im3x3(dcol, dx, n, h, w, c, kp, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_maxpool2_fwd(const void* x, void* y, int n, int h, int w, int c, void* stream) {
  return guarded([&] { dpl::maxpool2_fwd(x, y, n, h, w, c, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_maxpool2_relu_bwd(const void* x, const void* dy, void* dz, int n, int h, int w, int c, void* stream) {
  return guarded([&] { dpl::maxpool2_relu_bwd(x, dy, dz, n, h, w, c, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_relu_bwd(const void* y, const void* dy, void* dz, long long n, void* stream) {
  return guarded([&] { dpl::relu_bwd(y, dy, dz, n, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_sgd_apply(float* w32, float* g, void* w16, long long n, float lr, void* stream) {
  return guarded([&] { dpl::sgd_apply(w32, g, w16, n, lr, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_fill_uniform_bf16(void* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                            void* stream) {
  return guarded([&] { dpl::fill_uniform_bf16(dst, n, seed, tensor, idx0, scale, static_cast<cudaStream_t>(stream)); });
}

int dpl_k_fill_uniform_f32(float* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                           void* stream) {
  return guarded([&] { dpl::fill_uniform_f32(dst, n, seed, tensor, idx0, scale, static_cast<cudaStream_t>(stream)); });
}

}  // extern "C"
