// Stage layers for the executor: the per-layer forward / backward programs
// built from the sm_100a kernels.  A "layer" is one profile layer
// (LayerProfile, model.hpp:16-22): one Linear+ReLU for the MLP family, one
// pre-LN transformer block for BERT / GPT.
//
// Gradient contract between consecutive layers (also across the stage
// boundary, where it travels through Split-Concat):
//   * MLP:        grad w.r.t. the layer's *pre-activation* output (dZ); the
//                 consumer layer applies relu'(x) to the dX it produces, so
//                 the activation derivative is fused into the dgrad GEMM.
//   * transformer: grad w.r.t. the block output (residual stream).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "kernels/gemm.h"

namespace dpl {

using bf16 = __nv_bfloat16;

struct ModelSpec {
  std::string kind = "mlp";  // "mlp" | "bert" | "gpt"
  int layers = 16;
  int hidden = 1024;
  int heads = 16;
  int ffn = 4096;
  int seq = 1;  // tokens per sample (1 for the MLP)
  bool causal = false;
  float ln_eps = 1e-5f;
  int vocab = 0;  // > 0: GPT language model (token ids in, cross-entropy out)
  // VGG-19 (kind "vgg", config C3): NHWC images image x image x 3, conv
  // widths width x {1, 2, 4, 8, 8} (2, 2, 4, 4, 4 convs, 2x2 max pool after
  // each group), FC fc -> fc -> classes; cross-entropy over classes.
  // The same family with other groups ("convs" per group, width "mults",
  // "fcs" = 3: fc, fc, classes or 1: classes only) gives the deeper conv
  // stand-ins (C5's AmoebaNet-36 shape: 12 + 12 + 11 convs + classifier).
  int image = 224, width = 64, fc = 4096, classes = 1000;
  std::vector<int> convs = {2, 2, 4, 4, 4}, mults = {1, 2, 4, 8, 8};
  int fcs = 3;
  int conv_layers() const {
    int n = 0;
    for (int c : convs) n += c;
    return n;
  }
};

// One VGG profile layer: a 3x3 conv (+ReLU, + optional 2x2 pool) or an FC.
struct VggLayerShape {
  bool conv = false;
  int h = 0, w = 0, cin = 0, cout = 0, kp = 0;  // conv: input spatial size, channels, padded K = 9 cin
  bool pool = false;
  int fin = 0, fout = 0;  // fc
  bool relu = true;
};
VggLayerShape vgg_layer(const ModelSpec& spec, int l);
// activation elements per sample entering global layer l (l == layers: the model output)
long long elems_per_sample(const ModelSpec& spec, int l);

// Device memory owned by one stage replica (freed by the executor).
class DeviceMemory {
 public:
  ~DeviceMemory();
  void* alloc(size_t bytes);  // 256-byte aligned, zero-initialised on stream()
  size_t total() const { return total_; }
  void set_stream(cudaStream_t s) { stream_ = s; }

 private:
  cudaStream_t stream_ = nullptr;
  std::vector<void*> blocks_;
  size_t total_ = 0;
};

// Per-replica context shared by the layers of a stage.
struct StageContext {
  ModelSpec spec;
  int rows = 0;     // token rows per micro-batch slice (samples * seq)
  int samples = 0;  // samples per micro-batch slice
  int slots = 1;    // activation stash depth (phi of this stage)
  cudaStream_t stream = nullptr;
  // Weight-gradient side stream of the backward: the wgrad GEMMs of a
  // layer run there beside the dgrad chain on `stream`, forked and joined
  // with the two events below inside the layer (null: everything on stream)
  cudaStream_t wstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // run f(stream) on the side stream after everything issued so far on `stream`
  // (side-stream GEMM grids capped at wgrad_ctas CTAs when nonzero, so the
  // critical-path stream keeps SMs)
  int wgrad_ctas = 0;
  template <typename F>
  void on_side(F&& f) {
    if (!wstream) {
      f(stream);
      return;
    }
    cudaEventRecord(ev_fork, stream);
    cudaStreamWaitEvent(wstream, ev_fork, 0);
    gemms.max_ctas_override = wgrad_ctas;
    f(wstream);
    gemms.max_ctas_override = 0;
  }
  // `stream` waits for the side stream's work so far
  void join_side() {
    if (!wstream) return;
    cudaEventRecord(ev_join, wstream);
    cudaStreamWaitEvent(stream, ev_join, 0);
  }
  GemmCache gemms;
  DeviceMemory* mem = nullptr;
  // shared scratch (transformer backward / attention)
  float* scores = nullptr;  // fp32 [z][s][s]  (S in forward, dP in backward)
  bf16* dscores = nullptr;  // bf16 [z][s][s]
  bf16* t_h = nullptr;      // [R][H] scratch
  bf16* t_h2 = nullptr;     // [R][H] scratch
  bf16* t_h3 = nullptr;     // [R][H] scratch (head layout)
  bf16* t_qkv = nullptr;    // [R][3H]
  bf16* t_f = nullptr;      // [R][F]
  float* att_dsum = nullptr;  // attention backward workspaces: [z][S]
  float* att_dq = nullptr;    // [z][S][64]
  float* att_part = nullptr;  // causal forward split partials, flags (AttentionDesc::fwd_part / fwd_flags)
  int* att_flags = nullptr;
  float* ln_ws = nullptr;     // LayerNorm-backward partials [kLnBwdBlocks][2][H]
  bf16* conv_col = nullptr;   // VGG: im2col columns (max over the stage's convs)
  bf16* conv_dcol = nullptr;  // VGG: column gradients
  bf16* conv_dz = nullptr;    // VGG: gradient w.r.t. the conv / FC pre-activation
  const bf16* cur_y = nullptr;  // output of the layer whose backward runs (set by the executor)
  double flops_fwd = 0.0, flops_bwd = 0.0;  // per micro-batch slice (accounting)
};

class Layer {
 public:
  virtual ~Layer() = default;
  // number of fp32 parameters and their (tensor id, count, init scale) list
  virtual size_t param_count() const = 0;
  // binds parameter / gradient / bf16-copy views and initialises weights
  virtual void bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s) = 0;
  virtual void alloc_stash(StageContext& ctx) = 0;
  virtual void forward(StageContext& ctx, int slot, const bf16* x, bf16* y) = 0;
  // dx may be null (first layer of the model: no input gradient needed)
  virtual void backward(StageContext& ctx, int slot, const bf16* x, const bf16* dy, bf16* dx) = 0;
  virtual double flops_fwd(const StageContext& ctx) const = 0;
  virtual double flops_bwd(const StageContext& ctx, bool need_dx) const = 0;
  // named tensors for parity reads: (name, offset into the layer's params, count)
  struct Named {
    std::string name;
    size_t offset;
    size_t count;
  };
  virtual std::vector<Named> tensors() const = 0;
  // scratch the layer needs in StageContext (VGG): columns, dz (elements)
  virtual size_t col_elems(const StageContext&) const { return 0; }
  virtual size_t dz_elems(const StageContext&) const { return 0; }
  // a stashed intermediate the backward reads besides x / y (parity probes):
  // the post-ReLU pre-pool conv output of a pooling VGG layer
  virtual const bf16* probe_aux(int) const { return nullptr; }
  virtual size_t probe_aux_elems(const StageContext&) const { return 0; }
};

std::unique_ptr<Layer> make_layer(const ModelSpec& spec, int global_index);

// GPT language-model ends (config C4).  Not profile layers of their own:
// the embedding runs inside the first stage's F/B blocks before layer 0 /
// after its backward, the head inside the last stage's blocks after the
// last layer ("head on stage 7").
//   x = wte[tok] + wpe[pos]                       (TokenEmbedding)
//   loss = CE(LN_f(y) Wout^T, tgt)               (LmHead; Wout [V][H], untied)
class TokenEmbedding {
 public:
  explicit TokenEmbedding(const ModelSpec& spec) : v_(spec.vocab), h_(spec.hidden), seq_(spec.seq) {}
  size_t param_count() const { return static_cast<size_t>(v_) * h_ + static_cast<size_t>(seq_) * h_; }
  void bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s);
  void forward(StageContext& ctx, const int* tok, bf16* x);
  void backward(StageContext& ctx, const int* tok, const bf16* dx);
  std::vector<Layer::Named> tensors() const;

 private:
  int v_, h_, seq_;
  float* g32_ = nullptr;
  bf16* w16_ = nullptr;
};

class LmHead {
 public:
  // the vocabulary projection is stored with vp_ = vocab rounded up to 8 rows
  // (50257 -> 50264 for GPT-2): the padding rows stay zero, their logits are
  // masked out of the softmax and get no gradient
  explicit LmHead(const ModelSpec& spec)
      : v_(spec.vocab), vp_((spec.vocab + 7) / 8 * 8), h_(spec.hidden), eps_(spec.ln_eps) {}
  size_t param_count() const { return 2 * static_cast<size_t>(h_) + static_cast<size_t>(vp_) * h_; }
  void bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s);
  void alloc_stash(StageContext& ctx, int slots);
  // y: the last block's output; accumulates sum_rows CE into loss_acc and
  // leaves (softmax - onehot) * grad_scale of this slot for backward
  void forward(StageContext& ctx, int slot, const bf16* y, const int* tgt, float* loss_acc, float grad_scale);
  // dy <- gradient w.r.t. y; Wout / LN_f gradients accumulated
  void backward(StageContext& ctx, int slot, const bf16* y, bf16* dy);
  double flops_fwd(const StageContext& ctx) const { return 2.0 * ctx.rows * static_cast<double>(v_) * h_; }
  double flops_bwd(const StageContext& ctx) const { return 4.0 * ctx.rows * static_cast<double>(v_) * h_; }
  std::vector<Layer::Named> tensors() const;

 private:
  int v_, vp_, h_;
  float eps_;
  float* w32_ = nullptr;
  float* g32_ = nullptr;
  bf16* w16_ = nullptr;
  struct Slot {
    bf16* xn;
    float* mean;
    float* rstd;
    bf16* dlogits;  // [R][Vp]: logits, then in place their gradient
  };
  std::vector<Slot> slots_;
  bf16* dxn_ = nullptr;
};

// LM tensor ids (shared with oracle/executor_ref.py init_lm / lm_tokens)
constexpr uint64_t kTensorWte = 100;
constexpr uint64_t kTensorWpe = 101;
constexpr uint64_t kTensorWout = 112;

// Synthetic data tensor ids (shared with oracle/executor_ref.py).
constexpr uint64_t kTensorInput = 1;
constexpr uint64_t kTensorTarget = 2;
inline uint64_t param_tensor_id(int layer, int t) { return 1000ull + static_cast<uint64_t>(layer) * 16ull + t; }

}  // namespace dpl
