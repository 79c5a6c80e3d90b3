// Layer programs (see layers.h).  Every projection is the tcgen05 GEMM with
// bias, residual, GELU / ReLU and their derivatives, fp32 micro-batch
// gradient accumulation and the attention head split in its epilogue;
// attention itself is the fused flash kernel (kernels/attention.cu), so the
// only other kernels are LayerNorm and the bias-gradient column sums.
#include <cmath>
#include <cstdlib>
#include <stdexcept>

#include "kernels/attention.h"
#include "kernels/elementwise.h"
#include "kernels/conv.h"
#include "kernels/lm.h"
#include "layers.h"

namespace dpl {

DeviceMemory::~DeviceMemory() {
  cudaDeviceSynchronize();
  for (void* p : blocks_) cudaFree(p);
}

void* DeviceMemory::alloc(size_t bytes) {
  if (bytes == 0) bytes = 256;
  bytes = (bytes + 255) & ~size_t(255);
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error("dpl: cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  }
  // zero on a stream the executor orders against (it synchronises the
  // device before any other work), never on the legacy default stream
  if (cudaMemsetAsync(p, 0, bytes, stream_) != cudaSuccess) throw std::runtime_error("dpl: cudaMemsetAsync failed");
  blocks_.push_back(p);
  total_ += bytes;
  return p;
}

namespace {

template <typename T>
T* alloc_n(StageContext& ctx, size_t n) {
  return static_cast<T*>(ctx.mem->alloc(n * sizeof(T)));
}

GemmDesc plain(int M, int N, int K, const void* A, long long lda, bool a_mn, const void* B, long long ldb, bool b_mn,
               void* C, long long ldc, uint32_t epi) {
  GemmDesc d;
  d.M = M;
  d.N = N;
  d.K = K;
  d.A = A;
  d.lda = lda;
  d.a_mn_major = a_mn;
  d.B = B;
  d.ldb = ldb;
  d.b_mn_major = b_mn;
  d.C = C;
  d.ldc = ldc;
  d.s_zo = static_cast<long long>(M) * ldc;
  d.epi = epi;
  return d;
}

struct ParamInit {
  size_t offset;
  size_t count;
  int tid;
  float scale;  // U(-scale, scale); NaN = constant 1 (LayerNorm gamma)
};

void init_params(const std::vector<ParamInit>& plan, int layer, float* w32, bf16* w16, size_t total, uint64_t seed,
                 cudaStream_t s) {
  for (const ParamInit& p : plan) {
    if (std::isnan(p.scale)) {
      fill_const_f32(w32 + p.offset, static_cast<long long>(p.count), 1.0f, s);
    } else {
      fill_uniform_f32(w32 + p.offset, static_cast<long long>(p.count), seed, param_tensor_id(layer, p.tid), 0,
                       p.scale, s);
    }
  }
  cast_f32_bf16(w32, w16, static_cast<long long>(total), s);
}

// ------------------------------------------------------------------ MLP
// y = relu(x W^T + b) (no ReLU on the model's last layer); W [H][H].
class MlpLayer final : public Layer {
 public:
  MlpLayer(const ModelSpec& spec, int index)
      : h_(spec.hidden), index_(index), relu_(index != spec.layers - 1), in_relu_(index > 0) {}

  size_t param_count() const override { return static_cast<size_t>(h_) * h_ + h_; }

  void bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s) override {
    w32_ = w32;
    g32_ = g32;
    w16_ = w16;
    const size_t hh = static_cast<size_t>(h_) * h_;
    init_params({{0, hh, 0, std::sqrt(6.0f / h_)}, {hh, static_cast<size_t>(h_), 1, 0.05f}}, index_, w32, w16,
                param_count(), seed, s);
  }

  void alloc_stash(StageContext&) override {}

  void forward(StageContext& ctx, int, const bf16* x, bf16* y) override {
    GemmDesc d = plain(ctx.rows, h_, h_, x, h_, false, w16_, h_, false, y, h_, kBias | (relu_ ? kRelu : 0u));
    d.bias = bias32();
    ctx.gemms.run(d, ctx.stream);
  }

  void backward(StageContext& ctx, int, const bf16* x, const bf16* dz, bf16* dx) override {
    const int R = ctx.rows;
    // dW += dZ^T X  (both operands read transposed from their row-major forms),
    // db: on the weight-gradient side stream, joined below
    ctx.on_side([&](cudaStream_t s) {
      ctx.gemms.run(plain(h_, h_, R, dz, h_, true, x, h_, true, g32_, h_, kOutF32Acc), s);
      colsum_acc(dz, g32_ + static_cast<size_t>(h_) * h_, R, h_, s);
    });
    if (dx) {
      // dX = dZ W, with the previous layer's relu'(x) fused in the epilogue
      GemmDesc d = plain(R, h_, h_, dz, h_, false, w16_, h_, true, dx, h_, in_relu_ ? kDRelu : 0u);
      d.aux_in = x;
      ctx.gemms.run(d, ctx.stream);
    }
    ctx.join_side();
  }

  double flops_fwd(const StageContext& ctx) const override { return 2.0 * ctx.rows * h_ * h_; }
  double flops_bwd(const StageContext& ctx, bool need_dx) const override {
    return (need_dx ? 4.0 : 2.0) * ctx.rows * h_ * h_;
  }
  std::vector<Named> tensors() const override {
    return {{"W", 0, static_cast<size_t>(h_) * h_}, {"b", static_cast<size_t>(h_) * h_, static_cast<size_t>(h_)}};
  }

 private:
  const float* bias32() const { return w32_ + static_cast<size_t>(h_) * h_; }
  int h_, index_;
  bool relu_, in_relu_;
  float* w32_ = nullptr;
  float* g32_ = nullptr;
  bf16* w16_ = nullptr;
};

// ------------------------------------------------------------------ transformer
// Pre-LN block:  h = x + Wo·attn(LN1 x) + bo ;  y = h + W2·gelu(W1·LN2 h + b1) + b2
class TransformerLayer final : public Layer {
 public:
  TransformerLayer(const ModelSpec& spec, int index)
      : H_(spec.hidden), F_(spec.ffn), nh_(spec.heads), d_(spec.hidden / spec.heads), causal_(spec.causal),
        eps_(spec.ln_eps), index_(index) {
    if (H_ % nh_ != 0 || d_ % 32 != 0) throw std::invalid_argument("dpl: head dim must be a multiple of 32");
    size_t o = 0;
    auto add = [&](size_t n) {
      const size_t at = o;
      o += n;
      return at;
    };
    ln1g_ = add(H_);
    ln1b_ = add(H_);
    wqkv_ = add(3ull * H_ * H_);
    bqkv_ = add(3ull * H_);
    wo_ = add(1ull * H_ * H_);
    bo_ = add(H_);
    ln2g_ = add(H_);
    ln2b_ = add(H_);
    w1_ = add(1ull * F_ * H_);
    b1_ = add(F_);
    w2_ = add(1ull * H_ * F_);
    b2_ = add(H_);
    total_ = o;
  }

  size_t param_count() const override { return total_; }

  void bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s) override {
    w32_ = w32;
    g32_ = g32;
    w16_ = w16;
    const float nan = std::nanf("");
    const float sh = 1.0f / std::sqrt(static_cast<float>(H_));
    const float sf = 1.0f / std::sqrt(static_cast<float>(F_));
    init_params({{ln1g_, size_t(H_), 0, nan},
                 {ln1b_, size_t(H_), 1, 0.0f},
                 {wqkv_, 3ull * H_ * H_, 2, sh},
                 {bqkv_, 3ull * H_, 3, 0.02f},
                 {wo_, 1ull * H_ * H_, 4, sh},
                 {bo_, size_t(H_), 5, 0.02f},
                 {ln2g_, size_t(H_), 6, nan},
                 {ln2b_, size_t(H_), 7, 0.0f},
                 {w1_, 1ull * F_ * H_, 8, sh},
                 {b1_, size_t(F_), 9, 0.02f},
                 {w2_, 1ull * H_ * F_, 10, sf},
                 {b2_, size_t(H_), 11, 0.02f}},
                index_, w32, w16, total_, seed, s);
  }

  void alloc_stash(StageContext& ctx) override {
    const size_t R = ctx.rows;
    const size_t z = static_cast<size_t>(nh_) * ctx.samples;
    stash_.resize(ctx.slots);
    for (Stash& st : stash_) {
      st.ln1 = alloc_n<bf16>(ctx, R * H_);
      st.mean1 = alloc_n<float>(ctx, R);
      st.rstd1 = alloc_n<float>(ctx, R);
      st.qkv = alloc_n<bf16>(ctx, 3 * R * H_);
      st.lse = alloc_n<float>(ctx, z * ctx.spec.seq);
      st.ctx = alloc_n<bf16>(ctx, R * H_);
      st.h = alloc_n<bf16>(ctx, R * H_);
      st.ln2 = alloc_n<bf16>(ctx, R * H_);
      st.mean2 = alloc_n<float>(ctx, R);
      st.rstd2 = alloc_n<float>(ctx, R);
      st.z1 = alloc_n<bf16>(ctx, R * F_);
      st.g = alloc_n<bf16>(ctx, R * F_);
    }
  }

  void forward(StageContext& ctx, int slot, const bf16* x, bf16* y) override {
    Stash& st = stash_[slot];
    const int R = ctx.rows;
    cudaStream_t str = ctx.stream;
    layernorm_fwd(x, w32_ + ln1g_, w32_ + ln1b_, st.ln1, st.mean1, st.rstd1, R, H_, eps_, str);
    {  // QKV with head-split store: [3][heads][b][s][d]
      GemmDesc d = plain(R, 3 * H_, H_, st.ln1, H_, false, w16_ + wqkv_, H_, false, st.qkv, d_, kBias);
      d.ndiv = d_;
      d.s_no = static_cast<long long>(R) * d_;
      d.bias = w32_ + bqkv_;
      ctx.gemms.run(d, str);
    }
    // fused flash attention: context head-merged into [R][H], lse stashed
    attention(ctx, slot).forward(str);
    {  // h = x + ctx Wo^T + bo
      GemmDesc d = plain(R, H_, H_, st.ctx, H_, false, w16_ + wo_, H_, false, st.h, H_, kBias | kResid);
      d.bias = w32_ + bo_;
      d.resid = x;
      ctx.gemms.run(d, str);
    }
    layernorm_fwd(st.h, w32_ + ln2g_, w32_ + ln2b_, st.ln2, st.mean2, st.rstd2, R, H_, eps_, str);
    {  // g = gelu(ln2 W1^T + b1), z1 = pre-activation
      GemmDesc d = plain(R, F_, H_, st.ln2, H_, false, w16_ + w1_, H_, false, st.g, F_, kBias | kGelu | kAuxOut);
      d.bias = w32_ + b1_;
      d.aux_out = st.z1;
      ctx.gemms.run(d, str);
    }
    {  // y = h + g W2^T + b2
      GemmDesc d = plain(R, H_, F_, st.g, F_, false, w16_ + w2_, F_, false, y, H_, kBias | kResid);
      d.bias = w32_ + b2_;
      d.resid = st.h;
      ctx.gemms.run(d, str);
    }
  }

  void backward(StageContext& ctx, int slot, const bf16* x, const bf16* dy, bf16* dx) override {
    Stash& st = stash_[slot];
    const int R = ctx.rows;
    cudaStream_t str = ctx.stream;
    bf16* dz1 = ctx.t_f;
    bf16* dln = ctx.t_h;
    bf16* dh = ctx.t_h2;
    bf16* dctx_h = ctx.t_h3;
    bf16* dqkv = ctx.t_qkv;

    // Weight gradients go to the side stream (ctx.on_side) beside the dgrad
    // chain; each reads only buffers the chain does not write before the
    // join at the end of this layer, and they accumulate into W* gradients
    // the chain never touches.
    // FFN2: dW2 += dy^T g ; db2 ; dz1 = (dy W2) * gelu'(z1)
    ctx.on_side([&](cudaStream_t s) {
      ctx.gemms.run(plain(H_, F_, R, dy, H_, true, st.g, F_, true, g32_ + w2_, F_, kOutF32Acc), s);
    });
    {
      // db1 = colsum(dz1) accumulated by the epilogue from the staged chunks
      GemmDesc d = plain(R, F_, H_, dy, H_, false, w16_ + w2_, F_, true, dz1, F_, kDGelu | kColSum);
      d.aux_in = st.z1;
      d.colsum = g32_ + b1_;
      ctx.gemms.run(d, str);
    }
    // FFN1: dW1 += dz1^T ln2 ; dln2 = dz1 W1
    // With a full-machine side grid (4096-row slices), fork dW1 after the
    // LN2 backward so the persistent wgrad grid does not hold the SMs that
    // kernel needs (BERT-48 N=1 +0.8%, LN backward 26.9 -> 20.3 ms per step);
    // capped side grids (<= 2048-row slices) keep the early fork (GPT-2
    // -1.9% late).  DPL_WGRAD_LATE=0/1 forces either (A/B).
    static const int late_env = [] {
      const char* e = std::getenv("DPL_WGRAD_LATE");
      return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    const bool late = late_env >= 0 ? late_env == 1 : ctx.wgrad_ctas == 0;
    auto w1_grad = [&] {
      ctx.on_side([&](cudaStream_t s) {
        ctx.gemms.run(plain(F_, H_, R, dz1, F_, true, st.ln2, H_, true, g32_ + w1_, H_, kOutF32Acc), s);
      });
    };
    if (!late) w1_grad();
    ctx.gemms.run(plain(R, H_, F_, dz1, F_, false, w16_ + w1_, H_, true, dln, H_, kOutBf16), str);
    // LN2 backward (+ residual gradient dy); also db2 = colsum(dy) and
    // dbo = colsum(dh) from the rows it already holds
    layernorm_bwd(dln, st.h, st.mean2, st.rstd2, w32_ + ln2g_, dy, dh, g32_ + ln2g_, g32_ + ln2b_, R, H_, str,
                  ctx.ln_ws, g32_ + b2_, g32_ + bo_);
    if (late) w1_grad();
    // O projection: dWo += dh^T ctx ; dbo ; dctx = dh Wo (head-split store)
    ctx.on_side([&](cudaStream_t s) {
      ctx.gemms.run(plain(H_, H_, R, dh, H_, true, st.ctx, H_, true, g32_ + wo_, H_, kOutF32Acc), s);
    });
    {
      GemmDesc d = plain(R, H_, H_, dh, H_, false, w16_ + wo_, H_, true, dctx_h, d_, kOutBf16);
      d.ndiv = d_;
      d.s_no = static_cast<long long>(R) * d_;
      ctx.gemms.run(d, str);
    }
    // fused flash attention backward -> dQ, dK, dV head-merged into dqkv
    attention(ctx, slot).backward(str);
    // QKV: dWqkv += dqkv^T ln1 ; dbqkv ; dln1 = dqkv Wqkv
    ctx.on_side([&](cudaStream_t s) {
      ctx.gemms.run(plain(3 * H_, H_, R, dqkv, 3 * H_, true, st.ln1, H_, true, g32_ + wqkv_, H_, kOutF32Acc), s);
      colsum_acc(dqkv, g32_ + bqkv_, R, 3 * H_, s);
    });
    ctx.gemms.run(plain(R, H_, 3 * H_, dqkv, 3 * H_, false, w16_ + wqkv_, H_, true, dln, H_, kOutBf16), str);
    // LN1 backward (+ residual gradient dh); the model's first layer still
    // needs gamma/beta grads, its dx goes to scratch
    layernorm_bwd(dln, x, st.mean1, st.rstd1, w32_ + ln1g_, dh, dx ? dx : dctx_h, g32_ + ln1g_, g32_ + ln1b_, R, H_,
                  str, ctx.ln_ws);
    // the layer's weight gradients are final (and its scratch free) when the
    // next layer's backward starts
    ctx.join_side();
  }

  double flops_fwd(const StageContext& ctx) const override {
    const double R = ctx.rows, s = ctx.spec.seq, z = static_cast<double>(nh_) * ctx.samples;
    return 2.0 * R * (4.0 * H_ * H_ + 2.0 * H_ * F_) + 4.0 * z * s * s * d_;
  }
  double flops_bwd(const StageContext& ctx, bool) const override { return 2.0 * flops_fwd(ctx); }

  std::vector<Named> tensors() const override {
    return {{"ln1_g", ln1g_, size_t(H_)}, {"ln1_b", ln1b_, size_t(H_)},   {"Wqkv", wqkv_, 3ull * H_ * H_},
            {"bqkv", bqkv_, 3ull * H_},   {"Wo", wo_, 1ull * H_ * H_},     {"bo", bo_, size_t(H_)},
            {"ln2_g", ln2g_, size_t(H_)}, {"ln2_b", ln2b_, size_t(H_)},   {"W1", w1_, 1ull * F_ * H_},
            {"b1", b1_, size_t(F_)},      {"W2", w2_, 1ull * H_ * F_},     {"b2", b2_, size_t(H_)}};
  }

 private:
  struct Stash {
    bf16 *ln1, *qkv, *ctx, *h, *ln2, *z1, *g;
    float *mean1, *rstd1, *mean2, *rstd2, *lse;
    AttentionOp attn;
    bool attn_ready = false;
  };
  AttentionOp& attention(StageContext& ctx, int slot) {
    Stash& st = stash_[slot];
    if (!st.attn_ready) {
      AttentionDesc d;
      d.qkv = st.qkv;
      d.ctx = st.ctx;
      d.ldc = H_;
      d.lse = st.lse;
      d.samples = ctx.samples;
      d.seq = ctx.spec.seq;
      d.heads = nh_;
      d.head_dim = d_;
      d.causal = causal_;
      d.dout = ctx.t_h3;
      d.dqkv = ctx.t_qkv;
      d.dsum = ctx.att_dsum;
      d.dq_acc = ctx.att_dq;
      d.fwd_part = ctx.att_part;
      d.fwd_flags = ctx.att_flags;
      st.attn.prepare(d);
      st.attn_ready = true;
    }
    return st.attn;
  }
  int H_, F_, nh_, d_;
  bool causal_;
  float eps_;
  int index_;
  size_t ln1g_, ln1b_, wqkv_, bqkv_, wo_, bo_, ln2g_, ln2b_, w1_, b1_, w2_, b2_, total_;
  float* w32_ = nullptr;
  float* g32_ = nullptr;
  bf16* w16_ = nullptr;
  std::vector<Stash> stash_;
};

}  // namespace

// ------------------------------------------------------------------ VGG-19
// Profile layers 0..15: 3x3 convs (+ReLU; the last conv of each group also
// does the 2x2 max pool), 16..18: FC (ReLU, ReLU, logits).  Activations are
// NHWC; a conv is  y = relu(im2col(x) W^T + b)  on the tcgen05 GEMM with
// W [cout][kp], K ordered (kh, kw, c) and zero-padded to kp = ceil8(9 cin).
// Gradient contract: every VGG layer takes dL/d(its output) and returns
// dL/d(its input) (ReLU' and the pool backward are applied inside).
VggLayerShape vgg_layer(const ModelSpec& spec, int l) {
  VggLayerShape v;
  int idx = 0, hw = spec.image, cin = 3;
  for (size_t g = 0; g < spec.convs.size(); ++g) {
    for (int c = 0; c < spec.convs[g]; ++c, ++idx) {
      const int cout = spec.width * spec.mults[g];
      if (idx == l) {
        v.conv = true;
        v.h = v.w = hw;
        v.cin = cin;
        v.cout = cout;
        v.kp = (9 * cin + 7) / 8 * 8;
        v.pool = c == spec.convs[g] - 1;
        return v;
      }
      cin = cout;
    }
    hw /= 2;
  }
  const int flat = hw * hw * cin, nc = spec.conv_layers();
  if (l < nc || l >= nc + spec.fcs) throw std::out_of_range("vgg_layer: layer index");
  const int f = l - nc;  // FC index
  v.fin = f == 0 ? flat : spec.fc;
  v.fout = f == spec.fcs - 1 ? spec.classes : spec.fc;
  v.relu = f != spec.fcs - 1;
  return v;
}

long long elems_per_sample(const ModelSpec& spec, int l) {
  if (spec.kind != "vgg") return static_cast<long long>(spec.seq) * spec.hidden;
  if (l >= spec.layers) return spec.classes;
  const VggLayerShape v = vgg_layer(spec, l);
  return v.conv ? static_cast<long long>(v.h) * v.w * v.cin : v.fin;
}

class ConvLayer final : public Layer {
 public:
  ConvLayer(const ModelSpec& spec, int index) : v_(vgg_layer(spec, index)), index_(index) {}

  size_t param_count() const override { return static_cast<size_t>(v_.cout) * v_.kp + v_.cout; }
  void bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s) override {
    w32_ = w32;
    g32_ = g32;
    w16_ = w16;
    const size_t nw = static_cast<size_t>(v_.cout) * v_.kp;
    // the padding columns kp > 9 cin meet zero columns: they never act or learn
    init_params({{0, nw, 0, std::sqrt(6.0f / (9.0f * v_.cin))}, {nw, static_cast<size_t>(v_.cout), 1, 0.05f}},
                index_, w32, w16, param_count(), seed, s);
  }
  size_t col_elems(const StageContext& c) const override {  // dcol scratch (explicit backward data only)
    return implicit_dgrad() ? 0 : px(c) * v_.kp;
  }
  size_t dz_elems(const StageContext& c) const override { return px(c) * v_.cout; }
  const bf16* probe_aux(int slot) const override { return v_.pool ? yr_[slot] : nullptr; }
  size_t probe_aux_elems(const StageContext& c) const override { return v_.pool ? px(c) * v_.cout : 0; }
  void alloc_stash(StageContext& ctx) override {
    for (int k = 0; k < ctx.slots; ++k) {
      // explicit columns only where TMA's im2col mode cannot feed the GEMM
      // (cin % 64 != 0: the RGB input); kept for the weight gradient
      if (!implicit()) col_.push_back(alloc_n<bf16>(ctx, px(ctx) * v_.kp));
      if (v_.pool) yr_.push_back(alloc_n<bf16>(ctx, px(ctx) * v_.cout));  // post-ReLU, pre-pool output
    }
    if (implicit_dgrad()) wt_ = alloc_n<bf16>(ctx, static_cast<size_t>(v_.cin) * 9 * v_.cout);
  }
  void forward(StageContext& ctx, int slot, const bf16* x, bf16* y) override {
    const int n = ctx.samples;
    const int rows = static_cast<int>(px(ctx));
    bf16* out = v_.pool ? yr_[slot] : y;
    GemmDesc d;
    if (implicit()) {
      // implicit GEMM: the A tiles are TMA im2col loads of x itself
      d = plain(rows, v_.cout, v_.kp, x, v_.kp, false, w16_, v_.kp, false, out, v_.cout, kBias | kRelu);
      conv_operand(d, 1, x, n);
    } else {
      im2col3x3(x, col_[slot], n, v_.h, v_.w, v_.cin, v_.kp, ctx.stream);
      d = plain(rows, v_.cout, v_.kp, col_[slot], v_.kp, false, w16_, v_.kp, false, out, v_.cout, kBias | kRelu);
    }
    d.bias = w32_ + static_cast<size_t>(v_.cout) * v_.kp;
    ctx.gemms.run(d, ctx.stream);
    if (v_.pool) maxpool2_fwd(out, y, n, v_.h, v_.w, v_.cout, ctx.stream);
  }
  void backward(StageContext& ctx, int slot, const bf16* x, const bf16* dy, bf16* dx) override {
    const int n = ctx.samples;
    const int rows = static_cast<int>(px(ctx));
    if (v_.pool) maxpool2_relu_bwd(yr_[slot], dy, ctx.conv_dz, n, v_.h, v_.w, v_.cout, ctx.stream);
    else relu_bwd(ctx.cur_y, dy, ctx.conv_dz, static_cast<long long>(rows) * v_.cout, ctx.stream);
    float* gw = g32_;
    // db and dW += dz^T col (the B tiles are TMA im2col loads of the stashed
    // input; explicit columns from the forward for the RGB layer) on the
    // weight-gradient side stream; dz, x and the columns stay untouched until
    // the join at the end of this layer
    ctx.on_side([&](cudaStream_t s) {
      colsum_acc(ctx.conv_dz, gw + static_cast<size_t>(v_.cout) * v_.kp, rows, v_.cout, s);
      GemmDesc dw = plain(v_.cout, v_.kp, rows, ctx.conv_dz, v_.cout, true, implicit() ? x : col_[slot], v_.kp, true,
                          gw, v_.kp, kOutF32Acc);
      if (implicit()) conv_operand(dw, 2, x, n);
      ctx.gemms.run(dw, s);
    });
    if (dx && implicit_dgrad()) {
      // backward data as a forward conv of dz with the flipped, transposed
      // weights: dx = im2col(dz) wt^T, the A tiles TMA im2col loads of dz
      conv_weight_flip(w16_, wt_, v_.cin, v_.cout, v_.kp, ctx.stream);
      GemmDesc dd = plain(rows, v_.cin, 9 * v_.cout, ctx.conv_dz, 9 * v_.cout, false, wt_, 9 * v_.cout, false, dx,
                          v_.cin, kOutBf16);
      dd.conv_x = ctx.conv_dz;
      dd.conv_operand = 1;
      dd.conv_n = n;
      dd.conv_h = v_.h;
      dd.conv_w = v_.w;
      dd.conv_c = v_.cout;
      ctx.gemms.run(dd, ctx.stream);
    } else if (dx) {
      ctx.gemms.run(plain(rows, v_.kp, v_.cout, ctx.conv_dz, v_.cout, false, w16_, v_.kp, true, ctx.conv_dcol, v_.kp,
                          kOutBf16),
                    ctx.stream);
      col2im3x3(ctx.conv_dcol, dx, n, v_.h, v_.w, v_.cin, v_.kp, ctx.stream);
    }
    ctx.join_side();
  }
  double flops_fwd(const StageContext& ctx) const override { return 2.0 * px(ctx) * v_.cout * 9.0 * v_.cin; }
  double flops_bwd(const StageContext& ctx, bool need_dx) const override {
    return (need_dx ? 2.0 : 1.0) * flops_fwd(ctx);
  }
  std::vector<Named> tensors() const override {
    const size_t nw = static_cast<size_t>(v_.cout) * v_.kp;
    return {{"W", 0, nw}, {"b", nw, static_cast<size_t>(v_.cout)}};
  }

 private:
  size_t px(const StageContext& c) const { return static_cast<size_t>(c.samples) * v_.h * v_.w; }
  bool implicit() const { return v_.cin % 64 == 0; }
  bool implicit_dgrad() const { return v_.cout % 64 == 0 && v_.cin % 8 == 0; }
  void conv_operand(GemmDesc& d, int which, const bf16* x, int n) const {
    d.conv_x = x;
    d.conv_operand = which;
    d.conv_n = n;
    d.conv_h = v_.h;
    d.conv_w = v_.w;
    d.conv_c = v_.cin;
  }
  VggLayerShape v_;
  int index_;
  float* w32_ = nullptr;
  float* g32_ = nullptr;
  bf16* w16_ = nullptr;
  std::vector<bf16*> yr_;
  std::vector<bf16*> col_;  // per slot: im2col columns of the forward
  bf16* wt_ = nullptr;      // flipped / transposed weights for the backward-data conv
};

// y = x W^T + b (+ReLU), W [fout][fin]; takes / returns output / input gradients
class FcLayer final : public Layer {
 public:
  FcLayer(const ModelSpec& spec, int index) : v_(vgg_layer(spec, index)), index_(index) {}

  size_t param_count() const override { return static_cast<size_t>(v_.fout) * v_.fin + v_.fout; }
  void bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s) override {
    w32_ = w32;
    g32_ = g32;
    w16_ = w16;
    const size_t nw = static_cast<size_t>(v_.fout) * v_.fin;
    init_params({{0, nw, 0, std::sqrt(6.0f / v_.fin)}, {nw, static_cast<size_t>(v_.fout), 1, 0.05f}}, index_, w32,
                w16, param_count(), seed, s);
  }
  size_t dz_elems(const StageContext& c) const override { return static_cast<size_t>(c.samples) * v_.fout; }
  void alloc_stash(StageContext&) override {}
  void forward(StageContext& ctx, int, const bf16* x, bf16* y) override {
    GemmDesc d = plain(ctx.samples, v_.fout, v_.fin, x, v_.fin, false, w16_, v_.fin, false, y, v_.fout,
                       kBias | (v_.relu ? kRelu : 0u));
    d.bias = w32_ + static_cast<size_t>(v_.fout) * v_.fin;
    ctx.gemms.run(d, ctx.stream);
  }
  void backward(StageContext& ctx, int, const bf16* x, const bf16* dy, bf16* dx) override {
    const int n = ctx.samples;
    const bf16* dz = dy;
    if (v_.relu) {
      relu_bwd(ctx.cur_y, dy, ctx.conv_dz, static_cast<long long>(n) * v_.fout, ctx.stream);
      dz = ctx.conv_dz;
    }
    ctx.on_side([&](cudaStream_t s) {
      ctx.gemms.run(plain(v_.fout, v_.fin, n, dz, v_.fout, true, x, v_.fin, true, g32_, v_.fin, kOutF32Acc), s);
      colsum_acc(dz, g32_ + static_cast<size_t>(v_.fout) * v_.fin, n, v_.fout, s);
    });
    if (dx)
      ctx.gemms.run(plain(n, v_.fin, v_.fout, dz, v_.fout, false, w16_, v_.fin, true, dx, v_.fin, kOutBf16), ctx.stream);
    ctx.join_side();
  }
  double flops_fwd(const StageContext& ctx) const override { return 2.0 * ctx.samples * v_.fin * v_.fout; }
  double flops_bwd(const StageContext& ctx, bool need_dx) const override {
    return (need_dx ? 2.0 : 1.0) * flops_fwd(ctx);
  }
  std::vector<Named> tensors() const override {
    const size_t nw = static_cast<size_t>(v_.fout) * v_.fin;
    return {{"W", 0, nw}, {"b", nw, static_cast<size_t>(v_.fout)}};
  }

 private:
  VggLayerShape v_;
  int index_;
  float* w32_ = nullptr;
  float* g32_ = nullptr;
  bf16* w16_ = nullptr;
};

std::unique_ptr<Layer> make_layer(const ModelSpec& spec, int global_index) {
  if (spec.kind == "mlp") return std::make_unique<MlpLayer>(spec, global_index);
  if (spec.kind == "bert" || spec.kind == "gpt") return std::make_unique<TransformerLayer>(spec, global_index);
  if (spec.kind == "vgg") {
    if (global_index < spec.conv_layers()) return std::make_unique<ConvLayer>(spec, global_index);
    return std::make_unique<FcLayer>(spec, global_index);
  }
  throw std::invalid_argument("dpl: unknown model kind '" + spec.kind + "'");
}

// ------------------------------------------------------------------ LM ends
void TokenEmbedding::bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s) {
  g32_ = g32;
  w16_ = w16;
  const size_t nte = static_cast<size_t>(v_) * h_;
  fill_uniform_f32(w32, static_cast<long long>(nte), seed, kTensorWte, 0, 0.1f, s);
  fill_uniform_f32(w32 + nte, static_cast<long long>(seq_) * h_, seed, kTensorWpe, 0, 0.1f, s);
  cast_f32_bf16(w32, w16, static_cast<long long>(param_count()), s);
}

void TokenEmbedding::forward(StageContext& ctx, const int* tok, bf16* x) {
  embed_fwd(tok, w16_, w16_ + static_cast<size_t>(v_) * h_, x, ctx.rows, seq_, h_, ctx.stream);
}

void TokenEmbedding::backward(StageContext& ctx, const int* tok, const bf16* dx) {
  embed_bwd(tok, dx, g32_, g32_ + static_cast<size_t>(v_) * h_, ctx.rows, seq_, h_, ctx.stream);
}

std::vector<Layer::Named> TokenEmbedding::tensors() const {
  return {{"wte", 0, static_cast<size_t>(v_) * h_}, {"wpe", static_cast<size_t>(v_) * h_, static_cast<size_t>(seq_) * h_}};
}

// params: [lnf_g H][lnf_b H][Wout V*H]
void LmHead::bind(float* w32, float* g32, bf16* w16, uint64_t seed, cudaStream_t s) {
  w32_ = w32;
  g32_ = g32;
  w16_ = w16;
  fill_const_f32(w32, h_, 1.0f, s);
  fill_const_f32(w32 + h_, h_, 0.0f, s);
  fill_uniform_f32(w32 + 2 * h_, static_cast<long long>(v_) * h_, seed, kTensorWout, 0,
                   1.0f / std::sqrt(static_cast<float>(h_)), s);
  cast_f32_bf16(w32, w16, static_cast<long long>(param_count()), s);
}

void LmHead::alloc_stash(StageContext& ctx, int slots) {
  const size_t R = ctx.rows;
  for (int k = 0; k < slots; ++k) {
    Slot st;
    st.xn = alloc_n<bf16>(ctx, R * h_);
    st.mean = alloc_n<float>(ctx, R);
    st.rstd = alloc_n<float>(ctx, R);
    st.dlogits = alloc_n<bf16>(ctx, R * static_cast<size_t>(vp_));
    slots_.push_back(st);
  }
  dxn_ = alloc_n<bf16>(ctx, R * h_);
}

void LmHead::forward(StageContext& ctx, int slot, const bf16* y, const int* tgt, float* loss_acc, float grad_scale) {
  const Slot& st = slots_[slot];
  const int R = ctx.rows;
  layernorm_fwd(y, w32_, w32_ + h_, st.xn, st.mean, st.rstd, R, h_, eps_, ctx.stream);
  // logits [R][V] = xn Wout^T  (tcgen05, bf16 out)
  ctx.gemms.run(plain(R, vp_, h_, st.xn, h_, false, w16_ + 2 * h_, h_, false, st.dlogits, vp_, kOutBf16), ctx.stream);
  cross_entropy_fwd_bwd(st.dlogits, tgt, loss_acc, R, v_, grad_scale, ctx.stream, vp_);
}

void LmHead::backward(StageContext& ctx, int slot, const bf16* y, bf16* dy) {
  const Slot& st = slots_[slot];
  const int R = ctx.rows;
  // dWout += dlogits^T xn (side stream) ; dxn = dlogits Wout
  ctx.on_side([&](cudaStream_t s) {
    ctx.gemms.run(plain(vp_, h_, R, st.dlogits, vp_, true, st.xn, h_, true, g32_ + 2 * h_, h_, kOutF32Acc), s);
  });
  ctx.gemms.run(plain(R, h_, vp_, st.dlogits, vp_, false, w16_ + 2 * h_, h_, true, dxn_, h_, kOutBf16), ctx.stream);
  layernorm_bwd(dxn_, y, st.mean, st.rstd, w32_, nullptr, dy, g32_, g32_ + h_, R, h_, ctx.stream, ctx.ln_ws);
  ctx.join_side();
}

std::vector<Layer::Named> LmHead::tensors() const {
  return {{"lnf_g", 0, static_cast<size_t>(h_)},
          {"lnf_b", static_cast<size_t>(h_), static_cast<size_t>(h_)},
          {"Wout", 2 * static_cast<size_t>(h_), static_cast<size_t>(v_) * h_}};
}

}  // namespace dpl
