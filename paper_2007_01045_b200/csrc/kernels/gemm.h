// Host-side interface of the tcgen05 GEMM (gemm_tcgen05.cu).
//
//   C[z, m, n] = epilogue( alpha * sum_k A[z, m, k] * B[z, n, k] )
//
// A is stored K-major ([M][lda], k contiguous) or M-major ([K][lda], m
// contiguous); B likewise with N.  Output addressing is general enough to
// express the attention head split / merge without separate transpose
// kernels:
//   off(z, m, n) = (z / zdiv) * s_zo + (z % zdiv) * s_zi + m * ldc
//                + (n / ndiv) * s_no + (n % ndiv)
// aux_in / resid / aux_out share C's addressing.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

namespace dpl {

enum GemmEpilogue : uint32_t {
  kOutBf16 = 0,      // C bf16 = result
  kOutF32 = 1,       // C fp32 = result
  kOutF32Acc = 2,    // C fp32 += result   (micro-batch gradient accumulation)
  kOutMask = 3,
  kBias = 1u << 2,   // + bias[n] (fp32)
  kGelu = 1u << 3,   // gelu(.)
  kRelu = 1u << 4,   // relu(.)
  kAuxOut = 1u << 5, // also store the pre-activation (bf16) to aux_out
  kDGelu = 1u << 6,  // * gelu'(aux_in)
  kDRelu = 1u << 7,  // * relu'(aux_in)
  kResid = 1u << 8,  // + resid (bf16), added after bias, before activation
  kColSum = 1u << 9, // also colsum[n] += sum_m C[m][n] of the stored bf16 output (bias gradient)
};

struct GemmDesc {
  int M = 0, N = 0, K = 0, batch = 1;
  const void* A = nullptr;
  long long lda = 0, a_batch_stride = 0;
  int a_mn_major = 0;
  const void* B = nullptr;
  long long ldb = 0, b_batch_stride = 0;
  int b_mn_major = 0;
  void* C = nullptr;
  long long ldc = 0;
  int zdiv = 1;
  long long s_zo = 0, s_zi = 0;
  int ndiv = 1 << 30;
  long long s_no = 0;
  uint32_t epi = kOutBf16;
  float alpha = 1.0f;
  const float* bias = nullptr;
  const void* aux_in = nullptr;
  const void* resid = nullptr;
  void* aux_out = nullptr;
  int force_bn = 0;  // 0 = heuristic; else 64/128/256
  int force_1sm = 0; // 1 = never use the CTA-pair kernel
  unsigned long long* trace = nullptr;  // per-CTA phase timestamps (16 per CTA), diagnostics
  float* colsum = nullptr;              // kColSum target (fp32, N)
  // implicit-GEMM 3x3 / pad-1 convolution over NHWC conv_x [n][h][w][c] (c % 64 == 0):
  //   conv_operand 1: A[M = n*h*w][K = 9c] are its im2col columns (K-major, A unused)
  //   conv_operand 2: B[K = n*h*w][N = 9c] are its im2col columns (MN-major, B unused)
  const void* conv_x = nullptr;
  int conv_operand = 0, conv_n = 0, conv_h = 0, conv_w = 0, conv_c = 0;
  // fp32 scratch for split-K of bf16-output GEMMs with too few tiles (host
  // side only; the GemmCache fills it in): zero on entry and left zero
  float* split_ws = nullptr;
  size_t split_ws_bytes = 0;
  // cap on the persistent grid in CTAs (0: one per SM): a GEMM on a side
  // stream can leave SMs to the critical-path stream (host side only)
  int max_ctas = 0;
};

// Device-visible launch parameters (one per prepared GEMM).
struct alignas(64) GemmParams {
  CUtensorMap tma_a;
  CUtensorMap tma_b;
  // TMA epilogue (tma_epi): 5-D maps over C's addressing
  //   [n % inner][m][n / inner][z % zdiv][z / zdiv], box 32 x 32
  CUtensorMap tma_c;  // output: bulk store (bf16 / fp32) or fp32 bulk reduce-add
  CUtensorMap tma_x;  // residual / activation input (bulk load) or aux_out (bulk store)
  int tma_epi;
  int c_inner;
  int stages;          // smem ring depth (runtime: what the epilogue carve-out leaves)
  int epi_warp_bytes;  // TMA epilogue smem per epilogue warp
  int epi_out_bytes;   // one output chunk buffer (2 KB bf16 / 4 KB fp32)
  int epi_nx;          // extra-tensor chunk buffers per warp
  int epi_tile_cols;   // columns of one CTA tile (bias slice staged per warp)
  float* colsum;       // kColSum target (TMA epilogue; otherwise a colsum pass after the GEMM)
  int conv_operand, conv_h, conv_w, conv_c;  // implicit-GEMM convolution operand (GemmDesc)
  int M, N, K, batch;
  int a_mn_major, b_mn_major;
  int num_m_blocks, num_n_blocks, num_k_blocks, num_tiles;
  int k_splits, kb_per_split;  // split-K (fp32-accumulate outputs only)
  int two_sm;                  // cta_group::2 pair kernel (256 x 256 tiles)
  int split_tail;              // pair kernel: the last split_tail tiles run as two 256 x 128 halves each
  uint32_t epi;
  float alpha;
  void* C;
  long long ldc;
  int zdiv, ndiv;
  long long s_zo, s_zi, s_no;
  const float* bias;
  const __nv_bfloat16* aux_in;
  const __nv_bfloat16* resid;
  __nv_bfloat16* aux_out;
  int vec_ok;
  unsigned long long* trace;
};

// A prepared GEMM: tensor maps encoded once, launched many times (the
// executor prepares every layer's GEMMs at setup, so steps pay no host cost).
class GemmOp {
 public:
  GemmOp() = default;
  void prepare(const GemmDesc& d);
  void launch(cudaStream_t stream) const;
  void launch_kernel(cudaStream_t stream) const;
  int bn() const { return bn_; }
  bool two_sm() const { return params_.two_sm != 0; }
  int grid() const { return grid_; }
  double flops() const { return 2.0 * params_.M * params_.N * static_cast<double>(params_.K) * params_.batch; }
  const GemmParams& params() const { return params_; }
  bool ready() const { return bn_ != 0; }
  bool split_bf16() const { return split_ != nullptr; }

 private:
  GemmParams params_{};
  bool colsum_fallback_ = false;
  // split-K of a bf16-output GEMM: the fp32 reduce-add GEMM into the cache's
  // scratch, then split_epilogue (bias / residual / act' -> bf16, scratch zeroed)
  std::shared_ptr<GemmOp> split_;
  GemmDesc split_desc_{};
  int bn_ = 0;
  int grid_ = 0;
  size_t smem_ = 0;
};

// Kernel launches issued by libdapple (all kernels); bench/smoke evidence.
void count_launch(long long n = 1);
long long launch_count();

// Optional per-kernel timing of every libdapple launch (CUDA events on the
// launching stream), enabled for one profiled step by bench.py.
struct KernelTimer {
  struct Rec {
    const char* name;
    cudaEvent_t start, end;
    double flops;
  };
  bool enabled = false;
  bool capturing = false;  // records become external event nodes of a captured step
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t take();
};
KernelTimer& kernel_timer();
// RAII helper: brackets one launch when the timer is enabled
class TimedLaunch {
 public:
  TimedLaunch(const char* name, cudaStream_t s, double flops = 0.0);
  ~TimedLaunch();

 private:
  cudaStream_t s_;
  bool on_;
};

// Optional per-launch timing of GEMMs (CUDA events around each launch on the
// launching stream) used by bench.py for the live roofline number.
struct GemmProfile {
  bool enabled = false;
  struct Rec {
    cudaEvent_t start, end;
    double flops;
    int M, N, K, batch, bn;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t take();
  void reset() { recs.clear(); used = 0; }
};

// Prepared-GEMM cache keyed by the full descriptor (pointers included):
// tensor maps are encoded the first time a (layer, buffer) combination is
// seen and reused on every later step.
class GemmCache {
 public:
  const GemmOp& get(const GemmDesc& d);
  void run(const GemmDesc& d, cudaStream_t s);
  GemmProfile profile;
  size_t size() const;
  double flops_run = 0.0;  // flops launched through run() (accounting)
  // zero-initialised fp32 scratch shared by this cache's split-K bf16 GEMMs
  // (they all run on one stream, one after another); null disables them
  float* split_ws = nullptr;
  size_t split_ws_bytes = 0;
  // nonzero: GemmDesc::max_ctas for every GEMM fetched while it is set
  // (StageContext::on_side caps the weight-gradient stream's grids)
  int max_ctas_override = 0;

 private:
  struct Impl;
  std::shared_ptr<Impl> impl_;
};

int num_sms();

}  // namespace dpl
