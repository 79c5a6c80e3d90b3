/* dapple-b200 C-ABI (libdapple.so).
 *
 * The reference (proj/, C++20 namespace pipeplan) exposes its planner and
 * simulator as C++ value types and free functions (proj/include/pipeplan/
 * *.hpp) and has no FFI and no executor.  This header is the drop-in
 * boundary a non-C++ host binds:
 *
 *  1. dpl_host_call      -- the whole pipeplan surface as JSON requests:
 *       "plan"                 planner.hpp:71-73   (planner.cpp:306-421)
 *       "brute_force_plan"     planner.hpp:78-79   (planner.cpp:423-489)
 *       "simulate_plan"        planner.hpp:87-90   (planner.cpp:491-514)
 *       "build_stage_sequence" estimator.hpp:25-27 (estimator.cpp:13-37)
 *       "estimate"             estimator.hpp:35/41 (estimator.cpp:56-107)
 *       "schedule"             simulator.hpp:46-58 (simulator.cpp:153-179)
 *       "optimize_phi"         simulator.hpp:71-72 (simulator.cpp:233-286)
 *       "expand_plan_phi", "apply_recompute", "allreduce_time",
 *       "splitconcat_time", "aggregate_stage", "enumerate_placements",
 *       "memory_feasible", "load_profile", "load_cluster", "stage_chain",
 *       "timeline_svg"
 *     Errors come back as {"error":{"type":..., "what":...}} using the
 *     reference's exception classes (invalid_argument / out_of_range /
 *     logic_error / runtime_error) and messages.
 *
 *  2. dpl_exec_*         -- the executor entry point that mirrors
 *     simulate_plan (planner.hpp:87-90) but runs the step on B200s and
 *     returns a *measured* Timeline (one process per GPU; see
 *     include/pipeplan/executor.hpp for the C++ form).
 *
 *  3. dpl_k_*            -- the individual stage kernels, exported so tests
 *     can check each against the CPU oracle.
 *
 * Conventions: int status (0 = ok), dpl_last_error() for the message,
 * opaque handles, no C++ exceptions cross the ABI, bf16 tensors as void*.
 */
#ifndef DAPPLE_H_
#define DAPPLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- host */
const char* dpl_host_call(const char* request_json);
const char* dpl_last_error(void);
const char* dpl_version(void);

/* ---------------------------------------------------------------- kernels */
/* C[z,m,n] = epi(alpha * sum_k A[z,m,k] B[z,n,k]); see csrc/kernels/gemm.h */
typedef struct dpl_gemm_desc {
  int M, N, K, batch;
  const void* A;
  long long lda, a_batch_stride;
  int a_mn_major;
  const void* B;
  long long ldb, b_batch_stride;
  int b_mn_major;
  void* C;
  long long ldc;
  int zdiv;
  long long s_zo, s_zi;
  int ndiv;
  long long s_no;
  uint32_t epi; /* DPL_EPI_* flags */
  float alpha;
  const float* bias;
  const void* aux_in;
  const void* resid;
  void* aux_out;
  int force_bn;
  int force_1sm; /* 1: never use the cta_group::2 pair kernel */
  /* optional: per-CTA phase timestamps (SM clock64 cycles), 16 u64 per CTA:
   * entry, prologue done, first TMA issued, first MMA, last MMA committed,
   * epilogue start, epilogue end, exit, then (TMA epilogue, first epilogue
   * warp) input ready / store issued for its first 4 chunks.  NULL = off. */
  unsigned long long* trace;
  float* colsum; /* DPL_EPI_COLSUM target: colsum[n] += sum_m C[m][n] (bf16 C as stored) */
  /* implicit-GEMM 3x3 pad-1 convolution over NHWC conv_x [n][h][w][c], c % 64 == 0:
   * conv_operand 1 = A is im2col(conv_x) (M = n*h*w, K = 9c); 2 = B is im2col(conv_x)
   * MN-major (K = n*h*w, N = 9c); loaded by TMA in im2col mode, no column matrix */
  const void* conv_x;
  int conv_operand, conv_n, conv_h, conv_w, conv_c;
  /* optional zeroed fp32 scratch (>= M*N*4 bytes, left zeroed): a bf16-output
   * GEMM that would leave most CTA pairs idle runs as split-K fp32 reduce-add
   * into it plus a bf16 epilogue pass (bias / residual / gelu' only).
   * NULL = never split (the executor passes its stage scratch). */
  float* split_ws;
  size_t split_ws_bytes;
} dpl_gemm_desc;

#define DPL_EPI_OUT_BF16 0u
#define DPL_EPI_OUT_F32 1u
#define DPL_EPI_OUT_F32_ACC 2u
#define DPL_EPI_BIAS (1u << 2)
#define DPL_EPI_GELU (1u << 3)
#define DPL_EPI_RELU (1u << 4)
#define DPL_EPI_AUX_OUT (1u << 5)
#define DPL_EPI_DGELU (1u << 6)
#define DPL_EPI_DRELU (1u << 7)
#define DPL_EPI_RESID (1u << 8)
#define DPL_EPI_COLSUM (1u << 9) /* + column sums of the bf16 output into desc.colsum */

int dpl_k_gemm(const dpl_gemm_desc* desc, void* stream);
/* Fused attention forward, head dim 64: qkv head-split [3][heads][B][S][64],
 * ctx head-merged [B*S][ldc], lse [heads*B][S]. */
int dpl_k_attention_fwd(const void* qkv, void* ctx, long long ldc, float* lse, int samples, int seq, int heads,
                        int causal, void* stream);
/* Diagnostics: the same forward with 16 %globaltimer / %smid slots per CTA
 * written to trace (tools/attn_trace.py). */
int dpl_k_attention_fwd_traced(const void* qkv, void* ctx, long long ldc, float* lse, int samples, int seq,
                               int heads, int causal, long long* trace, void* stream);
/* Fused attention backward: recomputes P from lse, dO head-split
 * [heads][B][S][64]; writes dQ/dK/dV head-merged into dqkv [B*S][3H];
 * workspaces dsum [heads*B][S] and dq_acc [heads*B][S][64] fp32. */
int dpl_k_attention_bwd(const void* qkv, const void* ctx, long long ldc, const float* lse, const void* dout,
                        void* dqkv, float* dsum, float* dq_acc, int samples, int seq, int heads, int causal,
                        void* stream);
/* Diagnostics: the same backward with 16 %globaltimer / %smid slots per CTA
 * of the main kernel written to trace (tools/attn_trace.py --bwd). */
int dpl_k_attention_bwd_traced(const void* qkv, const void* ctx, long long ldc, const float* lse, const void* dout,
                               void* dqkv, float* dsum, float* dq_acc, int samples, int seq, int heads, int causal,
                               long long* trace, void* stream);
int dpl_k_layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y, float* mean, float* rstd,
                        int rows, int h, float eps, void* stream);
int dpl_k_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gamma,
                        const void* dresid, void* dx, float* dgamma, float* dbeta, int rows, int h, void* stream);
/* The same, also accumulating the column sums of dresid and (if dx_colsum)
 * of dx -- the bias gradients the executor folds into LayerNorm backward. */
int dpl_k_layernorm_bwd_colsum(const void* dy, const void* x, const float* mean, const float* rstd, const float* gamma,
                               const void* dresid, void* dx, float* dgamma, float* dbeta, float* dresid_colsum,
                               float* dx_colsum, int rows, int h, void* stream);
int dpl_k_softmax_fwd(const float* s, void* p, int rows, int len, int q_len, int causal, void* stream);
int dpl_k_softmax_bwd(const void* p, const float* dp, void* ds, int rows, int len, void* stream);
int dpl_k_colsum_acc(const void* dy, float* db, int rows, int cols, void* stream);
int dpl_k_mse_loss(const void* y, const void* t, void* dy, float* loss_acc, long long n, float grad_scale,
                   void* stream);
int dpl_k_sgd_apply(float* w32, float* g, void* w16, long long n, float lr, void* stream);
/* GPT language-model ends (config C4; no reference counterpart -- the
 * reference has no numerical executor).
 * tokens: dst[i] = (splitmix64(seed, tensor, idx0+i) >> 32) % vocab
 * embed:  x[r] = wte[tok[r]] + wpe[r % seq]; backward red.adds into fp32 grads
 * cross_entropy: per row loss_acc += lse(row) - row[tgt]; row <- (softmax - onehot) * grad_scale */
int dpl_k_fill_tokens(int* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, int vocab, void* stream);
int dpl_k_embed_fwd(const int* tok, const void* wte, const void* wpe, void* x, int rows, int seq, int h, void* stream);
int dpl_k_embed_bwd(const int* tok, const void* dx, float* gwte, float* gwpe, int rows, int seq, int h, void* stream);
/* the same over rows of stride ld >= vocab (ld % 8 == 0): columns past vocab
 * are padding, excluded from the softmax, gradient 0 */
int dpl_k_cross_entropy_padded(void* logits, const int* tgt, float* loss_acc, int rows, int vocab, int ld,
                               float grad_scale, void* stream);
int dpl_k_cross_entropy(void* logits, const int* tgt, float* loss_acc, int rows, int vocab, float grad_scale,
                        void* stream);
/* VGG convolution support (config C3; NHWC bf16, 3x3 stride-1 pad-1 convs as
 * GEMMs over columns col[(n*H+h)*W+w][(kh*3+kw)*C+c], row length kp >= 9C):
 * im2col / col2im (gather), 2x2 max pool and its backward fused with ReLU',
 * ReLU' alone. */
int dpl_k_im2col3x3(const void* x, void* col, int n, int h, int w, int c, int kp, void* stream);
int dpl_k_col2im3x3(const void* dcol, void* dx, int n, int h, int w, int c, int kp, void* stream);
int dpl_k_maxpool2_fwd(const void* x, void* y, int n, int h, int w, int c, void* stream);
int dpl_k_maxpool2_relu_bwd(const void* x, const void* dy, void* dz, int n, int h, int w, int c, void* stream);
int dpl_k_relu_bwd(const void* y, const void* dy, void* dz, long long n, void* stream);
int dpl_k_fill_uniform_bf16(void* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                            void* stream);
int dpl_k_fill_uniform_f32(float* dst, long long n, uint64_t seed, uint64_t tensor, long long idx0, float scale,
                           void* stream);
/* Kernel launches issued by this library since load (smoke/bench evidence). */
long long dpl_k_launch_count(void);

/* ---------------------------------------------------------------- executor */
typedef struct dpl_exec dpl_exec; /* one per process / GPU */

/* Creates the executor for this rank.  `config_json` carries the model
 * ({"model": "mlp"|"bert"|"gpt", dims...}), the plan (plan JSON as written
 * by plan_to_json), the profile and cluster JSON, M, GBS, lr, seed, rank and
 * world size.  Allocates parameters, gradients, activation stash and
 * Split-Concat receive buffers on `device`. */
int dpl_exec_create(const char* config_json, int device, dpl_exec** out);
/* Opaque blob (<= 256 bytes) this rank must share with every other rank:
 * CUDA IPC handles of its receive region (activations, gradients, flag
 * words, loss) and of its fp32 gradients, plus process id / device / raw
 * pointers so ranks living in one process (several ranks on one GPU) map
 * each other without IPC.  dpl_exec_connect takes the blobs of all ranks,
 * concatenated in rank order. */
int dpl_exec_export(dpl_exec* ex, void* blob, size_t cap, size_t* len);
int dpl_exec_connect(dpl_exec* ex, const void* blobs, size_t blob_len, int world);
/* NCCL (config "allreduce": "nccl" only; the default "peer" reduces the
 * replica group over peer memory): rank 0 of each stage group creates the id
 * (128 bytes), the group shares it, then every member initialises its
 * communicator. */
int dpl_exec_nccl_id(void* id128);
int dpl_exec_nccl_init(dpl_exec* ex, const void* id128);
/* One synchronous DAPPLE step: phi warm-up forwards, 1F1B steady state,
 * drain, per-layer AllReduce, SGD apply.  Host inputs may be NULL (inputs
 * generated on device from the seed).  *loss gets the global-batch loss on
 * last-stage ranks (NaN elsewhere). */
int dpl_exec_step(dpl_exec* ex, const void* host_input, const void* host_target, float* loss);
/* The same step split in two: launch enqueues it (a CUDA-graph replay) and
 * returns, finish waits for it.  Ranks sharing one process launch every
 * rank's step before finishing any. */
int dpl_exec_step_launch(dpl_exec* ex, const void* host_input, const void* host_target);
/* Captures and instantiates the step graphs (both flag banks, device data)
 * ahead of the first step; ranks sharing one process call it on every rank
 * before any rank steps. */
int dpl_exec_prepare(dpl_exec* ex);
int dpl_exec_step_finish(dpl_exec* ex, float* loss);
/* Measured timeline of the last step as JSON (same layout as the
 * simulator's Timeline, seconds), plus per-block kernel times. */
const char* dpl_exec_timeline(dpl_exec* ex);
/* Copies a parameter / gradient tensor (by name) to host, for parity. */
int dpl_exec_read_tensor(dpl_exec* ex, const char* name, int grad, void* host, size_t bytes);
/* Parity probes (executor created with "probe": true): the last
 * micro-batch's input "x", output "y", backward intermediate "aux" (pooling
 * convs: pre-pool output), output gradient "dy" or input gradient "dx" of a
 * layer on this stage, bf16, for teacher-forced layer checks. */
int dpl_exec_read_probe(dpl_exec* ex, int layer, const char* which, void* host, size_t bytes);
int dpl_exec_info(dpl_exec* ex, char* buf, size_t cap);
/* Cross-GPU timer calibration (collective over phases 1..world-1, a host
 * barrier between the responder's call and rank 0's): on rank 0 returns the
 * offset of rank `phase`'s %globaltimer relative to rank 0's. */
int dpl_exec_clock_calibrate(dpl_exec* ex, int phase, long long* offset_ns);
/* Per-launch GEMM timing (CUDA events around every GEMM launch of the next
 * steps) and its summary as JSON {launches, seconds, flops, shapes[]}. */
int dpl_exec_gemm_profile(dpl_exec* ex, int enable);
const char* dpl_exec_gemm_profile_json(dpl_exec* ex);
/* B200 layer profiler: times this rank's layers (F in order, then B in
 * reverse, one event between layers, median of `reps` chains) at this
 * replica's micro-batch slice and returns the reference's profile JSON
 * (profile_to_json, reference model.cpp:162-173; ingested by load_profile,
 * model.cpp:128-153).  NULL on error (dpl_last_error). */
const char* dpl_exec_layer_profile(dpl_exec* ex, int reps);
/* Multi-rank teardown: disconnect on every rank (unmaps peers' IPC regions,
 * destroys the NCCL communicator), barrier, then destroy. */
int dpl_exec_disconnect(dpl_exec* ex);
void dpl_exec_destroy(dpl_exec* ex);

#ifdef __cplusplus
}
#endif

#endif /* DAPPLE_H_ */
