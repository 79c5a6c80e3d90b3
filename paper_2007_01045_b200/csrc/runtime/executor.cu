// Per-GPU DAPPLE step executor (one process per GPU).
//
// The executor mirrors simulate_plan (reference planner.cpp:491-514): the
// same plan, the same phi resolution (planner.cpp:501-508) and the same
// per-stage block order (simulator.cpp:81-97, realised by
// pipeplan::stage_chain), but every block is a real stream program on a
// B200 and the returned Timeline is measured.
//
// Streams per rank
//   compute   the stage's F/B chain (all tcgen05 GEMMs + stage kernels)
//   send_act  Split-Concat forward hand-off  (peer copies over NVLink)
//   send_grad Split-Concat backward hand-off
//   reduce    per-layer replica AllReduce (peer memory, or NCCL) + SGD apply
//
// Cross-GPU dependencies never involve the host: a sender pushes its rows
// straight into the receiver's buffer (cudaMemcpyAsync to a CUDA-IPC
// mapping), then a one-thread kernel stores i+1 into the receiver's flag word
// for micro-batch i; the receiver's compute stream waits on that word with
// cuStreamWaitValue32(GEQ).  Flags live in two banks used by alternate steps;
// each rank clears its own bank at the end of the step that used it (safe:
// the bank is next signalled two steps later, after this rank's step end).
//
// The step is captured once into a CUDA graph per bank parity (and per host
// input buffer pair) and replayed with one cudaGraphLaunch per step, so the
// ~10^4 kernels of a BERT-48 step run back to back with no host launch gaps.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <unistd.h>
#include <stdexcept>
#include <string>
#include <vector>

#include "dapple.h"
#include "host/json.hpp"
#include "kernels/collective.h"
#include "kernels/elementwise.h"
#include "kernels/lm.h"
#include "layers.h"
#include "pipeplan/executor.hpp"
#include "pipeplan/io.hpp"
#include "pipeplan/simulator.hpp"

namespace dpl {

int fail(const std::string& what);

namespace {

using json::Value;

#define DPL_CUDA(x)                                                                                   \
  do {                                                                                                \
    const cudaError_t cuda_rc_ = (x);                                                                 \
    if (cuda_rc_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(cuda_rc_)); \
  } while (0)
#define DPL_NCCL(x)                                                                                   \
  do {                                                                                                \
    const ncclResult_t nccl_rc_ = (x);                                                                \
    if (nccl_rc_ != ncclSuccess) throw std::runtime_error(std::string(#x) + ": " + ncclGetErrorString(nccl_rc_)); \
  } while (0)

typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// cuStreamWriteValue32: the flag store of a hand-off as a stream memory
// operation -- executed in stream order by the GPU front end, no SM needed
// (a one-thread signal kernel can wait a whole persistent GEMM for a free SM)
StreamValueFn write_value_fn() {
  static StreamValueFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<StreamValueFn>(p);
  }();
  return fn;
}

StreamValueFn wait_value_fn() {
  static StreamValueFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<StreamValueFn>(p);
  }();
  return fn;
}

__global__ void signal_kernel(uint32_t* flag, uint32_t value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

// Fallback wait if stream memory operations are unavailable.
__global__ void wait_kernel(const uint32_t* flag, uint32_t value) {
  uint32_t v;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
  } while (static_cast<int32_t>(v - value) < 0);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Clock-offset ping-pong between rank 0 (initiator) and one peer (responder)
// over peer-mapped words; both kernels run at the same time on different
// GPUs.  out[k] = {t_send, t_peer, t_recv} on the initiator (t_peer copied
// back by the responder).
__global__ void clock_ping_kernel(volatile uint32_t* ping_remote, volatile uint32_t* pong_local,
                                  volatile unsigned long long* peer_time_local, unsigned long long* out, int rounds) {
  for (int k = 1; k <= rounds; ++k) {
    const unsigned long long t0 = globaltimer();
    *ping_remote = k;
    __threadfence_system();
    while (*pong_local != static_cast<uint32_t>(k)) {
    }
    const unsigned long long t2 = globaltimer();
    __threadfence_system();
    out[3 * (k - 1)] = t0;
    out[3 * (k - 1) + 1] = *peer_time_local;
    out[3 * (k - 1) + 2] = t2;
  }
}
__global__ void clock_pong_kernel(volatile uint32_t* ping_local, volatile uint32_t* pong_remote,
                                  volatile unsigned long long* peer_time_remote, int rounds) {
  for (int k = 1; k <= rounds; ++k) {
    while (*ping_local != static_cast<uint32_t>(k)) {
    }
    *peer_time_remote = globaltimer();
    __threadfence_system();
    *pong_remote = k;
    __threadfence_system();
  }
}

__global__ void stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

using Route = pipeplan::SplitConcatRoute;

// after the flag banks: {ping u32, pong u32, peer_time u64} for clock calibration,
// then the step's loss accumulator (a peer-reduced block on replicated last stages)
constexpr size_t kCalibBytes = 256;

// What a rank publishes so its peers can reach its receive region and (for
// replica peers) its fp32 gradients: CUDA-IPC handles for other processes,
// plain pointers for ranks living in the same process (one per GPU, or
// several ranks sharing one GPU in tests).
struct PeerBlob {
  cudaIpcMemHandle_t recv;
  cudaIpcMemHandle_t grads;
  long long pid;
  int device;
  int pad;
  unsigned long long recv_ptr;
  unsigned long long grads_ptr;
};

// stream memory operations (cuStreamWaitValue32) usable, process-wide
bool& memops_flag() {
  static bool ok = true;
  return ok;
}
bool memops_ok() { return memops_flag(); }

struct BlockEvents {
  cudaEvent_t start = nullptr, end = nullptr;
};

}  // namespace

class Executor {
 public:
  explicit Executor(const Value& cfg, int device);
  ~Executor();

  size_t export_blob(void* blob, size_t cap);
  void connect(const uint8_t* blobs, size_t blob_len, int world);
  void nccl_init(const void* id);
  void disconnect();
  bool shares_gpu() const;
  // ns to add to this rank's %globaltimer to express it on rank 0's timer
  long long calibrate_clock(int phase);
  float step(const void* host_input, const void* host_target);
  void step_launch(const void* host_input, const void* host_target);
  float step_finish();
  void prepare_graphs();
  void set_gemm_profile(bool on) {
    ctx_.gemms.profile.enabled = on;
    ctx_.gemms.profile.reset();
    kernel_timer().enabled = on;
    kernel_timer().recs.clear();
    kernel_timer().used = 0;
    // the profiled graph is captured afresh so its event records are current
    for (auto it = graphs_.begin(); it != graphs_.end();) {
      if (it->key.profile) {
        it->destroy();
        it = graphs_.erase(it);
      } else {
        ++it;
      }
    }
  }
  std::string gemm_profile_json() const;
  std::string layer_profile_json(int reps);
  std::string timeline_json() const;
  void read_tensor(const std::string& name, bool grad, void* host, size_t bytes);
  // one probe tensor (bf16) of a layer of this stage: x | y | aux | dy | dx
  void read_probe(int layer, const std::string& which, void* host, size_t bytes);
  std::string info() const;
  long long graph_count() const;

 private:
  // --- configuration
  ModelSpec spec_;
  pipeplan::PipelinePlan plan_;
  int M_ = 1, gbs_ = 1, B_ = 1, rank_ = 0, world_ = 1, device_ = 0;
  float lr_ = 1e-3f;
  uint64_t seed_ = 1234;
  int k_ = 0, S_ = 1, rep_ = 0, r_ = 1, lo_ = 0, hi_ = 1;
  int phi_ = 1;
  std::vector<int> phi_expanded_;
  std::vector<pipeplan::ChainOp> chain_;
  std::vector<Route> in_routes_, out_routes_;  // activations into / out of this rank
  long long numel_global_ = 0;
  bool timeline_ = true;
  bool apply_ = true;  // false: keep the accumulated gradients (parity reads)
  bool gpipe_ = false;      // all-forward-first chain (simulator.cpp:161-167)
  bool recompute_ = false;  // re-run the stage forward inside each backward (simulator.cpp:216-221)
  int stash_slots_ = 1;     // layer-internal activation sets kept alive
  // parity probes (config "probe"): every layer's input, output, backward
  // intermediate, output gradient and input gradient of the LAST micro-batch,
  // copied aside so tests can teacher-force the oracle layer by layer
  bool probe_ = false;
  struct Probe {
    bf16 *x = nullptr, *y = nullptr, *aux = nullptr, *dy = nullptr, *dx = nullptr;
    size_t nx = 0, ny = 0, naux = 0;
  };
  std::vector<Probe> probes_;
  void probe_copy(bf16* dst, const bf16* src, size_t n) {
    if (dst && src && n) DPL_CUDA(cudaMemcpyAsync(dst, src, n * 2, cudaMemcpyDeviceToDevice, compute_));
  }

  // --- device state
  DeviceMemory mem_;
  StageContext ctx_;
  std::vector<std::unique_ptr<Layer>> layers_;
  std::vector<size_t> param_off_;
  size_t n_params_ = 0;
  float* w32_ = nullptr;
  float* g32_ = nullptr;
  bf16* w16_ = nullptr;
  std::vector<std::vector<bf16*>> act_;  // [layer-in-stage 1..L-1][slot]
  std::vector<bf16*> in_;                // stage-0 input per slot
  std::vector<bf16*> out_;               // stage output per micro-batch
  std::vector<bf16*> target_, dloss_;    // last stage, per slot
  std::vector<bf16*> send_grad_;         // first-layer dX per micro-batch (stage > 0)
  // GPT language model (spec_.vocab > 0): embedding on the first stage,
  // LN_f + vocabulary projection + cross-entropy on the last
  std::unique_ptr<TokenEmbedding> emb_;
  std::unique_ptr<LmHead> head_;
  size_t emb_off_ = 0, head_off_ = 0;
  std::vector<int*> tok_, tgt_tok_;  // token ids / targets per slot
  cudaEvent_t emb_done_ = nullptr, head_done_ = nullptr;
  float loss_norm_ = 1.0f;  // loss = sum / loss_norm_ (MSE: GBS*seq*H elements, CE: GBS*seq tokens)
  bf16* gbuf_[2] = {nullptr, nullptr};
  bf16* rc_out_ = nullptr;  // output of the re-computed forward (discarded)
  float* loss_acc_ = nullptr;
  unsigned long long* t0_ = nullptr;
  // receive region (one cudaMalloc, exported over CUDA IPC):
  //   [recv_act M x R x H][recv_grad M x R x H][flags: bank[2] x {act[world], grad[world]}]
  uint8_t* recv_ = nullptr;
  size_t recv_bytes_ = 0, recv_grad_off_ = 0, flags_off_ = 0;
  std::vector<uint8_t*> peer_recv_;  // by rank (IPC-mapped or same-process), null if unused
  std::vector<float*> peer_g32_;     // by rank: replica peers' fp32 gradients (peer AllReduce)
  std::vector<void*> ipc_opened_;    // mappings to close on disconnect
  std::vector<char> colocated_;      // by rank: same process and same GPU as this rank
  std::vector<int> group_;           // global ranks of this stage's replicas, replica order
  bool peer_ar_ = true;              // replica AllReduce over peer memory (false: NCCL)
  int nblk_ = 1;                     // parameter blocks per stage in the flag layout (layers + emb + head + loss)
  long long clock_offset_ns_ = 0;
  std::vector<int> peer_samples_;    // samples per micro-batch slice of each rank
  std::vector<int> peer_stage_;      // stage of each rank

  cudaStream_t compute_ = nullptr, send_act_ = nullptr, send_grad_s_ = nullptr, reduce_ = nullptr;
  cudaStream_t wgrad_ = nullptr;  // weight gradients (StageContext::wstream)
  cudaEvent_t ev_wg_done_ = nullptr;
  ncclComm_t comm_ = nullptr;
  cudaEvent_t ev_begin_ = nullptr, ev_end_ = nullptr, ev_reduce_done_ = nullptr;
  cudaEvent_t ev_sa_done_ = nullptr, ev_sg_done_ = nullptr, ev_fork_ = nullptr, ev_last_bwd_ = nullptr;
  std::vector<BlockEvents> fwd_ev_, bwd_ev_, send_fwd_ev_, send_bwd_ev_;
  std::vector<BlockEvents> ar_ev_;        // per parameter block: the replica AllReduce on the reduce stream
  std::vector<long long> ar_bytes_;       // fp32 bytes reduced per block (0: not reduced this step)
  std::vector<cudaEvent_t> layer_done_, fwd_done_, bwd_done_;
  long long steps_done_ = 0;
  bool launched_ = false;
  int bank_ = 0;
  float last_loss_ = NAN;
  float* loss_host_ = nullptr;  // pinned
  bool use_graph_ = true, capturing_ = false;
  // One captured step per (flag bank, host inputs present, host targets
  // present, profiling).  Host buffers are not part of the key: the graph's
  // host->device copy nodes are re-pointed in place
  // (cudaGraphExecMemcpyNodeSetParams1D) when a caller passes a different
  // pinned buffer, so a data loader rotating buffers never re-captures.
  struct GraphKey {
    int bank;
    bool in, tgt, profile;
    bool operator==(const GraphKey& o) const {
      return bank == o.bank && in == o.in && tgt == o.tgt && profile == o.profile;
    }
  };
  struct HostCopy {
    cudaGraphNode_t node;
    int which;      // 0 input, 1 target
    size_t offset;  // bytes from the start of the host buffer
    void* dst;
    size_t bytes;
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long kernels = 0;  // kernel nodes (launch accounting per replay)
    std::vector<HostCopy> copies;
    const void* src[2] = {nullptr, nullptr};  // host buffers the copy nodes currently read
    void destroy() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      exec = nullptr;
      graph = nullptr;
    }
  };
  std::vector<GraphEntry> graphs_;
  // pageable host inputs are staged through executor-owned pinned buffers
  void* staging_[2] = {nullptr, nullptr};
  size_t staging_bytes_[2] = {0, 0};
  const void* stage_host(const void* p, int which);
 public:
  // host bytes of this rank's inputs / targets for one step ([M][slice]), 0 if none
  size_t input_bytes() const;
  size_t target_bytes() const;

 private:
  void capture_step(GraphEntry& g, const void* host_input, const void* host_target);
  void enqueue_step(const void* host_input, const void* host_target);
  // this rank's gradients of one parameter block are final: AllReduce over
  // the replica group and apply on the reduce stream
  void reduce_apply(cudaEvent_t ready, size_t off, size_t n, int blk);
  // peer-memory AllReduce of one block over the replica group on the reduce stream
  void peer_allreduce(const std::vector<float*>& peers, size_t n, int blk);
  double flops_per_step_ = 0.0;

  // --- helpers
  // first sample of replica j's slice in this rank's stage (or stage k)
  int slice_lo(int j, int r = 0) const { return static_cast<int>(1LL * B_ * j / (r ? r : r_)); }
  int L() const { return hi_ - lo_; }
  // activation elements per sample entering global layer l (model output at l == layers)
  long long elems(int l) const { return elems_per_sample(spec_, l); }
  bool classify() const { return spec_.kind == "vgg"; }  // labels + cross-entropy over classes
  // one micro-batch slice of this stage's input / output activation
  size_t in_elems() const { return static_cast<size_t>(ctx_.samples) * elems(lo_); }
  size_t out_elems() const { return static_cast<size_t>(ctx_.samples) * elems(hi_); }
  bf16* recv_act(int i) const { return reinterpret_cast<bf16*>(recv_) + static_cast<size_t>(i) * in_elems(); }
  bf16* recv_grad(int i) const {
    return reinterpret_cast<bf16*>(recv_ + recv_grad_off_) + static_cast<size_t>(i) * out_elems();
  }
  // flag bank of the current step (parity): [act world][grad world][ar_ready nblk x world][ar_done nblk x world]
  size_t bank_words() const { return 2 * static_cast<size_t>(world_) * (1 + nblk_); }
  uint32_t* flags() const { return reinterpret_cast<uint32_t*>(recv_ + flags_off_) + bank_ * bank_words(); }
  // flag word of (bank, region, index) in any rank's receive region
  uint32_t* flag_at(uint8_t* region, int rank, size_t word) const {
    return reinterpret_cast<uint32_t*>(region + layout_flags_off(rank)) + bank_ * bank_words() + word;
  }
  size_t ar_word(int done, int blk, int src) const {
    return 2 * static_cast<size_t>(world_) + (static_cast<size_t>(done) * nblk_ + blk) * world_ + src;
  }
  size_t loss_off(int rank) const { return layout_flags_off(rank) + 2 * bank_words() * 4 + kCalibBytes; }
  // receive-region layout of any rank (from the plan): [recv_act M x s x E_in][recv_grad M x s x E_out][flags]
  size_t layout_grad_off(int rank) const;
  size_t layout_flags_off(int rank) const;
  void wait_flag(cudaStream_t s, uint32_t* flag, uint32_t value);
  void signal(cudaStream_t s, uint32_t* remote_flag, uint32_t value);
  void forward(int i, uint32_t base);
  void backward(int i, uint32_t base);
  // timing events become event-record nodes when the step is captured
  void record(cudaEvent_t e, cudaStream_t s) {
    DPL_CUDA(capturing_ ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s));
  }
};

Executor::Executor(const Value& cfg, int device) : device_(device) {
  DPL_CUDA(cudaSetDevice(device_));
  const Value& m = cfg.at("model");
  spec_.kind = m.at("kind").as_string();
  spec_.layers = static_cast<int>(m.at("layers").as_int());
  spec_.hidden = m.contains("hidden") ? static_cast<int>(m.at("hidden").as_int()) : 8;
  if (m.contains("heads")) spec_.heads = static_cast<int>(m.at("heads").as_int());
  if (m.contains("ffn")) spec_.ffn = static_cast<int>(m.at("ffn").as_int());
  spec_.seq = m.contains("seq") ? static_cast<int>(m.at("seq").as_int()) : 1;
  spec_.causal = m.contains("causal") && m.at("causal").as_bool();
  if (spec_.kind == "mlp") spec_.seq = 1;
  if (spec_.kind == "gpt") spec_.causal = true;
  if (m.contains("vocab")) spec_.vocab = static_cast<int>(m.at("vocab").as_int());
  if (m.contains("image")) spec_.image = static_cast<int>(m.at("image").as_int());
  if (m.contains("width")) spec_.width = static_cast<int>(m.at("width").as_int());
  if (m.contains("fc")) spec_.fc = static_cast<int>(m.at("fc").as_int());
  if (m.contains("classes")) spec_.classes = static_cast<int>(m.at("classes").as_int());
  if (m.contains("convs")) spec_.convs = m.at("convs").as_int_vector();
  if (m.contains("mults")) spec_.mults = m.at("mults").as_int_vector();
  if (m.contains("fcs")) spec_.fcs = static_cast<int>(m.at("fcs").as_int());
  if (spec_.kind == "vgg") {
    const int pools = static_cast<int>(spec_.convs.size());
    if (spec_.convs.size() != spec_.mults.size() || spec_.convs.empty() || (spec_.fcs != 1 && spec_.fcs != 3) ||
        spec_.layers != spec_.conv_layers() + spec_.fcs || spec_.image % (1 << pools) || spec_.width % 8 ||
        spec_.classes % 8 || spec_.fc % 8)
      throw std::invalid_argument("dpl exec: conv net needs layers == sum(convs) + fcs (1 or 3), image divisible by "
                                  "2^groups, width / fc / classes % 8 == 0");
    spec_.seq = 1;
    spec_.hidden = spec_.classes;
  }
  if (spec_.vocab > 0 && spec_.kind != "gpt") throw std::invalid_argument("dpl exec: vocab needs kind gpt");

  plan_ = pipeplan::plan_from_json(cfg.at("plan").is_string() ? cfg.at("plan").as_string() : cfg.at("plan").dump());
  M_ = static_cast<int>(cfg.at("M").as_int());
  gbs_ = static_cast<int>(cfg.at("gbs").as_int());
  rank_ = cfg.contains("rank") ? static_cast<int>(cfg.at("rank").as_int()) : 0;
  world_ = cfg.contains("world") ? static_cast<int>(cfg.at("world").as_int()) : 1;
  if (cfg.contains("lr")) lr_ = static_cast<float>(cfg.at("lr").as_double());
  if (cfg.contains("seed")) seed_ = static_cast<uint64_t>(cfg.at("seed").as_int());
  if (cfg.contains("timeline")) timeline_ = cfg.at("timeline").as_bool();
  if (cfg.contains("apply")) apply_ = cfg.at("apply").as_bool();
  if (cfg.contains("graph")) use_graph_ = cfg.at("graph").as_bool();
  if (cfg.contains("schedule")) gpipe_ = cfg.at("schedule").as_string() == "gpipe";
  if (cfg.contains("recompute")) recompute_ = cfg.at("recompute").as_bool();
  if (cfg.contains("probe")) probe_ = cfg.at("probe").as_bool();
  if (cfg.contains("allreduce")) {
    const std::string ar = cfg.at("allreduce").as_string();
    if (ar != "peer" && ar != "nccl") throw std::invalid_argument("dpl exec: allreduce must be peer or nccl");
    peer_ar_ = ar == "peer";
  }
  if (M_ < 1 || gbs_ % M_ != 0) throw std::invalid_argument("dpl exec: GBS must be a multiple of M");
  B_ = gbs_ / M_;

  // plan checks (the profile-independent part of PipelinePlan::validate,
  // model.cpp:100-131): contiguous cover of the model's layers, non-empty,
  // non-negative and pairwise disjoint device sets
  S_ = plan_.compute_stage_count();
  if (S_ < 1) throw std::invalid_argument("dpl exec: empty plan");
  int expect = 0;
  k_ = -1;
  std::vector<int> owner(static_cast<size_t>(std::max(world_, 1)), -1);
  for (int k = 0; k < S_; ++k) {
    const pipeplan::Stage& st = plan_.stages[k];
    if (st.layer_lo != expect || st.layer_hi <= st.layer_lo)
      throw std::invalid_argument("dpl exec: plan stages must partition the layers");
    if (st.devices.empty()) throw std::invalid_argument("dpl exec: stage " + std::to_string(k) + " has no GPUs");
    for (int g : st.devices) {
      if (g < 0) throw std::invalid_argument("dpl exec: negative GPU id in the plan");
      if (g < world_) {
        if (owner[g] >= 0)
          throw std::invalid_argument("dpl exec: GPU " + std::to_string(g) + " appears in more than one stage slot");
        owner[g] = k;
      }
    }
    expect = st.layer_hi;
    // replica j owns samples [B*j/r, B*(j+1)/r) of every micro-batch
    // (uneven when r does not divide B, as the planner's
    // cost model allows, costmodel/model.cpp:228-229)
    if (B_ < st.replication())
      throw std::invalid_argument("dpl exec: micro-batch of " + std::to_string(B_) + " samples is smaller than " +
                                  std::to_string(st.replication()) + " replicas");
    for (size_t j = 0; j < st.devices.size(); ++j) {
      if (st.devices[j] >= world_) throw std::invalid_argument("dpl exec: plan uses GPU ids beyond the world size");
      if (st.devices[j] == rank_) {
        k_ = k;
        rep_ = static_cast<int>(j);
      }
    }
  }
  if (expect != spec_.layers) throw std::invalid_argument("dpl exec: plan does not cover the model's layers");
  if (k_ < 0) throw std::invalid_argument("dpl exec: rank " + std::to_string(rank_) + " has no stage in the plan");
  const pipeplan::Stage& mine = plan_.stages[k_];
  r_ = mine.replication();
  lo_ = mine.layer_lo;
  hi_ = mine.layer_hi;
  group_ = mine.devices;  // sorted (plan_from_json): replica j is devices[j]
  if (r_ > kMaxReplicas) throw std::invalid_argument("dpl exec: at most 16 replicas per stage");
  // parameter blocks of the widest stage (layers + embedding + LM head + loss): every rank can lay out any rank's flags
  for (int k = 0; k < S_; ++k) nblk_ = std::max(nblk_, plan_.stages[k].layer_hi - plan_.stages[k].layer_lo + 3);

  // phi resolution, planner.cpp:501-508 (preset A is cost-independent)
  const int Se = 2 * S_ - 1;
  if (static_cast<int>(plan_.phi_expanded.size()) == Se) {
    phi_expanded_ = plan_.phi_expanded;
  } else if (!plan_.phi.empty()) {
    phi_expanded_ = pipeplan::expand_plan_phi(plan_.phi);
  } else {
    phi_expanded_.resize(Se);
    for (int x = 0; x < Se; ++x) phi_expanded_[x] = std::min(Se - x, M_);
  }
  // every rank checks the whole vector (check_phi, simulator.cpp:118-133, after
  // clamping to M): a phi that grows toward the top stage or is < 1 would
  // deadlock the ranks' flag waits rather than fail
  if (static_cast<int>(phi_expanded_.size()) != Se)
    throw std::invalid_argument("dpl exec: phi must have one entry per expanded stage");
  for (int x = 0; x < Se; ++x) {
    const int px = std::min(phi_expanded_[x], M_);
    if (phi_expanded_[x] < 1) throw std::invalid_argument("dpl exec: phi entries must be >= 1");
    if (x > 0 && px > std::min(phi_expanded_[x - 1], M_))
      throw std::invalid_argument("dpl exec: phi must be non-increasing toward the top stage");
  }
  if (phi_expanded_.back() != 1) throw std::invalid_argument("dpl exec: phi of the topmost stage must be 1");
  phi_ = gpipe_ ? M_ : std::min(phi_expanded_[2 * k_], M_);
  chain_ = pipeplan::stage_chain(M_, phi_, gpipe_ ? pipeplan::ScheduleKind::gpipe : pipeplan::ScheduleKind::dapple);
  // live micro-batches per stage = phi (DAPPLE) or M (GPipe); with
  // re-computation only the stage inputs stay alive and one stash set is reused
  stash_slots_ = recompute_ ? 1 : phi_;

  if (k_ > 0) {
    for (const Route& r : pipeplan::splitconcat_routes(plan_.stages[k_ - 1], mine, B_, static_cast<int>(elems(lo_))))
      if (r.dst_gpu == rank_) in_routes_.push_back(r);
  }
  if (k_ + 1 < S_) {
    for (const Route& r : pipeplan::splitconcat_routes(mine, plan_.stages[k_ + 1], B_, static_cast<int>(elems(hi_))))
      if (r.src_gpu == rank_) out_routes_.push_back(r);
  }
  numel_global_ = 1LL * gbs_ * elems(spec_.layers);
  loss_norm_ = spec_.vocab > 0    ? static_cast<float>(1LL * gbs_ * spec_.seq)
               : classify()       ? static_cast<float>(gbs_)  // mean CE over the samples
                                  : static_cast<float>(numel_global_);

  // --- context, layers, parameters
  ctx_.spec = spec_;
  ctx_.samples = slice_lo(rep_ + 1) - slice_lo(rep_);
  ctx_.rows = ctx_.samples * spec_.seq;
  ctx_.slots = stash_slots_;
  ctx_.mem = &mem_;
  // The compute chain (and the replica AllReduce) at the highest stream
  // priority, the weight-gradient side stream at the lowest: when both have
  // CTAs waiting for SMs, the critical path's go first (DPL_STREAM_PRIO=0: off)
  int prio_low = 0, prio_high = 0;
  {
    const char* e = std::getenv("DPL_STREAM_PRIO");
    if (!(e && e[0] == '0')) DPL_CUDA(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
  }
  DPL_CUDA(cudaStreamCreateWithPriority(&compute_, cudaStreamNonBlocking, prio_high));
  mem_.set_stream(compute_);
  DPL_CUDA(cudaStreamCreateWithFlags(&send_act_, cudaStreamNonBlocking));
  DPL_CUDA(cudaStreamCreateWithFlags(&send_grad_s_, cudaStreamNonBlocking));
  DPL_CUDA(cudaStreamCreateWithPriority(&reduce_, cudaStreamNonBlocking, prio_high));
  ctx_.stream = compute_;
  {  // weight-gradient side stream of the backward (DPL_WGRAD_STREAM=0: off)
    const char* e = std::getenv("DPL_WGRAD_STREAM");
    const bool on = cfg.contains("wgrad_stream") ? cfg.at("wgrad_stream").as_bool() : !(e && e[0] == '0');
    if (on) {
      DPL_CUDA(cudaStreamCreateWithPriority(&wgrad_, cudaStreamNonBlocking, prio_low));
      // side-stream grid cap: measured +2.5% on GPT-2 1.5B (1024-row slices)
      // at 64 CTAs, -2.5% on BERT-48 (4096 rows); default on for transformer
      // slices of <= 2048 token rows
      const char* c = std::getenv("DPL_WGRAD_CTAS");
      ctx_.wgrad_ctas = cfg.contains("wgrad_ctas") ? static_cast<int>(cfg.at("wgrad_ctas").as_int())
                        : c                        ? std::atoi(c)
                        : (spec_.kind == "bert" || spec_.kind == "gpt") && ctx_.rows <= 2048 ? 64
                                                                                              : 0;
      DPL_CUDA(cudaEventCreateWithFlags(&ctx_.ev_fork, cudaEventDisableTiming));
      DPL_CUDA(cudaEventCreateWithFlags(&ctx_.ev_join, cudaEventDisableTiming));
      ctx_.wstream = wgrad_;
    }
  }

  for (int l = lo_; l < hi_; ++l) layers_.push_back(make_layer(spec_, l));
  for (auto& layer : layers_) {
    param_off_.push_back(n_params_);
    n_params_ += (layer->param_count() + 63) / 64 * 64;  // keep every layer 256B aligned
  }
  if (spec_.vocab > 0 && k_ == 0) {
    emb_ = std::make_unique<TokenEmbedding>(spec_);
    emb_off_ = n_params_;
    n_params_ += (emb_->param_count() + 63) / 64 * 64;
  }
  if (spec_.vocab > 0 && k_ == S_ - 1) {
    head_ = std::make_unique<LmHead>(spec_);
    head_off_ = n_params_;
    n_params_ += (head_->param_count() + 63) / 64 * 64;
  }
  w32_ = static_cast<float*>(mem_.alloc(n_params_ * 4));
  g32_ = static_cast<float*>(mem_.alloc(n_params_ * 4));
  w16_ = static_cast<bf16*>(mem_.alloc(n_params_ * 2));
  for (size_t li = 0; li < layers_.size(); ++li)
    layers_[li]->bind(w32_ + param_off_[li], g32_ + param_off_[li], w16_ + param_off_[li], seed_, compute_);
  if (emb_) emb_->bind(w32_ + emb_off_, g32_ + emb_off_, w16_ + emb_off_, seed_, compute_);
  if (head_) head_->bind(w32_ + head_off_, g32_ + head_off_, w16_ + head_off_, seed_, compute_);

  const size_t RH = static_cast<size_t>(ctx_.rows) * spec_.hidden;
  if (spec_.kind == "vgg") {
    size_t col = 0, dz = 0;
    for (auto& layer : layers_) {
      col = std::max(col, layer->col_elems(ctx_));
      dz = std::max(dz, layer->dz_elems(ctx_));
    }
    if (col) ctx_.conv_dcol = static_cast<bf16*>(mem_.alloc(col * 2));
    ctx_.conv_dz = static_cast<bf16*>(mem_.alloc(std::max<size_t>(dz, 8) * 2));
  } else if (spec_.kind != "mlp") {
    const size_t z = static_cast<size_t>(spec_.heads) * ctx_.samples;
    ctx_.att_dsum = static_cast<float*>(mem_.alloc(z * spec_.seq * 4));
    ctx_.att_dq = static_cast<float*>(mem_.alloc(RH * 4));
    if (spec_.causal) {
      const size_t tiles = z * (spec_.seq / 128);
      ctx_.att_part = static_cast<float*>(mem_.alloc(tiles * 2 * 66 * 128 * 4));
      ctx_.att_flags = static_cast<int*>(mem_.alloc(tiles * 4));
    }
    ctx_.ln_ws = static_cast<float*>(mem_.alloc(static_cast<size_t>(kLnBwdBlocks) * 4 * spec_.hidden * 4));
    ctx_.t_h = static_cast<bf16*>(mem_.alloc(RH * 2));
    ctx_.t_h2 = static_cast<bf16*>(mem_.alloc(RH * 2));
    ctx_.t_h3 = static_cast<bf16*>(mem_.alloc(RH * 2));
    ctx_.t_qkv = static_cast<bf16*>(mem_.alloc(RH * 3 * 2));
    ctx_.t_f = static_cast<bf16*>(mem_.alloc(static_cast<size_t>(ctx_.rows) * spec_.ffn * 2));
  }
  if (spec_.kind != "vgg") {
    // scratch for the split-K bf16 GEMMs of small replica slices (gemm_tcgen05.cu
    // split_bf16_candidate): one [rows][widest layer output] fp32 buffer, zero
    const int widest = spec_.kind == "mlp" ? spec_.hidden : std::max(spec_.hidden, spec_.ffn);
    ctx_.gemms.split_ws_bytes = static_cast<size_t>(ctx_.rows) * widest * 4;
    ctx_.gemms.split_ws = static_cast<float*>(mem_.alloc(ctx_.gemms.split_ws_bytes));
  }
  for (auto& layer : layers_) layer->alloc_stash(ctx_);
  act_.assign(L(), {});
  // activation buffers sized per boundary: layer l's input is samples x elems(l)
  const size_t smp = static_cast<size_t>(ctx_.samples);
  size_t gmax = 8;
  for (int li = 1; li < L(); ++li) {
    const size_t e = smp * elems(lo_ + li);
    gmax = std::max(gmax, e);
    for (int s = 0; s < stash_slots_; ++s) act_[li].push_back(static_cast<bf16*>(mem_.alloc(e * 2)));
  }
  if (recompute_) rc_out_ = static_cast<bf16*>(mem_.alloc(out_elems() * 2));
  if (k_ == 0)
    for (int s = 0; s < phi_; ++s) in_.push_back(static_cast<bf16*>(mem_.alloc(in_elems() * 2)));
  for (int i = 0; i < M_; ++i) out_.push_back(static_cast<bf16*>(mem_.alloc(out_elems() * 2)));
  if (k_ == S_ - 1) {
    for (int s = 0; s < phi_; ++s) {
      if (!head_ && !classify()) target_.push_back(static_cast<bf16*>(mem_.alloc(out_elems() * 2)));
      dloss_.push_back(static_cast<bf16*>(mem_.alloc(out_elems() * 2)));
    }
  }
  // the head's logits-gradient stash lives from F_i to B_i like the loss
  // gradient (phi slots, also under re-computation)
  if (head_) head_->alloc_stash(ctx_, phi_);
  for (int s = 0; s < phi_ && emb_; ++s) tok_.push_back(static_cast<int*>(mem_.alloc(ctx_.rows * 4)));
  for (int s = 0; s < phi_ && head_; ++s) tgt_tok_.push_back(static_cast<int*>(mem_.alloc(ctx_.rows * 4)));
  // classification labels: one class id per sample
  for (int s = 0; s < phi_ && classify() && k_ == S_ - 1; ++s)
    tgt_tok_.push_back(static_cast<int*>(mem_.alloc(smp * 4)));
  if (k_ > 0)
    for (int i = 0; i < M_; ++i) send_grad_.push_back(static_cast<bf16*>(mem_.alloc(in_elems() * 2)));
  if (probe_) {
    probes_.resize(L());
    for (int li = 0; li < L(); ++li) {
      Probe& p = probes_[li];
      p.nx = smp * elems(lo_ + li);
      p.ny = smp * elems(lo_ + li + 1);
      p.naux = layers_[li]->probe_aux_elems(ctx_);
      p.x = static_cast<bf16*>(mem_.alloc(p.nx * 2));
      p.dx = static_cast<bf16*>(mem_.alloc(p.nx * 2));
      p.y = static_cast<bf16*>(mem_.alloc(p.ny * 2));
      p.dy = static_cast<bf16*>(mem_.alloc(p.ny * 2));
      if (p.naux) p.aux = static_cast<bf16*>(mem_.alloc(p.naux * 2));
    }
  }
  if (emb_) gmax = std::max(gmax, in_elems());
  gbuf_[0] = static_cast<bf16*>(mem_.alloc(gmax * 2));
  gbuf_[1] = static_cast<bf16*>(mem_.alloc(gmax * 2));
  t0_ = static_cast<unsigned long long*>(mem_.alloc(8));

  // receive region: one allocation so a single IPC handle covers it
  peer_samples_.assign(world_, 0);
  peer_stage_.assign(world_, 0);
  for (int k = 0; k < S_; ++k)
    for (int j = 0; j < plan_.stages[k].replication(); ++j) {
      const int rk = plan_.stages[k].replication();
      peer_samples_[plan_.stages[k].devices[j]] = slice_lo(j + 1, rk) - slice_lo(j, rk);
      peer_stage_[plan_.stages[k].devices[j]] = k;
    }
  recv_grad_off_ = layout_grad_off(rank_);
  flags_off_ = layout_flags_off(rank_);
  recv_bytes_ = loss_off(rank_) + 256;
  recv_ = static_cast<uint8_t*>(mem_.alloc(recv_bytes_));
  loss_acc_ = reinterpret_cast<float*>(recv_ + loss_off(rank_));
  peer_recv_.assign(world_, nullptr);
  peer_g32_.assign(world_, nullptr);
  colocated_.assign(world_, 0);

  // events
  auto mk = [](cudaEvent_t* e) { DPL_CUDA(cudaEventCreate(e)); };
  auto mk_nt = [](cudaEvent_t* e) { DPL_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming)); };
  mk(&ev_begin_);
  mk(&ev_end_);
  mk_nt(&ev_reduce_done_);
  mk_nt(&ev_sa_done_);
  mk_nt(&ev_sg_done_);
  mk_nt(&ev_fork_);
  mk_nt(&ev_last_bwd_);
  mk_nt(&ev_wg_done_);
  fwd_ev_.resize(M_);
  bwd_ev_.resize(M_);
  send_fwd_ev_.resize(M_);
  send_bwd_ev_.resize(M_);
  for (auto* v : {&fwd_ev_, &bwd_ev_, &send_fwd_ev_, &send_bwd_ev_})
    for (BlockEvents& b : *v) {
      mk(&b.start);
      mk(&b.end);
    }
  layer_done_.resize(L());
  for (auto& e : layer_done_) mk_nt(&e);
  ar_ev_.resize(nblk_);
  ar_bytes_.assign(nblk_, 0);
  for (BlockEvents& b : ar_ev_) {
    mk(&b.start);
    mk(&b.end);
  }
  mk_nt(&emb_done_);
  mk_nt(&head_done_);
  fwd_done_.resize(M_);
  bwd_done_.resize(M_);
  for (auto& e : fwd_done_) mk_nt(&e);
  for (auto& e : bwd_done_) mk_nt(&e);

  for (size_t li = 0; li < layers_.size(); ++li) {
    const bool need_dx = !(k_ == 0 && li == 0) || emb_;
    flops_per_step_ += M_ * ((recompute_ ? 2 : 1) * layers_[li]->flops_fwd(ctx_) + layers_[li]->flops_bwd(ctx_, need_dx));
  }
  if (head_) flops_per_step_ += M_ * (head_->flops_fwd(ctx_) + head_->flops_bwd(ctx_));
  DPL_CUDA(cudaMallocHost(reinterpret_cast<void**>(&loss_host_), sizeof(float)));
  // parameters initialised and every buffer (incl. the IPC-exported flags)
  // zeroed before any peer can see this rank
  DPL_CUDA(cudaDeviceSynchronize());
}

size_t Executor::layout_grad_off(int rank) const {
  const pipeplan::Stage& st = plan_.stages[peer_stage_[rank]];
  const size_t bytes = static_cast<size_t>(M_) * peer_samples_[rank] * elems(st.layer_lo) * 2;
  return (bytes + 255) & ~size_t(255);
}
size_t Executor::layout_flags_off(int rank) const {
  const pipeplan::Stage& st = plan_.stages[peer_stage_[rank]];
  const size_t bytes = static_cast<size_t>(M_) * peer_samples_[rank] * elems(st.layer_hi) * 2;
  return layout_grad_off(rank) + ((bytes + 255) & ~size_t(255));
}

// Teardown is two-phase across ranks: every rank first unmaps its peers'
// regions and destroys its communicator (disconnect), the ranks barrier, and
// only then free memory -- freeing an exported region while another process
// still has it mapped is undefined behaviour in CUDA IPC.
void Executor::disconnect() {
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  // captured steps reference the communicator and the peer mappings
  for (auto& g : graphs_) g.destroy();
  graphs_.clear();
  if (comm_) {
    ncclCommDestroy(comm_);
    comm_ = nullptr;
  }
  for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
  ipc_opened_.clear();
  for (uint8_t*& p : peer_recv_) p = nullptr;
  for (float*& p : peer_g32_) p = nullptr;
}

Executor::~Executor() {
  disconnect();
  if (loss_host_) cudaFreeHost(loss_host_);
  for (void* p : staging_)
    if (p) cudaFreeHost(p);
  for (cudaEvent_t e : {ev_begin_, ev_end_, ev_reduce_done_, ev_sa_done_, ev_sg_done_, ev_fork_, ev_last_bwd_,
                        emb_done_, head_done_, ev_wg_done_, ctx_.ev_fork, ctx_.ev_join})
    if (e) cudaEventDestroy(e);
  for (auto* v : {&fwd_ev_, &bwd_ev_, &send_fwd_ev_, &send_bwd_ev_, &ar_ev_})
    for (BlockEvents& b : *v) {
      if (b.start) cudaEventDestroy(b.start);
      if (b.end) cudaEventDestroy(b.end);
    }
  for (auto* v : {&layer_done_, &fwd_done_, &bwd_done_})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {compute_, send_act_, send_grad_s_, reduce_, wgrad_})
    if (s) cudaStreamDestroy(s);
}

size_t Executor::input_bytes() const {
  if (k_ != 0) return 0;
  if (emb_) return static_cast<size_t>(M_) * ctx_.rows * 4;  // token ids
  return static_cast<size_t>(M_) * in_elems() * 2;
}

size_t Executor::target_bytes() const {
  if (k_ != S_ - 1) return 0;
  if (head_) return static_cast<size_t>(M_) * ctx_.rows * 4;        // next-token ids
  if (classify()) return static_cast<size_t>(M_) * ctx_.samples * 4;  // class labels
  return static_cast<size_t>(M_) * out_elems() * 2;
}

// Pinned (or registered) host memory is used in place; pageable memory is
// copied into an executor-owned pinned buffer first (a captured step can
// only read page-locked memory).
const void* Executor::stage_host(const void* p, int which) {
  if (!p) return nullptr;
  const size_t bytes = which == 0 ? input_bytes() : target_bytes();
  if (bytes == 0) return nullptr;  // this rank consumes no such tensor
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost) return p;
  cudaGetLastError();
  if (staging_bytes_[which] < bytes) {
    if (staging_[which]) DPL_CUDA(cudaFreeHost(staging_[which]));
    staging_[which] = nullptr;
    DPL_CUDA(cudaMallocHost(&staging_[which], bytes));
    staging_bytes_[which] = bytes;
  }
  std::memcpy(staging_[which], p, bytes);
  return staging_[which];
}

size_t Executor::export_blob(void* blob, size_t cap) {
  if (cap < sizeof(PeerBlob)) throw std::invalid_argument("dpl exec: export buffer too small");
  PeerBlob b{};
  DPL_CUDA(cudaIpcGetMemHandle(&b.recv, recv_));
  DPL_CUDA(cudaIpcGetMemHandle(&b.grads, g32_));
  b.pid = static_cast<long long>(getpid());
  b.device = device_;
  b.recv_ptr = reinterpret_cast<unsigned long long>(recv_);
  b.grads_ptr = reinterpret_cast<unsigned long long>(g32_);
  std::memcpy(blob, &b, sizeof b);
  return sizeof b;
}

void Executor::connect(const uint8_t* blobs, size_t blob_len, int world) {
  if (world != world_) throw std::invalid_argument("dpl exec: world size mismatch");
  if (blob_len < sizeof(PeerBlob)) throw std::invalid_argument("dpl exec: peer blobs too short");
  auto blob = [&](int p) {
    PeerBlob b;
    std::memcpy(&b, blobs + static_cast<size_t>(p) * blob_len, sizeof b);
    return b;
  };
  const long long me = static_cast<long long>(getpid());
  std::vector<int> peers;
  for (const Route& r : out_routes_) peers.push_back(r.dst_gpu);
  for (const Route& r : in_routes_) peers.push_back(r.src_gpu);
  if (rank_ == 0) {
    for (int p = 1; p < world_; ++p) peers.push_back(p);
  } else {
    peers.push_back(0);
  }
  for (int p : group_) peers.push_back(p);
  for (int p = 0; p < world_; ++p) {
    const PeerBlob b = blob(p);
    colocated_[p] = b.pid == me && b.device == device_;
  }
  for (int p : peers) {
    if (p == rank_ || peer_recv_[p]) continue;
    const PeerBlob b = blob(p);
    if (b.pid == me) {
      // a rank of this process: plain pointers (peer access for another GPU)
      if (b.device != device_) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) DPL_CUDA(e);
        cudaGetLastError();
      }
      peer_recv_[p] = reinterpret_cast<uint8_t*>(b.recv_ptr);
      peer_g32_[p] = reinterpret_cast<float*>(b.grads_ptr);
      continue;
    }
    void* ptr = nullptr;
    DPL_CUDA(cudaIpcOpenMemHandle(&ptr, b.recv, cudaIpcMemLazyEnablePeerAccess));
    peer_recv_[p] = static_cast<uint8_t*>(ptr);
    ipc_opened_.push_back(ptr);
    if (std::find(group_.begin(), group_.end(), p) != group_.end() && peer_ar_) {
      DPL_CUDA(cudaIpcOpenMemHandle(&ptr, b.grads, cudaIpcMemLazyEnablePeerAccess));
      peer_g32_[p] = static_cast<float*>(ptr);
      ipc_opened_.push_back(ptr);
    }
  }
  peer_g32_[rank_] = g32_;
  // the flag waits of ranks sharing one GPU must stay stream memory
  // operations: a spinning wait kernel could starve the kernel that would
  // release it
  for (int p = 0; p < world_; ++p)
    if (p != rank_ && colocated_[p] && !memops_ok())
      throw std::runtime_error("dpl exec: ranks sharing a GPU need stream memory operations (cuStreamWaitValue32)");
}

bool Executor::shares_gpu() const {
  for (int p = 0; p < world_; ++p)
    if (p != rank_ && colocated_[p]) return true;
  return false;
}

// Called collectively: phase p (1..world-1) calibrates rank p against rank 0;
// the host side barriers between phases.  Returns this rank's offset.
long long Executor::calibrate_clock(int phase) {
  if (world_ == 1 || (rank_ != 0 && rank_ != phase)) return clock_offset_ns_;
  // ranks on one GPU share its timer (and must not run the spinning ping-pong)
  if (colocated_[rank_ == 0 ? phase : 0]) return 0;
  constexpr int kRounds = 64;
  auto calib = [&](uint8_t* region, int rank) {
    uint8_t* base = region + layout_flags_off(rank) + 2 * bank_words() * 4;
    return base;
  };
  DPL_CUDA(cudaSetDevice(device_));
  // words start at zero (zeroed allocation) and are only ever counted up
  // 1..kRounds per responder, so no re-zeroing (and no zeroing race) is needed
  uint8_t* mine = calib(recv_, rank_);
  if (rank_ == 0) {
    uint8_t* peer = calib(peer_recv_[phase], phase);
    unsigned long long* out = nullptr;
    DPL_CUDA(cudaMalloc(&out, 3 * kRounds * sizeof(unsigned long long)));
    clock_ping_kernel<<<1, 1, 0, compute_>>>(reinterpret_cast<uint32_t*>(peer), reinterpret_cast<uint32_t*>(mine + 4),
                                             reinterpret_cast<unsigned long long*>(mine + 8), out, kRounds);
    DPL_CUDA(cudaStreamSynchronize(compute_));
    std::vector<unsigned long long> h(3 * kRounds);
    DPL_CUDA(cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(out);
    // offset of the peer relative to rank 0 from the tightest round trip
    long long best_rtt = -1, offset = 0;
    for (int k = 0; k < kRounds; ++k) {
      const long long t0 = h[3 * k], tp = h[3 * k + 1], t2 = h[3 * k + 2];
      if (best_rtt < 0 || t2 - t0 < best_rtt) {
        best_rtt = t2 - t0;
        offset = tp - (t0 + t2) / 2;
      }
    }
    return offset;  // rank 0 reports the peer's offset; the host forwards it
  }
  uint8_t* zero = calib(peer_recv_[0], 0);
  clock_pong_kernel<<<1, 1, 0, compute_>>>(reinterpret_cast<uint32_t*>(mine), reinterpret_cast<uint32_t*>(zero + 4),
                                           reinterpret_cast<unsigned long long*>(zero + 8), kRounds);
  DPL_CUDA(cudaStreamSynchronize(compute_));
  return 0;
}

void Executor::nccl_init(const void* id) {
  if (r_ == 1 || peer_ar_) return;
  for (int p : group_)
    if (p != rank_ && colocated_[p]) throw std::runtime_error("dpl exec: NCCL cannot reduce over ranks sharing a GPU");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  DPL_NCCL(ncclCommInitRank(&comm_, r_, uid, rep_));
}

void Executor::wait_flag(cudaStream_t s, uint32_t* flag, uint32_t value) {
  if (memops_ok()) {
    if (StreamValueFn fn = wait_value_fn()) {
      const CUresult rc = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value, 0x0 /*GEQ*/);
      if (rc == CUDA_SUCCESS) return;
    }
    // a spinning wait kernel could starve the kernel of a rank sharing this
    // GPU that would release it: those ranks need stream memory operations
    if (shares_gpu())
      throw std::runtime_error("dpl exec: ranks sharing a GPU need stream memory operations (cuStreamWaitValue32)");
    memops_flag() = false;  // not available / not capturable: one-thread acquire spin on this stream
  }
  count_launch();
  wait_kernel<<<1, 1, 0, s>>>(flag, value);
}

void Executor::signal(cudaStream_t s, uint32_t* remote_flag, uint32_t value) {
  // default flags (0): the write is ordered after the stream's earlier work
  // and that work's memory writes (the hand-off copy) are visible first
  if (memops_ok()) {
    if (StreamValueFn fn = write_value_fn()) {
      const CUresult rc =
          fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(remote_flag), value, 0x0 /*DEFAULT*/);
      if (rc == CUDA_SUCCESS) return;
    }
    memops_flag() = false;  // not available / not capturable: the capture is retried with kernels
  }
  count_launch();
  signal_kernel<<<1, 1, 0, s>>>(remote_flag, value);
}

void Executor::forward(int i, uint32_t base) {
  const int slot = i % phi_;                         // stage input / target / loss-grad buffers
  const int ss = recompute_ ? 0 : i % stash_slots_;  // layer-internal stash
  const bf16* x;
  if (k_ == 0) {
    x = in_[slot];
  } else {
    for (const Route& r : in_routes_) wait_flag(compute_, flags() + r.src_gpu, base + i + 1);
    x = recv_act(i);
  }
  record(fwd_ev_[i].start, compute_);
  if (emb_) emb_->forward(ctx_, tok_[slot], in_[slot]);
  const bool probe = probe_ && i == M_ - 1;
  for (int li = 0; li < L(); ++li) {
    bf16* y = li + 1 < L() ? act_[li + 1][ss] : out_[i];
    layers_[li]->forward(ctx_, ss, x, y);
    if (probe) {
      Probe& p = probes_[li];
      probe_copy(p.x, x, p.nx);
      probe_copy(p.y, y, p.ny);
      probe_copy(p.aux, layers_[li]->probe_aux(ss), p.naux);
    }
    x = y;
  }
  if (head_) {
    // causal-LM cross-entropy, mean over the global batch's tokens
    head_->forward(ctx_, slot, out_[i], tgt_tok_[slot], loss_acc_, 1.0f / loss_norm_);
  } else if (k_ == S_ - 1 && classify()) {
    // softmax cross-entropy over the classes, mean over the global batch
    DPL_CUDA(cudaMemcpyAsync(dloss_[slot], out_[i], out_elems() * 2, cudaMemcpyDeviceToDevice, compute_));
    cross_entropy_fwd_bwd(dloss_[slot], tgt_tok_[slot], loss_acc_, ctx_.samples, spec_.classes, 1.0f / loss_norm_,
                          compute_);
  } else if (k_ == S_ - 1) {
    // MSE over the whole global batch: loss = sum (y-t)^2 / numel, dY = 2 (y-t) / numel
    mse_loss(out_[i], target_[slot], dloss_[slot], loss_acc_, static_cast<long long>(out_elems()),
             2.0f / static_cast<float>(numel_global_), compute_);
  }
  record(fwd_ev_[i].end, compute_);
  if (!out_routes_.empty()) {
    DPL_CUDA(cudaEventRecord(fwd_done_[i], compute_));
    DPL_CUDA(cudaStreamWaitEvent(send_act_, fwd_done_[i], 0));
    record(send_fwd_ev_[i].start, send_act_);
    // routes are in activation elements (samples x elems(boundary))
    const size_t eb = static_cast<size_t>(elems(hi_));
    for (const Route& r : out_routes_) {
      uint8_t* peer = peer_recv_[r.dst_gpu];
      bf16* dst = reinterpret_cast<bf16*>(peer) + static_cast<size_t>(i) * peer_samples_[r.dst_gpu] * eb + r.dst_row;
      DPL_CUDA(cudaMemcpyAsync(dst, out_[i] + r.src_row, r.rows * 2, cudaMemcpyDeviceToDevice, send_act_));
      uint32_t* flag = flag_at(peer, r.dst_gpu, rank_);
      signal(send_act_, flag, base + i + 1);
    }
    record(send_fwd_ev_[i].end, send_act_);
  }
}

void Executor::backward(int i, uint32_t base) {
  const int slot = i % phi_;
  const int ss = recompute_ ? 0 : i % stash_slots_;
  const bf16* dy;
  if (k_ == S_ - 1) {
    dy = dloss_[slot];
  } else {
    for (const Route& r : out_routes_) wait_flag(compute_, flags() + world_ + r.dst_gpu, base + i + 1);
    dy = recv_grad(i);
  }
  record(bwd_ev_[i].start, compute_);
  const bool last_mb = i == M_ - 1;
  if (head_) {
    head_->backward(ctx_, slot, out_[i], dloss_[slot]);
    if (last_mb) reduce_apply(head_done_, head_off_, head_->param_count(), L() + 1);
  }
  if (recompute_) {
    // the backward block first re-runs the stage forward (B' = B + F)
    const bf16* x = k_ == 0 ? in_[slot] : recv_act(i);
    for (int li = 0; li < L(); ++li) {
      bf16* y = li + 1 < L() ? act_[li + 1][ss] : rc_out_;
      layers_[li]->forward(ctx_, ss, x, y);
      x = y;
    }
  }
  int pp = 0;
  for (int li = L() - 1; li >= 0; --li) {
    const bf16* x = li > 0 ? act_[li][ss] : (k_ == 0 ? in_[slot] : recv_act(i));
    bf16* dx = nullptr;
    if (li > 0) {
      dx = gbuf_[pp];
      pp ^= 1;
    } else if (k_ > 0) {
      dx = send_grad_[i];
    } else if (emb_) {
      dx = gbuf_[pp];
    }
    ctx_.cur_y = li + 1 < L() ? act_[li + 1][ss] : (recompute_ ? rc_out_ : out_[i]);
    if (probe_ && last_mb) probe_copy(probes_[li].dy, dy, probes_[li].ny);
    layers_[li]->backward(ctx_, ss, x, dy, dx);
    if (probe_ && last_mb) probe_copy(probes_[li].dx, dx, probes_[li].nx);
    dy = dx;
    // this layer's gradients are final: AllReduce + apply while the
    // remaining layers' backward runs
    if (last_mb) reduce_apply(layer_done_[li], param_off_[li], layers_[li]->param_count(), li);
  }
  if (emb_) {
    emb_->backward(ctx_, tok_[slot], dy);
    if (last_mb) reduce_apply(emb_done_, emb_off_, emb_->param_count(), L());
  }
  record(bwd_ev_[i].end, compute_);
  if (k_ > 0) {
    DPL_CUDA(cudaEventRecord(bwd_done_[i], compute_));
    DPL_CUDA(cudaStreamWaitEvent(send_grad_s_, bwd_done_[i], 0));
    record(send_bwd_ev_[i].start, send_grad_s_);
    const size_t eb = static_cast<size_t>(elems(lo_));
    for (const Route& r : in_routes_) {
      uint8_t* peer = peer_recv_[r.src_gpu];
      bf16* dst = reinterpret_cast<bf16*>(peer + layout_grad_off(r.src_gpu)) +
                  static_cast<size_t>(i) * peer_samples_[r.src_gpu] * eb + r.src_row;
      DPL_CUDA(cudaMemcpyAsync(dst, send_grad_[i] + r.dst_row, r.rows * 2, cudaMemcpyDeviceToDevice, send_grad_s_));
      uint32_t* flag = flag_at(peer, r.src_gpu, world_ + rank_);
      signal(send_grad_s_, flag, base + i + 1);
    }
    record(send_bwd_ev_[i].end, send_grad_s_);
  }
}

void Executor::reduce_apply(cudaEvent_t ready, size_t off, size_t n, int blk) {
  DPL_CUDA(cudaEventRecord(ready, compute_));
  DPL_CUDA(cudaStreamWaitEvent(reduce_, ready, 0));
  if (r_ > 1) {
    record(ar_ev_[blk].start, reduce_);
    ar_bytes_[blk] = static_cast<long long>(n) * 4;
  }
  if (r_ > 1 && peer_ar_) {
    std::vector<float*> peers(r_);
    for (int j = 0; j < r_; ++j) peers[j] = peer_g32_[group_[j]] + off;
    peer_allreduce(peers, n, blk);
  } else if (r_ > 1) {
    if (!comm_) throw std::runtime_error("dpl exec: replicated stage without an NCCL communicator");
    DPL_NCCL(ncclAllReduce(g32_ + off, g32_ + off, n, ncclFloat, ncclSum, comm_, reduce_));
  }
  if (r_ > 1) record(ar_ev_[blk].end, reduce_);
  if (apply_) sgd_apply(w32_ + off, g32_ + off, w16_ + off, static_cast<long long>(n), lr_, reduce_);
}

// Two flag rounds around one kernel (collective.cu): every replica announces
// that its block is final, replica j reduces chunk j across the group and
// stores the sum into every replica, and each replica waits until all
// chunks have landed before anything (SGD) reads the block.
void Executor::peer_allreduce(const std::vector<float*>& peers, size_t n, int blk) {
  if (static_cast<int>(peers.size()) != r_) throw std::logic_error("dpl exec: replica pointers");
  ReplicaPtrs rp{};
  for (int j = 0; j < r_; ++j) {
    if (!peers[j]) throw std::runtime_error("dpl exec: replica peer gradients not mapped (connect first)");
    rp.g[j] = peers[j];
  }
  for (int round = 0; round < 2; ++round) {
    if (round == 1) replica_allreduce_chunk(rp, r_, static_cast<long long>(n), rep_, reduce_);
    for (int p : group_)
      if (p != rank_) signal(reduce_, flag_at(peer_recv_[p], p, ar_word(round, blk, rank_)), 1u);
    for (int p : group_)
      if (p != rank_) wait_flag(reduce_, flags() + ar_word(round, blk, p), 1u);
  }
}

void Executor::enqueue_step(const void* host_input, const void* host_target) {
  const uint32_t base = 0;  // flag values are i+1 within the bank of this step
  count_launch();
  stamp_kernel<<<1, 1, 0, compute_>>>(t0_);
  record(ev_begin_, compute_);
  // fork every side stream from the compute stream (they join again at the
  // end), so a captured step always has one origin and one sink
  DPL_CUDA(cudaEventRecord(ev_fork_, compute_));
  for (cudaStream_t side : {send_act_, send_grad_s_, reduce_, wgrad_})
    if (side) DPL_CUDA(cudaStreamWaitEvent(side, ev_fork_, 0));
  DPL_CUDA(cudaMemsetAsync(loss_acc_, 0, 4, compute_));

  // sample rows [row0, row0 + samples) of micro-batch i owned by this replica
  const long long slice_first = slice_lo(rep_);
  for (const pipeplan::ChainOp& op : chain_) {
    const int i = op.micro_batch;
    const int slot = i % phi_;
    if (op.kind == pipeplan::BlockKind::forward) {
      const long long sample0 = 1LL * i * B_ + slice_first;
      const long long idx0 = sample0 * elems(0);
      const long long tidx0 = sample0 * elems(spec_.layers);
      const long long tok0 = sample0 * spec_.seq;
      const size_t rows = static_cast<size_t>(ctx_.rows);
      const size_t ein = in_elems(), eout = out_elems();
      if (emb_) {  // token ids: [M][rows] int32 on the host
        if (host_input) {
          DPL_CUDA(cudaMemcpyAsync(tok_[slot], static_cast<const int*>(host_input) + i * rows, rows * 4,
                                   cudaMemcpyHostToDevice, compute_));
        } else {
          fill_tokens(tok_[slot], static_cast<long long>(rows), seed_, kTensorInput, tok0, spec_.vocab, compute_);
        }
      } else if (k_ == 0) {
        if (host_input) {
          DPL_CUDA(cudaMemcpyAsync(in_[slot], static_cast<const bf16*>(host_input) + static_cast<size_t>(i) * ein,
                                   ein * 2, cudaMemcpyHostToDevice, compute_));
        } else {
          fill_uniform_bf16(in_[slot], static_cast<long long>(ein), seed_, kTensorInput, idx0, 1.0f, compute_);
        }
      }
      if (head_) {
        if (host_target) {
          DPL_CUDA(cudaMemcpyAsync(tgt_tok_[slot], static_cast<const int*>(host_target) + i * rows, rows * 4,
                                   cudaMemcpyHostToDevice, compute_));
        } else {
          fill_tokens(tgt_tok_[slot], static_cast<long long>(rows), seed_, kTensorTarget, tok0, spec_.vocab, compute_);
        }
      } else if (k_ == S_ - 1 && classify()) {  // class labels: [M][samples] int32 on the host
        const size_t smp = static_cast<size_t>(ctx_.samples);
        if (host_target) {
          DPL_CUDA(cudaMemcpyAsync(tgt_tok_[slot], static_cast<const int*>(host_target) + i * smp, smp * 4,
                                   cudaMemcpyHostToDevice, compute_));
        } else {
          fill_tokens(tgt_tok_[slot], static_cast<long long>(smp), seed_, kTensorTarget, sample0, spec_.classes,
                      compute_);
        }
      } else if (k_ == S_ - 1) {
        if (host_target) {
          DPL_CUDA(cudaMemcpyAsync(target_[slot], static_cast<const bf16*>(host_target) + static_cast<size_t>(i) * eout,
                                   eout * 2, cudaMemcpyHostToDevice, compute_));
        } else {
          fill_uniform_bf16(target_[slot], static_cast<long long>(eout), seed_, kTensorTarget, tidx0, 1.0f, compute_);
        }
      }
      forward(i, base);
    } else {
      backward(i, base);
    }
  }
  if (k_ == S_ - 1 && r_ > 1) {
    // sync (non-timing) event: timing events are external nodes in a
    // captured step and cannot carry dependencies
    DPL_CUDA(cudaEventRecord(ev_last_bwd_, compute_));
    DPL_CUDA(cudaStreamWaitEvent(reduce_, ev_last_bwd_, 0));
    if (peer_ar_) {
      std::vector<float*> peers(r_);
      for (int j = 0; j < r_; ++j)
        peers[j] = group_[j] == rank_ ? loss_acc_
                                      : reinterpret_cast<float*>(peer_recv_[group_[j]] + loss_off(group_[j]));
      peer_allreduce(peers, 1, L() + 2);
    } else {
      if (!comm_) throw std::runtime_error("dpl exec: replicated stage without an NCCL communicator");
      DPL_NCCL(ncclAllReduce(loss_acc_, loss_acc_, 1, ncclFloat, ncclSum, comm_, reduce_));
    }
  }
  DPL_CUDA(cudaEventRecord(ev_reduce_done_, reduce_));
  DPL_CUDA(cudaEventRecord(ev_sa_done_, send_act_));
  DPL_CUDA(cudaEventRecord(ev_sg_done_, send_grad_s_));
  DPL_CUDA(cudaStreamWaitEvent(compute_, ev_reduce_done_, 0));
  DPL_CUDA(cudaStreamWaitEvent(compute_, ev_sa_done_, 0));
  DPL_CUDA(cudaStreamWaitEvent(compute_, ev_sg_done_, 0));
  if (wgrad_) {  // joined after every layer already; a step without transformer work still rejoins it
    DPL_CUDA(cudaEventRecord(ev_wg_done_, wgrad_));
    DPL_CUDA(cudaStreamWaitEvent(compute_, ev_wg_done_, 0));
  }
  record(ev_end_, compute_);
  if (k_ == S_ - 1) DPL_CUDA(cudaMemcpyAsync(loss_host_, loss_acc_, 4, cudaMemcpyDeviceToHost, compute_));
  // clear this step's flag bank (signalled again two steps from now)
  DPL_CUDA(cudaMemsetAsync(flags(), 0, bank_words() * 4, compute_));
}

// Captures enqueue_step into g.  A stream memory op that cannot be captured
// invalidates the capture; wait_flag then switches to its kernel form and the
// capture is retried once.  Any other failure is rethrown as is.
void Executor::capture_step(GraphEntry& g, const void* host_input, const void* host_target) {
  for (int attempt = 0; attempt < 2; ++attempt) {
    cudaGraph_t graph = nullptr;
    const long long counted0 = launch_count();
    const bool memops_before = memops_ok();
    DPL_CUDA(cudaStreamBeginCapture(compute_, cudaStreamCaptureModeRelaxed));
    capturing_ = true;
    kernel_timer().capturing = true;
    std::string error;
    try {
      enqueue_step(host_input, host_target);
    } catch (const std::exception& e) {
      error = e.what();
    }
    capturing_ = false;
    kernel_timer().capturing = false;
    const cudaError_t end = cudaStreamEndCapture(compute_, &graph);
    // captured launches are not executions: the kernel nodes are counted on
    // every replay instead
    count_launch(counted0 - launch_count());
    if (error.empty() && end == cudaSuccess && graph) {
      g.graph = graph;
      DPL_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
      size_t n_nodes = 0;
      DPL_CUDA(cudaGraphGetNodes(graph, nullptr, &n_nodes));
      std::vector<cudaGraphNode_t> nodes(n_nodes);
      DPL_CUDA(cudaGraphGetNodes(graph, nodes.data(), &n_nodes));
      const void* bases[2] = {host_input, host_target};
      const size_t sizes[2] = {input_bytes(), target_bytes()};
      g.kernels = 0;
      for (cudaGraphNode_t nd : nodes) {
        // stream memory-op nodes (the flag waits) have no runtime-API type:
        // the query fails for them, which is fine -- only kernels and host
        // copies matter here
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nd, &t) != cudaSuccess) {
          cudaGetLastError();
          continue;
        }
        if (t == cudaGraphNodeTypeKernel) ++g.kernels;
        if (t != cudaGraphNodeTypeMemcpy) continue;
        cudaMemcpy3DParms mp{};
        if (cudaGraphMemcpyNodeGetParams(nd, &mp) != cudaSuccess) {
          cudaGetLastError();
          continue;
        }
        const char* src = static_cast<const char*>(mp.srcPtr.ptr);
        for (int w = 0; w < 2; ++w) {
          const char* b = static_cast<const char*>(bases[w]);
          if (b && src >= b && src < b + sizes[w])
            g.copies.push_back({nd, w, static_cast<size_t>(src - b), mp.dstPtr.ptr, mp.extent.width});
        }
      }
      g.src[0] = host_input;
      g.src[1] = host_target;
      return;
    }
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    const bool retry = memops_before && !memops_ok();  // the flag waits fell back to kernels
    if (!retry || attempt == 1)
      throw std::runtime_error("dpl exec: step capture failed: " +
                               (error.empty() ? std::string(cudaGetErrorString(end)) : error));
  }
}

float Executor::step(const void* host_input, const void* host_target) {
  step_launch(host_input, host_target);
  return step_finish();
}

// Enqueues one step (a graph replay) without waiting for it: ranks sharing
// this process launch every rank's step before finishing any of them.
void Executor::step_launch(const void* host_input, const void* host_target) {
  DPL_CUDA(cudaSetDevice(device_));
  if (launched_) throw std::logic_error("dpl exec: step_launch twice without step_finish");
  host_input = stage_host(host_input, 0);
  host_target = stage_host(host_target, 1);
  const bool profiling = ctx_.gemms.profile.enabled || kernel_timer().enabled;
  if (!use_graph_) {
    enqueue_step(host_input, host_target);
  } else {
    // a profiled step is its own graph (per-launch timing events inside);
    // its records are re-registered on every capture
    const GraphKey key{bank_, host_input != nullptr, host_target != nullptr, profiling};
    GraphEntry* g = nullptr;
    for (GraphEntry& e : graphs_)
      if (e.key == key) g = &e;
    if (!g) {
      GraphEntry fresh;
      fresh.key = key;
      capture_step(fresh, host_input, host_target);
      graphs_.push_back(std::move(fresh));
      g = &graphs_.back();
    }
    const void* now[2] = {host_input, host_target};
    for (const HostCopy& c : g->copies)
      if (now[c.which] != g->src[c.which])
        DPL_CUDA(cudaGraphExecMemcpyNodeSetParams1D(g->exec, c.node, c.dst,
                                                     static_cast<const char*>(now[c.which]) + c.offset, c.bytes,
                                                     cudaMemcpyHostToDevice));
    g->src[0] = host_input;
    g->src[1] = host_target;
    DPL_CUDA(cudaGraphLaunch(g->exec, compute_));
    count_launch(g->kernels);
  }
  launched_ = true;
}

float Executor::step_finish() {
  if (!launched_) throw std::logic_error("dpl exec: step_finish without step_launch");
  launched_ = false;
  DPL_CUDA(cudaSetDevice(device_));
  DPL_CUDA(cudaStreamSynchronize(compute_));
  DPL_CUDA(cudaGetLastError());
  ++steps_done_;
  bank_ ^= 1;
  float loss = NAN;
  if (k_ == S_ - 1) loss = *loss_host_ / loss_norm_;
  last_loss_ = loss;
  return loss;
}

long long Executor::graph_count() const { return static_cast<long long>(graphs_.size()); }

// Captures and instantiates the device-data step graphs of both flag banks
// now, so later steps only launch.  Ranks sharing one process must do this
// before any of them runs a step: a capture / instantiation while another
// rank's step is blocked on this rank can synchronise the context.
void Executor::prepare_graphs() {
  if (!use_graph_) return;
  DPL_CUDA(cudaSetDevice(device_));
  const bool profiling = ctx_.gemms.profile.enabled || kernel_timer().enabled;
  const int saved = bank_;
  for (int b = 0; b < 2; ++b) {
    const GraphKey key{b, false, false, profiling};
    bool have = false;
    for (const GraphEntry& e : graphs_) have = have || e.key == key;
    if (have) continue;
    bank_ = b;
    GraphEntry fresh;
    fresh.key = key;
    try {
      capture_step(fresh, nullptr, nullptr);
    } catch (...) {
      bank_ = saved;
      throw;
    }
    graphs_.push_back(std::move(fresh));
  }
  bank_ = saved;
  DPL_CUDA(cudaDeviceSynchronize());
}

std::string Executor::timeline_json() const {
  auto ms = [&](cudaEvent_t e) {
    float v = 0.f;
    if (cudaEventElapsedTime(&v, ev_begin_, e) != cudaSuccess) {
      cudaGetLastError();
      return -1.0;
    }
    return static_cast<double>(v) * 1e-3;
  };
  unsigned long long t0 = 0;
  cudaMemcpy(&t0, t0_, 8, cudaMemcpyDeviceToHost);
  Value out = Value::object();
  out["rank"] = rank_;
  out["stage"] = k_;
  out["replica"] = rep_;
  out["expanded_stage"] = 2 * k_;
  out["M"] = M_;
  out["phi"] = phi_;
  out["t0_ns"] = static_cast<long long>(t0);
  out["step_s"] = ms(ev_end_);
  out["flops"] = flops_per_step_;
  out["loss"] = std::isnan(last_loss_) ? Value() : Value(static_cast<double>(last_loss_));
  Value blocks = Value::array();
  auto add = [&](int stage, int mb, int kind, const BlockEvents& b) {
    Value row = Value::array();
    row.push_back(stage);
    row.push_back(mb);
    row.push_back(kind);
    row.push_back(ms(b.start));
    row.push_back(ms(b.end));
    blocks.push_back(std::move(row));
  };
  for (int i = 0; i < M_; ++i) add(2 * k_, i, 0, fwd_ev_[i]);
  for (int i = 0; i < M_; ++i) add(2 * k_, i, 1, bwd_ev_[i]);
  if (!out_routes_.empty())
    for (int i = 0; i < M_; ++i) add(2 * k_ + 1, i, 0, send_fwd_ev_[i]);
  if (k_ > 0)
    for (int i = 0; i < M_; ++i) add(2 * k_ - 1, i, 1, send_bwd_ev_[i]);
  out["blocks"] = std::move(blocks);
  // replica AllReduce per parameter block: [block, start_s, end_s, fp32 bytes]
  Value ars = Value::array();
  for (int b = 0; b < nblk_; ++b) {
    if (!ar_bytes_[b]) continue;
    Value row = Value::array();
    row.push_back(b);
    row.push_back(ms(ar_ev_[b].start));
    row.push_back(ms(ar_ev_[b].end));
    row.push_back(ar_bytes_[b]);
    ars.push_back(std::move(row));
  }
  out["allreduce"] = std::move(ars);
  out["replication"] = r_;
  out["allreduce_impl"] = r_ > 1 ? (peer_ar_ ? "peer" : "nccl") : "none";
  // Split-Concat bytes of one micro-batch hand-off out of / into this rank
  long long sent = 0, sent_back = 0;
  for (const Route& r : out_routes_) sent += r.rows * 2;
  for (const Route& r : in_routes_) sent_back += r.rows * 2;
  out["send_bytes"] = sent;          // activations, per forward send block
  out["send_back_bytes"] = sent_back;  // activation gradients, per backward send block
  return out.dump();
}

void Executor::read_tensor(const std::string& name, bool grad, void* host, size_t bytes) {
  // name = "<global layer>.<tensor>" ; only layers of this stage are readable
  const size_t dot = name.find('.');
  if (dot == std::string::npos) throw std::invalid_argument("dpl exec: tensor name must be <layer>.<name>");
  const std::string t = name.substr(dot + 1);
  const std::string owner = name.substr(0, dot);
  if (owner == "emb" || owner == "head") {
    const bool e = owner == "emb";
    if (e ? !emb_ : !head_) throw std::out_of_range("dpl exec: " + owner + " not on this stage");
    for (const Layer::Named& n : e ? emb_->tensors() : head_->tensors()) {
      if (n.name != t) continue;
      if (bytes != n.count * 4) throw std::invalid_argument("dpl exec: size mismatch for " + name);
      const float* src = (grad ? g32_ : w32_) + (e ? emb_off_ : head_off_) + n.offset;
      DPL_CUDA(cudaSetDevice(device_));
      DPL_CUDA(cudaDeviceSynchronize());
      DPL_CUDA(cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost));
      return;
    }
    throw std::invalid_argument("dpl exec: unknown tensor " + name);
  }
  const int layer = std::stoi(owner);
  if (layer < lo_ || layer >= hi_) throw std::out_of_range("dpl exec: layer not on this stage");
  const int li = layer - lo_;
  for (const Layer::Named& n : layers_[li]->tensors()) {
    if (n.name != t) continue;
    if (bytes != n.count * 4) throw std::invalid_argument("dpl exec: size mismatch for " + name);
    const float* src = (grad ? g32_ : w32_) + param_off_[li] + n.offset;
    DPL_CUDA(cudaSetDevice(device_));
    DPL_CUDA(cudaDeviceSynchronize());
    DPL_CUDA(cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost));
    return;
  }
  throw std::invalid_argument("dpl exec: unknown tensor " + name);
}

void Executor::read_probe(int layer, const std::string& which, void* host, size_t bytes) {
  if (!probe_) throw std::invalid_argument("dpl exec: executor built without \"probe\"");
  if (layer < lo_ || layer >= hi_) throw std::out_of_range("dpl exec: layer not on this stage");
  const Probe& p = probes_[layer - lo_];
  const bf16* src = which == "x" ? p.x : which == "y" ? p.y : which == "aux" ? p.aux : which == "dy" ? p.dy
                    : which == "dx" ? p.dx : nullptr;
  const size_t n = which == "x" || which == "dx" ? p.nx : which == "aux" ? p.naux : p.ny;
  if (!src) throw std::invalid_argument("dpl exec: no probe '" + which + "' for layer " + std::to_string(layer));
  if (bytes != n * 2) throw std::invalid_argument("dpl exec: probe size mismatch (" + std::to_string(n * 2) + " bytes)");
  DPL_CUDA(cudaSetDevice(device_));
  DPL_CUDA(cudaDeviceSynchronize());
  DPL_CUDA(cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost));
}

// B200 layer profiler (the reference only ingests
// profiles, model.cpp:128-153).  Runs this stage's layers on the compute
// stream in step order -- F of layer lo..hi-1 then B of hi-1..lo, loss
// included in the last layer's F -- with a timing event between layers, so
// each layer sees the L2 state it sees inside a step.  Median over `reps`
// chains.  Output: profile_to_json (model.cpp:162-173) at
// profile_batch_size = this replica's samples per micro-batch.
std::string Executor::layer_profile_json(int reps) {
  if (reps < 1) throw std::invalid_argument("layer_profile: reps must be >= 1");
  if (recompute_) throw std::invalid_argument("layer_profile: executor built with recompute");
  const int n = L();
  std::vector<cudaEvent_t> fe(n + 1), be(n + 1);
  for (auto* v : {&fe, &be})
    for (cudaEvent_t& e : *v) DPL_CUDA(cudaEventCreate(&e));
  std::vector<std::vector<float>> ft(n), bt(n);
  if (emb_) fill_tokens(tok_[0], ctx_.rows, seed_, kTensorInput, 0, spec_.vocab, compute_);
  else if (k_ == 0) fill_uniform_bf16(in_[0], static_cast<long long>(in_elems()), seed_, kTensorInput, 0, 1.0f, compute_);
  if (head_) fill_tokens(tgt_tok_[0], ctx_.rows, seed_, kTensorTarget, 0, spec_.vocab, compute_);
  else if (k_ == S_ - 1 && classify()) fill_tokens(tgt_tok_[0], ctx_.samples, seed_, kTensorTarget, 0, spec_.classes, compute_);
  else if (k_ == S_ - 1)
    fill_uniform_bf16(target_[0], static_cast<long long>(out_elems()), seed_, kTensorTarget, 0, 1.0f, compute_);
  const bf16* x0 = k_ == 0 ? in_[0] : recv_act(0);
  for (int rep = 0; rep < reps + 1; ++rep) {  // first chain is a warm-up
    const bf16* x = x0;
    DPL_CUDA(cudaEventRecord(fe[0], compute_));
    if (emb_) emb_->forward(ctx_, tok_[0], in_[0]);  // counted in layer 0 (profile layers are the blocks)
    for (int li = 0; li < n; ++li) {
      bf16* y = li + 1 < n ? act_[li + 1][0] : out_[0];
      layers_[li]->forward(ctx_, 0, x, y);
      if (li == n - 1 && head_)
        head_->forward(ctx_, 0, out_[0], tgt_tok_[0], loss_acc_, 1.0f / loss_norm_);  // counted in the last layer
      else if (li == n - 1 && k_ == S_ - 1 && classify()) {
        DPL_CUDA(cudaMemcpyAsync(dloss_[0], out_[0], out_elems() * 2, cudaMemcpyDeviceToDevice, compute_));
        cross_entropy_fwd_bwd(dloss_[0], tgt_tok_[0], loss_acc_, ctx_.samples, spec_.classes, 1.0f / loss_norm_,
                              compute_);
      } else if (li == n - 1 && k_ == S_ - 1)
        mse_loss(out_[0], target_[0], dloss_[0], loss_acc_, static_cast<long long>(out_elems()),
                 2.0f / static_cast<float>(numel_global_), compute_);
      DPL_CUDA(cudaEventRecord(fe[li + 1], compute_));
      x = y;
    }
    const bf16* dy = k_ == S_ - 1 ? dloss_[0] : recv_grad(0);
    int pp = 0;
    DPL_CUDA(cudaEventRecord(be[n], compute_));
    if (head_) head_->backward(ctx_, 0, out_[0], dloss_[0]);
    for (int li = n - 1; li >= 0; --li) {
      const bf16* xin = li > 0 ? act_[li][0] : x0;
      bf16* dx = li > 0 || emb_ ? gbuf_[pp] : (k_ > 0 ? send_grad_[0] : nullptr);
      pp ^= 1;
      ctx_.cur_y = li + 1 < n ? act_[li + 1][0] : out_[0];
      layers_[li]->backward(ctx_, 0, xin, dy, dx);
      if (li == 0 && emb_) emb_->backward(ctx_, tok_[0], dx);
      DPL_CUDA(cudaEventRecord(be[li], compute_));
      dy = dx;
    }
    DPL_CUDA(cudaStreamSynchronize(compute_));
    if (rep == 0) continue;
    for (int li = 0; li < n; ++li) {
      float a = 0, b = 0;
      DPL_CUDA(cudaEventElapsedTime(&a, fe[li], fe[li + 1]));
      DPL_CUDA(cudaEventElapsedTime(&b, be[li + 1], be[li]));
      ft[li].push_back(a);
      bt[li].push_back(b);
    }
  }
  for (auto* v : {&fe, &be})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  // the profiled chains accumulated into the gradient buffers: clear them
  DPL_CUDA(cudaMemsetAsync(g32_, 0, n_params_ * sizeof(float), compute_));
  DPL_CUDA(cudaStreamSynchronize(compute_));
  auto median = [](std::vector<float> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  pipeplan::ModelProfile prof;
  prof.profile_batch_size = ctx_.samples;
  for (int li = 0; li < n; ++li) {
    pipeplan::LayerProfile l;
    l.index = lo_ + li;
    l.fwd_time = median(ft[li]) * 1e-3;
    l.bwd_time = median(bt[li]) * 1e-3;
    l.activation_bytes = static_cast<std::int64_t>(ctx_.samples) * elems(lo_ + li + 1) * 2;  // bf16 output
    size_t np = layers_[li]->param_count();
    if (li == 0 && emb_) np += emb_->param_count();
    if (li == n - 1 && head_) np += head_->param_count();
    l.param_bytes = static_cast<std::int64_t>(np) * 4;  // fp32 master
    prof.layers.push_back(l);
  }
  return pipeplan::profile_to_json(prof);
}

std::string Executor::gemm_profile_json() const {
  // per-launch durations of the GEMMs of the last profiled step, grouped by shape
  struct Agg {
    int M, N, K, batch, bn;
    long long launches = 0;
    double flops = 0, seconds = 0;
  };
  std::vector<Agg> aggs;
  double total_s = 0, total_f = 0;
  for (const auto& r : ctx_.gemms.profile.recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.start, r.end);
    const double sec = ms * 1e-3;
    total_s += sec;
    total_f += r.flops;
    auto it = std::find_if(aggs.begin(), aggs.end(), [&](const Agg& a) {
      return a.M == r.M && a.N == r.N && a.K == r.K && a.batch == r.batch;
    });
    if (it == aggs.end()) {
      aggs.push_back({r.M, r.N, r.K, r.batch, r.bn});
      it = aggs.end() - 1;
    }
    it->launches++;
    it->flops += r.flops;
    it->seconds += sec;
  }
  Value out = Value::object();
  out["launches"] = static_cast<long long>(ctx_.gemms.profile.recs.size());
  out["seconds"] = total_s;
  out["flops"] = total_f;
  Value shapes = Value::array();
  for (const Agg& a : aggs) {
    Value e = Value::object();
    e["M"] = a.M;
    e["N"] = a.N;
    e["K"] = a.K;
    e["batch"] = a.batch;
    e["bn"] = a.bn;
    e["launches"] = a.launches;
    e["flops"] = a.flops;
    e["seconds"] = a.seconds;
    e["tflops"] = a.seconds > 0 ? a.flops / a.seconds * 1e-12 : 0.0;
    shapes.push_back(std::move(e));
  }
  out["shapes"] = std::move(shapes);
  // every libdapple kernel of the profiled step, grouped by kernel
  // "seconds" sums each launch's own duration; "busy_seconds" is the union of
  // the launches' intervals on the step's timeline (launches on the compute
  // and weight-gradient streams overlap, so the sum double-counts)
  struct K {
    std::string name;
    long long launches = 0;
    double seconds = 0, flops = 0;
    std::vector<std::pair<float, float>> spans;  // ms from the step's first event
  };
  std::vector<K> ks;
  for (const auto& r : kernel_timer().recs) {
    float ms = 0.f, a = 0.f, b = 0.f;
    cudaEventElapsedTime(&ms, r.start, r.end);
    auto it = std::find_if(ks.begin(), ks.end(), [&](const K& k) { return k.name == r.name; });
    if (it == ks.end()) {
      ks.push_back({r.name});
      it = ks.end() - 1;
    }
    it->launches++;
    it->seconds += ms * 1e-3;
    it->flops += r.flops;
    if (cudaEventElapsedTime(&a, ev_begin_, r.start) == cudaSuccess &&
        cudaEventElapsedTime(&b, ev_begin_, r.end) == cudaSuccess)
      it->spans.push_back({a, b});
    cudaGetLastError();
  }
  Value kernels = Value::array();
  for (K& k : ks) {
    Value e = Value::object();
    e["kernel"] = k.name;
    e["launches"] = k.launches;
    e["seconds"] = k.seconds;
    if (k.flops > 0) e["tflops"] = k.flops / k.seconds * 1e-12;
    std::sort(k.spans.begin(), k.spans.end());
    double busy = 0.0, lo = -1.0, hi = -1.0;
    for (const auto& [a, b] : k.spans) {
      if (a > hi) {
        if (hi > lo) busy += hi - lo;
        lo = a;
        hi = b;
      } else {
        hi = std::max<double>(hi, b);
      }
    }
    if (hi > lo) busy += hi - lo;
    e["busy_seconds"] = busy * 1e-3;
    if (k.flops > 0 && busy > 0) e["busy_tflops"] = k.flops / (busy * 1e-3) * 1e-12;
    kernels.push_back(std::move(e));
  }
  out["kernels"] = std::move(kernels);
  return out.dump();
}

std::string Executor::info() const {
  Value v = Value::object();
  v["rank"] = rank_;
  v["stage"] = k_;
  v["replica"] = rep_;
  v["replication"] = r_;
  v["layers"] = std::vector<int>{lo_, hi_};
  v["phi"] = phi_;
  v["phi_expanded"] = phi_expanded_;
  v["schedule"] = gpipe_ ? "gpipe" : "dapple";
  v["recompute"] = recompute_;
  v["stash_slots"] = stash_slots_;
  v["vocab"] = spec_.vocab;
  v["rows"] = ctx_.rows;
  v["micro_batch_samples"] = B_;
  v["params"] = static_cast<long long>(n_params_);
  v["device_bytes"] = static_cast<long long>(mem_.total());
  v["flops_per_step"] = flops_per_step_;
  v["gemm_plans"] = static_cast<long long>(ctx_.gemms.size());
  v["input_bytes"] = static_cast<long long>(input_bytes());
  v["target_bytes"] = static_cast<long long>(target_bytes());
  v["input_dtype"] = emb_ ? "int32" : "bfloat16";
  v["target_dtype"] = (head_ || classify()) ? "int32" : "bfloat16";
  v["graphs"] = graph_count();
  v["wgrad_stream"] = wgrad_ != nullptr;
  Value chain = Value::array();
  for (const auto& c : chain_) chain.push_back(std::string(c.kind == pipeplan::BlockKind::forward ? "F" : "B") +
                                               std::to_string(c.micro_batch));
  v["chain"] = std::move(chain);
  Value routes = Value::array();
  for (const auto* list : {&in_routes_, &out_routes_})
    for (const Route& r : *list) {
      Value e = Value::array();
      e.push_back(r.src_gpu);
      e.push_back(r.dst_gpu);
      e.push_back(static_cast<long long>(r.src_row));
      e.push_back(static_cast<long long>(r.dst_row));
      e.push_back(static_cast<long long>(r.rows));
      routes.push_back(std::move(e));
    }
  v["routes"] = std::move(routes);
  return v.dump();
}

}  // namespace dpl

// ------------------------------------------------------------------ C-ABI
struct dpl_exec {
  std::unique_ptr<dpl::Executor> impl;
  std::string reply;
};

namespace {
template <typename F>
int exec_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return dpl::fail(e.what());
  }
}
}  // namespace

extern "C" {

int dpl_exec_create(const char* config_json, int device, dpl_exec** out) {
  return exec_guard([&] {
    auto ex = std::make_unique<dpl_exec>();
    ex->impl = std::make_unique<dpl::Executor>(dpl::json::Value::parse(config_json), device);
    *out = ex.release();
  });
}

int dpl_exec_export(dpl_exec* ex, void* blob, size_t cap, size_t* len) {
  return exec_guard([&] { *len = ex->impl->export_blob(blob, cap); });
}

int dpl_exec_connect(dpl_exec* ex, const void* blobs, size_t blob_len, int world) {
  return exec_guard([&] { ex->impl->connect(static_cast<const uint8_t*>(blobs), blob_len, world); });
}

int dpl_exec_nccl_id(void* id128) {
  return exec_guard([&] {
    ncclUniqueId id;
    DPL_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof id);
  });
}

int dpl_exec_nccl_init(dpl_exec* ex, const void* id128) {
  return exec_guard([&] { ex->impl->nccl_init(id128); });
}

int dpl_exec_step(dpl_exec* ex, const void* host_input, const void* host_target, float* loss) {
  return exec_guard([&] {
    const float l = ex->impl->step(host_input, host_target);
    if (loss) *loss = l;
  });
}

int dpl_exec_step_launch(dpl_exec* ex, const void* host_input, const void* host_target) {
  return exec_guard([&] { ex->impl->step_launch(host_input, host_target); });
}

int dpl_exec_prepare(dpl_exec* ex) {
  return exec_guard([&] { ex->impl->prepare_graphs(); });
}

int dpl_exec_step_finish(dpl_exec* ex, float* loss) {
  return exec_guard([&] {
    const float l = ex->impl->step_finish();
    if (loss) *loss = l;
  });
}

const char* dpl_exec_timeline(dpl_exec* ex) {
  try {
    ex->reply = ex->impl->timeline_json();
  } catch (const std::exception& e) {
    ex->reply = std::string("{\"error\":\"") + e.what() + "\"}";
  }
  return ex->reply.c_str();
}

int dpl_exec_read_tensor(dpl_exec* ex, const char* name, int grad, void* host, size_t bytes) {
  return exec_guard([&] { ex->impl->read_tensor(name, grad != 0, host, bytes); });
}

int dpl_exec_read_probe(dpl_exec* ex, int layer, const char* which, void* host, size_t bytes) {
  return exec_guard([&] { ex->impl->read_probe(layer, which, host, bytes); });
}

int dpl_exec_info(dpl_exec* ex, char* buf, size_t cap) {
  return exec_guard([&] {
    const std::string s = ex->impl->info();
    if (s.size() + 1 > cap) throw std::invalid_argument("dpl exec: info buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int dpl_exec_gemm_profile(dpl_exec* ex, int enable) {
  return exec_guard([&] { ex->impl->set_gemm_profile(enable != 0); });
}

const char* dpl_exec_gemm_profile_json(dpl_exec* ex) {
  try {
    ex->reply = ex->impl->gemm_profile_json();
  } catch (const std::exception& e) {
    ex->reply = std::string("{\"error\":\"") + e.what() + "\"}";
  }
  return ex->reply.c_str();
}

const char* dpl_exec_layer_profile(dpl_exec* ex, int reps) {
  try {
    ex->reply = ex->impl->layer_profile_json(reps);
  } catch (const std::exception& e) {
    dpl::fail(e.what());
    return nullptr;
  }
  return ex->reply.c_str();
}

int dpl_exec_clock_calibrate(dpl_exec* ex, int phase, long long* offset_ns) {
  return exec_guard([&] { *offset_ns = ex->impl->calibrate_clock(phase); });
}

int dpl_exec_disconnect(dpl_exec* ex) {
  return exec_guard([&] { ex->impl->disconnect(); });
}

void dpl_exec_destroy(dpl_exec* ex) { delete ex; }

}  // extern "C"
