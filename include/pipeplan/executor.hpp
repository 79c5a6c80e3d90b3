// dapple-b200 executor API: the B200 counterpart of simulate_plan
// (reference planner.hpp:81-90, planner.cpp:491-514).  Same inputs, same
// phi resolution (planner.cpp:501-508), same per-stage block order
// (simulator.cpp:81-97); the returned Timeline is *measured* on the GPUs, so
// batch_latency / peak_activations / write_timeline_csv / write_timeline_svg
// apply to it unchanged.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "pipeplan/model.hpp"
#include "pipeplan/simulator.hpp"

namespace pipeplan {

/// One contiguous run of micro-batch rows moved between a replica of stage
/// k and a replica of stage k+1 (Split-Concat).  Rows
/// are token rows; offsets are relative to each replica's own slice.  The
/// interval-overlap mapping yields at most r_k + r_{k+1} - 1 flows (the cost
/// model charges r_k * r_{k+1} equal flows, costmodel.cpp:60-69).
struct SplitConcatRoute {
  int src_gpu = 0;
  int dst_gpu = 0;
  std::int64_t src_row = 0;
  std::int64_t dst_row = 0;
  std::int64_t rows = 0;
};

std::vector<SplitConcatRoute> splitconcat_routes(const Stage& from, const Stage& to, int micro_batch_samples,
                                                 int rows_per_sample);

struct ExecOptions {
  /// {"kind": "mlp"|"bert"|"gpt", "layers", "hidden", "heads", "ffn", "seq"}
  std::string model_json;
  int rank = 0;   // this process's global GPU id in the plan
  int world = 1;  // number of GPUs / processes
  int device = 0;
  int global_batch = 0;  // samples per step (multiple of micro_batches)
  double lr = 1e-3;
  std::uint64_t seed = 1234;
  bool apply = true;
  /// Block order: DAPPLE early-backward (default) or GPipe all-forward-first
  /// (stage_chain, simulator.cpp:161-167).
  ScheduleKind schedule = ScheduleKind::dapple;
  /// Keep only stage inputs; each backward block re-runs the stage forward
  /// (the executed counterpart of apply_recompute, simulator.cpp:216-221).
  bool recompute = false;
  /// Replica-group gradient AllReduce: "peer" (one reduce kernel over the
  /// replicas' peer-mapped gradients, collective.cu) or "nccl".
  std::string allreduce = "peer";
  /// Plumbing for world > 1: all-gather of one byte string per rank
  /// (CUDA-IPC handles, NCCL ids, timelines), e.g. over torch.distributed
  /// or MPI.  Must be collective and return the strings in rank order.
  std::function<std::vector<std::string>(const std::string&)> allgather;
};

struct PlanExecution {
  StageCostSequence seq;   // the plan's expanded cost sequence (as simulate_plan)
  Timeline timeline;       // measured, expanded stages, seconds from the first forward
  double latency = 0.0;    // measured L: first forward start -> last rank done
  double loss = 0.0;       // global-batch loss (NaN if no rank reported one)
  double bubble = 0.0;     // 1 - sum(busy) / (G * L)
};

/// Runs one synchronous DAPPLE step of `plan` on this rank's GPU.  Every
/// rank of the plan calls it collectively.
PlanExecution execute_plan(const PipelinePlan& plan, const ModelProfile& profile, const ClusterSpec& cluster,
                           int micro_batches, const ExecOptions& opts);

}  // namespace pipeplan
