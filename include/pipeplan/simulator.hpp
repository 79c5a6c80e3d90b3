// dapple-b200 host API -- drop-in for pipeplan/simulator.hpp
// (reference: proj/include/pipeplan/simulator.hpp:12-84).  The Timeline type
// is also what the B200 executor returns, filled with *measured* block times
// (see pipeplan/executor.hpp), so batch_latency / peak_activations /
// write_timeline_csv work unchanged on measurements.
#pragma once

#include <vector>

#include "pipeplan/model.hpp"

namespace pipeplan {

enum class BlockKind { forward, backward };

struct Block {
  int stage = 0;
  int micro_batch = 0;
  BlockKind kind = BlockKind::forward;
  double start = 0.0;
  double end = 0.0;
};

/// blocks[x*M + i] = forward(i, x); blocks[S*M + x*M + i] = backward(i, x).
struct Timeline {
  int micro_batches = 0;
  int stage_count = 0;
  std::vector<int> phi;
  std::vector<Block> blocks;

  const Block& forward(int micro_batch, int stage) const;
  const Block& backward(int micro_batch, int stage) const;
  Block& forward(int micro_batch, int stage);
  Block& backward(int micro_batch, int stage);
};

enum class ScheduleKind { dapple, gpipe };

Timeline dapple_schedule(const StageCostSequence& seq, int micro_batches,
                         const std::vector<int>& phi);
Timeline gpipe_schedule(const StageCostSequence& seq, int micro_batches);
double batch_latency(const Timeline& timeline, const StageCostSequence& seq);
std::vector<int> peak_activations(const Timeline& timeline);

enum class PhiStrategy { preset_a, preset_b, search };

struct PhiResult {
  std::vector<int> phi;
  double latency = 0.0;
};

PhiResult optimize_phi(const StageCostSequence& seq, int micro_batches,
                       PhiStrategy strategy, int max_injection);
std::vector<int> expand_plan_phi(const std::vector<int>& compute_phi);
StageCostSequence apply_recompute(StageCostSequence seq);

/// Per-stage execution order implied by the DAG for a given phi: a list of
/// (kind, micro_batch) for stage x.  The DAG fixes a total order per stage
/// independent of durations (simulator.cpp:81-97); the executor issues
/// exactly this chain on each stage's compute stream.
struct ChainOp {
  BlockKind kind;
  int micro_batch;
};
std::vector<ChainOp> stage_chain(int micro_batches, int phi_x, ScheduleKind kind = ScheduleKind::dapple);

}  // namespace pipeplan
