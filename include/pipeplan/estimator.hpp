// dapple-b200 host API -- drop-in for pipeplan/estimator.hpp
// (reference: proj/include/pipeplan/estimator.hpp:12-41).
#pragma once

#include "pipeplan/model.hpp"

namespace pipeplan {

/// total = warmup + steady + ending; steady = (M-1)(F_Q+B_Q).
struct LatencyBreakdown {
  double warmup = 0.0;
  double steady = 0.0;
  double ending = 0.0;
  double total = 0.0;
  int pivot = 0;
};

StageCostSequence build_stage_sequence(const PipelinePlan& plan,
                                       const ModelProfile& profile,
                                       const ClusterSpec& cluster);
int select_pivot(const StageCostSequence& seq, int micro_batches);
LatencyBreakdown estimate_latency(const StageCostSequence& seq, int micro_batches);
double compute_acr(const StageCostSequence& seq);

}  // namespace pipeplan
