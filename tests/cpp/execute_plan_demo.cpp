// C++ drop-in demo: the reference-style flow -- load a
// profile / cluster, take a plan, simulate it -- plus execute_plan on this
// GPU; the measured Timeline goes through the reference's helpers unchanged.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <iostream>
#include <sstream>

#include "pipeplan/executor.hpp"
#include "pipeplan/io.hpp"
#include "pipeplan/planner.hpp"

int main() {
  using namespace pipeplan;
  std::istringstream prof_json(
      R"({"profile_batch_size": 4, "layers": [
          {"fwd_time_us": 100, "bwd_time_us": 200, "activation_bytes": 1048576, "param_bytes": 2000000},
          {"fwd_time_us": 100, "bwd_time_us": 200, "activation_bytes": 1048576, "param_bytes": 2000000}]})");
  std::istringstream cluster_json(
      R"({"seps": [1], "intra_bw_gbps": 700, "inter_bw_gbps": 50, "intra_latency_us": 5,
          "inter_latency_us": 10, "per_gpu_memory_gb": 80})");
  const ModelProfile profile = load_profile(prof_json);
  const ClusterSpec cluster = load_cluster(cluster_json);
  const PipelinePlan plan = pipeplan::plan(profile, cluster, 4, PlannerOptions{});
  const PlanSimulation sim = simulate_plan(plan, profile, cluster, 4);

  ExecOptions o;
  o.model_json = R"({"kind":"bert","layers":2,"hidden":256,"heads":4,"ffn":1024,"seq":128})";
  o.global_batch = 8;
  const PlanExecution ex = execute_plan(plan, profile, cluster, 4, o);
  const double measured = batch_latency(ex.timeline, ex.seq);
  const std::vector<int> peaks = peak_activations(ex.timeline);
  std::ostringstream csv;
  write_timeline_csv(csv, ex.timeline);
  const std::string text = csv.str();
  std::printf("stages %zu sim_L %.6f measured_L %.6f loss %.6f peaks %zu csv_lines %ld\n", plan.stages.size(),
              sim.latency, measured, ex.loss, peaks.size(),
              static_cast<long>(std::count(text.begin(), text.end(), '\n')));
  return std::isfinite(ex.loss) && ex.loss > 0 && measured > 0 && ex.timeline.blocks.size() == 2u * 4 ? 0 : 1;
}
