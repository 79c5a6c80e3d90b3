// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A JSON-in / JSON-out C bridge around the *reference* pipeplan library
// (/root/reference/proj, compiled by oracle/Makefile into oracle/_ref/).  The
// product library exposes the same request vocabulary through
// dpl_host_call() (include/dapple.h), so tests/ can send one request to both
// and compare the parsed answers bit for bit.
//
// Request: {"op": "<name>", ...arguments...}; reply: JSON object, or
// {"error": {"type": "<std exception class>", "what": "..."}}.
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>

#include <nlohmann/json.hpp>

#include "pipeplan/costmodel.hpp"
#include "pipeplan/estimator.hpp"
#include "pipeplan/harness.hpp"
#include "pipeplan/io.hpp"
#include "pipeplan/model.hpp"
#include "pipeplan/planner.hpp"
#include "pipeplan/simulator.hpp"

using namespace pipeplan;
using nlohmann::json;

namespace {

StageCostSequence seq_from(const json& j) {
  StageCostSequence seq;
  for (const auto& e : j) {
    StageCost c;
    c.kind = e.value("kind", std::string("compute")) == "communication" ? StageKind::communication
                                                                         : StageKind::compute;
    c.fwd = e.at("fwd").get<double>();
    c.bwd = e.at("bwd").get<double>();
    c.param_bytes = e.value("param_bytes", std::int64_t{0});
    c.allreduce_time = e.value("allreduce", 0.0);
    c.activation_out_bytes = e.value("act", std::int64_t{0});
    seq.push_back(c);
  }
  return seq;
}

json seq_to(const StageCostSequence& seq) {
  json a = json::array();
  for (const auto& c : seq) {
    a.push_back({{"kind", c.kind == StageKind::compute ? "compute" : "communication"},
                 {"fwd", c.fwd},
                 {"bwd", c.bwd},
                 {"param_bytes", c.param_bytes},
                 {"allreduce", c.allreduce_time},
                 {"act", c.activation_out_bytes}});
  }
  return a;
}

json timeline_to(const Timeline& tl) {
  json blocks = json::array();
  for (const auto& b : tl.blocks) {
    blocks.push_back({b.stage, b.micro_batch, b.kind == BlockKind::forward ? 0 : 1, b.start, b.end});
  }
  return {{"M", tl.micro_batches}, {"S", tl.stage_count}, {"phi", tl.phi}, {"blocks", blocks}};
}

ModelProfile profile_from(const json& j) {
  std::istringstream in(j.is_string() ? j.get<std::string>() : j.dump());
  return load_profile(in);
}

ClusterSpec cluster_from(const json& j) {
  std::istringstream in(j.is_string() ? j.get<std::string>() : j.dump());
  return load_cluster(in);
}

PipelinePlan plan_from(const json& j) { return plan_from_json(j.is_string() ? j.get<std::string>() : j.dump()); }

PhiStrategy strategy_from(const json& req) {
  const std::string s = req.value("phi_strategy", std::string("preset_a"));
  if (s == "preset_b") return PhiStrategy::preset_b;
  if (s == "search") return PhiStrategy::search;
  return PhiStrategy::preset_a;
}

json plan_to(const PipelinePlan& p, const ModelProfile& prof, const ClusterSpec& cl) {
  const double acr = compute_acr(build_stage_sequence(p, prof, cl));
  json j = json::parse(plan_to_json(p, acr));
  // exact doubles next to the microsecond file fields
  j["est_latency_s"] = p.est_latency;
  if (p.sim_latency) j["sim_latency_s"] = *p.sim_latency;
  return j;
}

json dispatch(const json& req) {
  const std::string op = req.at("op").get<std::string>();
  if (op == "plan") {
    const ModelProfile prof = profile_from(req.at("profile"));
    const ClusterSpec cl = cluster_from(req.at("cluster"));
    PlannerOptions opts;
    opts.phi_strategy = strategy_from(req);
    opts.top_k = req.value("top_k", 8);
    opts.optimizer_multiplier = req.value("optimizer_multiplier", 8.0);
    SearchReport rep;
    const bool want_report = req.value("report", false);
    const PipelinePlan p = plan(prof, cl, req.at("M").get<int>(), opts, want_report ? &rep : nullptr);
    json out = {{"plan", plan_to(p, prof, cl)}};
    if (want_report) {
      json top = json::array();
      for (const auto& r : rep.top) {
        top.push_back({{"est", r.est_latency}, {"sim", r.sim_latency}, {"plan", plan_to(r.plan, prof, cl)}});
      }
      out["report"] = {{"states_evaluated", rep.states_evaluated}, {"top", top}};
    }
    return out;
  }
  if (op == "brute_force_plan") {
    const ModelProfile prof = profile_from(req.at("profile"));
    const ClusterSpec cl = cluster_from(req.at("cluster"));
    PlannerOptions opts;
    opts.phi_strategy = strategy_from(req);
    const PipelinePlan p = brute_force_plan(prof, cl, req.at("M").get<int>(), opts);
    return {{"plan", plan_to(p, prof, cl)}};
  }
  if (op == "simulate_plan") {
    const ModelProfile prof = profile_from(req.at("profile"));
    const ClusterSpec cl = cluster_from(req.at("cluster"));
    const PipelinePlan p = plan_from(req.at("plan"));
    const bool gpipe = req.value("schedule", std::string("dapple")) == "gpipe";
    const PlanSimulation sim = simulate_plan(p, prof, cl, req.at("M").get<int>(),
                                             gpipe ? ScheduleKind::gpipe : ScheduleKind::dapple,
                                             req.value("recompute", false));
    std::ostringstream csv;
    write_timeline_csv(csv, sim.timeline);
    return {{"latency", sim.latency}, {"seq", seq_to(sim.seq)}, {"timeline", timeline_to(sim.timeline)},
            {"peaks", peak_activations(sim.timeline)}, {"csv", csv.str()}};
  }
  if (op == "build_stage_sequence") {
    const ModelProfile prof = profile_from(req.at("profile"));
    const ClusterSpec cl = cluster_from(req.at("cluster"));
    return {{"seq", seq_to(build_stage_sequence(plan_from(req.at("plan")), prof, cl))}};
  }
  if (op == "schedule") {
    const StageCostSequence seq = seq_from(req.at("seq"));
    const int m = req.at("M").get<int>();
    const bool gpipe = req.value("schedule", std::string("dapple")) == "gpipe";
    const Timeline tl = gpipe ? gpipe_schedule(seq, m)
                              : dapple_schedule(seq, m, req.at("phi").get<std::vector<int>>());
    return {{"latency", batch_latency(tl, seq)}, {"timeline", timeline_to(tl)}, {"peaks", peak_activations(tl)}};
  }
  if (op == "estimate") {
    const StageCostSequence seq = seq_from(req.at("seq"));
    const LatencyBreakdown lb = estimate_latency(seq, req.at("M").get<int>());
    json out = {{"warmup", lb.warmup}, {"steady", lb.steady}, {"ending", lb.ending},
                {"total", lb.total}, {"pivot", lb.pivot},
                {"select_pivot", select_pivot(seq, req.at("M").get<int>())}};
    bool has_compute = false;
    for (const auto& c : seq) has_compute |= c.kind == StageKind::compute;
    if (has_compute) out["acr"] = compute_acr(seq);
    return out;
  }
  if (op == "optimize_phi") {
    const StageCostSequence seq = seq_from(req.at("seq"));
    const PhiResult r = optimize_phi(seq, req.at("M").get<int>(), strategy_from(req), req.at("D").get<int>());
    return {{"phi", r.phi}, {"latency", r.latency}};
  }
  if (op == "expand_plan_phi") return {{"phi", expand_plan_phi(req.at("phi").get<std::vector<int>>())}};
  if (op == "apply_recompute") return {{"seq", seq_to(apply_recompute(seq_from(req.at("seq"))))}};
  if (op == "allreduce_time") {
    return {{"t", allreduce_time(req.at("size").get<std::int64_t>(), req.at("devices").get<std::vector<int>>(),
                                 cluster_from(req.at("cluster")))}};
  }
  if (op == "splitconcat_time") {
    return {{"t", splitconcat_time(req.at("size").get<std::int64_t>(), req.at("src").get<std::vector<int>>(),
                                   req.at("dst").get<std::vector<int>>(), cluster_from(req.at("cluster")))}};
  }
  if (op == "aggregate_stage") {
    const StageCost c = aggregate_stage(profile_from(req.at("profile")), req.at("lo").get<int>(),
                                        req.at("hi").get<int>(), req.at("r").get<int>());
    return {{"seq", seq_to({c})}};
  }
  if (op == "enumerate_placements") {
    DeviceState st{cluster_from(req.at("cluster"))};
    if (req.contains("free")) st.free = req.at("free").get<std::vector<int>>();
    return {{"placements", enumerate_placements(st, req.at("count").get<int>())}};
  }
  if (op == "memory_feasible") {
    StageCost c;
    c.param_bytes = req.at("param_bytes").get<std::int64_t>();
    c.activation_out_bytes = req.at("act").get<std::int64_t>();
    return {{"ok", memory_feasible(c, req.at("injected").get<int>(), req.at("capacity").get<std::int64_t>(),
                                   req.value("optimizer_multiplier", 8.0))}};
  }
  if (op == "load_profile") {
    const ModelProfile p = profile_from(req.at("profile"));
    json layers = json::array();
    for (const auto& l : p.layers) layers.push_back({l.index, l.fwd_time, l.bwd_time, l.activation_bytes, l.param_bytes});
    return {{"profile_batch_size", p.profile_batch_size}, {"layers", layers}, {"json", profile_to_json(p)}};
  }
  if (op == "load_cluster") {
    const ClusterSpec c = cluster_from(req.at("cluster"));
    return {{"seps", c.seps}, {"intra_bw", c.intra_bw}, {"inter_bw", c.inter_bw},
            {"intra_latency", c.intra_latency}, {"inter_latency", c.inter_latency},
            {"per_gpu_memory", c.per_gpu_memory}, {"json", cluster_to_json(c)}};
  }
  if (op == "ranking_experiment") {
    const RankingReport r = ranking_experiment(req.at("pairs").get<long long>(), req.at("M").get<int>(),
                                               req.at("phi").get<std::vector<int>>(), req.value("total", 1.0),
                                               req.at("seed").get<std::uint64_t>(), 1.0 / 3.0,
                                               req.value("workers", 0));
    return {{"errors", r.errors}, {"pairs", r.pairs_tested}};
  }
  throw std::invalid_argument("unknown op " + op);
}

thread_local std::string g_reply;

}  // namespace

extern "C" __attribute__((visibility("default"))) const char* ref_call(const char* request) {
  json reply;
  try {
    reply = dispatch(json::parse(request));
  } catch (const std::invalid_argument& e) {
    reply = {{"error", {{"type", "invalid_argument"}, {"what", e.what()}}}};
  } catch (const std::out_of_range& e) {
    reply = {{"error", {{"type", "out_of_range"}, {"what", e.what()}}}};
  } catch (const std::logic_error& e) {
    reply = {{"error", {{"type", "logic_error"}, {"what", e.what()}}}};
  } catch (const std::runtime_error& e) {
    reply = {{"error", {{"type", "runtime_error"}, {"what", e.what()}}}};
  } catch (const std::exception& e) {
    reply = {{"error", {{"type", "exception"}, {"what", e.what()}}}};
  }
  g_reply = reply.dump();
  return g_reply.c_str();
}

#ifdef REF_CLI
// Line-oriented server: one JSON request per stdin line, one reply per
// stdout line.  Tests talk to this process so the reference library never
// shares an address space with the product library.
#include <iostream>
int main() {
  std::ios::sync_with_stdio(false);
  std::string line;
  while (std::getline(std::cin, line)) {
    if (line.empty()) continue;
    std::cout << ref_call(line.c_str()) << '\n' << std::flush;
  }
  return 0;
}
#endif
