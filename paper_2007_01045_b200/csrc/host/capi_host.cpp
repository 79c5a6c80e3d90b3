// C-ABI over the host planner/simulator (declared in include/dapple.h).
// One JSON request/reply entry point covers the whole pipeplan surface so
// that Python (paper_2007_01045_b200/pipeplan.py) and any other FFI can drive
// it with plain strings; C++ users call the pipeplan:: API directly.
// Errors never cross the ABI as exceptions: they come back as
// {"error": {"type": <std exception class>, "what": ...}}, matching the
// reference's exception conventions.
#include <sstream>
#include <stdexcept>
#include <string>

#include "json.hpp"
#include "pipeplan/costmodel.hpp"
#include "pipeplan/estimator.hpp"
#include "pipeplan/executor.hpp"
#include "pipeplan/io.hpp"
#include "pipeplan/model.hpp"
#include "pipeplan/planner.hpp"
#include "pipeplan/simulator.hpp"

using dpl::json::Value;

namespace pipeplan {
int& planner_threads_override();  // planner.cpp (not part of the reference API)
}
using namespace pipeplan;

namespace dpl {

Value seq_to_json(const StageCostSequence& seq) {
  Value a = Value::array();
  for (const StageCost& c : seq) {
    Value e = Value::object();
    e["kind"] = c.kind == StageKind::compute ? "compute" : "communication";
    e["fwd"] = c.fwd;
    e["bwd"] = c.bwd;
    e["param_bytes"] = static_cast<long long>(c.param_bytes);
    e["allreduce"] = c.allreduce_time;
    e["act"] = static_cast<long long>(c.activation_out_bytes);
    a.push_back(std::move(e));
  }
  return a;
}

StageCostSequence seq_from_json(const Value& a) {
  StageCostSequence seq;
  for (const Value& e : a.items()) {
    StageCost c;
    c.kind = e.contains("kind") && e.at("kind").as_string() == "communication" ? StageKind::communication
                                                                                : StageKind::compute;
    c.fwd = e.at("fwd").as_double();
    c.bwd = e.at("bwd").as_double();
    if (e.contains("param_bytes")) c.param_bytes = e.at("param_bytes").as_int();
    if (e.contains("allreduce")) c.allreduce_time = e.at("allreduce").as_double();
    if (e.contains("act")) c.activation_out_bytes = e.at("act").as_int();
    seq.push_back(c);
  }
  return seq;
}

Value timeline_to_json(const Timeline& tl) {
  Value blocks = Value::array();
  for (const Block& b : tl.blocks) {
    Value row = Value::array();
    row.push_back(b.stage);
    row.push_back(b.micro_batch);
    row.push_back(b.kind == BlockKind::forward ? 0 : 1);
    row.push_back(b.start);
    row.push_back(b.end);
    blocks.push_back(std::move(row));
  }
  Value t = Value::object();
  t["M"] = tl.micro_batches;
  t["S"] = tl.stage_count;
  t["phi"] = tl.phi;
  t["blocks"] = std::move(blocks);
  return t;
}

std::string text_of(const Value& v) { return v.is_string() ? v.as_string() : v.dump(); }

ModelProfile profile_of(const Value& v) {
  std::istringstream in(text_of(v));
  return load_profile(in);
}

ClusterSpec cluster_of(const Value& v) {
  std::istringstream in(text_of(v));
  return load_cluster(in);
}

PipelinePlan plan_of(const Value& v) { return plan_from_json(text_of(v)); }

namespace {

PhiStrategy strategy_of(const Value& req) {
  if (!req.contains("phi_strategy")) return PhiStrategy::preset_a;
  const std::string& s = req.at("phi_strategy").as_string();
  if (s == "preset_b") return PhiStrategy::preset_b;
  if (s == "search") return PhiStrategy::search;
  return PhiStrategy::preset_a;
}

int int_of(const Value& req, const char* key, int dflt) {
  return req.contains(key) ? static_cast<int>(req.at(key).as_int()) : dflt;
}
bool bool_of(const Value& req, const char* key) { return req.contains(key) && req.at(key).as_bool(); }
double dbl_of(const Value& req, const char* key, double dflt) {
  return req.contains(key) ? req.at(key).as_double() : dflt;
}
std::string str_of(const Value& req, const char* key, const char* dflt) {
  return req.contains(key) ? req.at(key).as_string() : std::string(dflt);
}

Value plan_json(const PipelinePlan& p, const ModelProfile& prof, const ClusterSpec& cl) {
  Value j = Value::parse(plan_to_json(p, compute_acr(build_stage_sequence(p, prof, cl))));
  j["est_latency_s"] = p.est_latency;
  if (p.sim_latency) j["sim_latency_s"] = *p.sim_latency;
  return j;
}

Value dispatch(const Value& req) {
  const std::string op = req.at("op").as_string();
  Value out = Value::object();
  if (op == "plan") {
    const ModelProfile prof = profile_of(req.at("profile"));
    const ClusterSpec cl = cluster_of(req.at("cluster"));
    PlannerOptions opts;
    opts.phi_strategy = strategy_of(req);
    opts.top_k = int_of(req, "top_k", 8);
    opts.optimizer_multiplier = dbl_of(req, "optimizer_multiplier", 8.0);
    SearchReport rep;
    const bool want = bool_of(req, "report");
    struct ThreadsScope {  // optional "threads": worker count of this search only (1 = sequential)
      explicit ThreadsScope(int n) { planner_threads_override() = n; }
      ~ThreadsScope() { planner_threads_override() = 0; }
    } threads_scope(int_of(req, "threads", 0));
    const PipelinePlan p = plan(prof, cl, int_of(req, "M", 1), opts, want ? &rep : nullptr);
    out["plan"] = plan_json(p, prof, cl);
    if (want) {
      Value top = Value::array();
      for (const RankedPlan& r : rep.top) {
        Value e = Value::object();
        e["est"] = r.est_latency;
        e["sim"] = r.sim_latency;
        e["plan"] = plan_json(r.plan, prof, cl);
        top.push_back(std::move(e));
      }
      Value r = Value::object();
      r["states_evaluated"] = rep.states_evaluated;
      r["top"] = std::move(top);
      out["report"] = std::move(r);
    }
    return out;
  }
  if (op == "brute_force_plan") {
    const ModelProfile prof = profile_of(req.at("profile"));
    const ClusterSpec cl = cluster_of(req.at("cluster"));
    PlannerOptions opts;
    opts.phi_strategy = strategy_of(req);
    out["plan"] = plan_json(brute_force_plan(prof, cl, int_of(req, "M", 1), opts), prof, cl);
    return out;
  }
  if (op == "simulate_plan") {
    const ModelProfile prof = profile_of(req.at("profile"));
    const ClusterSpec cl = cluster_of(req.at("cluster"));
    const bool gpipe = str_of(req, "schedule", "dapple") == "gpipe";
    const PlanSimulation sim = simulate_plan(plan_of(req.at("plan")), prof, cl, int_of(req, "M", 1),
                                             gpipe ? ScheduleKind::gpipe : ScheduleKind::dapple,
                                             bool_of(req, "recompute"));
    std::ostringstream csv;
    write_timeline_csv(csv, sim.timeline);
    out["latency"] = sim.latency;
    out["seq"] = seq_to_json(sim.seq);
    out["timeline"] = timeline_to_json(sim.timeline);
    out["peaks"] = peak_activations(sim.timeline);
    out["csv"] = csv.str();
    return out;
  }
  if (op == "build_stage_sequence") {
    out["seq"] = seq_to_json(build_stage_sequence(plan_of(req.at("plan")), profile_of(req.at("profile")),
                                                  cluster_of(req.at("cluster"))));
    return out;
  }
  if (op == "schedule") {
    const StageCostSequence seq = seq_from_json(req.at("seq"));
    const int m = int_of(req, "M", 1);
    const Timeline tl = str_of(req, "schedule", "dapple") == "gpipe"
                            ? gpipe_schedule(seq, m)
                            : dapple_schedule(seq, m, req.at("phi").as_int_vector());
    out["latency"] = batch_latency(tl, seq);
    out["timeline"] = timeline_to_json(tl);
    out["peaks"] = peak_activations(tl);
    return out;
  }
  if (op == "estimate") {
    const StageCostSequence seq = seq_from_json(req.at("seq"));
    const int m = int_of(req, "M", 1);
    const LatencyBreakdown lb = estimate_latency(seq, m);
    out["warmup"] = lb.warmup;
    out["steady"] = lb.steady;
    out["ending"] = lb.ending;
    out["total"] = lb.total;
    out["pivot"] = lb.pivot;
    out["select_pivot"] = select_pivot(seq, m);
    bool any_compute = false;
    for (const StageCost& c : seq) any_compute = any_compute || c.kind == StageKind::compute;
    if (any_compute) out["acr"] = compute_acr(seq);
    return out;
  }
  if (op == "optimize_phi") {
    const PhiResult r = optimize_phi(seq_from_json(req.at("seq")), int_of(req, "M", 1), strategy_of(req),
                                     int_of(req, "D", 1));
    out["phi"] = r.phi;
    out["latency"] = r.latency;
    return out;
  }
  if (op == "expand_plan_phi") {
    out["phi"] = expand_plan_phi(req.at("phi").as_int_vector());
    return out;
  }
  if (op == "apply_recompute") {
    out["seq"] = seq_to_json(apply_recompute(seq_from_json(req.at("seq"))));
    return out;
  }
  if (op == "allreduce_time") {
    out["t"] = allreduce_time(req.at("size").as_int(), req.at("devices").as_int_vector(), cluster_of(req.at("cluster")));
    return out;
  }
  if (op == "splitconcat_time") {
    out["t"] = splitconcat_time(req.at("size").as_int(), req.at("src").as_int_vector(), req.at("dst").as_int_vector(),
                                cluster_of(req.at("cluster")));
    return out;
  }
  if (op == "aggregate_stage") {
    out["seq"] = seq_to_json({aggregate_stage(profile_of(req.at("profile")), int_of(req, "lo", 0),
                                              int_of(req, "hi", 0), int_of(req, "r", 1))});
    return out;
  }
  if (op == "enumerate_placements") {
    DeviceState st{cluster_of(req.at("cluster"))};
    if (req.contains("free")) st.free = req.at("free").as_int_vector();
    Value sets = Value::array();
    for (const auto& s : enumerate_placements(st, int_of(req, "count", 1))) sets.push_back(Value(s));
    out["placements"] = std::move(sets);
    return out;
  }
  if (op == "memory_feasible") {
    StageCost c;
    c.param_bytes = req.at("param_bytes").as_int();
    c.activation_out_bytes = req.at("act").as_int();
    out["ok"] = memory_feasible(c, int_of(req, "injected", 1), req.at("capacity").as_int(),
                                dbl_of(req, "optimizer_multiplier", 8.0));
    return out;
  }
  if (op == "load_profile") {
    const ModelProfile p = profile_of(req.at("profile"));
    Value layers = Value::array();
    for (const LayerProfile& l : p.layers) {
      Value row = Value::array();
      row.push_back(l.index);
      row.push_back(l.fwd_time);
      row.push_back(l.bwd_time);
      row.push_back(static_cast<long long>(l.activation_bytes));
      row.push_back(static_cast<long long>(l.param_bytes));
      layers.push_back(std::move(row));
    }
    out["profile_batch_size"] = p.profile_batch_size;
    out["layers"] = std::move(layers);
    out["json"] = profile_to_json(p);
    return out;
  }
  if (op == "load_cluster") {
    const ClusterSpec c = cluster_of(req.at("cluster"));
    out["seps"] = c.seps;
    out["intra_bw"] = c.intra_bw;
    out["inter_bw"] = c.inter_bw;
    out["intra_latency"] = c.intra_latency;
    out["inter_latency"] = c.inter_latency;
    out["per_gpu_memory"] = static_cast<long long>(c.per_gpu_memory);
    out["json"] = cluster_to_json(c);
    return out;
  }
  if (op == "stage_chain") {
    Value chain = Value::array();
    const bool gpipe = str_of(req, "schedule", "dapple") == "gpipe";
    for (const ChainOp& c : stage_chain(int_of(req, "M", 1), int_of(req, "phi", 1),
                                        gpipe ? ScheduleKind::gpipe : ScheduleKind::dapple)) {
      Value e = Value::array();
      e.push_back(c.kind == BlockKind::forward ? 0 : 1);
      e.push_back(c.micro_batch);
      chain.push_back(std::move(e));
    }
    out["chain"] = std::move(chain);
    return out;
  }
  if (op == "splitconcat_routes") {
    const PipelinePlan p = plan_of(req.at("plan"));
    const int k = int_of(req, "boundary", 0);
    if (k < 0 || k + 1 >= p.compute_stage_count()) throw std::out_of_range("splitconcat_routes: bad boundary");
    Value routes = Value::array();
    for (const SplitConcatRoute& r :
         splitconcat_routes(p.stages[k], p.stages[k + 1], int_of(req, "micro_batch", 1), int_of(req, "rows_per_sample", 1))) {
      Value e = Value::array();
      e.push_back(r.src_gpu);
      e.push_back(r.dst_gpu);
      e.push_back(static_cast<long long>(r.src_row));
      e.push_back(static_cast<long long>(r.dst_row));
      e.push_back(static_cast<long long>(r.rows));
      routes.push_back(std::move(e));
    }
    out["routes"] = std::move(routes);
    return out;
  }
  if (op == "timeline_export") {
    // a measured (or any) timeline in timeline_to_json form -> the
    // reference's CSV / SVG writers (io.cpp) and its block-level metrics
    const Value& t = req.at("timeline");
    Timeline tl;
    tl.micro_batches = static_cast<int>(t.at("M").as_int());
    tl.stage_count = static_cast<int>(t.at("S").as_int());
    for (const Value& p : t.at("phi").items()) tl.phi.push_back(static_cast<int>(p.as_int()));
    tl.blocks.resize(static_cast<size_t>(2) * tl.micro_batches * tl.stage_count);
    for (const Value& b : t.at("blocks").items()) {
      const int x = static_cast<int>(b[0].as_int()), i = static_cast<int>(b[1].as_int());
      const bool fwd = b[2].as_int() == 0;
      if (x < 0 || x >= tl.stage_count || i < 0 || i >= tl.micro_batches)
        throw std::invalid_argument("timeline_export: block out of range");
      Block& blk = fwd ? tl.forward(i, x) : tl.backward(i, x);
      blk.stage = x;
      blk.micro_batch = i;
      blk.kind = fwd ? BlockKind::forward : BlockKind::backward;
      blk.start = b[3].as_double();
      blk.end = b[4].as_double();
    }
    std::ostringstream csv;
    write_timeline_csv(csv, tl);
    out["csv"] = csv.str();
    Value peaks = Value::array();
    for (int p : peak_activations(tl)) peaks.push_back(p);
    out["peak_activations"] = std::move(peaks);
    if (req.contains("plan")) {
      const StageCostSequence seq = build_stage_sequence(plan_of(req.at("plan")), profile_of(req.at("profile")),
                                                         cluster_of(req.at("cluster")));
      std::ostringstream svg;
      write_timeline_svg(svg, tl, seq);
      out["svg"] = svg.str();
      out["latency"] = batch_latency(tl, seq);
    }
    return out;
  }
  if (op == "timeline_svg") {
    const ModelProfile prof = profile_of(req.at("profile"));
    const ClusterSpec cl = cluster_of(req.at("cluster"));
    const PlanSimulation sim = simulate_plan(plan_of(req.at("plan")), prof, cl, int_of(req, "M", 1));
    std::ostringstream svg;
    write_timeline_svg(svg, sim.timeline, sim.seq);
    out["svg"] = svg.str();
    return out;
  }
  throw std::invalid_argument("unknown op " + op);
}

thread_local std::string g_reply;

Value error_reply(const char* type, const char* what) {
  Value e = Value::object();
  e["type"] = type;
  e["what"] = what;
  Value r = Value::object();
  r["error"] = std::move(e);
  return r;
}

}  // namespace
}  // namespace dpl

extern "C" const char* dpl_host_call(const char* request) {
  using dpl::error_reply;
  Value reply;
  try {
    reply = dpl::dispatch(Value::parse(request ? request : ""));
  } catch (const std::invalid_argument& e) {
    reply = error_reply("invalid_argument", e.what());
  } catch (const std::out_of_range& e) {
    reply = error_reply("out_of_range", e.what());
  } catch (const std::logic_error& e) {
    reply = error_reply("logic_error", e.what());
  } catch (const std::runtime_error& e) {
    reply = error_reply("runtime_error", e.what());
  } catch (const std::exception& e) {
    reply = error_reply("exception", e.what());
  }
  dpl::g_reply = reply.dump();
  return dpl::g_reply.c_str();
}
