// pipeplan::execute_plan -- the C++ drop-in entry point (executor.hpp),
// built on the C-ABI executor so the boundary stays the same for every host
// language.  Mirrors simulate_plan (planner.cpp:491-514).
#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>

#include "dapple.h"
#include "host/json.hpp"
#include "pipeplan/estimator.hpp"
#include "pipeplan/executor.hpp"
#include "pipeplan/io.hpp"
#include "pipeplan/planner.hpp"

namespace pipeplan {

namespace {

using dpl::json::Value;

void ok(int rc) {
  if (rc != 0) throw std::runtime_error(std::string("execute_plan: ") + dpl_last_error());
}

std::vector<std::string> gather(const ExecOptions& o, const std::string& mine) {
  if (o.world == 1) return {mine};
  if (!o.allgather) throw std::invalid_argument("execute_plan: world > 1 needs ExecOptions::allgather");
  std::vector<std::string> all = o.allgather(mine);
  if (static_cast<int>(all.size()) != o.world) throw std::runtime_error("execute_plan: allgather size mismatch");
  return all;
}

}  // namespace

PlanExecution execute_plan(const PipelinePlan& plan, const ModelProfile& profile, const ClusterSpec& cluster,
                           int micro_batches, const ExecOptions& opts) {
  PlanExecution out;
  out.seq = build_stage_sequence(plan, profile, cluster);  // validates the plan (model.cpp:100-131)
  const std::vector<int> phi = opts.schedule == ScheduleKind::gpipe
                                   ? std::vector<int>(out.seq.size(), micro_batches)  // simulator.cpp:164-166
                                   : resolve_phi(plan, out.seq, micro_batches);

  Value cfg = Value::object();
  cfg["model"] = Value::parse(opts.model_json);
  cfg["plan"] = Value::parse(plan_to_json(plan, 0.0));
  cfg["M"] = micro_batches;
  cfg["gbs"] = opts.global_batch;
  cfg["lr"] = opts.lr;
  cfg["seed"] = static_cast<long long>(opts.seed);
  cfg["rank"] = opts.rank;
  cfg["world"] = opts.world;
  cfg["apply"] = opts.apply;
  cfg["schedule"] = opts.schedule == ScheduleKind::gpipe ? "gpipe" : "dapple";
  cfg["recompute"] = opts.recompute;
  cfg["allreduce"] = opts.allreduce;
  dpl_exec* ex = nullptr;
  ok(dpl_exec_create(cfg.dump().c_str(), opts.device, &ex));
  try {
    if (opts.world > 1) {
      char blob[256];
      size_t len = 0;
      ok(dpl_exec_export(ex, blob, sizeof blob, &len));
      std::string all;
      for (const std::string& b : gather(opts, std::string(blob, len))) all += b;
      ok(dpl_exec_connect(ex, all.data(), len, opts.world));
      // one NCCL communicator per replicated stage; its lowest GPU makes the id
      const Stage* mine = nullptr;
      for (const Stage& s : plan.stages)
        if (std::find(s.devices.begin(), s.devices.end(), opts.rank) != s.devices.end()) mine = &s;
      if (!mine) throw std::invalid_argument("execute_plan: rank not in plan");
      std::string id;
      const bool nccl = mine->replication() > 1 && opts.allreduce == "nccl";
      if (nccl && mine->devices.front() == opts.rank) {
        char buf[128];
        ok(dpl_exec_nccl_id(buf));
        id.assign(buf, sizeof buf);
      }
      const std::vector<std::string> ids = gather(opts, id);
      if (nccl) ok(dpl_exec_nccl_init(ex, ids[mine->devices.front()].data()));
    }
    float loss = std::nanf("");
    ok(dpl_exec_step(ex, nullptr, nullptr, &loss));
    const std::vector<std::string> parts = gather(opts, dpl_exec_timeline(ex));

    // merge the per-rank measured blocks on the GPUs' global timer
    const int S = 2 * plan.compute_stage_count() - 1, M = micro_batches;
    long long t0 = std::numeric_limits<long long>::max();
    std::vector<Value> docs;
    for (const std::string& p : parts) {
      docs.push_back(Value::parse(p));
      t0 = std::min(t0, static_cast<long long>(docs.back().at("t0_ns").as_int()));
    }
    std::map<std::tuple<int, int, int>, std::pair<double, double>> span;
    double end = 0.0, busy = 0.0;
    out.loss = std::nan("");
    for (const Value& d : docs) {
      const double off = (d.at("t0_ns").as_int() - t0) * 1e-9;
      end = std::max(end, off + d.at("step_s").as_double());
      if (!d.at("loss").is_null()) out.loss = d.at("loss").as_double();
      for (const Value& b : d.at("blocks").items()) {
        const int x = static_cast<int>(b[0].as_int()), i = static_cast<int>(b[1].as_int()),
                  k = static_cast<int>(b[2].as_int());
        const double s = b[3].as_double() + off, e = b[4].as_double() + off;
        if (b[3].as_double() < 0) continue;
        if (x % 2 == 0) busy += e - s;
        auto key = std::make_tuple(x, i, k);
        auto it = span.find(key);
        if (it == span.end()) span[key] = {s, e};
        else it->second = {std::min(it->second.first, s), std::max(it->second.second, e)};
      }
    }
    double first = std::numeric_limits<double>::infinity();
    for (const auto& [key, se] : span)
      if (std::get<2>(key) == 0 && std::get<0>(key) % 2 == 0) first = std::min(first, se.first);
    Timeline& tl = out.timeline;
    tl.micro_batches = M;
    tl.stage_count = S;
    tl.phi = phi;
    tl.blocks.resize(static_cast<size_t>(2) * M * S);
    for (int x = 0; x < S; ++x)
      for (int i = 0; i < M; ++i)
        for (int k = 0; k < 2; ++k) {
          Block& b = k == 0 ? tl.forward(i, x) : tl.backward(i, x);
          b.stage = x;
          b.micro_batch = i;
          b.kind = k == 0 ? BlockKind::forward : BlockKind::backward;
          auto it = span.find(std::make_tuple(x, i, k));
          b.start = it == span.end() ? std::nan("") : it->second.first - first;
          b.end = it == span.end() ? std::nan("") : it->second.second - first;
        }
    out.latency = end - first;
    out.bubble = 1.0 - busy / (opts.world * out.latency);
    if (opts.world > 1) {
      ok(dpl_exec_disconnect(ex));
      gather(opts, "");  // barrier: every rank has unmapped its peers before anyone frees
    }
  } catch (...) {
    dpl_exec_destroy(ex);
    throw;
  }
  dpl_exec_destroy(ex);
  return out;
}

}  // namespace pipeplan
