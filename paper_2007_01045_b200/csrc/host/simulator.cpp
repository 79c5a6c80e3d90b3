// Exact schedule simulation (reference: proj/src/simulator.cpp).
//
// The reference solves the block DAG with Kahn's algorithm over explicit
// edges.  Here the DAG is exploited structurally: the intra-stage edges of
// both schedules form a *total order* per stage (stage_chain below), so each
// stage is a chain and the only cross-stage edges are f[i,x-1] -> f[i,x] and
// b[i,x+1] -> b[i,x].  A multi-pointer sweep over the S chains therefore
// visits every block once, in a topological order, and sets
// start = max(end of chain predecessor, end of cross-stage dependency),
// end = start + duration.  max() is exact in IEEE arithmetic, so the times
// equal the reference's bit for bit.  The same chains drive the GPU
// executor's per-stage stream programs.
#include "pipeplan/simulator.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>

namespace pipeplan {

namespace {

inline std::size_t fwd_slot(int i, int x, int m) { return static_cast<std::size_t>(x) * m + i; }
inline std::size_t bwd_slot(int i, int x, int m, int s) {
  return static_cast<std::size_t>(s) * m + static_cast<std::size_t>(x) * m + i;
}

// simulator.cpp:118-133 (same messages)
void validate_phi(const std::vector<int>& phi, int stages, int m) {
  if (static_cast<int>(phi.size()) != stages) {
    throw std::invalid_argument("phi: expected one entry per stage, got " + std::to_string(phi.size()) +
                                " for " + std::to_string(stages) + " stages");
  }
  for (int x = 0; x < stages; ++x) {
    if (phi[x] < 1 || phi[x] > m) throw std::invalid_argument("phi[" + std::to_string(x) + "] must be in [1, M]");
    if (x > 0 && phi[x] > phi[x - 1]) throw std::invalid_argument("phi must be non-increasing toward the top stage");
  }
  if (phi.back() != 1) throw std::invalid_argument("phi of the topmost stage must be 1");
}

Timeline sweep(const StageCostSequence& seq, int m, const std::vector<int>& phi, ScheduleKind kind) {
  const int s = static_cast<int>(seq.size());
  Timeline tl;
  tl.micro_batches = m;
  tl.stage_count = s;
  tl.phi = phi;
  tl.blocks.resize(static_cast<std::size_t>(2) * m * s);
  std::vector<char> done(tl.blocks.size(), 0);

  std::vector<std::vector<ChainOp>> chains(s);
  for (int x = 0; x < s; ++x) chains[x] = stage_chain(m, phi[x], kind);
  std::vector<std::size_t> cursor(s, 0);
  std::vector<double> last_end(s, 0.0);

  std::size_t remaining = tl.blocks.size();
  while (remaining > 0) {
    bool progressed = false;
    for (int x = 0; x < s; ++x) {
      while (cursor[x] < chains[x].size()) {
        const ChainOp op = chains[x][cursor[x]];
        const int i = op.micro_batch;
        const bool fwd = op.kind == BlockKind::forward;
        double dep = cursor[x] == 0 ? 0.0 : last_end[x];
        if (fwd && x > 0) {
          const std::size_t up = fwd_slot(i, x - 1, m);
          if (!done[up]) break;
          dep = std::max(dep, tl.blocks[up].end);
        }
        if (!fwd && x + 1 < s) {
          const std::size_t down = bwd_slot(i, x + 1, m, s);
          if (!done[down]) break;
          dep = std::max(dep, tl.blocks[down].end);
        }
        const std::size_t slot = fwd ? fwd_slot(i, x, m) : bwd_slot(i, x, m, s);
        Block& b = tl.blocks[slot];
        b.stage = x;
        b.micro_batch = i;
        b.kind = op.kind;
        b.start = dep;
        b.end = dep + (fwd ? seq[x].fwd : seq[x].bwd);
        done[slot] = 1;
        last_end[x] = b.end;
        ++cursor[x];
        --remaining;
        progressed = true;
      }
    }
    if (!progressed) throw std::logic_error("schedule dependency graph has a cycle");
  }
  return tl;
}

}  // namespace

// The per-stage total order implied by simulator.cpp:81-97.
// dapple: F_0..F_{phi-1}, then B_j, F_{j+phi} alternating, then the
// remaining backwards.  gpipe: all forwards, then all backwards.
std::vector<ChainOp> stage_chain(int m, int phi_x, ScheduleKind kind) {
  std::vector<ChainOp> chain;
  chain.reserve(static_cast<std::size_t>(2) * m);
  const int warm = kind == ScheduleKind::gpipe ? m : std::min(phi_x, m);
  for (int i = 0; i < warm; ++i) chain.push_back({BlockKind::forward, i});
  int next_f = warm;
  for (int j = 0; j < m; ++j) {
    chain.push_back({BlockKind::backward, j});
    if (next_f < m) chain.push_back({BlockKind::forward, next_f++});
  }
  return chain;
}

const Block& Timeline::forward(int micro_batch, int stage) const { return blocks[fwd_slot(micro_batch, stage, micro_batches)]; }
const Block& Timeline::backward(int micro_batch, int stage) const {
  return blocks[bwd_slot(micro_batch, stage, micro_batches, stage_count)];
}
Block& Timeline::forward(int micro_batch, int stage) { return blocks[fwd_slot(micro_batch, stage, micro_batches)]; }
Block& Timeline::backward(int micro_batch, int stage) {
  return blocks[bwd_slot(micro_batch, stage, micro_batches, stage_count)];
}

// simulator.cpp:153-159
Timeline dapple_schedule(const StageCostSequence& seq, int micro_batches, const std::vector<int>& phi) {
  if (seq.empty()) throw std::invalid_argument("dapple_schedule: empty stage sequence");
  if (micro_batches < 1) throw std::invalid_argument("dapple_schedule: M must be >= 1");
  validate_phi(phi, static_cast<int>(seq.size()), micro_batches);
  return sweep(seq, micro_batches, phi, ScheduleKind::dapple);
}

// simulator.cpp:161-167
Timeline gpipe_schedule(const StageCostSequence& seq, int micro_batches) {
  if (seq.empty()) throw std::invalid_argument("gpipe_schedule: empty stage sequence");
  if (micro_batches < 1) throw std::invalid_argument("gpipe_schedule: M must be >= 1");
  return sweep(seq, micro_batches, std::vector<int>(seq.size(), micro_batches), ScheduleKind::gpipe);
}

// simulator.cpp:169-179
double batch_latency(const Timeline& timeline, const StageCostSequence& seq) {
  if (static_cast<int>(seq.size()) != timeline.stage_count) {
    throw std::invalid_argument("batch_latency: sequence does not match timeline");
  }
  double latest = 0.0;
  for (int x = 0; x < timeline.stage_count; ++x) {
    latest = std::max(latest, timeline.backward(timeline.micro_batches - 1, x).end + seq[x].allreduce_time);
  }
  return latest;
}

// simulator.cpp:181-203: +1 when a forward ends, -1 when its backward ends;
// coincident events are applied together before the peak is sampled.
std::vector<int> peak_activations(const Timeline& timeline) {
  std::vector<int> peaks(timeline.stage_count, 0);
  std::vector<std::pair<double, int>> ev;
  for (int x = 0; x < timeline.stage_count; ++x) {
    ev.clear();
    for (int i = 0; i < timeline.micro_batches; ++i) {
      ev.emplace_back(timeline.forward(i, x).end, 1);
      ev.emplace_back(timeline.backward(i, x).end, -1);
    }
    std::sort(ev.begin(), ev.end());
    int live = 0, peak = 0;
    for (std::size_t k = 0; k < ev.size();) {
      const double t = ev[k].first;
      while (k < ev.size() && ev[k].first == t) live += ev[k++].second;
      peak = std::max(peak, live);
    }
    peaks[x] = peak;
  }
  return peaks;
}

// simulator.cpp:205-214: the comm stage between k and k+1 takes phi[k+1].
std::vector<int> expand_plan_phi(const std::vector<int>& compute_phi) {
  if (compute_phi.empty()) throw std::invalid_argument("expand_plan_phi: empty phi");
  std::vector<int> out;
  for (std::size_t k = 0; k < compute_phi.size(); ++k) {
    out.push_back(compute_phi[k]);
    if (k + 1 < compute_phi.size()) out.push_back(compute_phi[k + 1]);
  }
  return out;
}

// simulator.cpp:216-221
StageCostSequence apply_recompute(StageCostSequence seq) {
  for (StageCost& c : seq) {
    if (c.kind == StageKind::compute) c.bwd += c.fwd;
  }
  return seq;
}

// simulator.cpp:233-286
PhiResult optimize_phi(const StageCostSequence& seq, int micro_batches, PhiStrategy strategy, int max_injection) {
  if (seq.empty()) throw std::invalid_argument("optimize_phi: empty stage sequence");
  if (micro_batches < 1) throw std::invalid_argument("optimize_phi: M must be >= 1");
  if (max_injection < 1) throw std::invalid_argument("optimize_phi: injection cap D must be >= 1");
  const int s = static_cast<int>(seq.size());
  auto preset = [&](bool policy_b) {
    std::vector<int> phi(s);
    for (int i = 0; i < s; ++i) {
      const int lead = policy_b ? 2 * (s - i) - 1 : s - i;
      phi[i] = std::min({lead, max_injection, micro_batches});
    }
    return phi;
  };
  auto evaluate = [&](const std::vector<int>& phi) {
    return PhiResult{phi, batch_latency(dapple_schedule(seq, micro_batches, phi), seq)};
  };
  if (strategy == PhiStrategy::preset_a) return evaluate(preset(false));
  if (strategy == PhiStrategy::preset_b) return evaluate(preset(true));

  // exhaustive: non-increasing vectors bounded by preset B; best by
  // (latency, sum, lexicographic)
  const std::vector<int> bound = preset(true);
  std::vector<int> cur(s, 1);
  PhiResult best;
  long long best_sum = 0;
  bool have = false;
  auto visit = [&](auto&& self, int pos) -> void {
    if (pos == s) {
      PhiResult r = evaluate(cur);
      const long long sum = std::accumulate(cur.begin(), cur.end(), 0LL);
      if (!have || r.latency < best.latency ||
          (r.latency == best.latency && (sum < best_sum || (sum == best_sum && cur < best.phi)))) {
        best = std::move(r);
        best_sum = sum;
        have = true;
      }
      return;
    }
    const int top = pos == 0 ? bound[0] : std::min(bound[pos], cur[pos - 1]);
    for (int v = top; v >= 1; --v) {
      cur[pos] = v;
      self(self, pos + 1);
    }
  };
  visit(visit, 0);
  return best;
}

}  // namespace pipeplan
