// Split-Concat routing: which rows of a micro-batch move
// from each replica of stage k to each replica of stage k+1.
#include <algorithm>
#include <stdexcept>

#include "pipeplan/executor.hpp"

namespace pipeplan {

std::vector<SplitConcatRoute> splitconcat_routes(const Stage& from, const Stage& to, int micro_batch_samples,
                                                 int rows_per_sample) {
  const int ra = from.replication(), rb = to.replication();
  if (ra < 1 || rb < 1) throw std::invalid_argument("splitconcat_routes: empty device set");
  if (micro_batch_samples < ra || micro_batch_samples < rb)
    throw std::invalid_argument("splitconcat_routes: micro-batch has fewer samples than replicas");
  const std::int64_t B = micro_batch_samples;
  std::vector<SplitConcatRoute> out;
  for (int i = 0; i < ra; ++i) {
    const std::int64_t a0 = B * i / ra, a1 = B * (i + 1) / ra;  // samples owned by source replica i
    for (int j = 0; j < rb; ++j) {
      const std::int64_t b0 = B * j / rb, b1 = B * (j + 1) / rb;
      const std::int64_t lo = std::max(a0, b0), hi = std::min(a1, b1);
      if (hi <= lo) continue;
      out.push_back({from.devices[i], to.devices[j], (lo - a0) * rows_per_sample, (lo - b0) * rows_per_sample,
                     (hi - lo) * rows_per_sample});
    }
  }
  return out;
}

}  // namespace pipeplan
