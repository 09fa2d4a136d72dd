// Capacity planning from measured numbers (FastDecode Eq. 7-11): the
// reference's planner (planner.cpp:48-222, planner.hpp:25-109) as host C++
// over B200-measured inputs — T(B) from sd_bench_dense_block and R from
// sd_bench_attention_per_token.
#include "planner.h"

#include <algorithm>
#include <cmath>
#include <string>

namespace sd {

void validate_profile(const PerfProfile& p) {
  if (p.t_table.empty()) fail(SD_ERR_CONFIG, "profile: empty T(B) table");
  for (size_t i = 0; i < p.t_table.size(); ++i) {
    if (!(p.t_table[i].second > 0)) fail(SD_ERR_CONFIG, "profile: T(B) entries must be positive");
    if (i && p.t_table[i].first <= p.t_table[i - 1].first) {
      fail(SD_ERR_CONFIG, "profile: batch sizes must be strictly ascending");
    }
  }
  if (!(p.r_per_token > 0)) fail(SD_ERR_CONFIG, "profile: R must be positive");
  if (p.capacity_c < 1) fail(SD_ERR_CONFIG, "profile: capacity must be >= 1");
}

// T(B): piecewise-linear between measured batches; no extrapolation
double block_seconds(const PerfProfile& p, int batch) {
  const auto& t = p.t_table;
  if (batch < t.front().first) {
    fail(SD_ERR_CONFIG, "T(B): batch " + std::to_string(batch) + " below the measured range");
  }
  if (batch > t.back().first) {
    fail(SD_ERR_CONFIG, "T(B): batch " + std::to_string(batch) + " above the measured range (extrapolation refused)");
  }
  auto hi = std::lower_bound(t.begin(), t.end(), batch,
                             [](const std::pair<int, double>& e, int b) { return e.first < b; });
  if (hi->first == batch) return hi->second;
  const auto lo = hi - 1;
  const double frac = static_cast<double>(batch - lo->first) / (hi->first - lo->first);
  return lo->second + frac * (hi->second - lo->second);
}

double batch_efficiency(const PerfProfile& p, int batch) { return batch / block_seconds(p, batch); }

int plan_batch_size(const PerfProfile& p, const PlanRequest& r, int* tightest_out) {
  if (r.num_layers < 1 || r.target_len < 1) fail(SD_ERR_CONFIG, "plan request: layers and target length must be >= 1");
  std::vector<int> cand = r.candidates;
  if (cand.empty()) {
    for (const auto& e : p.t_table) cand.push_back(e.first);
  }
  std::sort(cand.begin(), cand.end());
  if (r.latency_budget > 0) {
    // largest batch whose full-sequence latency 2·N·S·T(B) fits the budget
    int best = -1, tight = cand.front();
    double tight_s = 0;
    for (size_t i = 0; i < cand.size(); ++i) {
      const double sec = 2.0 * r.num_layers * r.target_len * block_seconds(p, cand[i]);
      if (i == 0 || sec < tight_s) {
        tight = cand[i];
        tight_s = sec;
      }
      if (sec <= r.latency_budget) best = cand[i];
    }
    if (tightest_out) *tightest_out = tight;
    if (best < 0) {
      fail(SD_ERR_INFEASIBLE, "no candidate batch satisfies the latency budget; tightest is B=" +
                                  std::to_string(tight) + " at " + std::to_string(tight_s) + " s");
    }
    return best;
  }
  // knee: first step whose throughput gain per doubling of B falls below the threshold
  for (size_t i = 1; i < cand.size(); ++i) {
    const double e0 = batch_efficiency(p, cand[i - 1]), e1 = batch_efficiency(p, cand[i]);
    const double doublings = std::log2(static_cast<double>(cand[i]) / cand[i - 1]);
    if (std::pow(e1 / e0, 1.0 / doublings) - 1.0 < r.knee_threshold) return cand[i - 1];
  }
  return cand.back();
}

void plan_worker_count(const PerfProfile& p, int batch, int target_len, int* workers, double* estimate) {
  // attention of B sequences at mean length S/2 spread over P workers
  // matches one dense block: P = B·S·R / (2·T(B))
  const double est = static_cast<double>(batch) * target_len * p.r_per_token / (2.0 * block_seconds(p, batch));
  *estimate = est;
  *workers = std::max(1, static_cast<int>(std::ceil(est)));
}

void check_memory(int64_t batch, int64_t target_len, int64_t capacity, int64_t workers, bool* feasible,
                  int* min_workers) {
  if (batch < 1 || target_len < 1 || capacity < 1 || workers < 1) {
    fail(SD_ERR_CONFIG, "check_memory: all arguments must be >= 1");
  }
  const double need = static_cast<double>(batch) * target_len / 2.0;  // mean resident tokens
  *feasible = need <= static_cast<double>(capacity) * workers;
  *min_workers = *feasible ? static_cast<int>(workers) : static_cast<int>(std::ceil(need / capacity));
}

void check_balance(const PerfProfile& p, int batch, int target_len, int workers, double tolerance,
                   double* stage_seconds, double* residual, bool* accepted) {
  if (workers < 1) fail(SD_ERR_CONFIG, "check_balance: workers must be >= 1");
  const double t = block_seconds(p, batch);
  *stage_seconds = static_cast<double>(batch) * target_len * p.r_per_token / (2.0 * workers);
  *residual = std::fabs(*stage_seconds - t) / t;
  *accepted = *residual <= tolerance;
}

HardwarePlan plan(const PerfProfile& p, const PlanRequest& r) {
  validate_profile(p);
  HardwarePlan h;
  h.batch_size = plan_batch_size(p, r, &h.tightest_batch);
  h.binding = r.latency_budget > 0 ? kBindLatency : kBindKnee;
  plan_worker_count(p, h.batch_size, r.target_len, &h.worker_count, &h.worker_estimate);
  bool ok = false;
  int minw = 0;
  check_memory(h.batch_size, r.target_len, p.capacity_c, h.worker_count, &ok, &minw);
  if (!ok) {
    h.worker_count = minw;
    h.binding = kBindMemory;
  }
  const double t = block_seconds(p, h.batch_size);
  h.predicted_seq_seconds = 2.0 * r.num_layers * r.target_len * t;
  h.efficiency = h.batch_size / t;
  const double stage = static_cast<double>(h.batch_size) * r.target_len * p.r_per_token / (2.0 * h.worker_count);
  h.balance_residual = std::fabs(stage - t) / t;
  h.balanced = h.balance_residual <= r.balance_tolerance;
  return h;
}

}  // namespace sd
