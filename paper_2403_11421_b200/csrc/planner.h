// Capacity planner (planner.cpp) over measured T(B) and R.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "sd_common.h"

namespace sd {

struct PerfProfile {
  std::vector<std::pair<int, double>> t_table;  // (batch, seconds per block), ascending
  double r_per_token = 0;                       // seconds per token-position per layer per worker
  int64_t capacity_c = 0;                       // tokens of KV storage per worker
};

constexpr double kNoBudget = -1.0;
struct PlanRequest {
  int num_layers = 0;
  int target_len = 0;            // S
  double latency_budget = kNoBudget;  // seconds per full sequence (> 0), or kNoBudget
  std::vector<int> candidates;   // empty: the profile's table
  double knee_threshold = 0.10;
  double balance_tolerance = 0.15;
};

enum Binding : int { kBindLatency = 0, kBindKnee = 1, kBindMemory = 2 };

struct HardwarePlan {
  int batch_size = 0, worker_count = 0;
  double worker_estimate = 0, predicted_seq_seconds = 0, efficiency = 0, balance_residual = 0;
  bool balanced = false;
  int binding = kBindKnee;
  int tightest_batch = 0;
};

void validate_profile(const PerfProfile& p);
double block_seconds(const PerfProfile& p, int batch);
double batch_efficiency(const PerfProfile& p, int batch);
int plan_batch_size(const PerfProfile& p, const PlanRequest& r, int* tightest_out);
void plan_worker_count(const PerfProfile& p, int batch, int target_len, int* workers, double* estimate);
void check_memory(int64_t batch, int64_t target_len, int64_t capacity, int64_t workers, bool* feasible,
                  int* min_workers);
void check_balance(const PerfProfile& p, int batch, int target_len, int workers, double tolerance,
                   double* stage_seconds, double* residual, bool* accepted);
HardwarePlan plan(const PerfProfile& p, const PlanRequest& r);

}  // namespace sd
