// GPU measurements of the planner's inputs (perf_bench.cpp).
#pragma once

#include <cstdint>

#include "engine.h"
#include "kv_store.h"

namespace sd {

// T(B) for each batch (ascending) in seconds per block
void bench_dense_block(Weights& w, const int* batches, int n, int reps, double* seconds);
// R in seconds per token-position per layer for a shard holding all kv heads
double bench_attention_per_token(const Spec& spec, int fmt, int batch, int seq_len, int reps, int device);
// C: token positions of full-depth KV that fit in the device's free memory
int64_t kv_capacity_tokens(const Spec& spec, int fmt, int device, double reserve_bytes);

}  // namespace sd
