/*
 * A plain C program over include/sd_abi.h — the drop-in boundary exercised
 * the way a non-Python host (the reference's C++ driver, a cgo / JNI / FFI
 * binding) would call it: opaque handles, host pointers, int statuses and
 * sd_last_error(). Built by tests/test_abi_c.py with gcc against
 * libsd_b200.so.
 *
 *   sd_abi_test host       host-only entry points (no device needed):
 *                          specs, mix64 / prompt_token, ShardMap, the
 *                          scheduler, the distributed row plan, the planner,
 *                          typed errors
 *   sd_abi_test gpu GOLDEN the toy model end to end on cuda:0: product-side
 *                          seed_random_weights, KvShard, the StepComputation
 *                          driven by drive_schedule (sd_drive) must print the
 *                          reference's golden transcript byte for byte
 *                          (test_dense.cpp:173-190); one step through the
 *                          features entry point must pick the tokens the
 *                          token-id entry point picks
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sd_abi.h"

static int failures = 0;
#define CHECK(cond, ...)                                   \
  do {                                                     \
    if (!(cond)) {                                         \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);                        \
      fprintf(stderr, "\n");                               \
      ++failures;                                          \
    }                                                      \
  } while (0)
#define OK(call) CHECK((call) == SD_OK, "%s -> %s", #call, sd_last_error())

static void host_checks(void) {
  sd_model_spec s;
  OK(sd_make_model_spec(2, 64, 4, 256, 128, 0, &s));
  CHECK(s.head_dim == 16 && s.num_kv_heads == 4, "toy spec: hd %d kv %d", s.head_dim, s.num_kv_heads);
  /* ConfigError (core.cpp:11-30) with a message */
  CHECK(sd_make_model_spec(2, 63, 4, 256, 128, 0, &s) == SD_ERR_CONFIG, "D not divisible by H");
  CHECK(strstr(sd_last_error(), "divisible") != NULL, "message: %s", sd_last_error());

  /* mix64 / prompt_token (core.cpp:161-171); values pinned by the oracle tests */
  CHECK(sd_mix64(42) == 0xbdd732262feb6e95ull, "mix64(42)");
  CHECK(sd_prompt_token(0, 1, 128) == 30 && sd_prompt_token(0, 2, 128) == 52 && sd_prompt_token(0, 3, 128) == 23,
        "prompt tokens seed 0");
  CHECK(sd_prompt_token(7, 1, 32000) == 31666, "prompt token seed 7");

  /* ShardMap (test_transport.cpp:333-387): 1000 sequences over 4 workers */
  int32_t cnt[4] = {0, 0, 0, 0}, w = -1, a = 0, c = 0;
  for (uint64_t q = 1; q <= 1000; ++q) {
    OK(sd_shardmap_worker_for(SD_SHARD_BY_SEQUENCE, 8, 4, q, 0, &w));
    cnt[w] += 1;
  }
  CHECK(cnt[0] == 261 && cnt[1] == 241 && cnt[2] == 244 && cnt[3] == 254, "by-sequence counts %d %d %d %d", cnt[0],
        cnt[1], cnt[2], cnt[3]);
  OK(sd_shardmap_head_range(SD_SHARD_BY_HEAD, 8, 2, 1, &a, &c));
  CHECK(a == 4 && c == 4, "by-head 8/2 worker 1: [%d, +%d)", a, c);
  int32_t total = 0;
  for (int i = 0; i < 3; ++i) {
    OK(sd_shardmap_head_range(SD_SHARD_BY_HEAD, 7, 3, i, &a, &c));
    total += c;
    CHECK(c == (i == 0 ? 3 : 2), "by-head 7/3 worker %d count %d", i, c);
  }
  CHECK(total == 7, "by-head 7/3 covers every head");
  CHECK(sd_shardmap_head_range(SD_SHARD_BY_HEAD, 2, 4, 0, &a, &c) == SD_ERR_CONFIG, "more workers than heads");

  /* scheduler (scheduler.cpp:10-21): AdmissionError when B*F < S */
  int32_t mb = 0;
  OK(sd_micro_batch_size(1024, 16, 1024, &mb));
  CHECK(mb == 16, "micro_batch_size(1024, 16, 1024) = %d", mb);
  CHECK(sd_micro_batch_size(4, 2, 16, &mb) == SD_ERR_ADMISSION, "interval too short");
  CHECK(strstr(sd_last_error(), "interval too short") != NULL, "message: %s", sd_last_error());
  int64_t triples[3 * 64], n = 0;
  OK(sd_cold_start_schedule(6, 6, 2, 0, 12, triples, 64, &n));
  int64_t admitted = 0;
  for (int64_t i = 0; i < n; ++i) admitted += triples[3 * i + 1];
  CHECK(n > 0 && admitted >= 6, "cold start admits the batch (%lld rows in %lld admissions)", (long long)admitted,
        (long long)n);

  /* distributed row plan: every row has exactly one home; shard rows follow mix64 % world */
  uint64_t seqs[64];
  for (int i = 0; i < 64; ++i) seqs[i] = (uint64_t)i + 1;
  int32_t home[64], shard[64], nh = 0, ns = 0, sc[2], rc[2], homes = 0;
  for (int r = 0; r < 2; ++r) {
    OK(sd_dist_plan(2, r, 2, SD_SHARD_BY_SEQUENCE, 8, 64, seqs, home, &nh, shard, &ns, sc, rc));
    homes += nh;
    for (int i = 0; i < ns; ++i) CHECK((int)(sd_mix64(seqs[shard[i]]) % 2) == r, "shard row of rank %d", r);
  }
  CHECK(homes == 64, "homes cover the batch once (%d)", homes);

  /* planner (planner.cpp:48-222): a feasible plan on a toy profile */
  int32_t batch[3] = {1, 64, 1024};
  double secs[3] = {1e-3, 1.1e-3, 4e-3};
  sd_perf_profile prof = {batch, secs, 3, 1e-8, 100000000};
  sd_plan_request req;
  memset(&req, 0, sizeof(req));
  req.num_layers = 32;
  req.target_len = 1024;
  req.knee_threshold = 0.10;
  req.balance_tolerance = 0.15;
  sd_hardware_plan plan;
  const int prc = sd_plan(&prof, &req, &plan);
  CHECK(prc == SD_OK || prc == SD_ERR_INFEASIBLE, "sd_plan -> %d (%s)", prc, sd_last_error());
  CHECK(prc != SD_OK || (plan.batch_size >= 1 && plan.worker_count >= 1), "plan batch %d workers %d",
        plan.batch_size, plan.worker_count);

  /* typed errors on handles: a NULL KV store */
  int64_t tok = 0;
  CHECK(sd_kv_token_count(NULL, &tok) != SD_OK, "NULL handle rejected");
}

static int gpu_checks(const char* golden_path) {
  sd_model_spec s;
  OK(sd_make_model_spec(2, 64, 4, 256, 128, 0, &s));
  sd_weights* w = NULL;
  OK(sd_weights_seed_random(&s, 0, SD_DENSE_EXACT_F32, 0, &w));
  sd_kv* kv = NULL;
  OK(sd_kv_create(&s, 0, 4, 1 << 16, SD_KV_SINGLE, 0, NULL, &kv));
  sd_engine* e = NULL;
  OK(sd_engine_create(w, kv, &e));
  if (failures) return 1;

  /* drive_schedule (workers.cpp:547-684): batch 3, S = F = 20, 20 steps, seed 0 */
  sd_drive_config cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.batch = 3;
  cfg.target_len = 20;
  cfg.interval = 20;
  cfg.steps = 20;
  sd_drive_result* r = NULL;
  OK(sd_drive(e, &cfg, &r));
  char got[8192];
  size_t off = (size_t)snprintf(got, sizeof(got), "step,seq_id,token_id\n");
  for (int64_t i = 0; i < sd_drive_count(r); ++i) {
    int64_t st = 0;
    uint64_t q = 0;
    int32_t t = 0;
    OK(sd_drive_record(r, i, &st, &q, &t));
    off += (size_t)snprintf(got + off, sizeof(got) - off, "%lld,%llu,%d\n", (long long)st, (unsigned long long)q, t);
  }
  OK(sd_drive_destroy(r));
  FILE* f = fopen(golden_path, "rb");
  CHECK(f != NULL, "open %s", golden_path);
  if (f) {
    char want[8192];
    const size_t nw = fread(want, 1, sizeof(want) - 1, f);
    want[nw] = 0;
    fclose(f);
    CHECK(nw == off && memcmp(want, got, nw) == 0, "transcript differs from the golden fixture:\n%s", got);
  }

  /* one step through the features entry point (TokenBatch.features =
   * embedding columns, workers.cpp:629-638) against the token-id one */
  const int B = 3, D = s.model_dim;
  const uint64_t seqs_a[3] = {101, 102, 103}, seqs_b[3] = {201, 202, 203};
  const int32_t toks[3] = {5, 77, 127};
  float* emb = (float*)malloc(sizeof(float) * (size_t)D * s.vocab_size);
  float* x = (float*)malloc(sizeof(float) * (size_t)B * D);
  OK(sd_weights_export_embedding(w, emb, (size_t)D * s.vocab_size));
  for (int b = 0; b < B; ++b) memcpy(x + (size_t)b * D, emb + (size_t)toks[b] * D, sizeof(float) * (size_t)D);
  int32_t n1[3], n2[3];
  OK(sd_engine_step(e, B, seqs_a, toks, n1, NULL));
  OK(sd_engine_step_features(e, B, seqs_b, x, n2, NULL, NULL));
  CHECK(memcmp(n1, n2, sizeof(n1)) == 0, "features path tokens %d %d %d vs %d %d %d", n2[0], n2[1], n2[2], n1[0],
        n1[1], n1[2]);
  /* CapacityError / ConfigError come back as statuses, not crashes */
  const uint64_t dup[2] = {7, 7};
  CHECK(sd_engine_step(e, 2, dup, toks, n1, NULL) == SD_ERR_CONFIG, "duplicate sequence id");
  free(emb);
  free(x);
  OK(sd_engine_destroy(e));
  OK(sd_kv_destroy(kv));
  OK(sd_weights_destroy(w));
  return 0;
}

int main(int argc, char** argv) {
  CHECK(sd_abi_version() == SD_ABI_VERSION, "abi version");
  host_checks();
  if (argc > 2 && strcmp(argv[1], "gpu") == 0) gpu_checks(argv[2]);
  if (failures) {
    fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  printf("sd_abi_test ok (%s)\n", argc > 1 ? argv[1] : "host");
  return 0;
}
