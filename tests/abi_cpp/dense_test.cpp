// The reference's dense / drive tests (proj/tests/test_dense.cpp) restated
// against the C++ interface of include/sd_b200.hpp (exact fp32 S-Part): the
// same seeds, inputs and bitwise bars, run on a B200.
//   dense_test <golden_transcript_2x64_3seq_20.csv>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "sd_b200.hpp"

using namespace sd_b200;

namespace {

int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    ++g_checks;                                                   \
    if (!(cond)) {                                                \
      ++g_failed;                                                 \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

// random_matrix (test_dense.cpp:16-24): the mix64 chain fills Eigen's
// column-major storage; stored here row-major
Rows random_matrix(int rows, int cols, std::uint64_t salt) {
  Rows m(rows, cols);
  std::uint64_t state = salt;
  for (int i = 0; i < rows * cols; ++i) {
    state = mix64(state);
    m.row(i % rows)[i / rows] = 2.0f * (static_cast<float>(state >> 40) * 0x1p-24f) - 1.0f;
  }
  return m;
}
Rows one_row(const Rows& m, int r) {
  Rows o(1, m.cols);
  std::copy(m.row(r), m.row(r) + m.cols, o.row(0));
  return o;
}
bool same_row(const Rows& a, int ra, const Rows& b, int rb) {
  return a.cols == b.cols && std::equal(a.row(ra), a.row(ra) + a.cols, b.row(rb));
}

}  // namespace

int main(int argc, char** argv) {
  try {
    {  // "projection of one row is bitwise independent of the batch"
      const ModelSpec spec = make_model_spec(1, 32, 4, 32, 10);
      const WeightSet w(spec, 21);
      const Rows big = random_matrix(7, 32, 5);
      const QkvProjection pb = project_qkv(w, 0, big);
      const QkvProjection ps = project_qkv(w, 0, one_row(big, 2));
      CHECK(same_row(pb.q, 2, ps.q, 0));
      CHECK(same_row(pb.k, 2, ps.k, 0));
      CHECK(same_row(pb.v, 2, ps.v, 0));
    }
    {  // "argmax is invariant under positive rescaling of logits"
      const Rows l = random_matrix(1, 50, 91);
      std::vector<float> a(l.row(0), l.row(0) + 50), b = a, c = a;
      for (float& x : b) x *= 7.5f;
      for (float& x : c) x *= 0.001f;
      const int base = argmax_token(a);
      CHECK(argmax_token(b) == base);
      CHECK(argmax_token(c) == base);
    }
    {  // "monolithic decode step: batch of one equals the batched run bitwise"
      const ModelSpec spec = make_model_spec(2, 64, 4, 256, 128);
      WeightSet w(spec, 0);
      KvShard all_kv(spec, 0, spec.num_heads, 1 << 12), solo_kv(spec, 0, spec.num_heads, 1 << 12);
      StepComputation all(w, all_kv), solo(w, solo_kv);
      TokenBatch batch{{1, 2, 3}, Rows(3, 64)};
      for (int b = 0; b < 3; ++b) {
        const Vec e = w.embedding_column(b + 5);
        std::copy(e.begin(), e.end(), batch.features.row(b));
      }
      TokenBatch one{{2}, one_row(batch.features, 1)};
      for (int step = 0; step < 4; ++step) {
        const DecodeStepResult ra = all.compute(batch, step + 1);
        const DecodeStepResult ro = solo.compute(one, step + 1);
        CHECK(ra.next_tokens[1] == ro.next_tokens[0]);
        CHECK(same_row(ra.final_activations, 1, ro.final_activations, 0));
        for (int b = 0; b < 3; ++b) {
          const Vec e = w.embedding_column(ra.next_tokens[static_cast<std::size_t>(b)]);
          std::copy(e.begin(), e.end(), batch.features.row(b));
        }
        one.features = one_row(batch.features, 1);
      }
    }
    if (argc > 1) {  // "golden transcript fixture: 2 layers, 64 dim, 3 sequences, 20 steps"
      const ModelSpec spec = make_model_spec(2, 64, 4, 256, 128);
      WeightSet w(spec, 0);
      KvShard kv(spec, 0, spec.num_heads, 1 << 16);
      StepComputation comp(w, kv);
      GenerationConfig config;
      config.seed = 0;
      config.batch = 3;
      config.target_len = 20;
      config.interval = 20;
      config.steps = 20;
      std::ifstream f(argv[1]);
      std::stringstream ss;
      ss << f.rdbuf();
      CHECK(f.good() || !ss.str().empty());
      CHECK(transcript_csv(drive_schedule(config, comp)) == ss.str());
    }
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught: %s\n", e.what());
    return 1;
  }
  std::printf("dense: %d checks, %d failed\n", g_checks, g_failed);
  return g_failed == 0 ? 0 : 1;
}
