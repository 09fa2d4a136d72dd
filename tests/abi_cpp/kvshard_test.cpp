// The reference's KvShard tests (proj/tests/test_attention.cpp) restated
// against sd_b200::KvShard (include/sd_b200.hpp): the same cases, inputs,
// bars and exception types, run on a B200 through the C ABI. `host` runs the
// cases that need no device.
//   g++ -std=c++20 -O2 -I include tests/abi_cpp/kvshard_test.cpp -L paper_2403_11421_b200 -lsd_b200
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "sd_b200.hpp"

using namespace sd_b200;

namespace {

int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_failed;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)
template <class E, class F>
bool throws_as(F&& f, const char* contains = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return !contains || std::strstr(e.what(), contains) != nullptr;
  } catch (...) {
    return false;
  }
  return false;
}

std::uint64_t g_state = 7;
float next_unit_signed() {  // test_attention.cpp:13-19
  g_state = mix64(g_state);
  return 2.0f * (static_cast<float>(g_state >> 40) * 0x1p-24f) - 1.0f;
}
Vec random_vec(int n) {
  Vec v(static_cast<std::size_t>(n));
  for (float& x : v) x = next_unit_signed();
  return v;
}

// brute-force attention, double accumulation (test_attention.cpp:27-58)
std::vector<double> attention_oracle(const Vec& q, const std::vector<Vec>& ks, const std::vector<Vec>& vs,
                                     int num_heads, int head_dim) {
  const int width = num_heads * head_dim;
  std::vector<double> out(static_cast<std::size_t>(width), 0.0);
  const double inv_sqrt = 1.0 / std::sqrt(static_cast<double>(head_dim));
  for (int h = 0; h < num_heads; ++h) {
    std::vector<double> scores(ks.size());
    for (std::size_t j = 0; j < ks.size(); ++j) {
      double dot = 0;
      for (int d = 0; d < head_dim; ++d) dot += double(q[h * head_dim + d]) * double(ks[j][h * head_dim + d]);
      scores[j] = dot * inv_sqrt;
    }
    double mx = scores[0];
    for (double s : scores) mx = std::max(mx, s);
    double denom = 0;
    for (double& s : scores) {
      s = std::exp(s - mx);
      denom += s;
    }
    for (std::size_t j = 0; j < ks.size(); ++j) {
      const double a = scores[j] / denom;
      for (int d = 0; d < head_dim; ++d) out[h * head_dim + d] += a * double(vs[j][h * head_dim + d]);
    }
  }
  return out;
}

double max_abs_diff(const Vec& a, const std::vector<double>& b) {
  double w = 0;
  for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::fabs(double(a[i]) - b[i]));
  return w;
}
double max_abs_diff(const Vec& a, const Vec& b) {
  double w = 0;
  for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::fabs(double(a[i]) - double(b[i])));
  return w;
}

AttentionRequest one_item(SequenceId seq, std::uint32_t pos, const Vec& q, const Vec& k, const Vec& v,
                          int layer = 0) {
  AttentionRequest req;
  req.layer = layer;
  req.items.push_back(AttentionItem{seq, pos, q, k, v});
  return req;
}
std::span<const float> sp(const Vec& v) { return std::span<const float>(v.data(), v.size()); }

void host_cases() {
  // make_model_spec validation (core.cpp:11-30)
  CHECK(throws_as<ConfigError>([] { make_model_spec(2, 63, 4, 256, 128); }, "not divisible"));
  CHECK(throws_as<ConfigError>([] { make_model_spec(0, 64, 4, 256, 128); }));
  const ModelSpec s = make_model_spec(2, 64, 4, 256, 128);
  CHECK(s.head_dim == 16 && s.num_kv_heads == 4);
  // a shard's head range and capacity are validated before any device work
  CHECK(throws_as<ConfigError>([&] { KvShard bad(s, 3, 2, 64); }, "head range"));
  CHECK(throws_as<ConfigError>([&] { KvShard bad(s, 0, 4, 0); }, "capacity"));
}

void gpu_cases() {
  {  // "attending over a single stored token returns V exactly"
    const ModelSpec spec = make_model_spec(1, 16, 2, 8, 8);
    KvShard shard(spec, 0, 2, 64);
    const Vec q = random_vec(16), k = random_vec(16), v = random_vec(16);
    AttentionRequest req = one_item(7, 0, q, k, v);
    shard.append_request(req);
    const AttentionResponse resp = shard.attend(req);
    CHECK(resp.outputs.size() == 1);
    CHECK(resp.outputs[0].o == v);  // softmax over one element is exactly 1
  }
  {  // "q orthogonal to equal-norm keys averages the values"
    const ModelSpec spec = make_model_spec(1, 4, 1, 8, 8);
    KvShard shard(spec, 0, 1, 64);
    Vec k1(4, 0.0f), k2(4, 0.0f), q(4, 0.0f);
    k1[0] = 1.0f;
    k2[1] = 1.0f;
    q[3] = 5.0f;
    const Vec v1 = random_vec(4), v2 = random_vec(4);
    shard.append_request(one_item(1, 0, q, k1, v1));
    shard.append_request(one_item(1, 1, q, k2, v2));
    const AttentionResponse resp = shard.attend(one_item(1, 1, q, k2, v2));
    Vec mean(4);
    for (int i = 0; i < 4; ++i) mean[i] = 0.5f * v1[i] + 0.5f * v2[i];
    CHECK(max_abs_diff(resp.outputs[0].o, mean) < 1e-6);
  }
  {  // "17-token sequence matches the brute-force oracle"
    const ModelSpec spec = make_model_spec(1, 24, 3, 8, 8);
    KvShard shard(spec, 0, 3, 64);
    std::vector<Vec> ks, vs;
    Vec q;
    for (std::uint32_t pos = 0; pos < 17; ++pos) {
      q = random_vec(24);
      ks.push_back(random_vec(24));
      vs.push_back(random_vec(24));
      shard.append_request(one_item(1, pos, q, ks.back(), vs.back()));
    }
    const AttentionResponse resp = shard.attend(one_item(1, 16, q, ks.back(), vs.back()));
    CHECK(max_abs_diff(resp.outputs[0].o, attention_oracle(q, ks, vs, 3, 8)) < 1e-5);
  }
  {  // "softmax weights are nonnegative and sum to one per head"
    const int len = 12;
    const ModelSpec spec = make_model_spec(1, len, 1, 8, 8);
    KvShard shard(spec, 0, 1, 64);
    Vec q;
    for (int pos = 0; pos < len; ++pos) {
      q = random_vec(len);
      Vec v(static_cast<std::size_t>(len), 0.0f);
      v[static_cast<std::size_t>(pos)] = 1.0f;
      shard.append_request(one_item(1, static_cast<std::uint32_t>(pos), q, random_vec(len), v));
    }
    const AttentionResponse resp =
        shard.attend(one_item(1, len - 1, q, Vec(static_cast<std::size_t>(len), 0.0f), Vec(static_cast<std::size_t>(len), 0.0f)));
    double sum = 0;
    for (float w : resp.outputs[0].o) {
      CHECK(w >= 0.0f);
      sum += w;
    }
    CHECK(std::fabs(sum - 1.0) < 1e-6);
  }
  {  // "incremental cache equals from-scratch recomputation" (50 trials)
    const ModelSpec spec = make_model_spec(1, 32, 4, 8, 8);
    double worst = 0;
    for (int trial = 0; trial < 50; ++trial) {
      KvShard shard(spec, 0, 4, 256);
      std::vector<Vec> ks, vs;
      const int len = 1 + static_cast<int>(mix64(static_cast<std::uint64_t>(trial)) % 64);
      for (int pos = 0; pos < len; ++pos) {
        const Vec q = random_vec(32);
        ks.push_back(random_vec(32));
        vs.push_back(random_vec(32));
        AttentionRequest req = one_item(1, static_cast<std::uint32_t>(pos), q, ks.back(), vs.back());
        shard.append_request(req);
        worst = std::max(worst, max_abs_diff(shard.attend(req).outputs[0].o, attention_oracle(q, ks, vs, 4, 8)));
      }
    }
    CHECK(worst < 1e-5);
  }
  // "half / int8 storage stays within 2e-3 / 5e-2 of single storage"; int4
  // (the extension) within 0.5
  for (auto [fmt, bar, salt] : {std::tuple{KvFormat::kHalf, 2e-3, 1000}, std::tuple{KvFormat::kInt8, 5e-2, 2000},
                                std::tuple{KvFormat::kInt4, 0.5, 3000}}) {
    const ModelSpec spec = make_model_spec(1, 32, 4, 8, 8);
    double worst = 0;
    for (int trial = 0; trial < 200; ++trial) {
      KvShard single(spec, 0, 4, 256, KvFormat::kSingle);
      KvShard other(spec, 0, 4, 256, fmt);
      const int len = 1 + static_cast<int>(mix64(static_cast<std::uint64_t>(salt + trial)) % 32);
      AttentionRequest last;
      for (int pos = 0; pos < len; ++pos) {
        last = one_item(1, static_cast<std::uint32_t>(pos), random_vec(32), random_vec(32), random_vec(32));
        single.append_request(last);
        other.append_request(last);
      }
      worst = std::max(worst, max_abs_diff(single.attend(last).outputs[0].o, other.attend(last).outputs[0].o));
    }
    CHECK(worst < bar);
  }
  {  // "append grows per-sequence arrays and enforces capacity"
    const ModelSpec spec = make_model_spec(2, 8, 2, 8, 8);
    KvShard shard(spec, 0, 2, 4);
    const Vec k = random_vec(8), v = random_vec(8);
    shard.append(1, 0, 0, sp(k), sp(v));
    CHECK(shard.stored_length(1, 0) == 1);
    shard.append(1, 1, 0, sp(k), sp(v));
    CHECK(shard.token_count() == 1);
    for (std::uint32_t pos = 1; pos < 4; ++pos)
      for (int layer = 0; layer < 2; ++layer) shard.append(1, layer, pos, sp(k), sp(v));
    CHECK(shard.stored_length(1, 0) == 4);
    CHECK(shard.token_count() == 4);
    CHECK(throws_as<CapacityError>([&] { shard.append(1, 0, 4, sp(k), sp(v)); }, "capacity exceeded"));
  }
  {  // "position bookkeeping rejects holes and stale ids"
    const ModelSpec spec = make_model_spec(1, 8, 2, 8, 8);
    KvShard shard(spec, 0, 2, 64);
    const Vec k = random_vec(8), v = random_vec(8);
    CHECK(throws_as<UnknownSequenceError>([&] { shard.append(9, 0, 3, sp(k), sp(v)); }));
    shard.append(9, 0, 0, sp(k), sp(v));
    CHECK(throws_as<ProtocolError>([&] { shard.append(9, 0, 2, sp(k), sp(v)); }));
    CHECK(throws_as<ProtocolError>([&] { shard.append(9, 1, 1, sp(k), sp(v)); }, "layer index out of range"));
    CHECK(throws_as<ProtocolError>([&] { shard.append(9, 0, 1, sp(Vec(7)), sp(v)); }, "width"));
  }
  {  // "batch append is atomic against capacity"
    const ModelSpec spec = make_model_spec(1, 8, 2, 8, 8);
    KvShard shard(spec, 0, 2, 2);
    AttentionRequest req;
    for (int i = 0; i < 3; ++i)
      req.items.push_back(AttentionItem{static_cast<SequenceId>(i + 1), 0, random_vec(8), random_vec(8), random_vec(8)});
    CHECK(throws_as<CapacityError>([&] { shard.append_request(req); }));
    CHECK(shard.token_count() == 0);
    CHECK(!shard.has_sequence(1));
  }
  {  // "drop removes accounting and is a counted no-op when repeated"
    const ModelSpec spec = make_model_spec(2, 8, 2, 8, 8);
    KvShard shard(spec, 0, 2, 16);
    const Vec k = random_vec(8), v = random_vec(8);
    for (std::uint32_t pos = 0; pos < 3; ++pos)
      for (int layer = 0; layer < 2; ++layer) shard.append(4, layer, pos, sp(k), sp(v));
    CHECK(shard.token_count() == 3);
    shard.drop_sequence(4);
    CHECK(shard.token_count() == 0);
    CHECK(!shard.has_sequence(4));
    CHECK(shard.warning_count() == 0);
    shard.drop_sequence(4);
    CHECK(shard.warning_count() == 1);
    AttentionRequest req = one_item(4, 3, random_vec(8), k, v);
    CHECK(throws_as<UnknownSequenceError>([&] { shard.attend(req); }));
  }
  {  // attend on a layer the sequence never reached: std::logic_error (attention.cpp:223-225)
    const ModelSpec spec = make_model_spec(2, 8, 2, 8, 8);
    KvShard shard(spec, 0, 2, 16);
    const Vec k = random_vec(8), v = random_vec(8);
    shard.append(5, 1, 0, sp(k), sp(v));
    CHECK(throws_as<std::logic_error>([&] { shard.attend(one_item(5, 0, k, k, v, 0)); }, "empty cache"));
  }
  {  // bytes_per_token (attention.cpp:296-305)
    const ModelSpec spec = make_model_spec(1, 32, 4, 8, 8);
    CHECK(KvShard(spec, 0, 4, 8, KvFormat::kSingle).bytes_per_token() == 2 * 32 * 4);
    CHECK(KvShard(spec, 0, 4, 8, KvFormat::kHalf).bytes_per_token() == 2 * 32 * 2);
    CHECK(KvShard(spec, 0, 4, 8, KvFormat::kInt8).bytes_per_token() == 2 * (32 + 4 * 4));
    CHECK(KvShard(spec, 0, 4, 8, KvFormat::kInt4).bytes_per_token() == 2 * (16 + 4 * 4));
  }
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  try {
    host_cases();
    if (mode == "gpu") gpu_cases();
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught: %s\n", e.what());
    return 1;
  }
  std::printf("%s: %d checks, %d failed\n", mode.c_str(), g_checks, g_failed);
  return g_failed == 0 ? 0 : 1;
}
