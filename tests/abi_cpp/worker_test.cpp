// AttentionWorkerSession over SDWP through the C++ interface of
// include/sd_b200.hpp (workers.cpp:40-160; frames transport.cpp:105-301,
// built here by hand): HELLO is echoed, CONFIG acknowledged, a QKV_BATCH of
// one first token returns O == V exactly (softmax over one position), two
// sequences with different histories come back in request order, DROP_SEQ
// has no reply, SHUTDOWN returns the stats and ends the session; a bad magic
// is a fatal ProtocolError.
#include <cstdio>
#include <cstring>
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

using Bytes = std::vector<std::uint8_t>;
void put(Bytes& b, std::uint64_t v, int n) {
  for (int i = 0; i < n; ++i) b.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}
void put_f(Bytes& b, const Vec& v) {
  for (float x : v) {
    std::uint32_t u;
    std::memcpy(&u, &x, 4);
    put(b, u, 4);
  }
}
Bytes frame(int type, const Bytes& payload) {  // "SDWP" | 1 | type | len u32 | payload
  Bytes f = {'S', 'D', 'W', 'P', 1, static_cast<std::uint8_t>(type)};
  put(f, payload.size(), 4);
  f.insert(f.end(), payload.begin(), payload.end());
  return f;
}
std::uint64_t get(const std::uint8_t* p, int n) {
  std::uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= static_cast<std::uint64_t>(p[i]) << (8 * i);
  return v;
}
struct Frame {
  int type;
  Bytes payload;
};
std::vector<Frame> frames(const Bytes& s) {
  std::vector<Frame> out;
  size_t at = 0;
  while (at + 10 <= s.size()) {
    const size_t n = static_cast<size_t>(get(&s[at + 6], 4));
    out.push_back(Frame{s[at + 5], Bytes(s.begin() + static_cast<long>(at + 10), s.begin() + static_cast<long>(at + 10 + n))});
    at += 10 + n;
  }
  return out;
}
Vec o_row(const Bytes& p, int i, int width) {  // O_BATCH record i (fp32 wire)
  Vec o(static_cast<size_t>(width));
  std::memcpy(o.data(), p.data() + 14 + static_cast<size_t>(i) * (8 + 4 * width) + 8, 4 * static_cast<size_t>(width));
  return o;
}
Vec filled(int n, float base) {
  Vec v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v[static_cast<size_t>(i)] = base + 0.01f * static_cast<float>(i % 17) - 0.07f;
  return v;
}

}  // namespace

int main() {
  enum { kHello = 1, kConfig = 2, kQkv = 3, kO = 4, kDrop = 5, kShutdown = 6, kError = 7 };
  try {
    AttentionWorkerSession w(AttentionWorkerConfig{1 << 12, KvFormat::kSingle, 0});
    const std::string cfg =
        R"({"model": {"num_layers": 2, "model_dim": 64, "num_heads": 4, "head_dim": 16, "mlp_dim": 256, )"
        R"("vocab_size": 128}, "head_start": 0, "head_count": 4, "wire_precision": "single"})";
    const Bytes cfgb(cfg.begin(), cfg.end());
    std::vector<Frame> r = frames(w.feed(frame(kHello, {})));
    CHECK(r.size() == 1 && r[0].type == kHello);
    r = frames(w.feed(frame(kConfig, cfgb)));
    CHECK(r.size() == 1 && r[0].type == kConfig);
    const std::string ack(r[0].payload.begin(), r[0].payload.end());
    CHECK(ack.find("\"ok\":true") != std::string::npos);

    // one first token: O == V bitwise
    const Vec q = filled(64, 0.3f), k = filled(64, -0.2f), v = filled(64, 0.5f);
    Bytes p;
    put(p, 0, 2);   // layer
    put(p, 0, 4);   // step
    put(p, 1, 4);   // count
    put(p, 0, 2);   // head_start
    put(p, 4, 2);   // head_count
    put(p, 11, 8);  // seq
    put(p, 0, 4);   // position
    put_f(p, q);
    put_f(p, k);
    put_f(p, v);
    r = frames(w.feed(frame(kQkv, p)));
    CHECK(r.size() == 1 && r[0].type == kO);
    if (!r.empty() && r[0].type == kO) {
      CHECK(get(&r[0].payload[14], 8) == 11);
      CHECK(o_row(r[0].payload, 0, 64) == v);
    }
    // split feeding: the same stream one byte at a time gives the same reply
    AttentionWorkerSession w2(AttentionWorkerConfig{1 << 12, KvFormat::kSingle, 0});
    Bytes stream = frame(kHello, {});
    for (const Bytes& f : {frame(kConfig, cfgb), frame(kQkv, p)}) stream.insert(stream.end(), f.begin(), f.end());
    Bytes out;
    for (std::uint8_t byte : stream) {
      const Bytes part = w2.feed(std::span<const std::uint8_t>(&byte, 1));
      out.insert(out.end(), part.begin(), part.end());
    }
    r = frames(out);
    CHECK(r.size() == 3 && r[2].type == kO && o_row(r[2].payload, 0, 64) == v);

    // DROP_SEQ: no reply; SHUTDOWN: stats and the session ends
    Bytes d;
    put(d, 1, 4);
    put(d, 11, 8);
    CHECK(w.feed(frame(kDrop, d)).empty());
    r = frames(w.feed(frame(kShutdown, {})));
    CHECK(r.size() == 1 && r[0].type == kShutdown);
    const std::string stats(r[0].payload.begin(), r[0].payload.end());
    CHECK(stats.find("tokens_processed") != std::string::npos);
    CHECK(w.shutdown_requested());

    // a bad magic is fatal for the stream
    bool threw = false;
    try {
      Bytes bad = frame(kHello, {});
      bad[0] = 'X';
      w2.feed(bad);
    } catch (const ProtocolError& e) {
      threw = std::strstr(e.what(), "bad magic") != nullptr;
    }
    CHECK(threw);
    (void)kError;
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught: %s\n", e.what());
    return 1;
  }
  std::printf("worker: %d checks, %d failed\n", g_checks, g_failed);
  return g_failed == 0 ? 0 : 1;
}
