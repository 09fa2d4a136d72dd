// ============================================================================
// sd_oracle.cpp — CPU ORACLE (test infrastructure only; never the product).
//
// A plain-C++ (Eigen-free) restatement of the reference `splitdecode` decode
// hot path (FastDecode, arXiv 2403.11421), used ONLY by tests/, by
// __graft_entry__.smoke() as a checker, and by bench.py's cpu_baseline /
// --impl reference legs.  Nothing in the product path links or calls this.
//
// Build: g++ -O2 -std=c++20 -ffp-contract=off (the reference's flags,
//        proj/CMakeLists.txt:9-13), no -march, so scalar float arithmetic
//        rounds exactly like the reference's SSE2 build.
//
// Parity pinning (see tests/test_oracle_golden.py):
//   * weight_checksum == 0x138062486c631272 (proj/tests/test_core.cpp:55-63)
//   * golden transcript 2x64, 3 seq, 20 steps, byte-exact
//     (proj/tests/fixtures/golden_transcript_2x64_3seq_20.csv,
//      proj/tests/test_dense.cpp:173-190)
//   * int8 / fp16 known answers (proj/tests/test_attention.cpp:286-344)
//   * ShardMap cases (proj/tests/test_transport.cpp:333-387)
//   * scheduler worked examples (proj/tests/test_scheduler.cpp)
//
// Extension (NOT in the reference, parity unpinned): grouped-query attention
// via ModelSpec.num_kv_heads (query head h reads kv head h / (H / Hkv)).
// With num_kv_heads == num_heads every function is the reference's.
// Extension (NOT in the reference, parity unpinned): int4 KV storage, the
// paper's 4-bit quantization hook, following
// quantize_int8's rules with a +-7 range (quantize_int4 below).
//
// Layout at this C ABI: activations are row-major [rows][width]; weights
// keep the reference's Eigen column-major (out x in) storage, i.e. element
// w(j, k) lives at w[k * out + j] (proj/include/splitdecode/core.hpp:79-90).
// The per-element operation sequence — the only thing that decides the
// bits — is the reference's, so the memory layout of activations is free.
// ============================================================================

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors ---
// error codes match the C-ABI numbering of include/sd_abi.h
enum Err : int {
  kOk = 0,
  kProtocol = 3,      // ProtocolError        (transport.hpp:39-44 code 3)
  kCapacity = 4,      // CapacityError        (code 4)
  kUnknownSeq = 5,    // UnknownSequenceError (code 5)
  kInternal = 6,
  kLogic = 7,         // std::logic_error
  kConfig = 8,        // ConfigError
  kAdmission = 11,    // AdmissionError (scheduler.hpp:20-23)
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kInternal;
  }
}

// ------------------------------------------------------------ core types ---
struct Spec {  // core.hpp:43-50 (+ num_kv_heads extension)
  int num_layers, model_dim, num_heads, head_dim, mlp_dim, vocab_size,
      num_kv_heads;
};

// make_model_spec (core.cpp:11-30)
Spec make_spec(int L, int D, int H, int F, int V, int Hkv) {
  if (L < 1 || D < 1 || H < 1 || F < 1 || V < 1) {
    throw Error(kConfig, "model spec fields must all be >= 1");
  }
  if (D % H != 0) {
    throw Error(kConfig, "model_dim not divisible by heads (model_dim=" +
                             std::to_string(D) + ", num_heads=" +
                             std::to_string(H) + ")");
  }
  if (Hkv == 0) Hkv = H;
  if (Hkv < 1 || H % Hkv != 0) {
    throw Error(kConfig, "num_heads not divisible by num_kv_heads");
  }
  return Spec{L, D, H, D / H, F, V, Hkv};
}

// column-major out x in matrix, as Eigen::MatrixXf (core.hpp:79-90)
struct Mat {
  int rows = 0, cols = 0;
  std::vector<float> data;
  void resize(int r, int c) {
    rows = r;
    cols = c;
    data.assign(static_cast<size_t>(r) * c, 0.0f);
  }
  float at(int r, int c) const { return data[static_cast<size_t>(c) * rows + r]; }
};

struct Layer {
  Mat w_q, w_k, w_v, w_o, w_mlp_in, w_mlp_out;
};

struct Weights {
  Spec spec;
  Mat embedding;  // D x V, one column per token
  std::vector<Layer> layers;
  Mat head;  // V x D
};

// UniformSource (core.cpp:72-93): mt19937 seeded uint32(seed ^ seed>>32),
// u = (gen() >> 8) * 2^-24, value (2u - 1) * scale, memory order fill.
struct Uniform {
  std::mt19937 gen;
  explicit Uniform(uint64_t seed)
      : gen(static_cast<uint32_t>(seed ^ (seed >> 32))) {}
  float unit() { return static_cast<float>(gen() >> 8) * 0x1p-24f; }
  float signed_(float scale) { return (2.0f * unit() - 1.0f) * scale; }
  void fill(Mat& m, float scale) {
    for (float& x : m.data) x = signed_(scale);
  }
};

// seed_random_weights (core.cpp:97-127)
Weights seed_weights(const Spec& s, uint64_t seed) {
  Weights w;
  w.spec = s;
  Uniform src(seed);
  const float d_scale = 1.0f / std::sqrt(static_cast<float>(s.model_dim));
  const float m_scale = 1.0f / std::sqrt(static_cast<float>(s.mlp_dim));
  const int kvw = s.num_kv_heads * s.head_dim;
  w.embedding.resize(s.model_dim, s.vocab_size);
  src.fill(w.embedding, 1.0f);
  w.layers.resize(s.num_layers);
  for (Layer& l : w.layers) {
    l.w_q.resize(s.model_dim, s.model_dim);
    l.w_k.resize(kvw, s.model_dim);
    l.w_v.resize(kvw, s.model_dim);
    l.w_o.resize(s.model_dim, s.model_dim);
    l.w_mlp_in.resize(s.mlp_dim, s.model_dim);
    l.w_mlp_out.resize(s.model_dim, s.mlp_dim);
    src.fill(l.w_q, d_scale);
    src.fill(l.w_k, d_scale);
    src.fill(l.w_v, d_scale);
    src.fill(l.w_o, d_scale);
    src.fill(l.w_mlp_in, d_scale);
    src.fill(l.w_mlp_out, m_scale);
  }
  w.head.resize(s.vocab_size, s.model_dim);
  src.fill(w.head, d_scale);
  return w;
}

// weight_checksum: FNV-1a over raw float bytes (core.cpp:129-155)
void hash_mat(uint64_t& h, const Mat& m) {
  const auto* b = reinterpret_cast<const unsigned char*>(m.data.data());
  const size_t n = m.data.size() * sizeof(float);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
}
uint64_t checksum(const Weights& w) {
  uint64_t h = 0xcbf29ce484222325ull;
  hash_mat(h, w.embedding);
  for (const Layer& l : w.layers) {
    hash_mat(h, l.w_q);
    hash_mat(h, l.w_k);
    hash_mat(h, l.w_v);
    hash_mat(h, l.w_o);
    hash_mat(h, l.w_mlp_in);
    hash_mat(h, l.w_mlp_out);
  }
  hash_mat(h, w.head);
  return h;
}

// mix64 = SplitMix64 finalizer (core.cpp:161-166)
uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// prompt_token (core.cpp:168-171)
int prompt_token(uint64_t seed, uint64_t id, int vocab) {
  return static_cast<int>(mix64(seed ^ mix64(id)) % static_cast<uint64_t>(vocab));
}

// ---------------------------------------------------------------- codecs ---
// float_to_half_bits: IEEE binary16 round-to-nearest-even, the conversion
// Eigen::half(float) performs (attention.cpp:54-56).
uint16_t f2h(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) {  // inf / nan
    return static_cast<uint16_t>(sign | (ax > 0x7f800000u ? 0x7e00u : 0x7c00u));
  }
  if (ax >= 0x477ff000u) return static_cast<uint16_t>(sign | 0x7c00u);  // overflow
  if (ax < 0x38800000u) {  // subnormal half (or zero)
    // value = ax as float; half subnormal unit is 2^-24
    float a;
    std::memcpy(&a, &ax, 4);
    // exact: a * 2^24 then round-to-nearest-even to integer
    const float scaled = a * 0x1p24f;  // exact (power of two scale)
    const float r = std::nearbyint(scaled);
    return static_cast<uint16_t>(sign | static_cast<uint32_t>(r));
  }
  // normal: rebias exponent, round mantissa 23 -> 10 bits, RNE
  uint32_t mant_odd = (ax >> 13) & 1u;
  ax += 0xc8000fffu + mant_odd;  // (15-127)<<23 + rounding bias
  return static_cast<uint16_t>(sign | (ax >> 13));
}

float h2f(uint16_t h) {
  const uint32_t sign = (static_cast<uint32_t>(h) & 0x8000u) << 16;
  const uint32_t exp = (h >> 10) & 0x1fu;
  const uint32_t man = h & 0x3ffu;
  uint32_t bits;
  if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else {  // subnormal: man * 2^-24, exact in float
      float v = static_cast<float>(man) * 0x1p-24f;
      std::memcpy(&bits, &v, 4);
      bits |= sign;
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | (man << 13);
  } else {
    bits = sign | ((exp + 112u) << 23) | (man << 13);
  }
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

// quantize_int8 (attention.cpp:28-46)
float quantize_int8(const float* x, int n, int8_t* q) {
  float max_abs = 0.0f;
  for (int i = 0; i < n; ++i) max_abs = std::max(max_abs, std::fabs(x[i]));
  if (max_abs == 0.0f) {
    for (int i = 0; i < n; ++i) q[i] = 0;
    return 0.0f;
  }
  const float scale = max_abs / 127.0f;
  const double inv = 1.0 / static_cast<double>(scale);
  for (int i = 0; i < n; ++i) {
    double r = std::nearbyint(static_cast<double>(x[i]) * inv);
    r = std::clamp(r, -127.0, 127.0);
    q[i] = static_cast<int8_t>(r);
  }
  return scale;
}

// quantize_int4: the paper's quantization hook ("suppose
// that 4-bit integers are used to store K and V") in the shape of
// quantize_int8 — per-(position, head) scale max|x| / 7, round half to even,
// clamp to +-7 — stored two per byte, element 2i in the low nibble of byte
// i (two's complement). The reference has no 4-bit format: this extension is
// pinned to its int8 codec's rules, not to reference vectors.
float quantize_int4(const float* x, int n, uint8_t* packed) {
  float max_abs = 0.0f;
  for (int i = 0; i < n; ++i) max_abs = std::max(max_abs, std::fabs(x[i]));
  for (int i = 0; i < (n + 1) / 2; ++i) packed[i] = 0;
  if (max_abs == 0.0f) return 0.0f;
  const float scale = max_abs / 7.0f;
  const double inv = 1.0 / static_cast<double>(scale);
  for (int i = 0; i < n; ++i) {
    double r = std::nearbyint(static_cast<double>(x[i]) * inv);
    r = std::clamp(r, -7.0, 7.0);
    const uint8_t nib = static_cast<uint8_t>(static_cast<int>(r) & 0xF);
    packed[i / 2] = static_cast<uint8_t>(packed[i / 2] | (i & 1 ? nib << 4 : nib));
  }
  return scale;
}
int int4_at(const uint8_t* packed, int i) {
  const int nib = (packed[i / 2] >> (i & 1 ? 4 : 0)) & 0xF;
  return nib >= 8 ? nib - 16 : nib;
}

// ---------------------------------------------------------- dot products ---
// Eigen 3.x `a.dot(b)` for dynamic float vectors on an SSE2 build: linear
// vectorized redux with alignedStart 0 (the product expression has no
// direct access), two 4-lane packet accumulators over 8-element blocks, one
// optional trailing packet, predux (l0+l2)+(l1+l3), then a scalar tail.
// Used at attention.cpp:243/249 (qh.dot(kj)).
float eigen_dot(const float* a, const float* b, int n) {
  const int P = 4;
  const int aligned = (n / P) * P;
  const int aligned2 = (n / (2 * P)) * (2 * P);
  float res;
  if (aligned) {
    float r0[4], r1[4];
    for (int l = 0; l < 4; ++l) r0[l] = a[l] * b[l];
    if (aligned > P) {
      for (int l = 0; l < 4; ++l) r1[l] = a[P + l] * b[P + l];
      for (int i = 2 * P; i < aligned2; i += 2 * P) {
        for (int l = 0; l < 4; ++l) {
          r0[l] = r0[l] + a[i + l] * b[i + l];
          r1[l] = r1[l] + a[i + P + l] * b[i + P + l];
        }
      }
      for (int l = 0; l < 4; ++l) r0[l] = r0[l] + r1[l];
      if (aligned > aligned2) {
        for (int l = 0; l < 4; ++l) r0[l] = r0[l] + a[aligned2 + l] * b[aligned2 + l];
      }
    }
    res = (r0[0] + r0[2]) + (r0[1] + r0[3]);
    for (int i = aligned; i < n; ++i) res = res + a[i] * b[i];
  } else {
    res = a[0] * b[0];
    for (int i = 1; i < n; ++i) res = res + a[i] * b[i];
  }
  return res;
}

// ---------------------------------------------------------------- KvShard ---
enum Fmt : int { kSingle = 0, kHalf = 1, kInt8 = 2, kInt4 = 3 };

// KvShard (attention.hpp:68-140; attention.cpp:62-305). head_start /
// head_count index the shard's kv heads; the q width is derived from them.
class KvShard {
 public:
  KvShard(const Spec& s, int head_start, int head_count, long cap, int fmt)
      : s_(s), h0_(head_start), hc_(head_count), cap_(cap), fmt_(fmt) {
    // attention.cpp:66-72 (kv-head range under the GQA extension)
    if (head_start < 0 || head_count < 1 ||
        head_start + head_count > s.num_kv_heads) {
      throw Error(kConfig, "shard head range outside the model's heads");
    }
    if (cap < 1) throw Error(kConfig, "shard capacity must be >= 1");
    if (fmt < 0 || fmt > 3) throw Error(kConfig, "unknown kv storage format");
    if (fmt == kInt4 && s.head_dim % 2) throw Error(kConfig, "int4 kv storage needs an even head_dim");
  }
  int width() const { return hc_ * s_.head_dim; }  // kv width
  int head_start() const { return h0_; }
  const Spec& spec() const { return s_; }
  int group() const { return s_.num_heads / s_.num_kv_heads; }
  int q_width() const { return width() * group(); }
  long token_count() const { return total_ / s_.num_layers; }
  int warnings() const { return warn_; }
  bool has(uint64_t seq) const { return map_.count(seq) != 0; }
  int stored(uint64_t seq, int layer) const {
    const SeqLayer* sl = find(seq, layer);
    return sl ? sl->k.positions : 0;
  }
  size_t bytes_per_token() const {  // attention.cpp:296-305
    const size_t w = static_cast<size_t>(width());
    switch (fmt_) {
      case kSingle: return 2 * w * sizeof(float);
      case kHalf: return 2 * w * sizeof(uint16_t);
      case kInt4: return 2 * (w / 2 + static_cast<size_t>(hc_) * sizeof(float));
      default: return 2 * (w + static_cast<size_t>(hc_) * sizeof(float));
    }
  }

  // append (attention.cpp:139-170)
  void append(uint64_t seq, int layer, uint32_t pos, const float* k, const float* v) {
    if (layer < 0 || layer >= s_.num_layers) {
      throw Error(kProtocol, "append: layer index out of range");
    }
    if (total_ + 1 > cap_ * s_.num_layers) {
      throw Error(kCapacity, "capacity exceeded: shard holds " +
                                 std::to_string(token_count()) + " of " +
                                 std::to_string(cap_) + " tokens");
    }
    auto it = map_.find(seq);
    if (it == map_.end()) {
      if (pos != 0) {
        throw Error(kUnknownSeq, "unknown sequence " + std::to_string(seq) +
                                     " (non-zero position without prior tokens)");
      }
      it = map_.emplace(seq, std::vector<SeqLayer>(s_.num_layers)).first;
    }
    SeqLayer& sl = it->second[static_cast<size_t>(layer)];
    if (static_cast<uint32_t>(sl.k.positions) != pos) {
      throw Error(kProtocol, "append: position " + std::to_string(pos) +
                                 " does not match stored length " +
                                 std::to_string(sl.k.positions));
    }
    append_lane(sl.k, k);
    append_lane(sl.v, v);
    total_ += 1;
  }

  // append_request: all-or-nothing validation then sequential appends
  // (attention.cpp:172-202)
  void append_request(int layer, int n, const uint64_t* seqs, const uint32_t* pos,
                      const float* k, const float* v) {
    if (total_ + static_cast<long>(n) > cap_ * s_.num_layers) {
      throw Error(kCapacity, "capacity exceeded: batch of " + std::to_string(n) +
                                 " does not fit (shard at " +
                                 std::to_string(token_count()) + "/" +
                                 std::to_string(cap_) + " tokens)");
    }
    if (layer < 0 || layer >= s_.num_layers) {
      throw Error(kProtocol, "append: layer index out of range");
    }
    for (int i = 0; i < n; ++i) {
      const SeqLayer* sl = find(seqs[i], layer);
      const uint32_t st = sl ? static_cast<uint32_t>(sl->k.positions) : 0;
      if (!sl && pos[i] != 0) {
        throw Error(kUnknownSeq, "unknown sequence " + std::to_string(seqs[i]));
      }
      if (pos[i] != st) {
        throw Error(kProtocol, "append: position mismatch for sequence " +
                                   std::to_string(seqs[i]));
      }
    }
    const size_t w = static_cast<size_t>(width());
    for (int i = 0; i < n; ++i) append(seqs[i], layer, pos[i], k + i * w, v + i * w);
  }

  // attend (attention.cpp:204-282). q/o rows are q_width wide.
  void attend(int layer, int n, const uint64_t* seqs, const float* q, float* o) const {
    const int hd = s_.head_dim;
    const float inv_sqrt_d = 1.0f / std::sqrt(static_cast<float>(hd));
    const int G = group();
    const int qw = q_width();
    std::vector<float> row(static_cast<size_t>(hd));
    std::vector<float> scores;
    if (layer < 0 || layer >= s_.num_layers) {
      throw Error(kProtocol, "attend: layer index out of range");
    }
    for (int i = 0; i < n; ++i) {
      const SeqLayer* sl = find(seqs[i], layer);
      if (!sl) {
        throw Error(kUnknownSeq, "attend: unknown sequence " + std::to_string(seqs[i]));
      }
      const int len = sl->k.positions;
      if (len < 1) throw Error(kLogic, "attend: sequence has an empty cache");
      const float* qi = q + static_cast<size_t>(i) * qw;
      float* oi = o + static_cast<size_t>(i) * qw;
      std::fill(oi, oi + qw, 0.0f);
      scores.resize(static_cast<size_t>(len));
      for (int h = 0; h < hc_ * G; ++h) {  // local q head
        const int kh = h / G;               // local kv head
        const float* qh = qi + static_cast<size_t>(h) * hd;
        for (int j = 0; j < len; ++j) {
          const float* kj = decode(sl->k, j, kh, row.data());
          scores[j] = eigen_dot(qh, kj, hd) * inv_sqrt_d;
        }
        float mx = scores[0];
        for (int j = 1; j < len; ++j) mx = std::max(mx, scores[j]);
        float denom = 0.0f;
        for (int j = 0; j < len; ++j) {
          scores[j] = std::exp(scores[j] - mx);
          denom += scores[j];
        }
        const float inv_denom = 1.0f / denom;
        float* oh = oi + static_cast<size_t>(h) * hd;
        for (int j = 0; j < len; ++j) {
          const float* vj = decode(sl->v, j, kh, row.data());
          const float p = scores[j] * inv_denom;
          for (int d = 0; d < hd; ++d) oh[d] = oh[d] + p * vj[d];
        }
      }
    }
  }

  // drop_sequence (attention.cpp:284-294)
  void drop(uint64_t seq) {
    auto it = map_.find(seq);
    if (it == map_.end()) {
      warn_ += 1;
      return;
    }
    long removed = 0;
    for (const SeqLayer& sl : it->second) removed += sl.k.positions;
    total_ -= removed;
    map_.erase(it);
  }

  // raw storage bytes of one lane in the reference order [pos][head][d]
  // (attention.cpp:117-118) plus int8 scales [pos][head] (:129-130)
  size_t export_lane(uint64_t seq, int layer, int kv, void* out, size_t cap,
                     float* scales, size_t scap) const {
    const SeqLayer* sl = find(seq, layer);
    if (!sl) throw Error(kUnknownSeq, "export: unknown sequence");
    const Lane& ln = kv ? sl->v : sl->k;
    size_t bytes = 0;
    const void* src = nullptr;
    switch (fmt_) {
      case kSingle: bytes = ln.f32.size() * 4; src = ln.f32.data(); break;
      case kHalf: bytes = ln.f16.size() * 2; src = ln.f16.data(); break;
      case kInt4: bytes = ln.i4.size(); src = ln.i4.data(); break;
      default: bytes = ln.i8.size(); src = ln.i8.data(); break;
    }
    if (out && bytes <= cap && bytes) std::memcpy(out, src, bytes);
    if (scales && (fmt_ == kInt8 || fmt_ == kInt4) && ln.i8s.size() <= scap && !ln.i8s.empty()) {
      std::memcpy(scales, ln.i8s.data(), ln.i8s.size() * 4);
    }
    return bytes;
  }

 private:
  struct Lane {
    std::vector<float> f32;
    std::vector<uint16_t> f16;
    std::vector<int8_t> i8;
    std::vector<uint8_t> i4;  // int4: [pos][head][hd / 2] packed nibbles
    std::vector<float> i8s;   // int8 / int4 scales [pos][head]
    int positions = 0;
  };
  struct SeqLayer {
    Lane k, v;
  };
  const SeqLayer* find(uint64_t seq, int layer) const {
    auto it = map_.find(seq);
    if (it == map_.end()) return nullptr;
    if (layer < 0 || layer >= s_.num_layers) return nullptr;
    return &it->second[static_cast<size_t>(layer)];
  }
  // append_lane (attention.cpp:91-112)
  void append_lane(Lane& ln, const float* x) {
    const int w = width();
    switch (fmt_) {
      case kSingle: ln.f32.insert(ln.f32.end(), x, x + w); break;
      case kHalf:
        for (int i = 0; i < w; ++i) ln.f16.push_back(f2h(x[i]));
        break;
      case kInt4: {
        const int hd = s_.head_dim;
        std::vector<uint8_t> q(static_cast<size_t>(hd / 2));
        for (int h = 0; h < hc_; ++h) {
          const float sc = quantize_int4(x + h * hd, hd, q.data());
          ln.i4.insert(ln.i4.end(), q.begin(), q.end());
          ln.i8s.push_back(sc);
        }
        break;
      }
      default: {
        const int hd = s_.head_dim;
        std::vector<int8_t> q(static_cast<size_t>(hd));
        for (int h = 0; h < hc_; ++h) {
          const float sc = quantize_int8(x + h * hd, hd, q.data());
          ln.i8.insert(ln.i8.end(), q.begin(), q.end());
          ln.i8s.push_back(sc);
        }
      }
    }
    ln.positions += 1;
  }
  // decode_position_head (attention.cpp:114-137); fp32 returns in place
  const float* decode(const Lane& ln, int pos, int head, float* out) const {
    const int hd = s_.head_dim;
    const size_t off = static_cast<size_t>(pos) * width() + static_cast<size_t>(head) * hd;
    switch (fmt_) {
      case kSingle: return ln.f32.data() + off;
      case kHalf:
        for (int i = 0; i < hd; ++i) out[i] = h2f(ln.f16[off + i]);
        return out;
      case kInt4: {
        const float sc = ln.i8s[static_cast<size_t>(pos) * hc_ + head];
        const uint8_t* row = ln.i4.data() + off / 2;
        for (int i = 0; i < hd; ++i) out[i] = static_cast<float>(int4_at(row, i)) * sc;
        return out;
      }
      default: {
        const float sc = ln.i8s[static_cast<size_t>(pos) * hc_ + head];
        for (int i = 0; i < hd; ++i) out[i] = static_cast<float>(ln.i8[off + i]) * sc;
        return out;
      }
    }
  }

  Spec s_;
  int h0_, hc_;
  long cap_;
  int fmt_;
  long total_ = 0;
  int warn_ = 0;
  std::unordered_map<uint64_t, std::vector<SeqLayer>> map_;
};

// ----------------------------------------------------------------- dense ---
// apply_linear (dense.cpp:16-31): out(b, j) = sum_k w(j, k) * x(b, k), k
// ascending, one accumulator, multiply then add. Rows of x are row-major
// [B][in]; w is column-major out x in. Columns [j0, j1) only (threads split
// the output columns; per-element arithmetic is unchanged).
void apply_linear_cols(int B, int in, int out, const float* x, const float* w,
                       float* y, int j0, int j1) {
  for (int b = 0; b < B; ++b) {
    const float* xb = x + static_cast<size_t>(b) * in;
    float* yb = y + static_cast<size_t>(b) * out;
    for (int j = j0; j < j1; ++j) {
      float acc = 0.0f;
      for (int k = 0; k < in; ++k) acc = acc + w[static_cast<size_t>(k) * out + j] * xb[k];
      yb[j] = acc;
    }
  }
}

void apply_linear(int B, int in, int out, const float* x, const float* w, float* y,
                  int threads = 1) {
  if (threads <= 1 || out < 64) {
    apply_linear_cols(B, in, out, x, w, y, 0, out);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) {
    const int j0 = static_cast<int>(static_cast<long>(out) * t / threads);
    const int j1 = static_cast<int>(static_cast<long>(out) * (t + 1) / threads);
    ts.emplace_back(apply_linear_cols, B, in, out, x, w, y, j0, j1);
  }
  for (auto& t : ts) t.join();
}

void linear(const Mat& w, int B, const float* x, float* y, int threads = 1) {
  apply_linear(B, w.cols, w.rows, x, w.data.data(), y, threads);
}

// project_qkv (dense.cpp:33-43)
void project_qkv(const Weights& W, int layer, int B, const uint64_t* seqs,
                 const float* x, float* q, float* k, float* v, int threads = 1) {
  if (B == 0) throw Error(kConfig, "project_qkv: empty batch");
  std::unordered_set<uint64_t> seen;  // validate_batch (core.cpp:37-54)
  for (int b = 0; b < B; ++b) {
    if (!seen.insert(seqs[b]).second) {
      throw Error(kConfig, "token batch: duplicate sequence id " + std::to_string(seqs[b]));
    }
  }
  if (layer < 0 || layer >= W.spec.num_layers) throw Error(kConfig, "layer out of range");
  const Layer& l = W.layers[static_cast<size_t>(layer)];
  linear(l.w_q, B, x, q, threads);
  linear(l.w_k, B, x, k, threads);
  linear(l.w_v, B, x, v, threads);
}

float silu(float v) { return v / (1.0f + std::exp(-v)); }  // dense.cpp:47-49

// finish_block (dense.cpp:51-70)
void finish_block(const Weights& W, int layer, int B, const float* o,
                  const float* res, float* xout, int threads = 1) {
  if (layer < 0 || layer >= W.spec.num_layers) throw Error(kConfig, "layer out of range");
  const Layer& l = W.layers[static_cast<size_t>(layer)];
  const int D = W.spec.model_dim, F = W.spec.mlp_dim;
  std::vector<float> y(static_cast<size_t>(B) * D), hid(static_cast<size_t>(B) * F),
      mo(static_cast<size_t>(B) * D);
  linear(l.w_o, B, o, y.data(), threads);
  for (size_t i = 0; i < y.size(); ++i) y[i] = y[i] + res[i];
  linear(l.w_mlp_in, B, y.data(), hid.data(), threads);
  for (float& h : hid) h = silu(h);
  linear(l.w_mlp_out, B, hid.data(), mo.data(), threads);
  for (size_t i = 0; i < y.size(); ++i) xout[i] = y[i] + mo[i];
}

// argmax_token: first index wins ties (dense.cpp:78-88)
int argmax(const float* logits, int n) {
  int best = 0;
  float bv = logits[0];
  for (int i = 1; i < n; ++i) {
    if (logits[i] > bv) {
      bv = logits[i];
      best = i;
    }
  }
  return best;
}

// decode_step_monolithic (dense.cpp:90-129)
void decode_step(const Weights& W, KvShard& kv, int B, const uint64_t* seqs,
                 const float* x_in, int* tokens, float* final_x, float* logits_out,
                 int threads = 1) {
  const Spec& s = W.spec;
  const int D = s.model_dim, kvw = s.num_kv_heads * s.head_dim;
  std::vector<float> x(x_in, x_in + static_cast<size_t>(B) * D);
  std::vector<float> q(static_cast<size_t>(B) * D), k(static_cast<size_t>(B) * kvw),
      v(static_cast<size_t>(B) * kvw), o(static_cast<size_t>(B) * D),
      nx(static_cast<size_t>(B) * D);
  std::vector<uint32_t> pos(static_cast<size_t>(B));
  for (int layer = 0; layer < s.num_layers; ++layer) {
    project_qkv(W, layer, B, seqs, x.data(), q.data(), k.data(), v.data(), threads);
    for (int b = 0; b < B; ++b) pos[b] = static_cast<uint32_t>(kv.stored(seqs[b], layer));
    kv.append_request(layer, B, seqs, pos.data(), k.data(), v.data());
    kv.attend(layer, B, seqs, q.data(), o.data());
    finish_block(W, layer, B, o.data(), x.data(), nx.data(), threads);
    x.swap(nx);
  }
  if (final_x) std::copy(x.begin(), x.end(), final_x);
  std::vector<float> lg(static_cast<size_t>(B) * s.vocab_size);
  linear(W.head, B, x.data(), lg.data(), threads);
  for (int b = 0; b < B; ++b) tokens[b] = argmax(lg.data() + static_cast<size_t>(b) * s.vocab_size, s.vocab_size);
  if (logits_out) std::copy(lg.begin(), lg.end(), logits_out);
}

// -------------------------------------------------------------- ShardMap ---
// transport.cpp:319-380
std::pair<int, int> range_of(int index, int groups, int total) {
  const int base = total / groups, rem = total % groups;
  return {index * base + std::min(index, rem), base + (index < rem ? 1 : 0)};
}
int group_of_head(int head, int groups, int total) {
  for (int g = 0; g < groups; ++g) {
    auto [st, c] = range_of(g, groups, total);
    if (head >= st && head < st + c) return g;
  }
  throw Error(kConfig, "head index out of range");
}
struct ShardMap {
  int mode, heads, workers, head_groups;
  ShardMap(int m, int h, int w) : mode(m), heads(h), workers(w) {
    if (w < 1) throw Error(kConfig, "shard map needs at least one worker");
    if (h < 1) throw Error(kConfig, "shard map needs at least one head");
    if (m < 0 || m > 2) throw Error(kConfig, "invalid shard mode");
    if (m == 1 && w > h) throw Error(kConfig, "by-head sharding cannot use more workers than heads");
    head_groups = m == 2 ? std::gcd(w, h) : 1;
  }
  int worker_for(uint64_t seq, int head) const {
    if (head < 0 || head >= heads) throw Error(kConfig, "head index out of range");
    switch (mode) {
      case 0: return static_cast<int>(mix64(seq) % static_cast<uint64_t>(workers));
      case 1: return group_of_head(head, workers, heads);
      default: {
        const int sg_n = workers / head_groups;
        const int hg = group_of_head(head, head_groups, heads);
        const int sg = static_cast<int>(mix64(seq) % static_cast<uint64_t>(sg_n));
        return hg * sg_n + sg;
      }
    }
  }
  std::pair<int, int> head_range(int w) const {
    if (w < 0 || w >= workers) throw Error(kConfig, "worker index out of range");
    switch (mode) {
      case 0: return {0, heads};
      case 1: return range_of(w, workers, heads);
      default: return range_of(w / (workers / head_groups), head_groups, heads);
    }
  }
};

// ------------------------------------------------------------- scheduler ---
// scheduler.cpp:10-236
int micro_batch_size(int b, int f, int s) {
  if (b < 1 || f < 1 || s < 1) throw Error(kAdmission, "micro_batch_size: arguments must be >= 1");
  const long p = static_cast<long>(b) * f;
  if (p < s) {
    throw Error(kAdmission, "interval too short for target batch: B*F = " +
                                std::to_string(p) + " < S = " + std::to_string(s));
  }
  return static_cast<int>(std::max<long>(1, p / s));
}

struct MicroBatch {
  int id, size;
  long start, end;
  int target;
};
struct StepPlan {
  long step = 0;
  std::vector<int> active_ids, active_sizes;
  std::vector<long> active_len;
  long total_load = 0;
  std::vector<int> ending;
};

class LoadTracker {
 public:
  explicit LoadTracker(long limit) : limit_(limit) {
    if (limit < 1) throw Error(kAdmission, "load limit must be >= 1");
  }
  void set_limit(long l) {
    if (l < 1) throw Error(kAdmission, "load limit must be >= 1");
    limit_ = l;
  }
  long limit() const { return limit_; }
  long current() const { return cur_; }
  long earliest_start(int m, int s) const {
    if (m < 1 || s < 1) throw Error(kAdmission, "earliest_start: size and target length must be >= 1");
    if (static_cast<long>(m) * s > limit_) {
      throw Error(kAdmission, "micro-batch exceeds load limit: " +
                                  std::to_string(static_cast<long>(m) * s) + " > " +
                                  std::to_string(limit_));
    }
    long r = cur_;
    for (size_t i = 0; i < b_.size(); ++i) {
      const long x = (limit_ - w_[i]) / m;
      r = std::max(r, b_[i].end - x);
    }
    return r;
  }
  int add(long t, int m, int s) {
    if (m < 1 || s < 1) throw Error(kAdmission, "add_micro_batch: size and target length must be >= 1");
    if (t < cur_) {
      throw Error(kAdmission, "cannot admit in the past: step " + std::to_string(t) +
                                  " < current " + std::to_string(cur_));
    }
    const long own = static_cast<long>(m) * s;
    if (own > limit_) {
      throw Error(kAdmission, "admission rejected: batch workload " + std::to_string(own) +
                                  " exceeds limit " + std::to_string(limit_));
    }
    for (size_t i = 0; i < b_.size(); ++i) {
      if (b_[i].end > t && w_[i] + (b_[i].end - t) * m > limit_) {
        throw Error(kAdmission, "admission rejected: end-step workload of batch " +
                                    std::to_string(b_[i].id) + " would reach " +
                                    std::to_string(w_[i] + (b_[i].end - t) * m) + " > " +
                                    std::to_string(limit_));
      }
    }
    MicroBatch mb{next_id_++, m, t, t + s, s};
    for (size_t i = 0; i < b_.size(); ++i) {
      if (b_[i].end > t) w_[i] += (b_[i].end - t) * m;
    }
    b_.push_back(mb);
    w_.push_back(own);
    log_.push_back(mb);
    return mb.id;
  }
  StepPlan step() {
    cur_ += 1;
    StepPlan p;
    p.step = cur_;
    for (const MicroBatch& mb : b_) {
      if (mb.start < cur_ && cur_ <= mb.end) {
        p.active_ids.push_back(mb.id);
        p.active_sizes.push_back(mb.size);
        p.active_len.push_back(cur_ - mb.start);
        p.total_load += static_cast<long>(mb.size) * (cur_ - mb.start);
        if (mb.end == cur_) p.ending.push_back(mb.id);
      }
    }
    size_t keep = 0;
    for (size_t i = 0; i < b_.size(); ++i) {
      if (b_[i].end > cur_) {
        b_[keep] = b_[i];
        w_[keep] = w_[i];
        ++keep;
      }
    }
    b_.resize(keep);
    w_.resize(keep);
    return p;
  }
  long recomputed_load(long step) const {
    long load = 0;
    for (const MicroBatch& mb : log_) {
      if (mb.start < step && step <= mb.end) load += static_cast<long>(mb.size) * (step - mb.start);
    }
    return load;
  }
  const std::vector<long>& workloads() const { return w_; }
  const std::vector<MicroBatch>& batches() const { return b_; }

 private:
  long limit_;
  long cur_ = 0;
  int next_id_ = 0;
  std::vector<MicroBatch> b_;
  std::vector<long> w_;
  std::vector<MicroBatch> log_;
};

struct Admission {
  long step;
  int size, target;
};

int admission_size(long k, long b, long f, long s) {
  return static_cast<int>(((k + 1) * b * f) / s - (k * b * f) / s);
}
long ramp_limit(long u, long b, long s, long f) {
  const double steady = static_cast<double>(b) * (s + f) / 2.0;
  if (u >= s) return static_cast<long>(steady);
  const double bd = static_cast<double>(b);
  const double v = bd * f + bd * static_cast<double>(u) * (2.0 * s - f - u) / (2.0 * s);
  return static_cast<long>(std::floor(v + 1e-9));
}

// cold_start_schedule (scheduler.cpp:179-214); mode 0 fixed, 1 ramped
std::vector<Admission> cold_start(int b, int s, int f, int mode, long horizon) {
  micro_batch_size(b, f, s);
  std::vector<Admission> out;
  if (mode == 0) {
    long k = 0;
    for (long t = 0; t <= horizon; t += f, ++k) {
      const int m = admission_size(k, b, f, s);
      if (m > 0) out.push_back({t, m, s});
    }
    return out;
  }
  if (mode != 1) throw Error(kConfig, "unknown cold start mode");
  const long steady = static_cast<long>(b) * (s + f) / 2;
  LoadTracker tr(std::max<long>(1, ramp_limit(0, b, s, f)));
  long k = 0;
  for (long u = 0; u <= horizon; ++u) {
    tr.set_limit(std::max<long>(1, std::min(steady, ramp_limit(u, b, s, f))));
    for (;;) {
      const int m = admission_size(k, b, f, s);
      if (static_cast<long>(m) * s > tr.limit()) break;
      if (tr.earliest_start(m, s) != tr.current()) break;
      tr.add(tr.current(), m, s);
      out.push_back({tr.current(), m, s});
      ++k;
    }
    tr.step();
  }
  return out;
}

std::vector<StepPlan> run_schedule(const std::vector<Admission>& adm, long limit, long horizon) {
  LoadTracker tr(limit);
  size_t next = 0;
  std::vector<StepPlan> plans;
  while (next < adm.size() && adm[next].step == 0) {
    tr.add(0, adm[next].size, adm[next].target);
    ++next;
  }
  for (long u = 1; u <= horizon; ++u) {
    plans.push_back(tr.step());
    while (next < adm.size() && adm[next].step == u) {
      tr.add(u, adm[next].size, adm[next].target);
      ++next;
    }
  }
  return plans;
}

// ---------------------------------------------------------- drive (mono) ---
struct DriveConfig {
  int batch, target_len, interval;
  long steps;
  int cold_mode;
  long load_limit;
  uint64_t seed;
  int record_activations;
};
struct Record {
  long step;
  uint64_t seq;
  int token;
};
struct DriveResult {
  std::vector<Record> transcript;
  std::vector<float> activations;  // rows of D aligned with transcript when recorded
};

long default_load_limit(const DriveConfig& c) {  // workers.cpp:536-543
  if (c.load_limit > 0) return c.load_limit;
  const long b = c.batch, s = c.target_len, f = c.interval;
  if (s % f == 0 && (b * f) % s == 0) return b * (s + f) / 2;
  return b * s + b * f;
}

// drive_schedule (workers.cpp:547-684) over the monolithic computation
// (MonolithicComputation, workers.cpp:520-532).
DriveResult drive(const Weights& W, const DriveConfig& c, long capacity, int fmt, int threads) {
  if (c.batch < 1 || c.target_len < 1 || c.interval < 1) {
    throw Error(kConfig, "generation config: batch, target_len, interval must be >= 1");
  }
  const Spec& s = W.spec;
  KvShard kv(s, 0, s.num_kv_heads, capacity, fmt);
  const bool to_completion = c.steps <= 0;
  long adm_horizon;
  if (to_completion) {
    const int m = micro_batch_size(c.batch, c.interval, c.target_len);
    const long waves = std::max<long>(1, (c.batch + m - 1) / m);
    adm_horizon = (waves - 1) * c.interval;
  } else {
    adm_horizon = c.steps;
  }
  std::vector<Admission> adm = cold_start(c.batch, c.target_len, c.interval, c.cold_mode, adm_horizon);
  if (to_completion) {
    long total = 0;
    std::vector<Admission> trimmed;
    for (Admission a : adm) {
      if (total >= c.batch) break;
      a.size = static_cast<int>(std::min<long>(a.size, c.batch - total));
      total += a.size;
      trimmed.push_back(a);
    }
    adm = trimmed;
  }
  const long horizon = to_completion ? (adm.empty() ? 0 : adm.back().step + c.target_len) : c.steps;
  LoadTracker tr(default_load_limit(c));
  std::unordered_map<int, std::vector<uint64_t>> batch_seqs;
  struct St {
    int cur, target;
  };
  std::unordered_map<uint64_t, St> states;
  std::unordered_map<uint64_t, int> last;
  uint64_t next_id = 1;
  size_t next_adm = 0;
  auto admit_due = [&](long step) {
    while (next_adm < adm.size() && adm[next_adm].step == step) {
      const Admission& a = adm[next_adm];
      const int id = tr.add(a.step, a.size, a.target);
      auto& seqs = batch_seqs[id];
      for (int i = 0; i < a.size; ++i) {
        const uint64_t seq = next_id++;
        seqs.push_back(seq);
        states[seq] = St{0, a.target};
        last[seq] = prompt_token(c.seed, seq, s.vocab_size);
      }
      ++next_adm;
    }
  };
  DriveResult res;
  admit_due(0);
  const int D = s.model_dim;
  for (long u = 1; u <= horizon; ++u) {
    StepPlan plan = tr.step();
    if (plan.active_ids.empty() && next_adm >= adm.size()) break;
    if (!plan.active_ids.empty()) {
      std::vector<uint64_t> ids;
      for (int id : plan.active_ids) for (uint64_t q : batch_seqs[id]) ids.push_back(q);
      const int B = static_cast<int>(ids.size());
      std::vector<float> x(static_cast<size_t>(B) * D);
      for (int b = 0; b < B; ++b) {
        const int tok = last.at(ids[b]);
        for (int d = 0; d < D; ++d) x[static_cast<size_t>(b) * D + d] = W.embedding.at(d, tok);
      }
      std::vector<int> toks(static_cast<size_t>(B));
      std::vector<float> fx(static_cast<size_t>(B) * D);
      decode_step(W, kv, B, ids.data(), x.data(), toks.data(), fx.data(), nullptr, threads);
      for (int b = 0; b < B; ++b) {
        res.transcript.push_back({u, ids[b], toks[b]});
        last[ids[b]] = toks[b];
        St& st = states.at(ids[b]);
        st.cur += 1;
        if (st.cur > st.target) throw Error(kLogic, "sequence ran past its target length");
        if (c.record_activations) {
          res.activations.insert(res.activations.end(), fx.begin() + static_cast<long>(b) * D,
                                 fx.begin() + static_cast<long>(b + 1) * D);
        }
      }
    }
    if (!plan.ending.empty()) {
      for (int id : plan.ending) {
        auto it = batch_seqs.find(id);
        if (it == batch_seqs.end()) continue;
        for (uint64_t q : it->second) {
          if (states.at(q).cur != states.at(q).target) {
            throw Error(kLogic, "retiring a sequence short of its target");
          }
          kv.drop(q);
          last.erase(q);
          states.erase(q);
        }
        batch_seqs.erase(it);
      }
    }
    admit_due(u);
  }
  return res;
}

// ------------------------------------------------- synthetic KV (bench) ---
// Counter-based KV fill shared with the GPU bench: element idx
// of (seq slot, layer, pos, kv, i) gets 2u-1 with u = (mix64(0x5EED ^ idx)
// >> 40) * 2^-24.
inline float synth_value(uint64_t idx) {
  return 2.0f * (static_cast<float>(mix64(0x5EEDull ^ idx) >> 40) * 0x1p-24f) - 1.0f;
}

// Sequence-keyed element index of the synthetic prefill (the
// repo's fixed definition; not a reference function): sequence id, layer
// (< 4096), position (< 2^20), K (0) / V (1), global kv head h, element d.
inline uint64_t prefill_index(uint64_t seq, int layer, int pos, int kv, int h, int d, int kv_heads, int hd) {
  return ((((seq * 4096u + static_cast<uint64_t>(layer)) * 1048576u + static_cast<uint64_t>(pos)) * 2u +
           static_cast<uint64_t>(kv)) * static_cast<uint64_t>(kv_heads) + static_cast<uint64_t>(h)) *
             static_cast<uint64_t>(hd) + static_cast<uint64_t>(d);
}

}  // namespace orc

// ============================================================ C interface ===
using namespace orc;

extern "C" {

typedef struct {
  int num_layers, model_dim, num_heads, head_dim, mlp_dim, vocab_size, num_kv_heads;
} orc_spec;

static Spec to_spec(const orc_spec* s) {
  return make_spec(s->num_layers, s->model_dim, s->num_heads, s->mlp_dim, s->vocab_size,
                   s->num_kv_heads);
}

const char* orc_last_error() { return g_last_error.c_str(); }

int orc_make_spec(int L, int D, int H, int F, int V, int Hkv, orc_spec* out) {
  return guard([&] {
    Spec s = make_spec(L, D, H, F, V, Hkv);
    *out = orc_spec{s.num_layers, s.model_dim, s.num_heads, s.head_dim, s.mlp_dim,
                    s.vocab_size, s.num_kv_heads};
  });
}

uint64_t orc_mix64(uint64_t x) { return mix64(x); }
int orc_prompt_token(uint64_t seed, uint64_t id, int vocab) { return prompt_token(seed, id, vocab); }
uint16_t orc_f2h(float f) { return f2h(f); }
float orc_h2f(uint16_t h) { return h2f(h); }
float orc_quantize_int8(const float* x, int n, int8_t* q) { return quantize_int8(x, n, q); }
float orc_quantize_int4(const float* x, int n, uint8_t* packed) { return quantize_int4(x, n, packed); }
float orc_eigen_dot(const float* a, const float* b, int n) { return eigen_dot(a, b, n); }
float orc_synth_value(uint64_t idx) { return synth_value(idx); }

// ---- weights
int orc_weights_create(const orc_spec* s, uint64_t seed, void** out) {
  return guard([&] { *out = new Weights(seed_weights(to_spec(s), seed)); });
}
void orc_weights_destroy(void* w) { delete static_cast<Weights*>(w); }
uint64_t orc_weights_checksum(void* w) { return checksum(*static_cast<Weights*>(w)); }
// which: 0 embedding, 1 w_q, 2 w_k, 3 w_v, 4 w_o, 5 w_mlp_in, 6 w_mlp_out, 7 head
float* orc_weights_tensor(void* wp, int layer, int which, int* rows, int* cols) {
  Weights& w = *static_cast<Weights*>(wp);
  Mat* m = nullptr;
  if (which == 0) m = &w.embedding;
  else if (which == 7) m = &w.head;
  else {
    if (layer < 0 || layer >= w.spec.num_layers) return nullptr;
    Layer& l = w.layers[static_cast<size_t>(layer)];
    Mat* t[] = {&l.w_q, &l.w_k, &l.w_v, &l.w_o, &l.w_mlp_in, &l.w_mlp_out};
    if (which < 1 || which > 6) return nullptr;
    m = t[which - 1];
  }
  *rows = m->rows;
  *cols = m->cols;
  return m->data.data();
}

// ---- KvShard
int orc_kv_create(const orc_spec* s, int head_start, int head_count, long cap, int fmt, void** out) {
  return guard([&] { *out = new KvShard(to_spec(s), head_start, head_count, cap, fmt); });
}
void orc_kv_destroy(void* kv) { delete static_cast<KvShard*>(kv); }
int orc_kv_append(void* kv, uint64_t seq, int layer, uint32_t pos, const float* k, const float* v) {
  return guard([&] { static_cast<KvShard*>(kv)->append(seq, layer, pos, k, v); });
}
// Synthetic context of `length` positions for each sequence in every layer,
// appended through KvShard::append (so the stored bytes follow the reference
// conversions): K/V element (seq, layer, pos, kv, h0 + head, d) =
// synth_value(salt ^ prefill_index(...)).
int orc_kv_prefill_synthetic(void* kvp, int n, const uint64_t* seqs, int length, uint64_t salt) {
  return guard([&] {
    KvShard* kv = static_cast<KvShard*>(kvp);
    const Spec& sp = kv->spec();
    const int w = kv->width(), hd = sp.head_dim, h0 = kv->head_start();
    std::vector<float> k(static_cast<size_t>(w)), v(static_cast<size_t>(w));
    for (int i = 0; i < n; ++i) {
      for (int l = 0; l < sp.num_layers; ++l) {
        for (int pos = 0; pos < length; ++pos) {
          const uint64_t bk = prefill_index(seqs[i], l, pos, 0, h0, 0, sp.num_kv_heads, hd);
          const uint64_t bv = prefill_index(seqs[i], l, pos, 1, h0, 0, sp.num_kv_heads, hd);
          for (int e = 0; e < w; ++e) {
            k[static_cast<size_t>(e)] = synth_value(salt ^ (bk + static_cast<uint64_t>(e)));
            v[static_cast<size_t>(e)] = synth_value(salt ^ (bv + static_cast<uint64_t>(e)));
          }
          kv->append(seqs[i], l, static_cast<uint32_t>(pos), k.data(), v.data());
        }
      }
    }
  });
}
uint64_t orc_kv_prefill_index(uint64_t seq, int layer, int pos, int kv, int h, int d, int kv_heads, int hd) {
  return prefill_index(seq, layer, pos, kv, h, d, kv_heads, hd);
}
int orc_kv_append_request(void* kv, int layer, int n, const uint64_t* seqs, const uint32_t* pos,
                          const float* k, const float* v) {
  return guard([&] { static_cast<KvShard*>(kv)->append_request(layer, n, seqs, pos, k, v); });
}
int orc_kv_attend(void* kv, int layer, int n, const uint64_t* seqs, const float* q, float* o) {
  return guard([&] { static_cast<KvShard*>(kv)->attend(layer, n, seqs, q, o); });
}
void orc_kv_drop(void* kv, uint64_t seq) { static_cast<KvShard*>(kv)->drop(seq); }
int orc_kv_stored_length(void* kv, uint64_t seq, int layer) {
  return static_cast<KvShard*>(kv)->stored(seq, layer);
}
long orc_kv_token_count(void* kv) { return static_cast<KvShard*>(kv)->token_count(); }
int orc_kv_warning_count(void* kv) { return static_cast<KvShard*>(kv)->warnings(); }
int orc_kv_has_sequence(void* kv, uint64_t seq) { return static_cast<KvShard*>(kv)->has(seq); }
size_t orc_kv_bytes_per_token(void* kv) { return static_cast<KvShard*>(kv)->bytes_per_token(); }
long orc_kv_export_lane(void* kv, uint64_t seq, int layer, int which, void* out, size_t cap,
                        float* scales, size_t scap) {
  long r = -1;
  int rc = guard([&] {
    r = static_cast<long>(static_cast<KvShard*>(kv)->export_lane(seq, layer, which, out, cap, scales, scap));
  });
  return rc ? -rc : r;
}

// ---- dense
int orc_apply_linear(int B, int in, int out, const float* x, const float* w_colmajor, float* y,
                     int threads) {
  return guard([&] { apply_linear(B, in, out, x, w_colmajor, y, threads); });
}
int orc_project_qkv(void* w, int layer, int B, const uint64_t* seqs, const float* x, float* q,
                    float* k, float* v, int threads) {
  return guard([&] { project_qkv(*static_cast<Weights*>(w), layer, B, seqs, x, q, k, v, threads); });
}
int orc_finish_block(void* w, int layer, int B, const float* o, const float* res, float* xout,
                     int threads) {
  return guard([&] { finish_block(*static_cast<Weights*>(w), layer, B, o, res, xout, threads); });
}
int orc_output_logits(void* wp, int B, const float* x, float* logits, int threads) {
  return guard([&] { linear(static_cast<Weights*>(wp)->head, B, x, logits, threads); });
}
int orc_argmax(const float* logits, int n) { return argmax(logits, n); }
int orc_decode_step(void* w, void* kv, int B, const uint64_t* seqs, const float* x, int* tokens,
                    float* final_x, float* logits, int threads) {
  return guard([&] {
    decode_step(*static_cast<Weights*>(w), *static_cast<KvShard*>(kv), B, seqs, x, tokens, final_x,
                logits, threads);
  });
}

// ---- ShardMap
int orc_shardmap_worker_for(int mode, int heads, int workers, uint64_t seq, int head, int* out) {
  return guard([&] { *out = ShardMap(mode, heads, workers).worker_for(seq, head); });
}
int orc_shardmap_head_range(int mode, int heads, int workers, int w, int* start, int* count) {
  return guard([&] {
    auto r = ShardMap(mode, heads, workers).head_range(w);
    *start = r.first;
    *count = r.second;
  });
}

// ---- scheduler
int orc_micro_batch_size(int b, int f, int s, int* out) {
  return guard([&] { *out = micro_batch_size(b, f, s); });
}
// writes up to cap admissions as (step, size, target) triples; returns count via *n
int orc_cold_start_schedule(int b, int s, int f, int mode, long horizon, long* out, long cap, long* n) {
  return guard([&] {
    auto a = cold_start(b, s, f, mode, horizon);
    *n = static_cast<long>(a.size());
    for (size_t i = 0; i < a.size() && static_cast<long>(i) < cap; ++i) {
      out[3 * i] = a[i].step;
      out[3 * i + 1] = a[i].size;
      out[3 * i + 2] = a[i].target;
    }
  });
}
// run_schedule: per step (step, n_active, total_load, n_ending)
int orc_run_schedule(const long* adm, long n_adm, long limit, long horizon, long* out) {
  return guard([&] {
    std::vector<Admission> a;
    for (long i = 0; i < n_adm; ++i) {
      a.push_back({adm[3 * i], static_cast<int>(adm[3 * i + 1]), static_cast<int>(adm[3 * i + 2])});
    }
    auto plans = run_schedule(a, limit, horizon);
    for (size_t i = 0; i < plans.size(); ++i) {
      out[4 * i] = plans[i].step;
      out[4 * i + 1] = static_cast<long>(plans[i].active_ids.size());
      out[4 * i + 2] = plans[i].total_load;
      out[4 * i + 3] = static_cast<long>(plans[i].ending.size());
    }
  });
}
int orc_tracker_create(long limit, void** out) {
  return guard([&] { *out = new LoadTracker(limit); });
}
void orc_tracker_destroy(void* t) { delete static_cast<LoadTracker*>(t); }
int orc_tracker_earliest_start(void* t, int m, int s, long* out) {
  return guard([&] { *out = static_cast<LoadTracker*>(t)->earliest_start(m, s); });
}
int orc_tracker_add(void* t, long start, int m, int s, int* id) {
  return guard([&] { *id = static_cast<LoadTracker*>(t)->add(start, m, s); });
}
// returns total load; fills ending ids
long orc_tracker_step(void* t, int* n_active, int* ending, int cap, int* n_ending) {
  StepPlan p = static_cast<LoadTracker*>(t)->step();
  *n_active = static_cast<int>(p.active_ids.size());
  *n_ending = static_cast<int>(p.ending.size());
  for (int i = 0; i < *n_ending && i < cap; ++i) ending[i] = p.ending[static_cast<size_t>(i)];
  return p.total_load;
}
long orc_tracker_recomputed_load(void* t, long step) {
  return static_cast<LoadTracker*>(t)->recomputed_load(step);
}
long orc_tracker_current(void* t) { return static_cast<LoadTracker*>(t)->current(); }
int orc_tracker_num_batches(void* t) {
  return static_cast<int>(static_cast<LoadTracker*>(t)->batches().size());
}
void orc_tracker_batch(void* t, int i, long* end, long* workload) {
  auto* tr = static_cast<LoadTracker*>(t);
  *end = tr->batches()[static_cast<size_t>(i)].end;
  *workload = tr->workloads()[static_cast<size_t>(i)];
}
long orc_tracker_limit(void* t) { return static_cast<LoadTracker*>(t)->limit(); }

// ---- drive (monolithic oracle generation)
int orc_drive_monolithic(void* w, int batch, int target_len, int interval, long steps,
                         int cold_mode, long load_limit, uint64_t seed, int record, long capacity,
                         int fmt, int threads, void** out) {
  return guard([&] {
    DriveConfig c{batch, target_len, interval, steps, cold_mode, load_limit, seed, record};
    *out = new DriveResult(drive(*static_cast<Weights*>(w), c, capacity, fmt, threads));
  });
}
long orc_drive_count(void* r) { return static_cast<long>(static_cast<DriveResult*>(r)->transcript.size()); }
void orc_drive_record(void* r, long i, long* step, uint64_t* seq, int* token) {
  const Record& rec = static_cast<DriveResult*>(r)->transcript[static_cast<size_t>(i)];
  *step = rec.step;
  *seq = rec.seq;
  *token = rec.token;
}
const float* orc_drive_activations(void* r) {
  auto* d = static_cast<DriveResult*>(r);
  return d->activations.empty() ? nullptr : d->activations.data();
}
void orc_drive_destroy(void* r) { delete static_cast<DriveResult*>(r); }

// ---- CPU baselines (bench.py cpu_baseline / --impl reference legs)
//
// R-Part: one KvShard per host thread (the reference's single-owner model,
// SPEC.md:168); `batch` sequences of `seq_len` stored tokens filled with the
// counter-based synthetic values, sequences dealt round-robin to threads.
// Each rep times one attend() over every sequence (in parallel threads) at
// layer 0 of a 1-layer spec. Returns the median seconds per rep.
int orc_bench_attend(const orc_spec* sp, int batch, int seq_len, int fmt, int threads, int reps,
                     double* median_s) {
  return guard([&] {
    Spec s = to_spec(sp);
    s.num_layers = 1;
    if (threads < 1) threads = 1;
    const int kvw = s.num_kv_heads * s.head_dim;
    const int qw = s.num_heads * s.head_dim;
    struct Part {
      std::unique_ptr<KvShard> kv;
      std::vector<uint64_t> seqs;
      std::vector<float> q, o;
    };
    std::vector<Part> parts(static_cast<size_t>(threads));
    for (int b = 0; b < batch; ++b) parts[static_cast<size_t>(b % threads)].seqs.push_back(static_cast<uint64_t>(b + 1));
    auto build = [&](Part& p) {
      const long n = static_cast<long>(p.seqs.size());
      p.kv = std::make_unique<KvShard>(s, 0, s.num_kv_heads, std::max<long>(1, n * seq_len), fmt);
      std::vector<float> k(static_cast<size_t>(kvw)), v(static_cast<size_t>(kvw));
      for (uint64_t seq : p.seqs) {
        for (int pos = 0; pos < seq_len; ++pos) {
          const uint64_t base = ((seq * 1 + 0) * static_cast<uint64_t>(1 << 20) + pos) * 2ull * kvw;
          for (int i = 0; i < kvw; ++i) {
            k[i] = synth_value(base + i);
            v[i] = synth_value(base + kvw + i);
          }
          p.kv->append(seq, 0, static_cast<uint32_t>(pos), k.data(), v.data());
        }
      }
      p.q.resize(p.seqs.size() * static_cast<size_t>(qw));
      for (size_t i = 0; i < p.q.size(); ++i) p.q[i] = synth_value(0xABCDEF0000ull + i);
      p.o.resize(p.q.size());
    };
    {
      std::vector<std::thread> ts;
      for (auto& p : parts) ts.emplace_back(build, std::ref(p));
      for (auto& t : ts) t.join();
    }
    std::vector<double> samples;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> ts;
      for (auto& p : parts) {
        if (p.seqs.empty()) continue;
        ts.emplace_back([&p] {
          p.kv->attend(0, static_cast<int>(p.seqs.size()), p.seqs.data(), p.q.data(), p.o.data());
        });
      }
      for (auto& t : ts) t.join();
      samples.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(samples.begin(), samples.end());
    *median_s = samples[samples.size() / 2];
  });
}

// S-Part: bench_dense_block (dense.cpp:145-196) at one batch size with the
// output columns of every apply_linear split over `threads` host threads
// (per-element arithmetic unchanged). Weights are generated for a 1-layer
// spec (seed 7, the reference's choice). Median seconds per block.
int orc_bench_dense(const orc_spec* sp, int batch, int threads, int reps, double* median_s) {
  return guard([&] {
    Spec s = to_spec(sp);
    s.num_layers = 1;
    s.vocab_size = 1;  // head/embedding are not part of the block
    Weights w = seed_weights(s, 7);
    const int D = s.model_dim, kvw = s.num_kv_heads * s.head_dim;
    std::vector<float> x(static_cast<size_t>(batch) * D), q(x.size()), o(x.size()),
        k(static_cast<size_t>(batch) * kvw), v(k.size());
    uint64_t st = 0x5eedu + static_cast<uint64_t>(batch);
    for (float& e : x) {
      st = mix64(st);
      e = 2.0f * (static_cast<float>(st >> 40) * 0x1p-24f) - 1.0f;
    }
    std::vector<uint64_t> ids(static_cast<size_t>(batch));
    std::iota(ids.begin(), ids.end(), 1);
    std::vector<double> samples;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      project_qkv(w, 0, batch, ids.data(), x.data(), q.data(), k.data(), v.data(), threads);
      finish_block(w, 0, batch, q.data(), x.data(), o.data(), threads);
      samples.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(samples.begin(), samples.end());
    *median_s = samples[samples.size() / 2];
  });
}

}  // extern "C"
