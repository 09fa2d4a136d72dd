// sd_b200.hpp — the reference's R-Part C++ interface (splitdecode/attention.hpp,
// core.hpp) over the C ABI, header-only: a C++ host sees the same names,
// argument meanings and exception types as splitdecode::KvShard, backed by
// the B200 KV store. The reference's Eigen vectors become contiguous float
// vectors / spans (Eigen is not part of this boundary); everything else —
// construction, append / append_request (all or nothing), attend (outputs in
// item order), drop_sequence, the accounting queries, the error types and
// their messages — follows attention.hpp:68-140 and core.hpp:25-38.
//
// The ABI takes packed rows, so vector sizes are checked here, with the
// reference's messages; a request that is both mis-sized and invalid in
// another way reports the size first (the reference checks capacity first in
// append_request and the sequence first in attend).
//
// Link with libsd_b200.so; include/sd_abi.h documents each entry point.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sd_abi.h"

namespace sd_b200 {

// ---- errors (core.hpp:25-38, attention.hpp:19-22)
class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ProtocolError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class UnknownSequenceError : public ProtocolError {
 public:
  using ProtocolError::ProtocolError;
};
class CapacityError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
// CUDA / internal failures of the B200 backend (no reference counterpart)
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// status -> the reference's exception type, message from sd_last_error()
inline void check(int status) {
  if (status == SD_OK) return;
  const std::string msg = sd_last_error();
  switch (status) {
    case SD_ERR_PROTOCOL: throw ProtocolError(msg);
    case SD_ERR_CAPACITY: throw CapacityError(msg);
    case SD_ERR_UNKNOWN_SEQ: throw UnknownSequenceError(msg);
    case SD_ERR_LOGIC: throw std::logic_error(msg);
    case SD_ERR_CONFIG: throw ConfigError(msg);
    default: throw DeviceError(msg);
  }
}

using SequenceId = std::uint64_t;
using Vec = std::vector<float>;

// ---- geometry (core.hpp:43-58): head_dim = model_dim / num_heads;
// num_kv_heads (the GQA extension) defaults to num_heads
struct ModelSpec {
  int num_layers = 0, model_dim = 0, num_heads = 0, head_dim = 0, mlp_dim = 0, vocab_size = 0;
  int num_kv_heads = 0;
  sd_model_spec raw() const {
    return sd_model_spec{num_layers, model_dim, num_heads, head_dim, mlp_dim, vocab_size, num_kv_heads};
  }
};

inline ModelSpec make_model_spec(int num_layers, int model_dim, int num_heads, int mlp_dim, int vocab_size,
                                 int num_kv_heads = 0) {
  sd_model_spec s{};
  check(sd_make_model_spec(num_layers, model_dim, num_heads, mlp_dim, vocab_size, num_kv_heads, &s));
  return ModelSpec{s.num_layers, s.model_dim, s.num_heads, s.head_dim, s.mlp_dim, s.vocab_size, s.num_kv_heads};
}

inline std::uint64_t mix64(std::uint64_t x) { return sd_mix64(x); }

// ---- KvFormat (attention.hpp:24); kInt4 is the 4-bit hook extension
enum class KvFormat : std::uint8_t { kSingle, kHalf, kInt8, kInt4 };

// ---- requests (attention.hpp:44-60)
struct AttentionItem {
  SequenceId seq = 0;
  std::uint32_t position = 0;  // stored length before this token is appended
  Vec q, k, v;                 // q: q_width, k / v: width of the shard's head range
};
struct AttentionRequest {
  int layer = 0;
  std::vector<AttentionItem> items;
};
struct AttentionOutput {
  SequenceId seq = 0;
  Vec o;
};
struct AttentionResponse {
  int layer = 0;
  std::vector<AttentionOutput> outputs;  // same order as the request items
};

// ---- KvShard (attention.hpp:68-140) on a B200
class KvShard {
 public:
  KvShard(const ModelSpec& spec, int head_start, int head_count, long capacity_tokens,
          KvFormat format = KvFormat::kSingle, int device = 0)
      : spec_(spec), head_start_(head_start), head_count_(head_count), capacity_(capacity_tokens),
        format_(format) {
    const sd_model_spec s = spec.raw();
    check(sd_kv_create(&s, head_start, head_count, capacity_tokens, static_cast<int>(format), device, nullptr,
                       &h_));
    std::int32_t w = 0, qw = 0;
    check(sd_kv_width(h_, &w, &qw));
    width_ = w;
    q_width_ = qw;
  }
  ~KvShard() {
    if (h_) sd_kv_destroy(h_);
  }
  KvShard(const KvShard&) = delete;
  KvShard& operator=(const KvShard&) = delete;
  KvShard(KvShard&& o) noexcept { *this = std::move(o); }
  KvShard& operator=(KvShard&& o) noexcept {
    if (this != &o) {
      if (h_) sd_kv_destroy(h_);
      h_ = o.h_;
      o.h_ = nullptr;
      spec_ = o.spec_;
      head_start_ = o.head_start_;
      head_count_ = o.head_count_;
      capacity_ = o.capacity_;
      format_ = o.format_;
      width_ = o.width_;
      q_width_ = o.q_width_;
    }
    return *this;
  }

  int head_start() const { return head_start_; }
  int head_count() const { return head_count_; }
  int width() const { return width_; }
  int q_width() const { return q_width_; }
  KvFormat format() const { return format_; }
  long capacity() const { return capacity_; }

  long token_count() const {
    std::int64_t n = 0;
    check(sd_kv_token_count(h_, &n));
    return static_cast<long>(n);
  }
  bool has_sequence(SequenceId seq) const {
    std::int32_t b = 0;
    check(sd_kv_has_sequence(h_, seq, &b));
    return b != 0;
  }
  int stored_length(SequenceId seq, int layer) const {
    std::int32_t n = 0;
    check(sd_kv_stored_length(h_, seq, layer, &n));
    return n;
  }
  int warning_count() const {
    std::int32_t n = 0;
    check(sd_kv_warning_count(h_, &n));
    return n;
  }
  std::size_t bytes_per_token() const {
    std::int64_t n = 0;
    check(sd_kv_bytes_per_token(h_, &n));
    return static_cast<std::size_t>(n);
  }

  // attention.hpp:91-92
  void append(SequenceId seq, int layer, std::uint32_t position, std::span<const float> k,
              std::span<const float> v) {
    if (layer < 0 || layer >= spec_.num_layers) throw ProtocolError("append: layer index out of range");
    if (static_cast<int>(k.size()) != width_ || static_cast<int>(v.size()) != width_) {
      throw ProtocolError("append: K/V width does not match the shard's head range");
    }
    check(sd_kv_append(h_, seq, layer, position, k.data(), v.data()));
  }

  // attention.hpp:96: all or nothing
  void append_request(const AttentionRequest& r) {
    Packed p(r, width_, q_width_, false);
    check(sd_kv_append_request(h_, r.layer, p.n, p.seqs.data(), p.pos.data(), p.k.data(), p.v.data()));
  }

  // attention.hpp:102: one output per item, in item order
  AttentionResponse attend(const AttentionRequest& r) const {
    Packed p(r, width_, q_width_, true);
    std::vector<float> o(static_cast<std::size_t>(p.n) * q_width_);
    check(sd_kv_attend(h_, r.layer, p.n, p.seqs.data(), p.q.data(), o.data()));
    AttentionResponse resp;
    resp.layer = r.layer;
    resp.outputs.resize(r.items.size());
    for (std::size_t i = 0; i < r.items.size(); ++i) {
      resp.outputs[i].seq = r.items[i].seq;
      resp.outputs[i].o.assign(o.begin() + static_cast<std::ptrdiff_t>(i * q_width_),
                               o.begin() + static_cast<std::ptrdiff_t>((i + 1) * q_width_));
    }
    return resp;
  }

  // attention.hpp:106
  void drop_sequence(SequenceId seq) { check(sd_kv_drop(h_, 1, &seq)); }

  sd_kv* handle() const { return h_; }

 private:
  // items packed row-major for the ABI (the reference's per-item VectorXf)
  struct Packed {
    std::int32_t n = 0;
    std::vector<std::uint64_t> seqs;
    std::vector<std::uint32_t> pos;
    std::vector<float> q, k, v;
    Packed(const AttentionRequest& r, int width, int q_width, bool want_q) {
      n = static_cast<std::int32_t>(r.items.size());
      for (const AttentionItem& it : r.items) {
        seqs.push_back(it.seq);
        pos.push_back(it.position);
        if (want_q) {
          if (static_cast<int>(it.q.size()) != q_width) {
            throw ProtocolError("attend: Q width does not match the shard's head range");
          }
          q.insert(q.end(), it.q.begin(), it.q.end());
        } else {
          if (static_cast<int>(it.k.size()) != width || static_cast<int>(it.v.size()) != width) {
            throw ProtocolError("append: K/V width does not match the shard's head range");
          }
          k.insert(k.end(), it.k.begin(), it.k.end());
          v.insert(v.end(), it.v.begin(), it.v.end());
        }
      }
    }
  };

  sd_kv* h_ = nullptr;
  ModelSpec spec_;
  int head_start_ = 0, head_count_ = 0;
  long capacity_ = 0;
  KvFormat format_ = KvFormat::kSingle;
  int width_ = 0, q_width_ = 0;
};

// ---- S-Part (dense.hpp:16-50) over device-resident weights

// the S-Part arithmetic of a WeightSet (sd_dense_mode): kExact is the
// reference's fp32 per-element order (bitwise), the rest run on tcgen05
enum class DenseMode : int { kExact = SD_DENSE_EXACT_F32, kBf16 = SD_DENSE_BF16, kTf32 = SD_DENSE_TF32, kFp16 = SD_DENSE_F16 };

// Row-major [rows][cols] float matrix (the reference's MatrixXf rows)
struct Rows {
  int rows = 0, cols = 0;
  std::vector<float> data;
  Rows() = default;
  Rows(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0f) {}
  float* row(int r) { return data.data() + static_cast<std::size_t>(r) * cols; }
  const float* row(int r) const { return data.data() + static_cast<std::size_t>(r) * cols; }
};

// seed_random_weights (core.cpp:97-127) generated on the device: the
// reference's mt19937 tensors bit for bit, in the requested dense mode
class WeightSet {
 public:
  WeightSet(const ModelSpec& spec, std::uint64_t seed, DenseMode mode = DenseMode::kExact, int device = 0)
      : spec_(spec) {
    const sd_model_spec s = spec.raw();
    check(sd_weights_seed_random(&s, seed, static_cast<int>(mode), device, &h_));
  }
  ~WeightSet() {
    if (h_) sd_weights_destroy(h_);
  }
  WeightSet(const WeightSet&) = delete;
  WeightSet& operator=(const WeightSet&) = delete;
  const ModelSpec& spec() const { return spec_; }
  sd_weights* handle() const { return h_; }
  // embedding.col(token) (workers.cpp:636)
  Vec embedding_column(int token) const {
    if (emb_.empty()) {
      emb_.resize(static_cast<std::size_t>(spec_.model_dim) * spec_.vocab_size);
      check(sd_weights_export_embedding(h_, emb_.data(), emb_.size()));
    }
    const float* c = emb_.data() + static_cast<std::size_t>(token) * spec_.model_dim;
    return Vec(c, c + spec_.model_dim);
  }

 private:
  ModelSpec spec_;
  sd_weights* h_ = nullptr;
  mutable std::vector<float> emb_;
};

struct QkvProjection {  // dense.hpp:22-27
  Rows q, k, v;
};
// project_qkv (dense.cpp:33-43): features [B][D] -> q [B][q width], k / v [B][kv width]
inline QkvProjection project_qkv(const WeightSet& w, int layer, const Rows& x) {
  const ModelSpec& s = w.spec();
  const int kvw = (s.num_kv_heads > 0 ? s.num_kv_heads : s.num_heads) * s.head_dim;
  QkvProjection r{Rows(x.rows, s.num_heads * s.head_dim), Rows(x.rows, kvw), Rows(x.rows, kvw)};
  check(sd_s_project_qkv(w.handle(), layer, x.rows, x.data.data(), r.q.data.data(), r.k.data.data(), r.v.data.data()));
  return r;
}
// finish_block (dense.cpp:51-70): o and the residual [B][D] -> the block's output
inline Rows finish_block(const WeightSet& w, int layer, const Rows& o, const Rows& residual) {
  Rows x(o.rows, w.spec().model_dim);
  check(sd_s_finish_block(w.handle(), layer, o.rows, o.data.data(), residual.data.data(), x.data.data()));
  return x;
}
// output_logits + argmax_token (dense.cpp:72-88)
inline Rows output_logits(const WeightSet& w, const Rows& x) {
  Rows l(x.rows, w.spec().vocab_size);
  std::vector<std::int32_t> t(static_cast<std::size_t>(x.rows));
  check(sd_s_logits_argmax(w.handle(), x.rows, x.data.data(), l.data.data(), t.data()));
  return l;
}
inline int argmax_token(std::span<const float> logits) {  // first maximum wins
  int best = 0;
  for (int j = 1; j < static_cast<int>(logits.size()); ++j)
    if (logits[static_cast<std::size_t>(j)] > logits[static_cast<std::size_t>(best)]) best = j;
  return best;
}

// ---- the runtime seam (workers.hpp:151-158): the GPU StepComputation

struct TokenBatch {  // core.hpp:66-72
  std::vector<SequenceId> seq_ids;
  Rows features;  // batch x model_dim
  int size() const { return static_cast<int>(seq_ids.size()); }
};
struct DecodeStepResult {  // dense.hpp:40-43
  std::vector<int> next_tokens;
  Rows final_activations;
};

class StepComputation {
 public:
  StepComputation(WeightSet& w, KvShard& kv) : spec_(w.spec()) { check(sd_engine_create(w.handle(), kv.handle(), &h_)); }
  ~StepComputation() {
    if (h_) sd_engine_destroy(h_);
  }
  StepComputation(const StepComputation&) = delete;
  StepComputation& operator=(const StepComputation&) = delete;
  // compute(batch, step) (workers.hpp:155): one decode step of every layer
  DecodeStepResult compute(const TokenBatch& batch, long /*step*/) {
    DecodeStepResult r;
    r.next_tokens.resize(batch.seq_ids.size());
    r.final_activations = Rows(batch.size(), spec_.model_dim);
    std::vector<std::int32_t> t(batch.seq_ids.size());
    check(sd_engine_step_features(h_, batch.size(), batch.seq_ids.data(), batch.features.data.data(), t.data(),
                                  r.final_activations.data.data(), nullptr));
    for (std::size_t i = 0; i < t.size(); ++i) r.next_tokens[i] = t[i];
    return r;
  }
  void retire(const std::vector<SequenceId>& seqs) {  // workers.hpp:157
    check(sd_engine_retire(h_, static_cast<std::int32_t>(seqs.size()), seqs.data()));
  }
  sd_engine* handle() const { return h_; }

 private:
  ModelSpec spec_;
  sd_engine* h_ = nullptr;
};

// ---- drive_schedule (workers.cpp:547-684) over a StepComputation, host C++
struct GenerationConfig {  // workers.hpp:115-129 (the fields drive_schedule reads)
  int batch = 0, target_len = 0, interval = 0;
  long steps = 0;  // <= 0: run to completion
  std::uint64_t seed = 0;
  int cold_start = 0;  // 0 fixed-interval, 1 ramped-limit
  long load_limit = 0;
};
struct GenerationRecord {  // workers.hpp:131-135
  long step = 0;
  SequenceId seq = 0;
  int token = 0;
};
namespace detail {
inline sd_drive_config drive_config(const GenerationConfig& c) {
  return sd_drive_config{c.batch, c.target_len, c.interval, c.cold_start, c.steps, c.load_limit, c.seed, 0};
}
inline std::vector<GenerationRecord> records(sd_drive_result* r) {
  std::vector<GenerationRecord> out(static_cast<std::size_t>(sd_drive_count(r)));
  for (std::size_t i = 0; i < out.size(); ++i) {
    std::int64_t st = 0;
    std::uint64_t sq = 0;
    std::int32_t tk = 0;
    const int rc = sd_drive_record(r, static_cast<std::int64_t>(i), &st, &sq, &tk);
    if (rc != SD_OK) {
      sd_drive_destroy(r);
      check(rc);
    }
    out[i] = GenerationRecord{static_cast<long>(st), sq, tk};
  }
  sd_drive_destroy(r);
  return out;
}
}  // namespace detail

inline std::vector<GenerationRecord> drive_schedule(const GenerationConfig& c, StepComputation& comp) {
  const sd_drive_config cfg = detail::drive_config(c);
  sd_drive_result* r = nullptr;
  check(sd_drive(comp.handle(), &cfg, &r));
  return detail::records(r);
}

// ---- DistributedComputation (workers.cpp:264-501) on NVLink peer memory:
// one process per rank (several may share a device). The peer exchange is
// connected before the first step: setup() writes this rank's CUDA IPC
// handles (SD_DIST_IPC_BYTES), the caller gathers every rank's in rank order
// over its own channel, connect() maps the peers.
enum class ShardMode : int { kBySequence = SD_SHARD_BY_SEQUENCE, kByHead = SD_SHARD_BY_HEAD, kHybrid = SD_SHARD_HYBRID };

// ShardMap::range_of (transport.cpp:354-376): the kv heads a rank's shard holds
inline std::pair<int, int> shard_head_range(ShardMode mode, int heads, int workers, int rank) {
  int h0 = 0, hc = 0;
  check(sd_shardmap_head_range(static_cast<int>(mode), heads, workers, rank, &h0, &hc));
  return {h0, hc};
}

class DistributedComputation {
 public:
  // weights: the S-ranks' weight set (nullptr on pure R-ranks); s_ranks 1 is
  // the paper's single S-worker, s_ranks == world data-parallel S-ranks
  DistributedComputation(WeightSet* weights, KvShard& kv, int rank, int world, int s_ranks,
                         ShardMode mode = ShardMode::kBySequence)
      : world_(world) {
    check(sd_dist_create(weights ? weights->handle() : nullptr, kv.handle(), rank, world, nullptr, s_ranks,
                         static_cast<int>(mode), &h_));
  }
  ~DistributedComputation() {
    if (h_) sd_dist_destroy(h_);
  }
  DistributedComputation(const DistributedComputation&) = delete;
  DistributedComputation& operator=(const DistributedComputation&) = delete;
  std::vector<std::uint8_t> setup(int max_rows) {
    std::vector<std::uint8_t> mine(SD_DIST_IPC_BYTES);
    check(sd_dist_p2p_setup(h_, max_rows, mine.data()));
    return mine;
  }
  void connect(const std::vector<std::uint8_t>& all_ranks) {
    if (all_ranks.size() != static_cast<std::size_t>(world_) * SD_DIST_IPC_BYTES) {
      throw ConfigError("connect: expected world x SD_DIST_IPC_BYTES of handles");
    }
    check(sd_dist_p2p_connect(h_, all_ranks.data()));
  }
  // the reference's pipelined_ (two interleaved mini-batches, seq % 2)
  void set_pipelined(bool on) { check(sd_dist_pipeline(h_, on ? 1 : 0)); }
  sd_dist* handle() const { return h_; }

 private:
  int world_;
  sd_dist* h_ = nullptr;
};

// drive_schedule over the distributed computation: the rows this rank
// produced (its home rows)
inline std::vector<GenerationRecord> drive_schedule(const GenerationConfig& c, DistributedComputation& comp) {
  const sd_drive_config cfg = detail::drive_config(c);
  sd_drive_result* r = nullptr;
  check(sd_dist_drive(comp.handle(), &cfg, &r));
  return detail::records(r);
}

// ---- the remote R-worker (workers.hpp:27-112): an AttentionWorkerSession
// speaking SDWP over a KvShard in HBM, and the blocking serve loop
struct AttentionWorkerConfig {  // workers.hpp:27-30 (+ the device)
  long capacity_tokens = 1 << 20;
  KvFormat storage = KvFormat::kSingle;
  int device = 0;
};
class AttentionWorkerSession {
 public:
  explicit AttentionWorkerSession(const AttentionWorkerConfig& c) {
    check(sd_rworker_create(c.capacity_tokens, static_cast<int>(c.storage), c.device, &h_));
  }
  ~AttentionWorkerSession() {
    if (h_) sd_rworker_destroy(h_);
  }
  AttentionWorkerSession(const AttentionWorkerSession&) = delete;
  AttentionWorkerSession& operator=(const AttentionWorkerSession&) = delete;
  // stream bytes in (any split), the reply frames' bytes out; a fatal
  // framing error (bad magic, oversized frame) throws ProtocolError
  std::vector<std::uint8_t> feed(std::span<const std::uint8_t> bytes) {
    const std::uint8_t* out = nullptr;
    std::size_t n = 0;
    check(sd_rworker_feed(h_, bytes.data(), bytes.size(), &out, &n));
    return std::vector<std::uint8_t>(out, out + n);
  }
  bool shutdown_requested() const {
    std::int32_t b = 0;
    check(sd_rworker_shutdown_requested(h_, &b));
    return b != 0;
  }

 private:
  sd_rworker* h_ = nullptr;
};
struct ServeOptions {  // workers.hpp:68-74
  std::string listen_addr = "127.0.0.1:0";
  std::string port_file;
  bool once = false;
  double recv_timeout_seconds = 0;
  AttentionWorkerConfig worker;
};
// serve_attention_worker (workers.cpp:162-214)
inline int serve_attention_worker(const ServeOptions& o) {
  check(sd_rworker_serve(o.listen_addr.c_str(), o.port_file.empty() ? nullptr : o.port_file.c_str(),
                         o.worker.capacity_tokens, static_cast<int>(o.worker.storage), o.worker.device, o.once ? 1 : 0,
                         o.recv_timeout_seconds));
  return 0;
}

// transcript_csv (workers.cpp:746-755): "step,seq_id,token_id" rows
inline std::string transcript_csv(const std::vector<GenerationRecord>& transcript) {
  std::string csv = "step,seq_id,token_id\n";
  for (const GenerationRecord& rec : transcript) {
    csv += std::to_string(rec.step) + "," + std::to_string(rec.seq) + "," + std::to_string(rec.token) + "\n";
  }
  return csv;
}

}  // namespace sd_b200
