// SDWP, the reference's binary wire protocol between the dense (S) worker
// and the attention (R) workers (transport.hpp / transport.cpp:105-301), and
// a GPU-backed attention-worker session speaking it (AttentionWorkerSession,
// workers.cpp:40-160; serve loop workers.cpp:162-214). A reference
// DistributedComputation on CPUs can drive a B200 R-worker over TCP with
// this: QKV_BATCH frames in, O_BATCH frames out, the KV cache in HBM.
//
//   frame = "SDWP" | version u8 | msg_type u8 | payload_len u32 | payload   (little-endian)
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "kv_store.h"

namespace sd {
namespace sdwp {

constexpr uint8_t kVersion = 1;
constexpr size_t kHeaderBytes = 10;
constexpr size_t kMaxPayload = size_t{64} << 20;

enum MsgType : uint8_t { kHello = 1, kConfig = 2, kQkvBatch = 3, kOBatch = 4, kDropSeq = 5, kShutdown = 6, kError = 7 };
// ERROR payload codes (transport.hpp); equal to the C-ABI status numbering
enum ErrCode : uint16_t {
  kErrBadVersion = 1,
  kErrUnknownType = 2,
  kErrMalformed = 3,
  kErrCapacity = 4,
  kErrUnknownSequence = 5,
  kErrInternal = 6
};
enum Precision : uint8_t { kSingle = 0, kHalf = 1 };

struct Message {
  uint8_t version = kVersion;
  uint8_t type = 0;  // kept raw so unknown values round-trip
  std::vector<uint8_t> payload;
};

std::vector<uint8_t> encode_frame(const Message& m);

// Incremental frame extraction: every prefix of a stream yields complete
// frames followed by need-more or exactly one fatal error (bad magic,
// oversized length); no silent misparse.
class FrameDecoder {
 public:
  enum Status { kFrame, kNeedMore, kFatal };
  void feed(const uint8_t* bytes, size_t n);
  Status poll(Message& out);
  const std::string& error() const { return error_; }

 private:
  std::vector<uint8_t> buf_;
  size_t used_ = 0;
  bool fatal_ = false;
  std::string error_;
};

// QKV_BATCH / O_BATCH payloads: layer u16 | step u32 | count u32 | head_start
// u16 | head_count u16, then per record seq u64 (| position u32) and the
// vectors (fp32, or fp16 RNE bits under kHalf). Rows are kept row-major.
struct Batch {
  uint16_t layer = 0;
  uint32_t step = 0;
  uint16_t head_start = 0, head_count = 0;
  std::vector<uint64_t> seqs;
  std::vector<uint32_t> positions;  // QKV only
  std::vector<float> q, k, v;       // QKV: [n][qw], [n][kw], [n][kw]
  std::vector<float> o;             // O: [n][qw]
};
std::vector<uint8_t> encode_qkv(const Batch& b, int q_width, int kv_width, Precision p);
Batch decode_qkv(const uint8_t* bytes, size_t n, int head_dim, int group, Precision p);
std::vector<uint8_t> encode_o(const Batch& b, int q_width, Precision p);
Batch decode_o(const uint8_t* bytes, size_t n, int head_dim, int group, Precision p);
std::vector<uint8_t> encode_drop(const std::vector<uint64_t>& seqs);
std::vector<uint64_t> decode_drop(const uint8_t* bytes, size_t n);
std::vector<uint8_t> encode_error(uint16_t code, const std::string& message);
Message make_error(uint16_t code, const std::string& message);

// IEEE binary16 round-to-nearest-even (the reference's Eigen::half), host side
uint16_t float_to_half(float f);
float half_to_float(uint16_t h);

// The attention worker backed by a KvStore on `device` (the reference's
// AttentionWorkerConfig: capacity_tokens, storage format).
class WorkerSession {
 public:
  WorkerSession(int64_t capacity_tokens, int kv_format, int device);
  std::vector<Message> handle(const Message& m);
  bool shutdown_requested() const { return shutdown_; }
  void note_idle(double s) { idle_s_ += s; }
  const KvStore* shard() const { return shard_.get(); }

 private:
  std::vector<Message> handle_inner(const Message& m);
  int64_t cap_;
  int fmt_, device_;
  Spec spec_{};
  Precision prec_ = kSingle;
  std::unique_ptr<KvStore> shard_;
  DevBuf dq_, dk_, dv_, doo_;
  bool shutdown_ = false;
  double busy_s_ = 0, idle_s_ = 0;
  int64_t tokens_ = 0;
};

// Blocking TCP service loop (serve_attention_worker, workers.cpp:162-214):
// listen on host:port (port 0 = any), write the bound port to port_file
// when given, serve one connection at a time; once = return after the first
// session ends. Returns 0, or throws sd::Error.
// recv_timeout_seconds > 0: a connection idle that long ends its session
// (ServeOptions::recv_timeout_seconds); 0 blocks forever.
int serve(const std::string& listen_addr, const std::string& port_file, int64_t capacity_tokens, int kv_format,
          int device, bool once, double recv_timeout_seconds = 0);

}  // namespace sdwp
}  // namespace sd
