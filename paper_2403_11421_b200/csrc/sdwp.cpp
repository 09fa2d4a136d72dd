// SDWP codecs and the GPU attention-worker session (see sdwp.h).
#include "sdwp.h"

#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>

namespace sd {
namespace sdwp {

namespace {

const uint8_t kMagic[4] = {'S', 'D', 'W', 'P'};

// ---- little-endian byte streams (ProtocolError on truncation)
struct Writer {
  std::vector<uint8_t>& out;
  void u8(uint8_t v) { out.push_back(v); }
  void u16(uint16_t v) {
    out.push_back(static_cast<uint8_t>(v));
    out.push_back(static_cast<uint8_t>(v >> 8));
  }
  void u32(uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
  }
  void u64(uint64_t v) {
    for (int i = 0; i < 8; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
  }
  void vec(const float* x, int n, Precision p) {
    for (int i = 0; i < n; ++i) {
      if (p == kSingle) {
        uint32_t b;
        std::memcpy(&b, &x[i], 4);
        u32(b);
      } else {
        u16(float_to_half(x[i]));
      }
    }
  }
};

struct Reader {
  const uint8_t* p;
  size_t n, at = 0;
  size_t left() const { return n - at; }
  void need(size_t k) const {
    if (left() < k) fail(SD_ERR_PROTOCOL, "payload truncated");
  }
  uint64_t le(int bytes) {
    need(static_cast<size_t>(bytes));
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(p[at + i]) << (8 * i);
    at += static_cast<size_t>(bytes);
    return v;
  }
  void vec(float* x, int w, Precision pr) {
    for (int i = 0; i < w; ++i) {
      if (pr == kSingle) {
        const uint32_t b = static_cast<uint32_t>(le(4));
        std::memcpy(&x[i], &b, 4);
      } else {
        x[i] = half_to_float(static_cast<uint16_t>(le(2)));
      }
    }
  }
};

void write_prefix(Writer& w, const Batch& b) {
  w.u16(b.layer);
  w.u32(b.step);
  w.u32(static_cast<uint32_t>(b.seqs.size()));
  w.u16(b.head_start);
  w.u16(b.head_count);
}

uint32_t read_prefix(Reader& r, Batch& b, const char* what) {
  b.layer = static_cast<uint16_t>(r.le(2));
  b.step = static_cast<uint32_t>(r.le(4));
  const uint32_t count = static_cast<uint32_t>(r.le(4));
  b.head_start = static_cast<uint16_t>(r.le(2));
  b.head_count = static_cast<uint16_t>(r.le(2));
  if (b.head_count == 0) fail(SD_ERR_PROTOCOL, std::string(what) + ": zero head range");
  return count;
}

// ---- a minimal JSON reader for CONFIG (objects, strings, numbers, bools)
struct Json {
  enum Kind { kNull, kBool, kNum, kStr, kObj } kind = kNull;
  double num = 0;
  bool b = false;
  std::string str;
  std::map<std::string, Json> obj;
  const Json* get(const std::string& k) const {
    auto it = obj.find(k);
    return it == obj.end() ? nullptr : &it->second;
  }
};

struct JsonParser {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r')) ++p;
  }
  [[noreturn]] void bad() { fail(SD_ERR_PROTOCOL, "bad config: malformed JSON"); }
  std::string string() {
    if (p >= e || *p != '"') bad();
    std::string s;
    for (++p; p < e && *p != '"'; ++p) {
      if (*p == '\\') {
        if (++p >= e) bad();
        s += *p == 'n' ? '\n' : *p == 't' ? '\t' : *p;
      } else {
        s += *p;
      }
    }
    if (p >= e) bad();
    ++p;
    return s;
  }
  Json value() {
    ws();
    Json j;
    if (p >= e) bad();
    if (*p == '{') {
      j.kind = Json::kObj;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return j;
      }
      for (;;) {
        ws();
        const std::string k = string();
        ws();
        if (p >= e || *p != ':') bad();
        ++p;
        j.obj[k] = value();
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return j;
        }
        bad();
      }
    }
    if (*p == '"') {
      j.kind = Json::kStr;
      j.str = string();
      return j;
    }
    if (e - p >= 4 && std::strncmp(p, "true", 4) == 0) {
      j.kind = Json::kBool;
      j.b = true;
      p += 4;
      return j;
    }
    if (e - p >= 5 && std::strncmp(p, "false", 5) == 0) {
      j.kind = Json::kBool;
      p += 5;
      return j;
    }
    if (e - p >= 4 && std::strncmp(p, "null", 4) == 0) {
      p += 4;
      return j;
    }
    char* end = nullptr;
    const std::string rest(p, e);
    j.num = std::strtod(rest.c_str(), &end);
    if (end == rest.c_str()) bad();
    j.kind = Json::kNum;
    p += end - rest.c_str();
    return j;
  }
};

int json_int(const Json& j, const char* key) {
  const Json* v = j.get(key);
  if (!v || v->kind != Json::kNum || v->num != std::floor(v->num)) {
    fail(SD_ERR_PROTOCOL, std::string("bad config: missing or non-integer '") + key + "'");
  }
  return static_cast<int>(v->num);
}

const char* format_name(int fmt) {
  return fmt == SD_KV_SINGLE ? "single" : fmt == SD_KV_HALF ? "half" : fmt == SD_KV_INT8 ? "int8" : "int4";
}

// nlohmann::json::dump() of a flat object: keys sorted, no spaces
std::string dump_sorted(const std::map<std::string, std::string>& kv) {
  std::string s = "{";
  for (const auto& [k, v] : kv) {
    if (s.size() > 1) s += ",";
    s += "\"" + k + "\":" + v;
  }
  return s + "}";
}

std::string num(double x) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", x);
  return b;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// IEEE binary16, round to nearest even
uint16_t float_to_half(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t mag = x & 0x7FFFFFFFu;
  if (mag >= 0x7F800000u) return static_cast<uint16_t>(sign | (mag > 0x7F800000u ? 0x7E00u : 0x7C00u));
  if (mag >= 0x477FF000u) return static_cast<uint16_t>(sign | 0x7C00u);  // rounds to >= 65520: inf
  if (mag < 0x38800000u) {                                                // subnormal half (or zero)
    const uint32_t shift = 126u - (mag >> 23);
    if (shift > 24) return static_cast<uint16_t>(sign);
    const uint32_t m = (mag & 0x7FFFFFu) | 0x800000u;
    uint32_t h = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1u))) ++h;
    return static_cast<uint16_t>(sign | h);
  }
  uint32_t h = ((mag >> 13) - (112u << 10));
  const uint32_t rem = mag & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return static_cast<uint16_t>(sign | h);
}

float half_to_float(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1Fu, man = h & 0x3FFu, x;
  if (exp == 0) {
    if (man == 0) {
      x = sign;
    } else {
      int e = -1;
      do {
        ++e;
        man <<= 1;
      } while (!(man & 0x400u));
      x = sign | ((112u - static_cast<uint32_t>(e)) << 23) | ((man & 0x3FFu) << 13);
    }
  } else if (exp == 31) {
    x = sign | 0x7F800000u | (man << 13);
  } else {
    x = sign | ((exp + 112u) << 23) | (man << 13);
  }
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}

std::vector<uint8_t> encode_frame(const Message& m) {
  if (m.payload.size() > kMaxPayload) fail(SD_ERR_PROTOCOL, "payload exceeds the frame size limit");
  std::vector<uint8_t> out(kMagic, kMagic + 4);
  out.reserve(kHeaderBytes + m.payload.size());
  Writer w{out};
  w.u8(m.version);
  w.u8(m.type);
  w.u32(static_cast<uint32_t>(m.payload.size()));
  out.insert(out.end(), m.payload.begin(), m.payload.end());
  return out;
}

void FrameDecoder::feed(const uint8_t* bytes, size_t n) {
  if (used_ > 0 && used_ == buf_.size()) {
    buf_.clear();
    used_ = 0;
  }
  buf_.insert(buf_.end(), bytes, bytes + n);
}

FrameDecoder::Status FrameDecoder::poll(Message& out) {
  if (fatal_) return kFatal;
  const size_t avail = buf_.size() - used_;
  if (avail < kHeaderBytes) return kNeedMore;
  const uint8_t* p = buf_.data() + used_;
  if (std::memcmp(p, kMagic, 4) != 0) {
    fatal_ = true;
    error_ = "bad magic";
    return kFatal;
  }
  uint32_t len = 0;
  for (int i = 0; i < 4; ++i) len |= static_cast<uint32_t>(p[6 + i]) << (8 * i);
  if (len > kMaxPayload) {
    fatal_ = true;
    error_ = "frame length " + std::to_string(len) + " exceeds the limit";
    return kFatal;
  }
  if (avail < kHeaderBytes + len) return kNeedMore;
  out.version = p[4];
  out.type = p[5];
  out.payload.assign(p + kHeaderBytes, p + kHeaderBytes + len);
  used_ += kHeaderBytes + len;
  return kFrame;
}

std::vector<uint8_t> encode_qkv(const Batch& b, int qw, int kw, Precision p) {
  std::vector<uint8_t> out;
  Writer w{out};
  write_prefix(w, b);
  for (size_t i = 0; i < b.seqs.size(); ++i) {
    w.u64(b.seqs[i]);
    w.u32(b.positions[i]);
    w.vec(b.q.data() + i * qw, qw, p);
    w.vec(b.k.data() + i * kw, kw, p);
    w.vec(b.v.data() + i * kw, kw, p);
  }
  return out;
}

Batch decode_qkv(const uint8_t* bytes, size_t n, int head_dim, int group, Precision p) {
  Reader r{bytes, n};
  Batch b;
  const uint32_t count = read_prefix(r, b, "qkv batch");
  const int kw = b.head_count * head_dim, qw = kw * group;
  const size_t rec = 12 + static_cast<size_t>(qw + 2 * kw) * (p == kSingle ? 4 : 2);
  if (r.left() != count * rec) fail(SD_ERR_PROTOCOL, "qkv batch: payload size does not match count");
  b.seqs.resize(count);
  b.positions.resize(count);
  b.q.resize(static_cast<size_t>(count) * qw);
  b.k.resize(static_cast<size_t>(count) * kw);
  b.v.resize(static_cast<size_t>(count) * kw);
  for (uint32_t i = 0; i < count; ++i) {
    b.seqs[i] = r.le(8);
    b.positions[i] = static_cast<uint32_t>(r.le(4));
    r.vec(b.q.data() + static_cast<size_t>(i) * qw, qw, p);
    r.vec(b.k.data() + static_cast<size_t>(i) * kw, kw, p);
    r.vec(b.v.data() + static_cast<size_t>(i) * kw, kw, p);
  }
  return b;
}

std::vector<uint8_t> encode_o(const Batch& b, int qw, Precision p) {
  std::vector<uint8_t> out;
  Writer w{out};
  write_prefix(w, b);
  for (size_t i = 0; i < b.seqs.size(); ++i) {
    w.u64(b.seqs[i]);
    w.vec(b.o.data() + i * qw, qw, p);
  }
  return out;
}

Batch decode_o(const uint8_t* bytes, size_t n, int head_dim, int group, Precision p) {
  Reader r{bytes, n};
  Batch b;
  const uint32_t count = read_prefix(r, b, "o batch");
  const int qw = b.head_count * head_dim * group;
  const size_t rec = 8 + static_cast<size_t>(qw) * (p == kSingle ? 4 : 2);
  if (r.left() != count * rec) fail(SD_ERR_PROTOCOL, "o batch: payload size does not match count");
  b.seqs.resize(count);
  b.o.resize(static_cast<size_t>(count) * qw);
  for (uint32_t i = 0; i < count; ++i) {
    b.seqs[i] = r.le(8);
    r.vec(b.o.data() + static_cast<size_t>(i) * qw, qw, p);
  }
  return b;
}

std::vector<uint8_t> encode_drop(const std::vector<uint64_t>& seqs) {
  std::vector<uint8_t> out;
  Writer w{out};
  w.u32(static_cast<uint32_t>(seqs.size()));
  for (uint64_t q : seqs) w.u64(q);
  return out;
}

std::vector<uint64_t> decode_drop(const uint8_t* bytes, size_t n) {
  Reader r{bytes, n};
  const uint32_t count = static_cast<uint32_t>(r.le(4));
  if (r.left() != static_cast<size_t>(count) * 8u) fail(SD_ERR_PROTOCOL, "drop: payload size does not match count");
  std::vector<uint64_t> seqs(count);
  for (uint32_t i = 0; i < count; ++i) seqs[i] = r.le(8);
  return seqs;
}

std::vector<uint8_t> encode_error(uint16_t code, const std::string& message) {
  std::vector<uint8_t> out;
  Writer w{out};
  w.u16(code);
  w.u32(static_cast<uint32_t>(message.size()));
  out.insert(out.end(), message.begin(), message.end());
  return out;
}

Message make_error(uint16_t code, const std::string& message) {
  Message m;
  m.type = kError;
  m.payload = encode_error(code, message);
  return m;
}

// ------------------------------------------------------------- session ---
WorkerSession::WorkerSession(int64_t capacity_tokens, int kv_format, int device)
    : cap_(capacity_tokens), fmt_(kv_format), device_(device) {
  if (capacity_tokens < 1) fail(SD_ERR_CONFIG, "shard capacity must be >= 1");
  if (kv_format < SD_KV_SINGLE || kv_format > SD_KV_INT4) fail(SD_ERR_CONFIG, "unknown kv storage format");
}

std::vector<Message> WorkerSession::handle(const Message& m) {
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<Message> r = handle_inner(m);
  busy_s_ += seconds_since(t0);
  return r;
}

std::vector<Message> WorkerSession::handle_inner(const Message& m) {
  if (m.version != kVersion) {
    return {make_error(kErrBadVersion, "unsupported version " + std::to_string(m.version) +
                                           "; this worker speaks version " + std::to_string(kVersion))};
  }
  Message reply;
  switch (m.type) {
    case kHello:
      reply.type = kHello;
      return {reply};
    case kConfig: {
      try {
        JsonParser jp{reinterpret_cast<const char*>(m.payload.data()),
                      reinterpret_cast<const char*>(m.payload.data()) + m.payload.size()};
        const Json j = jp.value();
        const Json* model = j.get("model");
        if (!model || model->kind != Json::kObj) fail(SD_ERR_PROTOCOL, "bad config: missing 'model'");
        const int hkv = model->get("num_kv_heads") ? json_int(*model, "num_kv_heads") : 0;  // GQA extension
        spec_ = make_spec(json_int(*model, "num_layers"), json_int(*model, "model_dim"), json_int(*model, "num_heads"),
                          json_int(*model, "mlp_dim"), json_int(*model, "vocab_size"), hkv);
        if (model->get("head_dim") && json_int(*model, "head_dim") != spec_.hd) {
          fail(SD_ERR_CONFIG, "head_dim inconsistent with model_dim / num_heads");
        }
        const int h0 = json_int(j, "head_start"), hc = json_int(j, "head_count");
        const Json* wp = j.get("wire_precision");
        prec_ = kSingle;
        if (wp) {
          if (wp->kind != Json::kStr || (wp->str != "single" && wp->str != "half")) {
            fail(SD_ERR_CONFIG, "unknown wire precision: " + (wp->kind == Json::kStr ? wp->str : std::string("?")));
          }
          prec_ = wp->str == "half" ? kHalf : kSingle;
        }
        shard_.reset();
        shard_ = std::make_unique<KvStore>(spec_, h0, hc, cap_, fmt_, device_, nullptr);
        const std::string ack = dump_sorted({{"capacity_tokens", std::to_string(cap_)},
                                             {"ok", "true"},
                                             {"storage_format", std::string("\"") + format_name(fmt_) + "\""},
                                             {"width", std::to_string(shard_->width())}});
        reply.type = kConfig;
        reply.payload.assign(ack.begin(), ack.end());
        return {reply};
      } catch (const Error& e) {
        return {make_error(kErrMalformed, std::string("bad config: ") + e.what())};
      }
    }
    case kQkvBatch: {
      if (!shard_) return {make_error(kErrMalformed, "QKV before CONFIG")};
      try {
        const int G = shard_->group_size();
        Batch b = decode_qkv(m.payload.data(), m.payload.size(), spec_.hd, G, prec_);
        if (b.head_start != shard_->head_start() || b.head_count * spec_.hd != shard_->width()) {
          return {make_error(kErrMalformed, "head range does not match this shard")};
        }
        const int n = static_cast<int>(b.seqs.size());
        const int kw = shard_->width(), qw = shard_->q_width();
        Batch o;
        o.layer = b.layer;
        o.step = b.step;
        o.head_start = b.head_start;
        o.head_count = b.head_count;
        o.seqs = b.seqs;
        o.o.assign(static_cast<size_t>(n) * qw, 0.0f);
        if (n > 0) {
          DeviceGuard dg(device_);
          float* dq = static_cast<float*>(dq_.get(b.q.size() * 4));
          float* dk = static_cast<float*>(dk_.get(b.k.size() * 4));
          float* dv = static_cast<float*>(dv_.get(b.v.size() * 4));
          float* dout = static_cast<float*>(doo_.get(o.o.size() * 4));
          SD_CUDA(cudaMemcpy(dq, b.q.data(), b.q.size() * 4, cudaMemcpyHostToDevice));
          SD_CUDA(cudaMemcpy(dk, b.k.data(), b.k.size() * 4, cudaMemcpyHostToDevice));
          SD_CUDA(cudaMemcpy(dv, b.v.data(), b.v.size() * 4, cudaMemcpyHostToDevice));
          // append_request then attend (the worker's QKV handler, workers.cpp:110-111)
          shard_->append(b.layer, n, b.seqs.data(), b.positions.data(), dk, kw, dv, kw, nullptr);
          shard_->attend(b.layer, n, b.seqs.data(), dq, qw, dout, qw, nullptr);
          SD_CUDA(cudaMemcpy(o.o.data(), dout, o.o.size() * 4, cudaMemcpyDeviceToHost));
        }
        tokens_ += n;
        reply.type = kOBatch;
        reply.payload = encode_o(o, qw, prec_);
        return {reply};
      } catch (const Error& e) {
        const uint16_t code = e.code == SD_ERR_CAPACITY     ? kErrCapacity
                              : e.code == SD_ERR_UNKNOWN_SEQ ? kErrUnknownSequence
                              : e.code == SD_ERR_PROTOCOL    ? kErrMalformed
                                                             : kErrInternal;
        if (code == kErrInternal) throw;
        return {make_error(code, e.what())};
      }
    }
    case kDropSeq: {
      if (!shard_) return {};
      try {
        for (uint64_t q : decode_drop(m.payload.data(), m.payload.size())) shard_->drop(q);
      } catch (const Error& e) {
        return {make_error(kErrMalformed, e.what())};
      }
      return {};  // fire-and-forget
    }
    case kShutdown: {
      shutdown_ = true;
      const std::string stats = dump_sorted({{"busy_seconds", num(busy_s_)},
                                             {"drop_warnings", std::to_string(shard_ ? shard_->warnings() : 0)},
                                             {"idle_seconds", num(idle_s_)},
                                             {"tokens_processed", std::to_string(tokens_)}});
      reply.type = kShutdown;
      reply.payload.assign(stats.begin(), stats.end());
      return {reply};
    }
    case kError:
      return {};  // peer-reported problem; nothing to reply
    case kOBatch:
      return {make_error(kErrUnknownType, "unexpected O_BATCH at the worker")};
    default:
      return {make_error(kErrUnknownType, "unknown message type " + std::to_string(m.type))};
  }
}

// ---------------------------------------------------------------- serve ---
int serve(const std::string& listen_addr, const std::string& port_file, int64_t capacity_tokens, int kv_format,
          int device, bool once, double recv_timeout_seconds) {
  const size_t colon = listen_addr.rfind(':');
  if (colon == std::string::npos) fail(SD_ERR_CONFIG, "listen address must be host:port");
  const std::string host = listen_addr.substr(0, colon);
  const int port = std::atoi(listen_addr.c_str() + colon + 1);
  const int lfd = ::socket(AF_INET, SOCK_STREAM, 0);
  if (lfd < 0) fail(SD_ERR_PROTOCOL, std::string("socket: ") + std::strerror(errno));
  const int one = 1;
  ::setsockopt(lfd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
  sockaddr_in addr{};
  addr.sin_family = AF_INET;
  addr.sin_port = htons(static_cast<uint16_t>(port));
  if (inet_pton(AF_INET, host.c_str(), &addr.sin_addr) != 1) {
    ::close(lfd);
    fail(SD_ERR_CONFIG, "invalid address: " + host);
  }
  if (::bind(lfd, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0 || ::listen(lfd, 4) != 0) {
    const std::string err = std::strerror(errno);
    ::close(lfd);
    fail(SD_ERR_PROTOCOL, "bind/listen " + listen_addr + ": " + err);
  }
  socklen_t alen = sizeof(addr);
  ::getsockname(lfd, reinterpret_cast<sockaddr*>(&addr), &alen);
  if (!port_file.empty()) {
    std::ofstream f(port_file);
    f << ntohs(addr.sin_port) << "\n";
  }
  std::fprintf(stderr, "attention worker (B200) listening on port %d (capacity %lld, %s)\n", ntohs(addr.sin_port),
               static_cast<long long>(capacity_tokens), format_name(kv_format));
  std::vector<uint8_t> buf(1 << 16);
  for (;;) {
    const int fd = ::accept(lfd, nullptr, nullptr);
    if (fd < 0) {
      if (errno == EINTR) continue;
      ::close(lfd);
      fail(SD_ERR_PROTOCOL, std::string("accept: ") + std::strerror(errno));
    }
    ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
    WorkerSession session(capacity_tokens, kv_format, device);
    FrameDecoder dec;
    bool over = false;
    while (!over) {
      const auto t0 = std::chrono::steady_clock::now();
      if (recv_timeout_seconds > 0) {
        pollfd pfd{fd, POLLIN, 0};
        const int pr = ::poll(&pfd, 1, static_cast<int>(recv_timeout_seconds * 1000.0));
        if (pr == 0) {
          std::fprintf(stderr, "worker: receive timed out after %.1f s\n", recv_timeout_seconds);
          break;
        }
      }
      const ssize_t n = ::recv(fd, buf.data(), buf.size(), 0);
      session.note_idle(seconds_since(t0));
      if (n <= 0) break;  // peer closed (or error)
      dec.feed(buf.data(), static_cast<size_t>(n));
      Message m;
      for (;;) {
        const FrameDecoder::Status st = dec.poll(m);
        if (st == FrameDecoder::kNeedMore) break;
        if (st == FrameDecoder::kFatal) {
          std::fprintf(stderr, "worker: fatal protocol error: %s\n", dec.error().c_str());
          over = true;
          break;
        }
        for (const Message& r : session.handle(m)) {
          const std::vector<uint8_t> bytes = encode_frame(r);
          size_t sent = 0;
          while (sent < bytes.size()) {
            const ssize_t k = ::send(fd, bytes.data() + sent, bytes.size() - sent, MSG_NOSIGNAL);
            if (k <= 0) {
              over = true;
              break;
            }
            sent += static_cast<size_t>(k);
          }
        }
        if (session.shutdown_requested()) {
          over = true;
          break;
        }
      }
    }
    ::close(fd);
    if (once) break;
  }
  ::close(lfd);
  return 0;
}

}  // namespace sdwp
}  // namespace sd
