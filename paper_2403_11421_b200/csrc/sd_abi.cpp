// extern "C" boundary (include/sd_abi.h): argument checks, exception ->
// status mapping, host<->device staging for the host-pointer entry points.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "dist.h"
#include "perf_bench.h"
#include "planner.h"
#include "engine.h"
#include "sdwp.h"
#include "kv_store.h"
#include "sd_common.h"

struct sd_rworker {
  std::unique_ptr<sd::sdwp::WorkerSession> s;
  sd::sdwp::FrameDecoder dec;
  std::vector<uint8_t> out;  // reply frames of the last feed
};
struct sd_kv {
  std::unique_ptr<sd::KvStore> s;
  sd::DevBuf qb, kb, vb, ob;  // staging for host-pointer calls
};
struct sd_weights {
  std::unique_ptr<sd::Weights> w;
};
struct sd_engine {
  std::unique_ptr<sd::Engine> e;
  sd_weights* w;
  sd_kv* kv;
};
struct sd_drive_result {
  sd::DriveResult r;
};
struct sd_dist {
  std::unique_ptr<sd::DistEngine> d;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SD_OK;
  } catch (const sd::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SD_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SD_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) sd::fail(SD_ERR_CONFIG, std::string("null argument: ") + what);
}

// copy host rows to a device staging buffer
float* stage(sd::DevBuf& b, const float* host, size_t floats) {
  float* d = static_cast<float*>(b.get(floats * 4 + 16));
  if (floats) SD_CUDA(cudaMemcpy(d, host, floats * 4, cudaMemcpyHostToDevice));
  return d;
}

}  // namespace

extern "C" {

const char* sd_last_error(void) { return g_err.c_str(); }
int sd_abi_version(void) { return SD_ABI_VERSION; }

int sd_make_model_spec(int L, int D, int H, int F, int V, int Hkv, sd_model_spec* out) {
  return guard([&] {
    need(out, "out");
    sd::Spec s = sd::make_spec(L, D, H, F, V, Hkv);
    *out = sd_model_spec{s.L, s.D, s.H, s.hd, s.F, s.V, s.Hkv};
  });
}

uint64_t sd_mix64(uint64_t x) { return sd::mix64(x); }
int sd_prompt_token(uint64_t seed, uint64_t seq, int vocab) {
  if (vocab < 1) return -1;
  return static_cast<int>(sd::mix64(seed ^ sd::mix64(seq)) % static_cast<uint64_t>(vocab));
}

// ------------------------------------------------------------------ KV ----
int sd_kv_create(const sd_model_spec* spec, int head_start, int head_count, int64_t cap,
                 int fmt, int device, const sd_kv_options* opts, sd_kv** out) {
  return guard([&] {
    need(out, "out");
    sd::Spec s = sd::from_abi(spec);
    auto h = std::make_unique<sd_kv>();
    h->s = std::make_unique<sd::KvStore>(s, head_start, head_count, cap, fmt, device, opts);
    *out = h.release();
  });
}

int sd_kv_destroy(sd_kv* kv) {
  return guard([&] {
    if (!kv) return;
    sd::DeviceGuard dg(kv->s->device());
    delete kv;
  });
}

int sd_kv_append(sd_kv* kv, uint64_t seq, int layer, uint32_t position, const float* k,
                 const float* v) {
  return guard([&] {
    need(kv, "kv");
    need(k, "k");
    need(v, "v");
    sd::DeviceGuard dg(kv->s->device());
    const int w = kv->s->width();
    float* dk = stage(kv->kb, k, static_cast<size_t>(w));
    float* dv = stage(kv->vb, v, static_cast<size_t>(w));
    kv->s->append(layer, 1, &seq, &position, dk, w, dv, w, nullptr);
    SD_CUDA(cudaDeviceSynchronize());
  });
}

int sd_kv_append_request(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                         const uint32_t* pos, const float* k, const float* v) {
  return guard([&] {
    need(kv, "kv");
    if (n < 0) sd::fail(SD_ERR_CONFIG, "negative item count");
    if (n > 0) {
      need(seqs, "seqs");
      need(pos, "positions");
      need(k, "k");
      need(v, "v");
    }
    sd::DeviceGuard dg(kv->s->device());
    const int w = kv->s->width();
    float* dk = stage(kv->kb, k, static_cast<size_t>(n) * w);
    float* dv = stage(kv->vb, v, static_cast<size_t>(n) * w);
    int rc = SD_OK;
    std::string msg;
    try {
      kv->s->append(layer, n, seqs, pos, dk, w, dv, w, nullptr);
    } catch (const sd::Error& e) {
      rc = e.code;
      msg = e.what();
    }
    SD_CUDA(cudaDeviceSynchronize());
    if (rc) sd::fail(rc, msg);
  });
}

int sd_kv_attend(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs, const float* q,
                 float* o) {
  return guard([&] {
    need(kv, "kv");
    if (n < 0) sd::fail(SD_ERR_CONFIG, "negative item count");
    if (n > 0) {
      need(seqs, "seqs");
      need(q, "q");
      need(o, "o");
    }
    sd::DeviceGuard dg(kv->s->device());
    const int qw = kv->s->q_width();
    float* dq = stage(kv->qb, q, static_cast<size_t>(n) * qw);
    float* dout = static_cast<float*>(kv->ob.get(static_cast<size_t>(n) * qw * 4 + 16));
    kv->s->attend(layer, n, seqs, dq, qw, dout, qw, nullptr);
    if (n) SD_CUDA(cudaMemcpy(o, dout, static_cast<size_t>(n) * qw * 4, cudaMemcpyDeviceToHost));
    SD_CUDA(cudaDeviceSynchronize());
  });
}

int sd_kv_append_attend(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                        const uint32_t* pos, const float* q, const float* k, const float* v,
                        float* o) {
  const int rc = sd_kv_append_request(kv, layer, n, seqs, pos, k, v);
  if (rc) return rc;
  return sd_kv_attend(kv, layer, n, seqs, q, o);
}

int sd_kv_append_request_dev(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                             const uint32_t* pos, const float* k, const float* v, void* stream) {
  return guard([&] {
    need(kv, "kv");
    if (n < 0) sd::fail(SD_ERR_CONFIG, "negative item count");
    sd::DeviceGuard dg(kv->s->device());
    const int w = kv->s->width();
    kv->s->append(layer, n, seqs, pos, k, w, v, w, static_cast<cudaStream_t>(stream));
  });
}

int sd_kv_attend_dev(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs, const float* q,
                     float* o, void* stream) {
  return guard([&] {
    need(kv, "kv");
    if (n < 0) sd::fail(SD_ERR_CONFIG, "negative item count");
    sd::DeviceGuard dg(kv->s->device());
    const int qw = kv->s->q_width();
    kv->s->attend(layer, n, seqs, q, qw, o, qw, static_cast<cudaStream_t>(stream));
  });
}

int sd_kv_append_attend_dev(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                            const uint32_t* pos, const float* q, const float* k, const float* v,
                            float* o, void* stream) {
  const int rc = sd_kv_append_request_dev(kv, layer, n, seqs, pos, k, v, stream);
  if (rc) return rc;
  return sd_kv_attend_dev(kv, layer, n, seqs, q, o, stream);
}

int sd_kv_drop(sd_kv* kv, int32_t n, const uint64_t* seqs) {
  return guard([&] {
    need(kv, "kv");
    for (int i = 0; i < n; ++i) kv->s->drop(seqs[i]);
  });
}

int sd_kv_stored_length(const sd_kv* kv, uint64_t seq, int layer, int32_t* out) {
  return guard([&] {
    need(kv, "kv");
    need(out, "out");
    *out = kv->s->stored(seq, layer);
  });
}
int sd_kv_has_sequence(const sd_kv* kv, uint64_t seq, int32_t* out) {
  return guard([&] {
    need(kv, "kv");
    need(out, "out");
    *out = kv->s->has(seq) ? 1 : 0;
  });
}
int sd_kv_token_count(const sd_kv* kv, int64_t* out) {
  return guard([&] {
    need(kv, "kv");
    need(out, "out");
    *out = kv->s->token_count();
  });
}
int sd_kv_warning_count(const sd_kv* kv, int32_t* out) {
  return guard([&] {
    need(kv, "kv");
    need(out, "out");
    *out = kv->s->warnings();
  });
}
int sd_kv_bytes_per_token(const sd_kv* kv, int64_t* out) {
  return guard([&] {
    need(kv, "kv");
    need(out, "out");
    *out = kv->s->bytes_per_token();
  });
}
int sd_kv_width(const sd_kv* kv, int32_t* width, int32_t* q_width) {
  return guard([&] {
    need(kv, "kv");
    if (width) *width = kv->s->width();
    if (q_width) *q_width = kv->s->q_width();
  });
}

int64_t sd_kv_export_lane(const sd_kv* kv, uint64_t seq, int layer, int which, void* host,
                          size_t host_bytes, float* scales, size_t scales_count) {
  int64_t r = 0;
  const int rc = guard([&] {
    need(kv, "kv");
    r = kv->s->export_lane(seq, layer, which, host, host_bytes, scales, scales_count);
  });
  return rc ? -rc : r;
}

int sd_kv_prefill_synthetic(sd_kv* kv, int32_t n, const uint64_t* seqs, int32_t length,
                            uint64_t salt) {
  return guard([&] {
    need(kv, "kv");
    sd::DeviceGuard dg(kv->s->device());
    kv->s->prefill_synthetic(n, seqs, length, salt, nullptr);
  });
}

int sd_kv_timing(sd_kv* kv, int enable) {
  return guard([&] {
    need(kv, "kv");
    kv->s->set_timing(enable < 0 ? 0 : enable);
  });
}

int sd_kv_timing_read(sd_kv* kv, double* ms, int64_t* launches, double* bytes, int reset) {
  return guard([&] {
    need(kv, "kv");
    kv->s->read_timing(ms, launches, bytes, reset != 0);
  });
}

// --------------------------------------------------------------- S-Part ---
int sd_weights_upload(const sd_model_spec* spec, const float* const* tensors, int mode,
                      int device, sd_weights** out) {
  return guard([&] {
    need(out, "out");
    sd::Spec s = sd::from_abi(spec);
    auto h = std::make_unique<sd_weights>();
    if (tensors) {
      for (int i = 0; i < 2 + 6 * s.L; ++i) need(tensors[i], "tensor");
      h->w = std::make_unique<sd::Weights>(s, tensors, mode, device);
    } else {
      // NULL tensors: device-generated synthetic weights (seed 0)
      h->w = std::make_unique<sd::Weights>(s, mode, 0, device);
    }
    *out = h.release();
  });
}

int sd_weights_destroy(sd_weights* w) {
  return guard([&] { delete w; });
}

namespace {
struct Scratch {
  sd::DevBuf a, b, c, d, ab, cb;
};
thread_local Scratch g_scr;

// run one linear from host buffers: y = x W^T (+epi)
void host_linear(sd_weights* w, int layer, int which, int B, const float* x, float* y, int epi,
                 const float* res) {
  const sd::Weights& W = *w->w;
  sd::DeviceGuard dg(W.device());
  const int in = W.in_dim(which), out = W.out_dim(which);
  const size_t bp = static_cast<size_t>((B + 127) / 128 * 128);
  float* dx = static_cast<float*>(g_scr.a.get(bp * in * 4));
  SD_CUDA(cudaMemset(dx, 0, bp * in * 4));
  SD_CUDA(cudaMemcpy(dx, x, static_cast<size_t>(B) * in * 4, cudaMemcpyHostToDevice));
  float* dy = static_cast<float*>(g_scr.b.get(bp * out * 4));
  const float* dr = nullptr;
  if (res) dr = stage(g_scr.c, res, static_cast<size_t>(B) * out);
  sd::act16* dxb = nullptr;
  if (W.mode() == SD_DENSE_BF16 || W.mode() == SD_DENSE_F16) {
    dxb = static_cast<sd::act16*>(g_scr.ab.get(bp * in * 2));
    SD_CUDA(cudaMemset(dxb, 0, bp * in * 2));
    sd::launch_to_16(B, in, dx, in, dxb, in, W.mode() == SD_DENSE_F16, nullptr);
  }
  W.linear(layer, which, B, dx, in, dxb, in, dy, out, nullptr, 0, epi, dr, out, nullptr);
  SD_CUDA(cudaMemcpy(y, dy, static_cast<size_t>(B) * out * 4, cudaMemcpyDeviceToHost));
  SD_CUDA(cudaDeviceSynchronize());
}
}  // namespace

int sd_s_project_qkv(sd_weights* w, int layer, int32_t B, const float* x, float* q, float* k,
                     float* v) {
  return guard([&] {
    need(w, "weights");
    if (B < 1) sd::fail(SD_ERR_CONFIG, "project_qkv: empty batch");
    const sd::Spec& s = w->w->spec();
    std::vector<float> y(static_cast<size_t>(B) * s.qkv_width());
    host_linear(w, layer, 0, B, x, y.data(), sd::kEpiNone, nullptr);
    const int D = s.D, kvw = s.kv_width(), qw = s.qkv_width();
    for (int b = 0; b < B; ++b) {
      std::memcpy(q + static_cast<size_t>(b) * D, y.data() + static_cast<size_t>(b) * qw, D * 4);
      std::memcpy(k + static_cast<size_t>(b) * kvw, y.data() + static_cast<size_t>(b) * qw + D, kvw * 4);
      std::memcpy(v + static_cast<size_t>(b) * kvw, y.data() + static_cast<size_t>(b) * qw + D + kvw, kvw * 4);
    }
  });
}

int sd_s_finish_block(sd_weights* w, int layer, int32_t B, const float* o, const float* res,
                      float* x_out) {
  return guard([&] {
    need(w, "weights");
    const sd::Spec& s = w->w->spec();
    std::vector<float> y(static_cast<size_t>(B) * s.D), h(static_cast<size_t>(B) * s.F);
    host_linear(w, layer, 4, B, o, y.data(), sd::kEpiResidual, res);
    host_linear(w, layer, 5, B, y.data(), h.data(), sd::kEpiSilu, nullptr);
    host_linear(w, layer, 6, B, h.data(), x_out, sd::kEpiResidual, y.data());
  });
}

int sd_s_logits_argmax(sd_weights* w, int32_t B, const float* x, float* logits, int32_t* tokens) {
  return guard([&] {
    need(w, "weights");
    const sd::Spec& s = w->w->spec();
    std::vector<float> lg(static_cast<size_t>(B) * s.V);
    host_linear(w, 0, 7, B, x, lg.data(), sd::kEpiNone, nullptr);
    if (logits) std::memcpy(logits, lg.data(), lg.size() * 4);
    if (tokens) {
      sd::DeviceGuard dg(w->w->device());
      float* dl = stage(g_scr.d, lg.data(), lg.size());
      int32_t* dt = static_cast<int32_t*>(g_scr.cb.get(static_cast<size_t>(B) * 4 + 16));
      sd::launch_argmax(B, s.V, dl, s.V, dt, nullptr);
      SD_CUDA(cudaMemcpy(tokens, dt, static_cast<size_t>(B) * 4, cudaMemcpyDeviceToHost));
    }
  });
}

int sd_s_apply_linear(sd_weights* w, int layer, int which, int32_t B, const float* x, float* y) {
  return guard([&] {
    need(w, "weights");
    if (which < 0 || which > 7) sd::fail(SD_ERR_CONFIG, "bad weight index");
    if (which >= 1 && which <= 3) {
      const sd::Spec& s = w->w->spec();
      std::vector<float> q(static_cast<size_t>(B) * s.D), k(static_cast<size_t>(B) * s.kv_width()),
          v(k.size());
      int rc = sd_s_project_qkv(w, layer, B, x, q.data(), k.data(), v.data());
      if (rc) sd::fail(rc, g_err);
      const std::vector<float>& src = which == 1 ? q : which == 2 ? k : v;
      std::memcpy(y, src.data(), src.size() * 4);
      return;
    }
    host_linear(w, layer, which, B, x, y, sd::kEpiNone, nullptr);
  });
}

int sd_gemm_dev(int kind, int M, int N, int K, const void* A, int64_t lda, const void* B,
                int64_t ldb, float* C, int64_t ldc, void* Cb, int64_t ldcb, int epi,
                const float* res, int64_t ldr, void* stream) {
  return guard([&] {
    sd::GemmArgs g{};
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.B = B;
    g.ldb = ldb;
    g.C = C;
    g.ldc = ldc;
    g.Cb = static_cast<sd::act16*>(Cb);
    g.ldcb = ldcb;
    g.epi = epi;
    g.res = res;
    g.ldr = ldr;
    g.kind = kind;
    if (!sd::gemm_sm100_supported(g)) sd::fail(SD_ERR_CONFIG, "sd_gemm_dev: unsupported shape/alignment");
    if (epi == sd::kEpiResidual && !res) sd::fail(SD_ERR_CONFIG, "sd_gemm_dev: residual epilogue needs res");
    sd::launch_gemm_sm100(g, static_cast<cudaStream_t>(stream));
  });
}

// --------------------------------------------------------------- engine ---
int sd_engine_create(sd_weights* w, sd_kv* kv, sd_engine** out) {
  return guard([&] {
    need(w, "weights");
    need(kv, "kv");
    need(out, "out");
    auto h = std::make_unique<sd_engine>();
    h->e = std::make_unique<sd::Engine>(w->w.get(), kv->s.get());
    h->w = w;
    h->kv = kv;
    *out = h.release();
  });
}

int sd_engine_destroy(sd_engine* e) {
  return guard([&] { delete e; });
}

int sd_engine_step(sd_engine* e, int32_t B, const uint64_t* seqs, const int32_t* tokens,
                   int32_t* next, float* final_x) {
  return guard([&] {
    need(e, "engine");
    need(tokens, "tokens");
    e->e->step(B, seqs, tokens, nullptr, next, final_x, nullptr);
  });
}

int sd_engine_step_features(sd_engine* e, int32_t B, const uint64_t* seqs, const float* x,
                            int32_t* next, float* final_x, float* logits) {
  return guard([&] {
    need(e, "engine");
    need(x, "features");
    e->e->step(B, seqs, nullptr, x, next, final_x, logits);
  });
}

int sd_engine_retire(sd_engine* e, int32_t n, const uint64_t* seqs) {
  return guard([&] {
    need(e, "engine");
    e->e->retire(n, seqs);
  });
}

int sd_engine_bench(sd_engine* e, int32_t B, const uint64_t* seqs, const int32_t* tokens,
                    int32_t steps, int32_t* next, double* ms) {
  return guard([&] {
    need(e, "engine");
    need(ms, "ms");
    *ms = e->e->bench(B, seqs, tokens, steps, next);
  });
}

int sd_engine_timing(sd_engine* e, int enable) {
  return guard([&] {
    need(e, "engine");
    e->e->set_timing(enable < 0 ? 0 : enable);
  });
}

int sd_engine_timing_read(sd_engine* e, double* ms, double* flops, int64_t* launches, int reset) {
  return guard([&] {
    need(e, "engine");
    e->e->read_timing(ms, flops, launches, reset != 0);
  });
}

int64_t sd_launch_count(void) { return sd::g_launches.load(); }

int sd_engine_pipeline(sd_engine* e, int enable, int r_sms) {
  return guard([&] {
    need(e, "engine");
    e->e->set_pipeline(enable != 0, r_sms);
  });
}

int sd_tune(const char* name, int value) {
  return guard([&] {
    need(name, "name");
    sd::Tuning& t = sd::tuning();
    const std::string n(name);
    int* f = n == "gemm_bn"        ? &t.gemm_bn
             : n == "gemm_pair"    ? &t.gemm_pair
             : n == "fused_append" ? &t.fused_append
             : n == "fused_argmax" ? &t.fused_argmax
             : n == "dist_fuse"    ? &t.dist_fuse
             : n == "attn_mma"     ? &t.attn_mma
             : n == "pdl"          ? &t.pdl
             : n == "dist_phases"  ? &t.dist_phases
             : n == "attn_i8_quad" ? &t.attn_i8_quad
             : n == "attn_l2_prefetch" ? &t.attn_l2_prefetch
             : n == "attn_max_stages" ? &t.attn_max_stages
             : n == "attn_imma"    ? &t.attn_imma
             : n == "attn_rps8"    ? &t.attn_rps8
             : n == "attn_ivalue"  ? &t.attn_ivalue
                                   : nullptr;
    if (!f) sd::fail(SD_ERR_CONFIG, "sd_tune: unknown switch " + n);
    *f = value;
  });
}

int sd_weights_seed_random(const sd_model_spec* spec, uint64_t seed, int mode, int device, sd_weights** out) {
  return guard([&] {
    need(out, "out");
    sd::Spec s = sd::from_abi(spec);
    auto h = std::make_unique<sd_weights>();
    h->w = std::make_unique<sd::Weights>(s, mode, seed, device, sd::Weights::SeedRandom{});
    *out = h.release();
  });
}

int sd_weights_export_embedding(const sd_weights* w, float* host, size_t count) {
  return guard([&] {
    need(w, "weights");
    need(host, "host");
    const sd::Spec& s = w->w->spec();
    const size_t n = static_cast<size_t>(s.D) * s.V;
    if (count < n) sd::fail(SD_ERR_CONFIG, "export_embedding: buffer holds fewer than model_dim * vocab floats");
    sd::DeviceGuard dg(w->w->device());
    SD_CUDA(cudaMemcpy(host, w->w->embedding(), n * 4, cudaMemcpyDeviceToHost));
  });
}

int sd_weights_synthetic(const sd_model_spec* spec, int mode, uint64_t seed, int device,
                         sd_weights** out) {
  return guard([&] {
    need(out, "out");
    sd::Spec s = sd::from_abi(spec);
    auto h = std::make_unique<sd_weights>();
    h->w = std::make_unique<sd::Weights>(s, mode, seed, device);
    *out = h.release();
  });
}

int sd_drive(sd_engine* e, const sd_drive_config* cfg, sd_drive_result** out) {
  return guard([&] {
    need(e, "engine");
    need(cfg, "config");
    need(out, "out");
    auto r = std::make_unique<sd_drive_result>();
    r->r = sd::drive(*e->e, *cfg);
    *out = r.release();
  });
}

int64_t sd_drive_count(const sd_drive_result* r) {
  return r ? static_cast<int64_t>(r->r.tokens.size()) : 0;
}

int sd_drive_record(const sd_drive_result* r, int64_t i, int64_t* step, uint64_t* seq,
                    int32_t* token) {
  return guard([&] {
    need(r, "result");
    if (i < 0 || i >= static_cast<int64_t>(r->r.tokens.size())) sd::fail(SD_ERR_CONFIG, "index out of range");
    *step = r->r.steps[static_cast<size_t>(i)];
    *seq = r->r.seqs[static_cast<size_t>(i)];
    *token = r->r.tokens[static_cast<size_t>(i)];
  });
}

const float* sd_drive_activations(const sd_drive_result* r) {
  return (r && !r->r.activations.empty()) ? r->r.activations.data() : nullptr;
}

double sd_drive_wall_seconds(const sd_drive_result* r) { return r ? r->r.wall_seconds : 0.0; }

int sd_drive_destroy(sd_drive_result* r) {
  return guard([&] { delete r; });
}

// ------------------------------------------------------------ multi-GPU ---
int sd_nccl_unique_id(void* out, size_t bytes) {
  return guard([&] {
    need(out, "out");
    if (bytes < sizeof(ncclUniqueId)) sd::fail(SD_ERR_CONFIG, "nccl id buffer too small");
    ncclUniqueId id;
    sd::nccl_unique_id(&id);
    std::memcpy(out, &id, sizeof(id));
  });
}

int sd_dist_create(sd_weights* w, sd_kv* kv, int rank, int world, const void* nccl_id, int s_ranks,
                   int shard_mode, sd_dist** out) {
  return guard([&] {
    need(kv, "kv");
    need(out, "out");
    auto h = std::make_unique<sd_dist>();
    h->d = std::make_unique<sd::DistEngine>(w ? w->w.get() : nullptr, kv->s.get(), rank, world, nccl_id,
                                            s_ranks, shard_mode);
    *out = h.release();
  });
}

int sd_dist_pipeline(sd_dist* d, int enable) {
  return guard([&] {
    need(d, "dist");
    d->d->set_pipeline(enable != 0);
  });
}

int sd_dist_destroy(sd_dist* d) {
  return guard([&] { delete d; });
}

int sd_dist_step(sd_dist* d, int32_t B, const uint64_t* seqs, const int32_t* tokens, int32_t* next,
                 float* final_x) {
  return guard([&] {
    need(d, "dist");
    need(seqs, "seqs");
    need(tokens, "tokens");
    need(next, "next_tokens");
    d->d->compute(B, seqs, tokens, next, final_x);
  });
}

int sd_dist_retire(sd_dist* d, int32_t n, const uint64_t* seqs) {
  return guard([&] {
    need(d, "dist");
    d->d->retire(n, seqs);
  });
}

int sd_dist_bench(sd_dist* d, int32_t B, const uint64_t* seqs, const int32_t* tokens, int32_t steps,
                  double* ms) {
  return guard([&] {
    need(d, "dist");
    need(ms, "ms");
    *ms = d->d->bench(B, seqs, tokens, steps);
  });
}

int sd_dist_drive(sd_dist* d, const sd_drive_config* cfg, sd_drive_result** out) {
  return guard([&] {
    need(d, "dist");
    need(cfg, "config");
    need(out, "out");
    auto r = std::make_unique<sd_drive_result>();
    r->r = sd::drive(*d->d, *cfg);
    *out = r.release();
  });
}

int sd_dist_timing(sd_dist* d, int enable) {
  return guard([&] {
    need(d, "dist");
    d->d->set_timing(enable != 0);
  });
}

int sd_dist_timing_read(sd_dist* d, double* ms, double* bytes, int reset) {
  return guard([&] {
    need(d, "dist");
    d->d->read_timing(ms, bytes, reset != 0);
  });
}

int sd_dist_p2p_setup(sd_dist* d, int32_t max_rows, void* handles_out) {
  static_assert(sd::DistEngine::kIpcBytes == SD_DIST_IPC_BYTES, "IPC handle block size");
  return guard([&] {
    need(d, "dist");
    need(handles_out, "handles_out");
    d->d->p2p_setup(max_rows, handles_out);
  });
}

int sd_dist_p2p_connect(sd_dist* d, const void* all_handles) {
  return guard([&] {
    need(d, "dist");
    need(all_handles, "all_handles");
    d->d->p2p_connect(all_handles);
  });
}

int sd_dist_plan(int world, int rank, int s_ranks, int shard_mode, int heads, int32_t B, const uint64_t* seqs,
                 int32_t* home_rows, int32_t* n_home, int32_t* shard_rows, int32_t* n_shard, int32_t* send_counts,
                 int32_t* recv_counts) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) sd::fail(SD_ERR_CONFIG, "bad rank / world");
    sd::DistPlan p;
    sd::make_plan(world, rank, s_ranks, B, seqs, p, shard_mode, heads);
    if (n_home) *n_home = static_cast<int32_t>(p.home_rows.size());
    if (n_shard) *n_shard = static_cast<int32_t>(p.shard_rows.size());
    if (home_rows) std::copy(p.home_rows.begin(), p.home_rows.end(), home_rows);
    if (shard_rows) std::copy(p.shard_rows.begin(), p.shard_rows.end(), shard_rows);
    if (send_counts) std::copy(p.send_cnt.begin(), p.send_cnt.end(), send_counts);
    if (recv_counts) std::copy(p.recv_cnt.begin(), p.recv_cnt.end(), recv_counts);
  });
}

// ------------------------------------------------------ shardmap / load ---
int sd_shardmap_worker_for(int mode, int heads, int workers, uint64_t seq, int head,
                           int32_t* out) {
  return guard([&] {
    need(out, "out");
    *out = sd::shard_worker_for(mode, heads, workers, seq, head);
  });
}

int sd_shardmap_head_range(int mode, int heads, int workers, int worker, int32_t* start,
                           int32_t* count) {
  return guard([&] {
    auto r = sd::shard_head_range(mode, heads, workers, worker);
    if (start) *start = r.first;
    if (count) *count = r.second;
  });
}

int sd_micro_batch_size(int batch, int interval, int target_len, int32_t* out) {
  return guard([&] {
    need(out, "out");
    *out = sd::micro_batch_size(batch, interval, target_len);
  });
}

int sd_cold_start_schedule(int batch, int target_len, int interval, int mode, int64_t horizon,
                           int64_t* triples, int64_t capacity, int64_t* count) {
  return guard([&] {
    need(count, "count");
    auto a = sd::cold_start_schedule(batch, target_len, interval, mode, horizon);
    *count = static_cast<int64_t>(a.size());
    for (size_t i = 0; i < a.size() && static_cast<int64_t>(i) < capacity && triples; ++i) {
      triples[3 * i] = a[i].step;
      triples[3 * i + 1] = a[i].size;
      triples[3 * i + 2] = a[i].target;
    }
  });
}

// ------------------------------------------------- SDWP attention worker
int sd_rworker_create(int64_t capacity_tokens, int kv_format, int device, sd_rworker** out) {
  return guard([&] {
    need(out, "out");
    auto h = std::make_unique<sd_rworker>();
    h->s = std::make_unique<sd::sdwp::WorkerSession>(capacity_tokens, kv_format, device);
    *out = h.release();
  });
}

int sd_rworker_destroy(sd_rworker* w) {
  return guard([&] { delete w; });
}

int sd_rworker_feed(sd_rworker* w, const uint8_t* bytes, size_t n, const uint8_t** replies, size_t* replies_len) {
  return guard([&] {
    need(w, "worker");
    w->out.clear();
    if (n) {
      need(bytes, "bytes");
      w->dec.feed(bytes, n);
    }
    sd::sdwp::Message m;
    for (;;) {
      const auto st = w->dec.poll(m);
      if (st == sd::sdwp::FrameDecoder::kNeedMore) break;
      if (st == sd::sdwp::FrameDecoder::kFatal) sd::fail(SD_ERR_PROTOCOL, "fatal protocol error: " + w->dec.error());
      for (const sd::sdwp::Message& r : w->s->handle(m)) {
        const std::vector<uint8_t> f = sd::sdwp::encode_frame(r);
        w->out.insert(w->out.end(), f.begin(), f.end());
      }
      if (w->s->shutdown_requested()) break;
    }
    if (replies) *replies = w->out.data();
    if (replies_len) *replies_len = w->out.size();
  });
}

int sd_rworker_shutdown_requested(const sd_rworker* w, int32_t* out) {
  return guard([&] {
    need(w, "worker");
    need(out, "out");
    *out = w->s->shutdown_requested() ? 1 : 0;
  });
}

int sd_rworker_serve(const char* listen_addr, const char* port_file, int64_t capacity_tokens, int kv_format,
                     int device, int once, double recv_timeout_seconds) {
  return guard([&] {
    need(listen_addr, "listen_addr");
    sd::sdwp::serve(listen_addr, port_file ? port_file : "", capacity_tokens, kv_format, device, once != 0,
                    recv_timeout_seconds);
  });
}

}  // extern "C"

// ------------------------------------------------------- planner and inputs
namespace {
sd::PerfProfile to_profile(const sd_perf_profile* p) {
  need(p, "profile");
  sd::PerfProfile r;
  if (p->n > 0) {
    need(p->batch, "profile.batch");
    need(p->seconds, "profile.seconds");
  }
  for (int i = 0; i < p->n; ++i) r.t_table.emplace_back(p->batch[i], p->seconds[i]);
  r.r_per_token = p->r_per_token;
  r.capacity_c = p->capacity_c;
  return r;
}
sd::PlanRequest to_request(const sd_plan_request* q) {
  need(q, "request");
  sd::PlanRequest r;
  r.num_layers = q->num_layers;
  r.target_len = q->target_len;
  if (q->has_latency_budget && !(q->latency_budget > 0)) {
    sd::fail(SD_ERR_CONFIG, "plan request: latency budget must be positive");
  }
  r.latency_budget = q->has_latency_budget ? q->latency_budget : sd::kNoBudget;
  if (q->candidates && q->n_candidates > 0) r.candidates.assign(q->candidates, q->candidates + q->n_candidates);
  r.knee_threshold = q->knee_threshold;
  r.balance_tolerance = q->balance_tolerance;
  return r;
}
}  // namespace

int sd_bench_dense_block(sd_weights* w, const int32_t* batches, int32_t n, int32_t reps, double* seconds_out) {
  return guard([&] {
    need(w, "weights");
    need(batches, "batches");
    need(seconds_out, "seconds_out");
    sd::bench_dense_block(*w->w, batches, n, reps, seconds_out);
  });
}

int sd_bench_attention_per_token(const sd_model_spec* spec, int kv_format, int32_t batch, int32_t seq_len,
                                 int32_t reps, int device, double* r_out) {
  return guard([&] {
    need(spec, "spec");
    need(r_out, "r_out");
    *r_out = sd::bench_attention_per_token(sd::from_abi(spec), kv_format, batch, seq_len, reps, device);
  });
}

int sd_kv_capacity_tokens(const sd_model_spec* spec, int kv_format, int device, double reserve_bytes,
                          int64_t* tokens_out) {
  return guard([&] {
    need(spec, "spec");
    need(tokens_out, "tokens_out");
    *tokens_out = sd::kv_capacity_tokens(sd::from_abi(spec), kv_format, device, reserve_bytes);
  });
}

int sd_plan(const sd_perf_profile* profile, const sd_plan_request* request, sd_hardware_plan* out) {
  return guard([&] {
    need(out, "out");
    const sd::PerfProfile p = to_profile(profile);
    const sd::PlanRequest q = to_request(request);
    *out = sd_hardware_plan{};
    try {
      const sd::HardwarePlan h = sd::plan(p, q);
      out->batch_size = h.batch_size;
      out->worker_count = h.worker_count;
      out->worker_estimate = h.worker_estimate;
      out->predicted_seq_seconds = h.predicted_seq_seconds;
      out->efficiency = h.efficiency;
      out->balance_residual = h.balance_residual;
      out->balanced = h.balanced ? 1 : 0;
      out->binding_constraint = h.binding;
      out->tightest_batch = h.tightest_batch;
    } catch (const sd::Error& e) {
      if (e.code == SD_ERR_INFEASIBLE) {
        int t = 0;
        try {
          sd::plan_batch_size(p, q, &t);
        } catch (const sd::Error&) {
        }
        out->tightest_batch = t;
      }
      throw;
    }
  });
}

int sd_plan_batch_size(const sd_perf_profile* profile, const sd_plan_request* request, int32_t* batch_out,
                       int32_t* tightest_out) {
  return guard([&] {
    need(batch_out, "batch_out");
    int t = 0;
    const sd::PerfProfile p = to_profile(profile);
    sd::validate_profile(p);
    try {
      *batch_out = sd::plan_batch_size(p, to_request(request), &t);
    } catch (const sd::Error&) {
      if (tightest_out) *tightest_out = t;
      throw;
    }
    if (tightest_out) *tightest_out = t;
  });
}

int sd_plan_block_seconds(const sd_perf_profile* profile, int32_t batch, double* seconds_out) {
  return guard([&] {
    need(seconds_out, "seconds_out");
    const sd::PerfProfile p = to_profile(profile);
    if (p.t_table.empty()) sd::fail(SD_ERR_CONFIG, "profile: empty T(B) table");
    *seconds_out = sd::block_seconds(p, batch);
  });
}

int sd_plan_worker_count(const sd_perf_profile* profile, int32_t batch, int32_t target_len, int32_t* workers,
                         double* estimate) {
  return guard([&] {
    need(workers, "workers");
    need(estimate, "estimate");
    const sd::PerfProfile p = to_profile(profile);
    if (p.t_table.empty()) sd::fail(SD_ERR_CONFIG, "profile: empty T(B) table");
    int w = 0;
    sd::plan_worker_count(p, batch, target_len, &w, estimate);
    *workers = w;
  });
}

int sd_plan_check_memory(int64_t batch, int64_t target_len, int64_t capacity, int64_t workers, int32_t* feasible,
                         int32_t* min_workers) {
  return guard([&] {
    need(feasible, "feasible");
    need(min_workers, "min_workers");
    bool f = false;
    int m = 0;
    sd::check_memory(batch, target_len, capacity, workers, &f, &m);
    *feasible = f ? 1 : 0;
    *min_workers = m;
  });
}

int sd_plan_check_balance(const sd_perf_profile* profile, int32_t batch, int32_t target_len, int32_t workers,
                          double tolerance, double* stage_seconds, double* residual, int32_t* accepted) {
  return guard([&] {
    need(stage_seconds, "stage_seconds");
    need(residual, "residual");
    need(accepted, "accepted");
    const sd::PerfProfile p = to_profile(profile);
    if (p.t_table.empty()) sd::fail(SD_ERR_CONFIG, "profile: empty T(B) table");
    bool ok = false;
    sd::check_balance(p, batch, target_len, workers, tolerance, stage_seconds, residual, &ok);
    *accepted = ok ? 1 : 0;
  });
}
