// The GPU StepComputation: decode_step_monolithic (dense.cpp:90-129), run
// either as one batch on one stream or as the reference's two interleaved
// mini-batches (DistributedComputation::compute, workers.cpp:399-480) on an
// S stream and an R stream, so that the R-Part of one mini-batch (HBM-bound
// attention) overlaps the S-Part of the other (tensor-core GEMMs) on
// disjoint SM partitions — FastDecode's S/R split inside one B200.
#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_set>

#include "engine.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace sd {

Engine::Engine(Weights* w, KvStore* kv) : w_(w), kv_(kv) {
  if (w->device() != kv->device()) fail(SD_ERR_CONFIG, "weights and KV store on different devices");
  const Spec& a = w->spec();
  const Spec& b = kv->spec();
  if (a.L != b.L || a.D != b.D || a.H != b.H || a.Hkv != b.Hkv || a.hd != b.hd) {
    fail(SD_ERR_CONFIG, "weights and KV store specs differ");
  }
  if (kv->width() != a.kv_width()) fail(SD_ERR_CONFIG, "engine needs a KV store over all kv heads");
  DeviceGuard dg(w->device());
  SD_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  SD_CUDA(cudaStreamCreateWithFlags(&stream_r_, cudaStreamNonBlocking));
  for (Group& g : groups_) {
    SD_CUDA(cudaEventCreateWithFlags(&g.ev_s, cudaEventDisableTiming));
    SD_CUDA(cudaEventCreateWithFlags(&g.ev_r, cudaEventDisableTiming));
  }
  SD_CUDA(cudaEventCreateWithFlags(&ev_final_, cudaEventDisableTiming));
}

void Engine::free_group(Group& g) {
  for (void* p : {static_cast<void*>(g.x), static_cast<void*>(g.qkv), static_cast<void*>(g.o),
                  static_cast<void*>(g.y), static_cast<void*>(g.h), static_cast<void*>(g.logits),
                  static_cast<void*>(g.xb), static_cast<void*>(g.ob), static_cast<void*>(g.yb),
                  static_cast<void*>(g.hb), static_cast<void*>(g.tok), static_cast<void*>(g.amax)}) {
    if (p) cudaFree(p);
  }
  g.x = g.qkv = g.o = g.y = g.h = g.logits = nullptr;
  g.xb = g.ob = g.yb = g.hb = nullptr;
  g.tok = nullptr;
  g.amax = nullptr;
  g.cap = 0;
}

Engine::~Engine() {
  DeviceGuard dg(w_->device());
  cudaStreamSynchronize(stream_);
  cudaStreamSynchronize(stream_r_);
  for (Group& g : groups_) {
    free_group(g);
    cudaEventDestroy(g.ev_s);
    cudaEventDestroy(g.ev_r);
  }
  for (auto& e : ev_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  cudaEventDestroy(ev_final_);
  cudaStreamDestroy(stream_);
  cudaStreamDestroy(stream_r_);
}

void Engine::set_pipeline(bool on, int r_sms) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, w_->device());
  pipeline_ = on;
  r_sms_ = on ? std::max(1, std::min(r_sms, nsm - 1)) : 0;
  s_sms_ = on ? nsm - r_sms_ : 0;
  kv_->set_grid_limit(r_sms_);
}

void Engine::ensure(Group& g, int n) {
  if (n <= g.cap) return;
  DeviceGuard dg(w_->device());
  SD_CUDA(cudaStreamSynchronize(stream_));
  SD_CUDA(cudaStreamSynchronize(stream_r_));
  free_group(g);
  const Spec& s = w_->spec();
  // rows padded to 128 so tensor-core tiles never read past the buffers
  const size_t bp = (static_cast<size_t>(n) + 127) / 128 * 128;
  auto zalloc = [&](auto** p, size_t bytes) {
    SD_CUDA(cudaMalloc(reinterpret_cast<void**>(p), bytes));
    SD_CUDA(cudaMemset(*p, 0, bytes));
  };
  zalloc(&g.x, bp * s.D * 4);
  zalloc(&g.qkv, bp * s.qkv_width() * 4);
  zalloc(&g.o, bp * s.D * 4);
  zalloc(&g.y, bp * s.D * 4);
  zalloc(&g.h, bp * s.F * 4);
  zalloc(&g.logits, bp * s.V * 4);
  zalloc(&g.xb, bp * s.D * 2);
  zalloc(&g.ob, bp * s.D * 2);
  zalloc(&g.yb, bp * s.D * 2);
  zalloc(&g.hb, bp * s.F * 2);
  zalloc(&g.tok, bp * 4);
  zalloc(&g.amax, bp * 8);
  // cudaMemset runs on the legacy stream, which does not order with the
  // engine's non-blocking streams: finish it before any kernel touches g
  SD_CUDA(cudaDeviceSynchronize());
  g.cap = n;
}

// Mini-batches by sequence id parity, merged when one is empty
// (workers.cpp:405-420); without the pipeline, one batch in row order.
int Engine::split(int B, const uint64_t* seqs) {
  for (Group& g : groups_) {
    g.rows.clear();
    g.seqs.clear();
  }
  if (pipeline_) {
    for (int b = 0; b < B; ++b) groups_[seqs[b] % 2].rows.push_back(b);
    if (groups_[0].rows.empty() || groups_[1].rows.empty()) {
      std::vector<int> all;
      for (Group& g : groups_) all.insert(all.end(), g.rows.begin(), g.rows.end());
      std::sort(all.begin(), all.end());
      groups_[0].rows = all;
      groups_[1].rows.clear();
    }
  } else {
    for (int b = 0; b < B; ++b) groups_[0].rows.push_back(b);
  }
  int ng = 0;
  for (Group& g : groups_) {
    if (g.rows.empty()) continue;
    for (int r : g.rows) g.seqs.push_back(seqs[r]);
    ensure(g, static_cast<int>(g.rows.size()));
    g.pos.resize(g.rows.size());
    ++ng;
  }
  return ng;
}

void Engine::gemm(int layer, int which, int B, const float* x, int64_t ldx,
                  const act16* xb, int64_t ldxb, float* y, int64_t ldy, act16* yb,
                  int64_t ldyb, int epi, const float* res, int64_t ldr, unsigned long long* amax,
                  const KvAppendOut* kvapp) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool timed = timing_ && (which == 7 || layer % timing_every_ == 0);
  if (timed) {
    for (cudaEvent_t* e : {&e0, &e1}) {
      if (ev_pool_.empty()) {
        SD_CUDA(cudaEventCreate(e));
      } else {
        *e = ev_pool_.back();
        ev_pool_.pop_back();
      }
    }
    SD_CUDA(cudaEventRecord(e0, stream_));
  }
  if (amax) {
    GemmArgs ga = w_->gemm_args(layer, which, B, x, ldx, xb, ldxb, nullptr, ldy, nullptr, 0, epi, res, ldr, s_sms_);
    ga.amax = amax;
    launch_gemm_sm100(ga, stream_);
  } else if (kvapp) {
    GemmArgs ga = w_->gemm_args(layer, which, B, x, ldx, xb, ldxb, y, ldy, yb, ldyb, epi, res, ldr, s_sms_);
    ga.kvapp = kvapp;
    launch_gemm_sm100(ga, stream_);
  } else {
    w_->linear(layer, which, B, x, ldx, xb, ldxb, y, ldy, yb, ldyb, epi, res, ldr, stream_, s_sms_);
  }
  if (timed) {
    SD_CUDA(cudaEventRecord(e1, stream_));
    ev_.emplace_back(e0, e1);
    ev_flops_.push_back(2.0 * B * w_->out_dim(which) * w_->in_dim(which));
  }
}

void Engine::read_timing(double* ms, double* flops, int64_t* launches, bool reset) {
  for (size_t i = 0; i < ev_.size(); ++i) {
    SD_CUDA(cudaEventSynchronize(ev_[i].second));
    float t = 0;
    SD_CUDA(cudaEventElapsedTime(&t, ev_[i].first, ev_[i].second));
    t_ms_ += t;
    t_flops_ += ev_flops_[i];
    t_n_ += 1;
    ev_pool_.push_back(ev_[i].first);
    ev_pool_.push_back(ev_[i].second);
  }
  ev_.clear();
  ev_flops_.clear();
  if (ms) *ms = t_ms_;
  if (flops) *flops = t_flops_;
  if (launches) *launches = t_n_;
  if (reset) {
    t_ms_ = t_flops_ = 0;
    t_n_ = 0;
  }
}

bool Engine::qkv_fused_append(int layer, Group& g) {
  const Spec& s = w_->spec();
  const int n = static_cast<int>(g.rows.size());
  if (!tuning().fused_append || pipeline_ || w_->mode() == SD_DENSE_EXACT_F32 || n == 0) return false;
  // the epilogue's K/V stores need the TMA-store path and 16-column-aligned
  // fp16 K/V rows: decided before anything is staged
  if (s.D % 16 || s.kv_width() % 16 || s.qkv_width() % 4) return false;
  for (int i = 0; i < n; ++i) {
    g.pos[static_cast<size_t>(i)] = static_cast<uint32_t>(kv_->stored(g.seqs[static_cast<size_t>(i)], layer));
  }
  KvAppendOut ka{};
  if (!kv_->stage_fused_append(layer, n, g.seqs.data(), g.pos.data(), &ka)) return false;
  ka.col_k = s.D;
  ka.width = s.kv_width();
  try {
    gemm(layer, 0, n, g.x, s.D, g.xb, s.D, g.qkv, s.qkv_width(), nullptr, 0, kEpiNone, nullptr, 0, nullptr, &ka);
  } catch (...) {
    kv_->abort_fused_append();  // lengths back: a later append / attend sees the store as before
    throw;
  }
  kv_->end_fused_append(stream_);
  return true;
}

// One decode step over the `ng` groups; embed = features from g.tok (else
// g.x/g.xb already hold them). Per group and layer: S_pre (finish_block of
// the previous layer + project_qkv) on the S stream, then the R-Part
// (append + attend) on the R stream; the S stream of a group waits for its
// own R-Part only, so group A's attention overlaps group B's GEMMs.
void Engine::run(int ng, bool embed) {
  const Spec& s = w_->spec();
  const int D = s.D, F = s.F, qkvw = s.qkv_width(), kvw = s.kv_width();
  // kind::f16 modes keep 16-bit copies of the GEMM A operands (bf16 or fp16)
  const bool bf = w_->mode() == SD_DENSE_BF16 || w_->mode() == SD_DENSE_F16;
  const int f16 = w_->mode() == SD_DENSE_F16 ? 1 : 0;
  cudaStream_t rs = pipeline_ ? stream_r_ : stream_;
  for (int gi = 0; gi < ng; ++gi) {
    Group& g = groups_[gi];
    const int n = static_cast<int>(g.rows.size());
    if (embed) launch_embed(n, D, g.tok, w_->embedding(), g.x, D, bf ? g.xb : nullptr, f16, stream_);
    gemm(0, 0, n, g.x, D, g.xb, D, g.qkv, qkvw, nullptr, 0, kEpiNone, nullptr, 0);
    if (pipeline_) SD_CUDA(cudaEventRecord(g.ev_s, stream_));
  }
  for (int gi = 0; gi < ng; ++gi) groups_[gi].appended.assign(static_cast<size_t>(s.L), 0);
  for (int l = 0; l < s.L; ++l) {
    for (int gi = 0; gi < ng; ++gi) {
      Group& g = groups_[gi];
      const int n = static_cast<int>(g.rows.size());
      if (pipeline_) SD_CUDA(cudaStreamWaitEvent(rs, g.ev_s, 0));
      if (!g.appended[static_cast<size_t>(l)]) {
        for (int i = 0; i < n; ++i) {
          g.pos[static_cast<size_t>(i)] = static_cast<uint32_t>(kv_->stored(g.seqs[static_cast<size_t>(i)], l));
        }
        kv_->append(l, n, g.seqs.data(), g.pos.data(), g.qkv + D, qkvw, g.qkv + D + kvw, qkvw, rs);
      }
      // the attention also writes the 16-bit copy of o that W_o consumes, and
      // prefetches W_o's weights into L2 at its end
      if (tuning().attn_l2_prefetch && w_->mode() != SD_DENSE_EXACT_F32) {
        kv_->set_l2_prefetch(w_->weight_ptr(l, 4), w_->weight_bytes(4));
      }
      kv_->attend(l, n, g.seqs.data(), g.qkv, qkvw, g.o, D, rs, gi, bf ? g.ob : nullptr, D, nullptr, f16);
      if (pipeline_) {
        SD_CUDA(cudaEventRecord(g.ev_r, rs));
        SD_CUDA(cudaStreamWaitEvent(stream_, g.ev_r, 0));
      }
      // finish_block (dense.cpp:51-70), then the next layer's project_qkv
      gemm(l, 4, n, g.o, D, g.ob, D, g.y, D, bf ? g.yb : nullptr, D, kEpiResidual, g.x, D);
      gemm(l, 5, n, g.y, D, g.yb, D, bf ? nullptr : g.h, F, bf ? g.hb : nullptr, F, kEpiSilu, nullptr, 0);
      gemm(l, 6, n, g.h, F, g.hb, F, g.x, D, bf ? g.xb : nullptr, D, kEpiResidual, g.y, D);
      if (l + 1 < s.L) {
        if (qkv_fused_append(l + 1, g)) {
          g.appended[static_cast<size_t>(l + 1)] = 1;
        } else {
          gemm(l + 1, 0, n, g.x, D, g.xb, D, g.qkv, qkvw, nullptr, 0, kEpiNone, nullptr, 0);
        }
        if (pipeline_) SD_CUDA(cudaEventRecord(g.ev_s, stream_));
      }
    }
  }
  if (early_final_ && ng == 1) {  // final activations leave while the head runs
    SD_CUDA(cudaEventRecord(ev_final_, stream_));
    SD_CUDA(cudaStreamWaitEvent(stream_r_, ev_final_, 0));
    SD_CUDA(cudaMemcpyAsync(early_final_, groups_[0].x, groups_[0].rows.size() * static_cast<size_t>(D) * 4,
                            cudaMemcpyDeviceToHost, stream_r_));
  }
  for (int gi = 0; gi < ng; ++gi) {  // output_logits + argmax_token (dense.cpp:72-88)
    Group& g = groups_[gi];
    const int n = static_cast<int>(g.rows.size());
    // tensor-core modes: argmax_token folded into the head GEMM's epilogue
    // (no logits round trip through HBM) unless the caller wants the logits
    if (!want_logits_ && tuning().fused_argmax && w_->mode() != SD_DENSE_EXACT_F32) {
      gemm(0, 7, n, g.x, D, g.xb, D, g.logits, s.V, nullptr, 0, kEpiNone, nullptr, 0, g.amax);
      launch_argmax_keys(n, g.amax, g.tok, stream_);
      continue;
    }
    gemm(0, 7, n, g.x, D, g.xb, D, g.logits, s.V, nullptr, 0, kEpiNone, nullptr, 0);
    launch_argmax(n, s.V, g.logits, s.V, g.tok, stream_);
  }
}

void Engine::step(int B, const uint64_t* seqs, const int32_t* tokens_host, const float* x_host,
                  int32_t* next_host, float* final_host, float* logits_host) {
  const Spec& s = w_->spec();
  if (B == 0) fail(SD_ERR_CONFIG, "project_qkv: empty batch");
  {
    std::unordered_set<uint64_t> seen;  // validate_batch (core.cpp:37-54)
    for (int i = 0; i < B; ++i) {
      if (!seen.insert(seqs[i]).second) {
        fail(SD_ERR_CONFIG, "token batch: duplicate sequence id " + std::to_string(seqs[i]));
      }
    }
  }
  if (tokens_host) {
    for (int i = 0; i < B; ++i) {
      if (tokens_host[i] < 0 || tokens_host[i] >= s.V) fail(SD_ERR_CONFIG, "token out of the vocabulary");
    }
  }
  DeviceGuard dg(w_->device());
  const int ng = split(B, seqs);
  const bool bf = w_->mode() == SD_DENSE_BF16 || w_->mode() == SD_DENSE_F16;
  const int f16 = w_->mode() == SD_DENSE_F16 ? 1 : 0;
  std::vector<float> xrows;
  for (int gi = 0; gi < ng; ++gi) {
    Group& g = groups_[gi];
    const int n = static_cast<int>(g.rows.size());
    if (tokens_host) {
      g.host_tok.resize(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) g.host_tok[static_cast<size_t>(i)] = tokens_host[g.rows[static_cast<size_t>(i)]];
      SD_CUDA(cudaMemcpyAsync(g.tok, g.host_tok.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, stream_));
    } else if (ng == 1) {
      // one group holds the batch in row order: the caller's rows go
      // straight to the device (a DMA from pinned memory when it is pinned)
      SD_CUDA(cudaMemcpyAsync(g.x, x_host, static_cast<size_t>(n) * s.D * 4, cudaMemcpyHostToDevice, stream_));
      if (bf) launch_to_16(n, s.D, g.x, s.D, g.xb, s.D, f16, stream_);
    } else {
      xrows.resize(static_cast<size_t>(n) * s.D);
      for (int i = 0; i < n; ++i) {
        std::memcpy(xrows.data() + static_cast<size_t>(i) * s.D, x_host + static_cast<size_t>(g.rows[static_cast<size_t>(i)]) * s.D,
                    static_cast<size_t>(s.D) * 4);
      }
      SD_CUDA(cudaMemcpyAsync(g.x, xrows.data(), xrows.size() * 4, cudaMemcpyHostToDevice, stream_));
      SD_CUDA(cudaStreamSynchronize(stream_));  // xrows is reused by the next group
      if (bf) launch_to_16(n, s.D, g.x, s.D, g.xb, s.D, f16, stream_);
    }
  }
  want_logits_ = logits_host != nullptr;
  early_final_ = ng == 1 ? final_host : nullptr;
  try {
    run(ng, tokens_host != nullptr);
  } catch (...) {
    early_final_ = nullptr;
    want_logits_ = false;
    throw;
  }
  const bool final_done = early_final_ != nullptr;
  early_final_ = nullptr;
  want_logits_ = false;
  if (final_done) SD_CUDA(cudaStreamSynchronize(stream_r_));
  std::vector<int32_t> nt;
  std::vector<float> buf;
  for (int gi = 0; gi < ng; ++gi) {
    Group& g = groups_[gi];
    const int n = static_cast<int>(g.rows.size());
    nt.resize(static_cast<size_t>(n));
    SD_CUDA(cudaMemcpyAsync(nt.data(), g.tok, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, stream_));
    SD_CUDA(cudaStreamSynchronize(stream_));
    for (int i = 0; i < n; ++i) {
      if (next_host) next_host[g.rows[static_cast<size_t>(i)]] = nt[static_cast<size_t>(i)];
    }
    auto scatter = [&](const float* dev, int width, float* dst) {
      if (ng == 1) {  // rows in batch order: straight into the caller's buffer
        SD_CUDA(cudaMemcpyAsync(dst, dev, static_cast<size_t>(n) * width * 4, cudaMemcpyDeviceToHost, stream_));
        SD_CUDA(cudaStreamSynchronize(stream_));
        return;
      }
      buf.resize(static_cast<size_t>(n) * width);
      SD_CUDA(cudaMemcpy(buf.data(), dev, buf.size() * 4, cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) {
        std::memcpy(dst + static_cast<size_t>(g.rows[static_cast<size_t>(i)]) * width,
                    buf.data() + static_cast<size_t>(i) * width, static_cast<size_t>(width) * 4);
      }
    };
    if (final_host && !final_done) scatter(g.x, s.D, final_host);
    if (logits_host) scatter(g.logits, s.V, logits_host);
  }
}

double Engine::bench(int B, const uint64_t* seqs, const int32_t* tokens_host, int steps,
                     int32_t* next_host) {
  DeviceGuard dg(w_->device());
  const int ng = split(B, seqs);
  for (int gi = 0; gi < ng; ++gi) {
    Group& g = groups_[gi];
    const int n = static_cast<int>(g.rows.size());
    g.host_tok.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) g.host_tok[static_cast<size_t>(i)] = tokens_host[g.rows[static_cast<size_t>(i)]];
    SD_CUDA(cudaMemcpyAsync(g.tok, g.host_tok.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, stream_));
  }
  cudaEvent_t e0, e1;
  SD_CUDA(cudaEventCreate(&e0));
  SD_CUDA(cudaEventCreate(&e1));
  SD_CUDA(cudaStreamSynchronize(stream_));
  SD_CUDA(cudaEventRecord(e0, stream_));
  for (int i = 0; i < steps; ++i) run(ng, true);  // tokens fed back on device
  SD_CUDA(cudaEventRecord(e1, stream_));
  SD_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  SD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (next_host) {
    for (int gi = 0; gi < ng; ++gi) {
      Group& g = groups_[gi];
      const int n = static_cast<int>(g.rows.size());
      SD_CUDA(cudaMemcpy(g.host_tok.data(), g.tok, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) next_host[g.rows[static_cast<size_t>(i)]] = g.host_tok[static_cast<size_t>(i)];
    }
  }
  return ms;
}

void Engine::retire(int n, const uint64_t* seqs) {
  for (int i = 0; i < n; ++i) kv_->drop(seqs[i]);
}

}  // namespace sd
