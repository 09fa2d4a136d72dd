// S-Part weights, the GPU StepComputation (engine) and the host scheduler.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <unordered_map>
#include <vector>

#include "dense_kernels.cuh"
#include "kv_store.h"
#include "sd_common.h"

namespace sd {

// WeightSet on the device (core.hpp:79-90). Exact mode keeps the reference
// storage W^T = [in][out] fp32; tensor-core modes keep W = [out][in]
// (K-major) in bf16 (kind::f16) or fp32 (kind::tf32). Q/K/V are fused into
// one [qkv_width] output projection; the per-element arithmetic is unchanged.
class Weights {
 public:
  Weights(const Spec& spec, const float* const* tensors, int mode, int device);
  // Counter-based synthetic weights of the same distribution (uniform
  // +-1/sqrt(fan_in)); generated on device for the full-size benchmark.
  Weights(const Spec& spec, int mode, uint64_t seed, int device);
  // seed_random_weights (core.cpp:97-127): the reference's mt19937 stream,
  // bit-identical to its WeightSet, generated on the host and uploaded.
  struct SeedRandom {};
  Weights(const Spec& spec, int mode, uint64_t seed, int device, SeedRandom);
  ~Weights();
  Weights(const Weights&) = delete;
  Weights& operator=(const Weights&) = delete;

  const Spec& spec() const { return spec_; }
  int mode() const { return mode_; }
  int device() const { return device_; }

  // y[B][out] = x . W^T (+ epilogue). which: 0 = qkv (fused), 4 = w_o,
  // 5 = w_mlp_in, 6 = w_mlp_out, 7 = head, 1/2/3 = q/k/v slices.
  // x_bf16 is required in BF16 mode (A operand), ignored otherwise.
  // the tensor-core GEMM of linear() without launching it (chained S-Part)
  GemmArgs gemm_args(int layer, int which, int B, const float* x, int64_t ldx, const act16* xb,
                     int64_t ldxb, float* y, int64_t ldy, act16* yb, int64_t ldyb, int epi,
                     const float* res, int64_t ldr, int max_ctas = 0) const;
  void linear(int layer, int which, int B, const float* x, int64_t ldx,
              const act16* xb, int64_t ldxb, float* y, int64_t ldy, act16* yb,
              int64_t ldyb, int epi, const float* res, int64_t ldr, cudaStream_t s,
              int max_ctas = 0) const;
  const float* embedding() const { return emb_; }  // fp32 D x V column-major (the reference storage)
  // the device tensor of (layer, which) and its bytes (L2 prefetch of the next GEMM's weights)
  const void* weight_ptr(int layer, int which) const { return tensor(layer, which); }
  int64_t weight_bytes(int which) const;
  int out_dim(int which) const;
  int in_dim(int which) const;

 private:
  void alloc();
  const void* tensor(int layer, int which) const;

  Spec spec_;
  int mode_, device_;
  float* emb_ = nullptr;        // D x V column-major ([V][D])
  void* blob_ = nullptr;        // all layer tensors + head
  std::vector<size_t> off_;     // per (layer, which) byte offsets
  size_t head_off_ = 0;
};

// StepComputation (workers.hpp:151-158): the per-step hook drive_schedule
// runs against. `owns` tells the driver which rows' tokens this process
// produced (all of them single-GPU; the home rows of a rank when
// distributed).
class StepComputation {
 public:
  virtual ~StepComputation() = default;
  virtual void compute(int B, const uint64_t* seqs, const int32_t* tokens, int32_t* next,
                       float* final_x) = 0;
  virtual void retire(int n, const uint64_t* seqs) = 0;
  virtual bool owns(uint64_t /*seq*/) const { return true; }
  virtual int model_dim() const = 0;
  virtual int vocab() const = 0;
};

// The GPU StepComputation: decode_step_monolithic (dense.cpp:90-129) with the
// S-Part on tensor cores / CUDA cores and the R-Part on the KvStore, all on
// one device stream.
class Engine : public StepComputation {
 public:
  Engine(Weights* w, KvStore* kv);
  ~Engine() override;
  void compute(int B, const uint64_t* seqs, const int32_t* tokens, int32_t* next,
               float* final_x) override {
    step(B, seqs, tokens, nullptr, next, final_x, nullptr);
  }
  int model_dim() const override { return w_->spec().D; }
  int vocab() const override { return w_->spec().V; }
  // features from token ids (workers.cpp:629-638) or explicit [B][D]
  void step(int B, const uint64_t* seqs, const int32_t* tokens_host, const float* x_host,
            int32_t* next_host, float* final_host, float* logits_host);
  void retire(int n, const uint64_t* seqs) override;
  double bench(int B, const uint64_t* seqs, const int32_t* tokens_host, int steps,
               int32_t* next_host);
  cudaStream_t stream() const { return stream_; }
  // CUDA-event timing of the S-Part GEMMs (on the S stream)
  // every = 0: off; 1: every GEMM; k > 1: the GEMMs of every k-th layer
  void set_timing(int every) {
    timing_ = every > 0;
    timing_every_ = every > 0 ? every : 1;
  }
  void read_timing(double* ms, double* flops, int64_t* launches, bool reset);
  // Two-mini-batch pipeline (workers.cpp:405-452): rows split by seq % 2;
  // the R-Part of one mini-batch (r_sms SMs, R stream) runs beside the
  // S-Part of the other (the remaining SMs, S stream). Off: one batch, one
  // stream, every kernel on every SM.
  void set_pipeline(bool on, int r_sms);

 private:
  struct Group {  // one mini-batch in flight (DistributedComputation::GroupState)
    std::vector<int> rows;
    std::vector<uint64_t> seqs;
    int cap = 0;
    float *x = nullptr, *qkv = nullptr, *o = nullptr, *y = nullptr, *h = nullptr, *logits = nullptr;
    act16 *xb = nullptr, *ob = nullptr, *yb = nullptr, *hb = nullptr;
    int32_t* tok = nullptr;
    unsigned long long* amax = nullptr;  // fused-argmax keys of the head GEMM
    std::vector<char> appended;          // per layer: K/V already stored by the QKV GEMM
    cudaEvent_t ev_s = nullptr, ev_r = nullptr;
    std::vector<uint32_t> pos;
    std::vector<int32_t> host_tok;
  };
  int split(int B, const uint64_t* seqs);  // fills groups_, returns the group count
  void ensure(Group& g, int n);
  void free_group(Group& g);
  void run(int ng, bool embed);
  int timing_every_ = 1;
  void gemm(int layer, int which, int B, const float* x, int64_t ldx, const act16* xb,
            int64_t ldxb, float* y, int64_t ldy, act16* yb, int64_t ldyb, int epi,
            const float* res, int64_t ldr, unsigned long long* amax = nullptr,
            const KvAppendOut* kvapp = nullptr);
  // the next layer's project_qkv with append_lane folded into its epilogue
  // when the KV store allows it (returns whether it did)
  bool qkv_fused_append(int layer, Group& g);
  bool want_logits_ = false;  // this step returns the logits (else the head's argmax is fused)
  // step(): the final activations' D2H copy, issued on the R stream as soon
  // as the last block is done, overlaps the head GEMM (one group only)
  float* early_final_ = nullptr;
  cudaEvent_t ev_final_ = nullptr;

  bool timing_ = false;
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_;
  std::vector<double> ev_flops_;
  double t_ms_ = 0, t_flops_ = 0;
  int64_t t_n_ = 0;

  Weights* w_;
  KvStore* kv_;
  cudaStream_t stream_ = nullptr;    // S stream (the only stream without the pipeline)
  cudaStream_t stream_r_ = nullptr;  // R stream
  bool pipeline_ = false;
  int r_sms_ = 0, s_sms_ = 0;
  Group groups_[2];
};

// ---- scheduler (scheduler.cpp:10-236), kept in host C++
int micro_batch_size(int batch, int interval, int target_len);
struct Admission {
  int64_t step;
  int size, target;
};
std::vector<Admission> cold_start_schedule(int batch, int target_len, int interval, int mode,
                                           int64_t horizon);
class LoadTracker {
 public:
  explicit LoadTracker(int64_t limit);
  int add(int64_t start, int size, int target);
  struct Plan {
    int64_t step = 0, total_load = 0;
    std::vector<int> active_ids, ending;
  };
  Plan step();
  int64_t earliest_start(int size, int target) const;
  int64_t current() const { return cur_; }
  void set_limit(int64_t l) {
    if (l < 1) fail(SD_ERR_ADMISSION, "load limit must be >= 1");
    limit_ = l;
  }

 private:
  struct MB {
    int id, size;
    int64_t start, end;
  };
  int64_t limit_, cur_ = 0;
  int next_id_ = 0;
  std::vector<MB> b_;
  std::vector<int64_t> w_;
};

// ShardMap (transport.cpp:319-380)
int shard_worker_for(int mode, int heads, int workers, uint64_t seq, int head);
std::pair<int, int> shard_head_range(int mode, int heads, int workers, int worker);

// drive_schedule (workers.cpp:547-684) over the engine
struct DriveResult {
  std::vector<int64_t> steps;
  std::vector<uint64_t> seqs;
  std::vector<int32_t> tokens;
  std::vector<float> activations;
  double wall_seconds = 0;
};
DriveResult drive(StepComputation& e, const sd_drive_config& c);

}  // namespace sd
