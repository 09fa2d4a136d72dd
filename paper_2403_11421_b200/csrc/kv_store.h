// KvStore: the B200 KvShard. Host-side mirror of per-(sequence, layer)
// stored lengths gives the reference's validation and error behaviour
// (attention.cpp:139-305); K/V live in a paged HBM pool written and read by
// the kernels in kv_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <unordered_map>
#include <vector>

#include "kv_kernels.cuh"
#include "sd_common.h"

namespace sd {

class KvStore {
 public:
  KvStore(const Spec& spec, int head_start, int head_count, int64_t capacity_tokens, int fmt,
          int device, const sd_kv_options* opts);
  ~KvStore();
  KvStore(const KvStore&) = delete;
  KvStore& operator=(const KvStore&) = delete;

  // ---- reference queries (attention.hpp:73-111)
  int width() const { return geom_.width; }
  int head_start() const { return head_start_; }
  int q_width() const { return geom_.width * G_; }
  int group_size() const { return G_; }
  int64_t capacity() const { return cap_; }
  int format() const { return geom_.fmt; }
  int64_t token_count() const { return total_ / spec_.L; }
  int warnings() const { return warnings_; }
  bool has(uint64_t seq) const { return slot_of_.count(seq) != 0; }
  int stored(uint64_t seq, int layer) const;
  int64_t bytes_per_token() const;
  int device() const { return device_; }
  const Spec& spec() const { return spec_; }

  // ---- operations (device pointers; host `seqs`/`positions`)
  // KvShard::append_request semantics (attention.cpp:172-202), including the
  // reference's partial commit when a later item of the batch fails inside
  // the sequential append loop (e.g. a duplicated sequence).
  void append(int layer, int n, const uint64_t* seqs, const uint32_t* positions,
              const float* k_dev, int64_t k_stride, const float* v_dev, int64_t v_stride,
              cudaStream_t s);
  // The same append with its stores left to the producer of k and v (the
  // QKV GEMM's epilogue): only on the lockstep fast path (every target page
  // open, the previous call at another layer with the same sequences and
  // positions) with fp16 pages. Returns false, changing nothing, otherwise.
  // On true the call is committed; `out` locates every row's page and the
  // producer must run on `s` before end_fused_append(s).
  bool stage_fused_append(int layer, int n, const uint64_t* seqs, const uint32_t* positions,
                          struct KvAppendOut* out);
  void end_fused_append(cudaStream_t s);
  // undo a staged append whose producer could not be launched (lengths,
  // totals and the fast-path layer return to their state before staging)
  void abort_fused_append();
  // KvShard::attend semantics (attention.cpp:204-282).
  // `slot` selects one of the cached split plans (one per interleaved
  // mini-batch, so alternating batches do not rebuild each other's plan).
  // `ob` (optional): also write o in bf16 (the W_o GEMM operand).
  void attend(int layer, int n, const uint64_t* seqs, const float* q_dev, int64_t q_stride,
              float* o_dev, int64_t o_stride, cudaStream_t s, int slot = 0,
              act16* ob = nullptr, int64_t ob_stride = 0, const ORoute* oroute = nullptr, int ob_f16 = 0);
  bool tensor_core_path() const { return use_mma_; }
  // SM budget of the attention grid (0 = every SM): the R-Part's share when
  // it runs beside the S-Part of the other mini-batch
  void set_grid_limit(int sms) { grid_limit_ = sms; }
  // bytes the next attend() launch prefetches into L2 at its end (the
  // following GEMM's weights; tensor-core path only)
  void set_l2_prefetch(const void* p, int64_t bytes) {
    l2pf_ = static_cast<const uint8_t*>(p);
    l2pf_bytes_ = bytes;
  }
  // KvShard::drop_sequence (attention.cpp:284-294)
  void drop(uint64_t seq);
  int64_t export_lane(uint64_t seq, int layer, int which, void* host, size_t host_bytes,
                      float* scales, size_t scales_count);
  void prefill_synthetic(int n, const uint64_t* seqs, int length, uint64_t salt,
                         cudaStream_t s);

  // ---- timing of the attention kernel (CUDA events on the launching stream)
  // every = 0: off; 1: every attention launch; k > 1: launches of every
  // k-th layer (layers are identical; fewer events perturb the step less)
  void set_timing(int every);
  void read_timing(double* ms, int64_t* launches, double* bytes, bool reset);

 private:
  struct Blob {  // one staged descriptor upload
    HostBuf host;
    DevBuf dev;
    cudaEvent_t done = nullptr;
  };
  Blob& next_blob();
  int slot_for_new(uint64_t seq);
  void release_slot(int slot);
  int alloc_group();
  void upload(Blob& b, size_t bytes, cudaStream_t s);
  struct Plan {
    std::vector<int32_t> slots, lens;
    int npieces = 0, grid = 0, ncombine = 0, sms = 0;
    int64_t positions = 0;
    Blob blob;
    size_t off_slot = 0, off_pieces = 0, off_cta = 0, off_comb = 0;
    DevBuf part_acc, part_ml, comb_cnt;
  };
  static constexpr int kPlanSlots = 2;
  void launch_attention_plan(Plan& P, int layer, const float* q, int64_t qs, float* o, int64_t os,
                             act16* ob, int64_t obs, cudaStream_t s, const ORoute* oroute, int ob_f16);

  Spec spec_;
  int head_start_, head_count_, G_;
  int64_t cap_;
  int device_;
  int nsm_ = 148;
  KvGeom geom_{};
  int T_ = 1, nstages_ = 2, stage_region_ = 0, sc_region_ = 0;
  size_t attn_smem_ = 0;
  bool use_mma_ = false;  // tensor-core GQA kernel (kv_mma.cu)
  int max_seqs_ = 0, max_len_ = 0, pool_groups_ = 0;

  // host mirror
  std::unordered_map<uint64_t, int> slot_of_;
  std::vector<int32_t> len_;     // [max_seqs][L]
  std::vector<int32_t> pages_;   // [max_seqs][max_pages], -1 = none
  std::vector<int32_t> npages_;  // [max_seqs]
  std::vector<int32_t> free_slots_, free_groups_;
  int64_t total_ = 0;
  int warnings_ = 0;

  // staging
  std::vector<Blob> ring_;
  size_t ring_next_ = 0;
  // cached attention plan (reused while (slots, lengths) repeat, e.g. across
  // the layers of one lockstep decode step)
  Plan plans_[kPlanSlots];
  int grid_limit_ = 0;
  // recent appends (lockstep fast path across the layers of a decode step;
  // two entries for the two interleaved mini-batches)
  struct Fast {
    bool valid = false;
    int n = 0, layer = -1;
    uint64_t used = 0;
    std::vector<uint64_t> seqs;
    std::vector<uint32_t> pos;
    std::vector<int32_t> slots;
    Blob* blob = nullptr;
  };
  Fast fast_[2];
  Fast* fused_pending_ = nullptr;
  const uint8_t* l2pf_ = nullptr;
  int64_t l2pf_bytes_ = 0;
  int fused_prev_layer_ = -1;
  uint64_t fast_clock_ = 0;
  const Fast* fast_match(int n, const uint64_t* seqs) const;

  // timing
  bool timing_ = false;
  int timing_every_ = 1;
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending_;
  std::vector<double> ev_bytes_;
  double t_ms_ = 0, t_bytes_ = 0;
  int64_t t_launches_ = 0;
};

}  // namespace sd
