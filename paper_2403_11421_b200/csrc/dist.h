// Multi-GPU decode: the reference's DistributedComputation (workers.cpp:264-501)
// on NVLink. Every rank is an R-shard holding the KV of the sequences the
// ShardMap assigns it (mix64(seq) % world, transport.cpp:352-353); S-ranks
// hold the weights and run the S-Part for their home rows. Per layer the
// Q/K/V rows of each home row go to the owning shard and the attention
// outputs come back (send_layer / receive_layer, workers.cpp:324-391), as
// NCCL grouped send/recv on the compute stream.
#pragma once

#include <nccl.h>

#include <unordered_set>
#include <vector>

#include "dist_p2p.cuh"
#include "engine.h"

namespace sd {

// S-rank of a sequence: rank 0 when s_ranks == 1 (the paper's single
// S-worker), else seq % s_ranks (data-parallel S-workers).
inline int home_of(uint64_t seq, int s_ranks) {
  return s_ranks <= 1 ? 0 : static_cast<int>(seq % static_cast<uint64_t>(s_ranks));
}
inline int shard_of(uint64_t seq, int world) {
  return static_cast<int>(mix64(seq) % static_cast<uint64_t>(world));
}

// Row plan of one step, identical on every rank (computed from the batch).
// ShardMap modes (transport.cpp:319-380): worker w = hg * SG + sg holds the
// kv heads of head group hg for the sequences of sequence group
// sg = mix64(seq) % SG. By-sequence: HG = 1, SG = world (the default); by
// head: HG = world, SG = 1; hybrid: HG = gcd(world, heads), SG = world / HG.
// Home rows are ordered by sg, so the rows a worker receives from an S-rank
// are one contiguous block (send_layer's per-worker filter, workers.cpp:336-351).
struct DistPlan {
  int mode = 0, hg = 1, sg = 1;     // shard mode, head groups, sequence groups
  std::vector<int32_t> home;        // home rank of every batch row
  std::vector<int32_t> home_rows;   // batch rows this rank runs the S-Part for, grouped by seq group
  std::vector<int32_t> send_cnt, send_off;  // per destination worker: block of home rows
  std::vector<int32_t> shard_rows;  // batch rows whose KV lives here, grouped by source S-rank
  std::vector<int32_t> recv_cnt, recv_off;
  std::vector<uint64_t> shard_seqs;
  std::vector<int32_t> head_start, head_count;  // per worker, in (kv) heads
};
void make_plan(int world, int rank, int s_ranks, int B, const uint64_t* seqs, DistPlan& p, int mode = 0,
               int heads = 1);
void nccl_unique_id(ncclUniqueId* id);

class DistEngine : public StepComputation {
 public:
  // shard_mode: SD_SHARD_BY_SEQUENCE (default), _BY_HEAD or _HYBRID over kv
  // heads; the KV store must hold this rank's head range (by-head / hybrid
  // need the peer exchange)
  DistEngine(Weights* w, KvStore* kv, int rank, int world, const void* nccl_id, int s_ranks,
             int shard_mode = 0);
  ~DistEngine() override;
  void compute(int B, const uint64_t* seqs, const int32_t* tokens, int32_t* next,
               float* final_x) override;
  void retire(int n, const uint64_t* seqs) override;
  // whether this rank's R-shard stores `seq` (ShardMap mode and rank)
  bool holds(uint64_t seq) const;
  // whether this rank produced `seq`'s token in the last step (homes are
  // assigned per step batch)
  bool owns(uint64_t seq) const override { return home_set_.count(seq) != 0; }
  int shard_mode() const { return mode_; }
  int model_dim() const override { return spec_.D; }
  int vocab() const override { return spec_.V; }
  // device-timed loop of `steps` steps over a fixed batch; tokens fed back on device
  double bench(int B, const uint64_t* seqs, const int32_t* tokens, int steps);
  void set_timing(bool on) { timing_ = on; }
  void read_timing(double* exch_ms, double* exch_bytes, bool reset);
  // The reference's two interleaved mini-batches (workers.cpp:405-452):
  // rows split by seq % 2 (merged when one is empty); every rank runs, per
  // layer and mini-batch, its shard's attention, then the S-Part of that
  // mini-batch's home rows, then its next QKV, so one mini-batch's attention
  // on the R-shards overlaps the other's dense work on the S-ranks. Needs
  // the peer exchange (sends never block there) when world > 1.
  void set_pipeline(bool on);
  // Peer-memory exchange (dist_p2p.cu): allocate fixed receive buffers for
  // up to `max_rows` rows per mini-batch and export their CUDA IPC handles
  // (kIpcBytes); connect() maps every rank's buffers (world x kIpcBytes, rank
  // order).
  // [rx_qkv | rx_o | flags | rx_ob | rx_tok handles][int32 dense mode of this rank, -1 none][pad]
  static constexpr int kIpcHandles = 5;
  static constexpr size_t kIpcBytes = kIpcHandles * sizeof(cudaIpcMemHandle_t) + 64;
  // flag slots: kind + 3 * mini-batch (kind 0 Q/K/V rows, 1 attention rows); 2 next tokens
  static constexpr int kFlagSlots = 6, kTokSlot = 2;
  static int slot(int kind, int g) { return kind + 3 * g; }
  void p2p_setup(int max_rows, void* handles_out);
  void p2p_connect(const void* all_handles);
  bool p2p() const { return p2p_; }

 private:
  // one mini-batch of the step (DistributedComputation::GroupState)
  struct Group {
    std::vector<int32_t> rows;  // batch rows, in batch order
    std::vector<uint64_t> seqs;
    DistPlan plan;              // over this mini-batch's rows
    int cap = 0;
    float *x = nullptr, *qkv_h = nullptr, *qkv_s = nullptr, *o_s = nullptr, *o_h = nullptr, *y = nullptr,
          *h = nullptr, *logits = nullptr;
    act16 *xb = nullptr, *ob = nullptr, *yb = nullptr, *hb = nullptr;
    int32_t* tok = nullptr;               // next tokens of the home rows (home order)
    int32_t* home_idx = nullptr;          // batch row of each home row
    unsigned long long* amax = nullptr;   // fused-argmax keys of the head GEMM
    std::vector<uint32_t> pos;
    std::vector<int32_t> host_tok;
    // peer exchange: this rank's rows' offsets in each peer's region of this
    // mini-batch, the fused routes, and who exchanges with whom
    std::vector<int32_t> peer_qkv_off, peer_o_off;
    DevBuf route;  // [qkv rank | qkv row | o rank | o row] int32 tables
    uint32_t to_shards = 0, from_homes = 0, to_homes = 0, from_shards = 0;
  };
  void ensure(int B);
  void free_group(Group& g);
  void plan_for(int B, const uint64_t* seqs);
  void run_step();
  // the reference's per-mini-batch phases (workers.cpp:405-452)
  void layer_in(int g, int l);    // project_qkv (+ embedding at l = 0 outside) and send_layer
  void shard_part(int g, int l);  // receive Q/K/V, append + attend this shard's rows, send O
  void layer_out(int g, int l);   // receive_layer + finish_block
  void head(int g);
  int64_t epoch_of(int l) const { return (steps_run_ - 1) * spec_.L + l + 1; }
  void exchange(const float* send, const std::vector<int32_t>& sc, const std::vector<int32_t>& so,
                float* recv, const std::vector<int32_t>& rc, const std::vector<int32_t>& ro, int width);
  // kind 0: Q/K/V rows home -> shard; kind 1: attention rows shard -> home
  double kind_bytes(const Group& G, int kind) const;
  void timed_wait(int slot, uint32_t expect, int64_t epoch, double bytes);
  void scatter_p2p(int g, int kind, int64_t epoch);
  // SD_DIST_PHASES=1: per-phase CUDA events on every 8th layer, summed into
  // ph_ms_ and printed to stderr per rank when the engine is destroyed
  void mark(int phase);
  void flush_phases();
  bool phases_ = false, ph_on_ = false;
  std::vector<std::pair<int, cudaEvent_t>> ph_;
  double ph_ms_[12] = {};
  int64_t ph_layers_ = 0;

  Spec spec_;
  Weights* w_;
  KvStore* kv_;
  int rank_, world_, s_ranks_, device_, mode_ = 0;
  ncclComm_t comm_ = nullptr;
  cudaStream_t stream_ = nullptr;
  Group groups_[2];
  int ngroups_ = 1;
  bool pipelined_ = false;
  int64_t steps_run_ = 0;
  int home_flags_ = 0;  // SD_HOME_MODULO or 0
  std::unordered_set<uint64_t> home_set_;
  std::vector<uint64_t> plan_key_;
  int cap_ = 0;
  int32_t* all_tok_ = nullptr;   // [B] next tokens of the whole batch (NCCL path)
  bool timing_ = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_;
  std::vector<double> ev_bytes_;
  double x_ms_ = 0, x_bytes_ = 0;
  // peer-memory exchange state: receive buffers hold two regions (one per
  // mini-batch) of rx_rows_ rows
  bool p2p_ = false;
  int p2p_cap_ = 0, rx_rows_ = 0;
  float *rx_qkv_ = nullptr, *rx_o_ = nullptr;  // receive buffers (shard rows / home rows)
  act16* rx_ob_ = nullptr;                     // home rows' attention output as the 16-bit W_o operand
  // fused exchange: the QKV GEMM and the attention store rows straight into
  // the peers' buffers (RowRoute / ORoute) and publish the epoch themselves.
  // Decided from rank-independent facts (a sender may still use the scatter
  // kernel, e.g. an exact-mode S-rank: receivers only see buffers and flags)
  bool fused_ = false;
  int32_t* gemm_done_ = nullptr;  // arrival counters of the routed launches
  int32_t* attn_done_ = nullptr;
  void build_routes(Group& G);
  int64_t* flags_ = nullptr;  // [kFlagSlots][kMaxWorld] epochs published by sources
  int32_t* done_ = nullptr;
  float* peer_qkv_[kMaxWorld] = {};
  float* peer_o_[kMaxWorld] = {};
  act16* peer_ob_[kMaxWorld] = {};
  int peer_mode_[kMaxWorld] = {};  // each rank's dense mode (-1: no weights)
  int64_t* peer_flags_[kMaxWorld] = {};
  int32_t* rx_tok_ = nullptr;  // [2][tok_rows_] next tokens of the batch (double-buffered)
  int32_t* peer_tok_[kMaxWorld] = {};
  int tok_rows_ = 0;
  int64_t tok_epoch_ = 0;
  std::vector<void*> opened_;
};

}  // namespace sd
