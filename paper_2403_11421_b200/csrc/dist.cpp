// DistEngine: sequence-sharded R-Part over NCCL (see dist.h).
#include "dist.h"

#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>

namespace sd {

namespace {

// NCCL is resolved at run time: inside a torch process this binds the NCCL
// torch already loaded (one NCCL per process), else the system libnccl.so.2.
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static Nccl& get() {
    static Nccl n;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) {
        err = dlerror() ? dlerror() : "dlopen failed";
        return;
      }
#define SD_SYM(f) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, "nccl" #f))
      SD_SYM(GetUniqueId);
      SD_SYM(CommInitRank);
      SD_SYM(CommDestroy);
      SD_SYM(GroupStart);
      SD_SYM(GroupEnd);
      SD_SYM(Send);
      SD_SYM(Recv);
      SD_SYM(AllReduce);
      SD_SYM(GetErrorString);
#undef SD_SYM
    });
    if (!n.Send || !n.Recv || !n.CommInitRank || !n.AllReduce) fail(SD_ERR_NCCL, "libnccl.so.2 unavailable: " + err);
    return n;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    fail(SD_ERR_NCCL, std::string(what) + ": " + Nccl::get().GetErrorString(r));
  }
}

}  // namespace

void nccl_unique_id(ncclUniqueId* id) { nccl_check(Nccl::get().GetUniqueId(id), "ncclGetUniqueId"); }

// Home rank of every batch row. s_ranks == 1: rank 0 (the paper's single
// S-worker). Data-parallel S-ranks under by-sequence sharding: each rank is
// home to a balanced quota (floor/ceil of B / world), filled first with the
// rows whose KV it holds, in batch order; the overflow rows of the heavier
// shards fill the remaining quotas in rank order. Every rank derives the same
// assignment from the batch. SD_HOME_MODULO (and the other shard modes):
// seq % s_ranks.
static void assign_homes(int world, int s_ranks, int B, const uint64_t* seqs, int mode, bool modulo,
                         std::vector<int32_t>& home) {
  home.assign(static_cast<size_t>(B), 0);
  if (s_ranks <= 1) return;
  if (modulo || mode != SD_SHARD_BY_SEQUENCE || s_ranks != world) {
    for (int i = 0; i < B; ++i) home[static_cast<size_t>(i)] = home_of(seqs[i], s_ranks);
    return;
  }
  std::vector<int32_t> quota(static_cast<size_t>(world)), cnt(static_cast<size_t>(world), 0);
  for (int r = 0; r < world; ++r) quota[static_cast<size_t>(r)] = B / world + (r < B % world ? 1 : 0);
  std::vector<int32_t> overflow;
  for (int i = 0; i < B; ++i) {
    const size_t pref = static_cast<size_t>(shard_of(seqs[i], world));
    if (cnt[pref] < quota[pref]) {
      home[static_cast<size_t>(i)] = static_cast<int32_t>(pref);
      ++cnt[pref];
    } else {
      overflow.push_back(i);
    }
  }
  size_t r = 0;
  for (int32_t i : overflow) {
    while (cnt[r] >= quota[r]) ++r;
    home[static_cast<size_t>(i)] = static_cast<int32_t>(r);
    ++cnt[r];
  }
}

void make_plan(int world, int rank, int s_ranks, int B, const uint64_t* seqs, DistPlan& p, int mode, int heads) {
  const bool modulo = (mode & SD_HOME_MODULO) != 0;
  mode &= ~SD_HOME_MODULO;
  if (mode == SD_SHARD_BY_SEQUENCE) {
    p.hg = 1;
    p.sg = world;
  } else if (mode == SD_SHARD_BY_HEAD) {
    if (world > heads) fail(SD_ERR_CONFIG, "by-head sharding cannot use more workers than heads");
    p.hg = world;
    p.sg = 1;
  } else if (mode == SD_SHARD_HYBRID) {
    p.hg = std::gcd(world, heads);
    p.sg = world / p.hg;
  } else {
    fail(SD_ERR_CONFIG, "invalid shard mode");
  }
  p.mode = mode;
  const size_t W = static_cast<size_t>(world);
  p.head_start.assign(W, 0);
  p.head_count.assign(W, heads);
  for (int w = 0; w < world; ++w) {
    if (mode == SD_SHARD_BY_SEQUENCE) continue;
    const auto r = shard_head_range(mode, heads, world, w);
    p.head_start[static_cast<size_t>(w)] = r.first;
    p.head_count[static_cast<size_t>(w)] = r.second;
  }
  auto sg_of = [&](uint64_t seq) {
    return p.sg == 1 ? 0 : static_cast<int>(mix64(seq) % static_cast<uint64_t>(p.sg));
  };
  assign_homes(world, s_ranks, B, seqs, mode, modulo, p.home);
  p.home_rows.clear();
  p.shard_rows.clear();
  p.shard_seqs.clear();
  p.send_cnt.assign(W, 0);
  p.send_off.assign(W, 0);
  p.recv_cnt.assign(W, 0);
  p.recv_off.assign(W, 0);
  // home rows grouped by sequence group (batch order inside a group); each
  // worker of group sg receives the group's block with its head slice
  std::vector<int32_t> blk_off(static_cast<size_t>(p.sg), 0), blk_cnt(static_cast<size_t>(p.sg), 0);
  for (int g = 0; g < p.sg; ++g) {
    blk_off[static_cast<size_t>(g)] = static_cast<int32_t>(p.home_rows.size());
    for (int i = 0; i < B; ++i) {
      if (p.home[static_cast<size_t>(i)] == rank && sg_of(seqs[i]) == g) p.home_rows.push_back(i);
    }
    blk_cnt[static_cast<size_t>(g)] = static_cast<int32_t>(p.home_rows.size()) - blk_off[static_cast<size_t>(g)];
  }
  for (int w = 0; w < world; ++w) {
    p.send_off[static_cast<size_t>(w)] = blk_off[static_cast<size_t>(w % p.sg)];
    p.send_cnt[static_cast<size_t>(w)] = blk_cnt[static_cast<size_t>(w % p.sg)];
  }
  // shard rows: this worker's sequence group from every source S-rank, each
  // in that source's send order
  const int my_sg = rank % p.sg;
  for (int src = 0; src < world; ++src) {
    p.recv_off[static_cast<size_t>(src)] = static_cast<int32_t>(p.shard_rows.size());
    for (int i = 0; i < B; ++i) {
      if (p.home[static_cast<size_t>(i)] == src && sg_of(seqs[i]) == my_sg) {
        p.shard_rows.push_back(i);
        p.shard_seqs.push_back(seqs[i]);
      }
    }
    p.recv_cnt[static_cast<size_t>(src)] = static_cast<int32_t>(p.shard_rows.size()) - p.recv_off[static_cast<size_t>(src)];
  }
}

DistEngine::DistEngine(Weights* w, KvStore* kv, int rank, int world, const void* nccl_id, int s_ranks,
                       int shard_mode)
    : spec_(kv->spec()), w_(w), kv_(kv), rank_(rank), world_(world), s_ranks_(s_ranks),
      device_(kv->device()), mode_(shard_mode & ~SD_HOME_MODULO), home_flags_(shard_mode & SD_HOME_MODULO) {
  if (world < 1 || rank < 0 || rank >= world) fail(SD_ERR_CONFIG, "bad rank / world");
  if (s_ranks != 1 && s_ranks != world) fail(SD_ERR_CONFIG, "s_ranks must be 1 or world");
  const bool s_rank = s_ranks == world || rank == 0;
  if (s_rank && !w) fail(SD_ERR_CONFIG, "an S-rank needs weights");
  if (w && w->device() != device_) fail(SD_ERR_CONFIG, "weights and KV store on different devices");
  {
    // the shard's kv-head range must be this worker's (ShardMap head_range)
    DistPlan probe;
    const uint64_t one = 1;
    make_plan(world, rank, s_ranks, 1, &one, probe, shard_mode, spec_.Hkv);
    const int h0 = probe.head_start[static_cast<size_t>(rank)], hc = probe.head_count[static_cast<size_t>(rank)];
    if (kv->head_start() != h0 || kv->width() != hc * spec_.hd) {
      fail(SD_ERR_CONFIG, "R-shard must hold kv heads [" + std::to_string(h0) + ", " + std::to_string(h0 + hc) +
                              ") for this shard mode and rank");
    }
  }
  DeviceGuard dg(device_);
  phases_ = tuning().dist_phases != 0;
  SD_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  if (world > 1 && nccl_id) {  // NULL: no communicator, the peer exchange carries everything
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    nccl_check(Nccl::get().CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
}

DistEngine::~DistEngine() {
  DeviceGuard dg(device_);
  cudaStreamSynchronize(stream_);
  if (phases_ && !ph_.empty()) {
    try {
      flush_phases();
    } catch (...) {
    }
  }
  if (phases_ && ph_layers_) {
    static const char* names[] = {"", "qkv", "recv_qkv", "append", "attend", "recv_o", "to_bf16", "w_o", "mlp_in", "mlp_out"};
    std::string line = "[dist phases] rank " + std::to_string(rank_) + ", " + std::to_string(ph_layers_) +
                       " layers, ms/layer:";
    for (int i = 1; i < 10; ++i) {
      char b[48];
      std::snprintf(b, sizeof(b), " %s=%.4f", names[i], ph_ms_[i] / static_cast<double>(ph_layers_));
      line += b;
    }
    line += "\n";
    std::fputs(line.c_str(), stderr);  // one write: ranks share the terminal
  }
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  for (void* p : {static_cast<void*>(rx_qkv_), static_cast<void*>(rx_o_), static_cast<void*>(flags_),
                  static_cast<void*>(done_), static_cast<void*>(gemm_done_),
                  static_cast<void*>(attn_done_), static_cast<void*>(rx_ob_), static_cast<void*>(rx_tok_)}) {
    if (p) cudaFree(p);
  }
  if (comm_) Nccl::get().CommDestroy(comm_);
  for (void* p : {static_cast<void*>(x_), static_cast<void*>(qkv_h_), static_cast<void*>(qkv_s_),
                  static_cast<void*>(o_s_), static_cast<void*>(o_h_), static_cast<void*>(y_),
                  static_cast<void*>(h_), static_cast<void*>(logits_), static_cast<void*>(xb_),
                  static_cast<void*>(ob_), static_cast<void*>(yb_), static_cast<void*>(hb_),
                  static_cast<void*>(tok_), static_cast<void*>(all_tok_), static_cast<void*>(home_idx_),
                  static_cast<void*>(amax_)}) {
    if (p) cudaFree(p);
  }
  for (auto& e : ev_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  cudaStreamDestroy(stream_);
}

void DistEngine::ensure(int B) {
  if (B <= cap_) return;
  DeviceGuard dg(device_);
  SD_CUDA(cudaStreamSynchronize(stream_));
  for (void* p : {static_cast<void*>(x_), static_cast<void*>(qkv_h_), static_cast<void*>(qkv_s_),
                  static_cast<void*>(o_s_), static_cast<void*>(o_h_), static_cast<void*>(y_),
                  static_cast<void*>(h_), static_cast<void*>(logits_), static_cast<void*>(xb_),
                  static_cast<void*>(ob_), static_cast<void*>(yb_), static_cast<void*>(hb_),
                  static_cast<void*>(tok_), static_cast<void*>(all_tok_), static_cast<void*>(home_idx_),
                  static_cast<void*>(amax_)}) {
    if (p) cudaFree(p);
  }
  const size_t bp = (static_cast<size_t>(B) + 127) / 128 * 128;
  const Spec& s = spec_;
  auto zalloc = [&](void** p, size_t bytes) {
    SD_CUDA(cudaMalloc(p, bytes));
    SD_CUDA(cudaMemset(*p, 0, bytes));
  };
  zalloc(reinterpret_cast<void**>(&x_), bp * s.D * 4);
  zalloc(reinterpret_cast<void**>(&qkv_h_), bp * s.qkv_width() * 4);
  zalloc(reinterpret_cast<void**>(&qkv_s_), bp * s.qkv_width() * 4);
  zalloc(reinterpret_cast<void**>(&o_s_), bp * s.D * 4);
  zalloc(reinterpret_cast<void**>(&o_h_), bp * s.D * 4);
  zalloc(reinterpret_cast<void**>(&y_), bp * s.D * 4);
  zalloc(reinterpret_cast<void**>(&h_), bp * s.F * 4);
  zalloc(reinterpret_cast<void**>(&logits_), bp * s.V * 4);
  zalloc(reinterpret_cast<void**>(&xb_), bp * s.D * 2);
  zalloc(reinterpret_cast<void**>(&ob_), bp * s.D * 2);
  zalloc(reinterpret_cast<void**>(&yb_), bp * s.D * 2);
  zalloc(reinterpret_cast<void**>(&hb_), bp * s.F * 2);
  zalloc(reinterpret_cast<void**>(&tok_), bp * 4);
  zalloc(reinterpret_cast<void**>(&all_tok_), bp * 4);
  zalloc(reinterpret_cast<void**>(&home_idx_), bp * 4);
  zalloc(reinterpret_cast<void**>(&amax_), bp * 8);
  SD_CUDA(cudaDeviceSynchronize());  // legacy-stream memsets before non-blocking-stream use
  cap_ = B;
}

void DistEngine::plan_for(int B, const uint64_t* seqs) {
  if (plan_key_.size() == static_cast<size_t>(B) && std::equal(plan_key_.begin(), plan_key_.end(), seqs)) return;
  make_plan(world_, rank_, s_ranks_, B, seqs, plan_, mode_ | home_flags_, spec_.Hkv);
  home_set_.clear();
  for (int32_t i : plan_.home_rows) home_set_.insert(seqs[i]);
  if (!plan_.home_rows.empty()) {
    SD_CUDA(cudaMemcpyAsync(home_idx_, plan_.home_rows.data(), plan_.home_rows.size() * 4, cudaMemcpyHostToDevice,
                            stream_));
  }
  plan_key_.assign(seqs, seqs + B);
  if (mode_ != SD_SHARD_BY_SEQUENCE && !p2p_) {
    fail(SD_ERR_CONFIG, "by-head / hybrid sharding needs the peer exchange (sd_dist_p2p_connect)");
  }
  if (world_ > 1 && !comm_ && !p2p_) {
    fail(SD_ERR_CONFIG, "a distributed engine without an NCCL id needs the peer exchange (sd_dist_p2p_connect)");
  }
  if (p2p_) {
    // where this rank's rows land in each peer's receive buffers (every rank
    // derives every plan from the same batch)
    peer_qkv_off_.assign(static_cast<size_t>(world_), 0);
    peer_o_off_.assign(static_cast<size_t>(world_), 0);
    DistPlan q;
    for (int d = 0; d < world_; ++d) {
      make_plan(world_, d, s_ranks_, B, seqs, q, mode_ | home_flags_, spec_.Hkv);
      peer_qkv_off_[static_cast<size_t>(d)] = q.recv_off[static_cast<size_t>(rank_)];
      peer_o_off_[static_cast<size_t>(d)] = q.send_off[static_cast<size_t>(rank_)];
      if (static_cast<int>(q.home_rows.size()) > p2p_cap_ || static_cast<int>(q.shard_rows.size()) > p2p_cap_) {
        fail(SD_ERR_CAPACITY, "peer exchange: batch exceeds the p2p_setup row capacity");
      }
    }
    if (fused_) build_routes();
  }
}

// device tables of the fused exchange: home row -> (shard rank, row in its
// receive buffer) and shard row -> (home rank, row in its receive buffer)
void DistEngine::build_routes() {
  const size_t nh = plan_.home_rows.size(), ns = plan_.shard_rows.size();
  std::vector<int32_t> t(2 * nh + 2 * ns + 1, 0);
  for (int d = 0; d < world_; ++d) {
    const size_t u = static_cast<size_t>(d);
    for (int j = 0; j < plan_.send_cnt[u]; ++j) {
      const size_t i = static_cast<size_t>(plan_.send_off[u] + j);
      t[i] = d;
      t[nh + i] = peer_qkv_off_[u] + j;
    }
    for (int j = 0; j < plan_.recv_cnt[u]; ++j) {
      const size_t i = static_cast<size_t>(plan_.recv_off[u] + j);
      t[2 * nh + i] = d;
      t[2 * nh + ns + i] = peer_o_off_[u] + j;
    }
  }
  route_.get(t.size() * 4);
  SD_CUDA(cudaMemcpy(route_.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
}

void DistEngine::p2p_setup(int max_rows, void* handles_out) {
  if (world_ > kMaxWorld) fail(SD_ERR_CONFIG, "peer exchange supports at most 8 ranks");
  if (max_rows < 1) fail(SD_ERR_CONFIG, "p2p_setup: max_rows must be positive");
  DeviceGuard dg(device_);
  SD_CUDA(cudaStreamSynchronize(stream_));
  for (void* p : {static_cast<void*>(rx_qkv_), static_cast<void*>(rx_o_), static_cast<void*>(flags_),
                  static_cast<void*>(done_), static_cast<void*>(gemm_done_),
                  static_cast<void*>(attn_done_), static_cast<void*>(rx_ob_), static_cast<void*>(rx_tok_)}) {
    if (p) cudaFree(p);
  }
  const size_t rows = (static_cast<size_t>(max_rows) + 127) / 128 * 128;
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_qkv_), rows * spec_.qkv_width() * 4));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_o_), rows * spec_.D * 4));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_ob_), rows * spec_.D * 2));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_tok_), 2 * rows * sizeof(int32_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&flags_), kFlagSlots * kMaxWorld * sizeof(int64_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&done_), sizeof(int32_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&gemm_done_), sizeof(int32_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&attn_done_), sizeof(int32_t)));
  SD_CUDA(cudaMemset(gemm_done_, 0, sizeof(int32_t)));
  SD_CUDA(cudaMemset(attn_done_, 0, sizeof(int32_t)));
  SD_CUDA(cudaMemset(rx_qkv_, 0, rows * spec_.qkv_width() * 4));
  SD_CUDA(cudaMemset(rx_o_, 0, rows * spec_.D * 4));
  SD_CUDA(cudaMemset(flags_, 0, kFlagSlots * kMaxWorld * sizeof(int64_t)));
  SD_CUDA(cudaMemset(rx_tok_, 0, 2 * rows * sizeof(int32_t)));
  SD_CUDA(cudaMemset(done_, 0, sizeof(int32_t)));
  SD_CUDA(cudaDeviceSynchronize());
  SD_CUDA(cudaMemset(rx_ob_, 0, rows * spec_.D * 2));
  cudaIpcMemHandle_t h[kIpcHandles];
  SD_CUDA(cudaIpcGetMemHandle(&h[4], rx_tok_));
  SD_CUDA(cudaIpcGetMemHandle(&h[0], rx_qkv_));
  SD_CUDA(cudaIpcGetMemHandle(&h[1], rx_o_));
  SD_CUDA(cudaIpcGetMemHandle(&h[2], flags_));
  SD_CUDA(cudaIpcGetMemHandle(&h[3], rx_ob_));
  std::memset(handles_out, 0, kIpcBytes);
  std::memcpy(handles_out, h, sizeof(h));
  const int32_t mode = w_ ? w_->mode() : -1;
  std::memcpy(static_cast<uint8_t*>(handles_out) + sizeof(h), &mode, sizeof(mode));
  p2p_cap_ = max_rows;
  tok_rows_ = static_cast<int>(rows);
  epoch_ = 0;
  tok_epoch_ = 0;
}

void DistEngine::p2p_connect(const void* all_handles) {
  if (!rx_qkv_) fail(SD_ERR_CONFIG, "p2p_connect before p2p_setup");
  DeviceGuard dg(device_);
  const auto* hb = static_cast<const uint8_t*>(all_handles);
  for (int p = 0; p < world_; ++p) {
    cudaIpcMemHandle_t h[kIpcHandles];
    std::memcpy(h, hb + static_cast<size_t>(p) * kIpcBytes, sizeof(h));
    std::memcpy(&peer_mode_[p], hb + static_cast<size_t>(p) * kIpcBytes + sizeof(h), sizeof(int32_t));
    if (p == rank_) {
      peer_qkv_[p] = rx_qkv_;
      peer_o_[p] = rx_o_;
      peer_flags_[p] = flags_;
      peer_ob_[p] = rx_ob_;
      peer_tok_[p] = rx_tok_;
      continue;
    }
    void* ptr[kIpcHandles];
    for (int i = 0; i < kIpcHandles; ++i) {
      SD_CUDA(cudaIpcOpenMemHandle(&ptr[i], h[i], cudaIpcMemLazyEnablePeerAccess));
      opened_.push_back(ptr[i]);
    }
    peer_qkv_[p] = static_cast<float*>(ptr[0]);
    peer_o_[p] = static_cast<float*>(ptr[1]);
    peer_flags_[p] = static_cast<int64_t*>(ptr[2]);
    peer_ob_[p] = static_cast<act16*>(ptr[3]);
    peer_tok_[p] = static_cast<int32_t*>(ptr[4]);
  }
  p2p_ = true;
  // the exchange is fused into the producers when both have a routed form
  fused_ = tuning().dist_fuse != 0 && mode_ == SD_SHARD_BY_SEQUENCE && kv_->tensor_core_path();
  plan_key_.clear();  // recompute the peer offsets
}

void DistEngine::exchange_p2p(int kind) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timing_) {
    SD_CUDA(cudaEventCreate(&e0));
    SD_CUDA(cudaEventCreate(&e1));
    SD_CUDA(cudaEventRecord(e0, stream_));
  }
  const int hd = spec_.hd, G = spec_.H / spec_.Hkv, D = spec_.D, kvw = spec_.kv_width();
  const int my_hc = plan_.head_count[static_cast<size_t>(rank_)], my_h0 = plan_.head_start[static_cast<size_t>(rank_)];
  P2PScatter a{};
  a.world = world_;
  a.self = rank_;
  a.slot = kind;
  a.epoch = ++epoch_;
  a.done = done_;
  const std::vector<int32_t>& sc = kind == 0 ? plan_.send_cnt : plan_.recv_cnt;
  const std::vector<int32_t>& so = kind == 0 ? plan_.send_off : plan_.recv_off;
  const std::vector<int32_t>& rc = kind == 0 ? plan_.recv_cnt : plan_.send_cnt;
  // kind 0: home rows (full q|k|v width) -> each worker's head slice packed
  //         as [q slice | k slice | v slice];
  // kind 1: shard rows (this worker's o slice) -> the home rows' o columns
  a.src = kind == 0 ? qkv_h_ : o_s_;
  a.src_stride = kind == 0 ? spec_.qkv_width() : static_cast<int64_t>(my_hc) * G * hd;
  double bytes = 0;
  uint32_t expect = 0;
  for (int d = 0; d < world_; ++d) {
    const size_t u = static_cast<size_t>(d);
    const int h0 = plan_.head_start[u], hc = plan_.head_count[u];
    a.cnt[d] = sc[u];
    a.src_off[d] = so[u];
    a.dst_off[d] = kind == 0 ? peer_qkv_off_[u] : peer_o_off_[u];
    a.dst[d] = kind == 0 ? peer_qkv_[d] : peer_o_[d];
    a.flag[d] = peer_flags_[d];
    if (kind == 0) {
      const int qw = hc * G * hd, kw = hc * hd;
      a.dst_stride[d] = qw + 2 * kw;
      a.nseg[d] = 3;
      a.seg_src[d][0] = h0 * G * hd, a.seg_dst[d][0] = 0, a.seg_n[d][0] = qw;
      a.seg_src[d][1] = D + h0 * hd, a.seg_dst[d][1] = qw, a.seg_n[d][1] = kw;
      a.seg_src[d][2] = D + kvw + h0 * hd, a.seg_dst[d][2] = qw + kw, a.seg_n[d][2] = kw;
    } else {
      a.dst_stride[d] = D;
      a.nseg[d] = 1;
      a.seg_src[d][0] = 0, a.seg_dst[d][0] = my_h0 * G * hd, a.seg_n[d][0] = my_hc * G * hd;
    }
    if (d != rank_ && sc[u] > 0) {
      a.notify |= 1u << d;
      int w = 0;
      for (int q = 0; q < a.nseg[d]; ++q) w += a.seg_n[d][q];
      bytes += static_cast<double>(sc[u]) * w * 4;
    }
    if (d != rank_ && rc[u] > 0) expect |= 1u << d;
  }
  launch_p2p_scatter(a, stream_);
  launch_p2p_wait(flags_, kind, expect, world_, a.epoch, stream_);
  if (timing_) {
    SD_CUDA(cudaEventRecord(e1, stream_));
    ev_.emplace_back(e0, e1);
    ev_bytes_.push_back(bytes);
  }
}

// per-destination grouped send/recv (the scatter of send_layer and the
// gather of receive_layer); the rank's own rows are a device copy
void DistEngine::exchange(const float* send, const std::vector<int32_t>& sc, const std::vector<int32_t>& so,
                          float* recv, const std::vector<int32_t>& rc, const std::vector<int32_t>& ro,
                          int width) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double bytes = 0;
  if (timing_) {
    SD_CUDA(cudaEventCreate(&e0));
    SD_CUDA(cudaEventCreate(&e1));
    SD_CUDA(cudaEventRecord(e0, stream_));
  }
  const size_t w = static_cast<size_t>(width);
  const int self = rank_;
  if (sc[static_cast<size_t>(self)]) {
    SD_CUDA(cudaMemcpyAsync(recv + ro[static_cast<size_t>(self)] * w, send + so[static_cast<size_t>(self)] * w,
                            static_cast<size_t>(sc[static_cast<size_t>(self)]) * w * 4, cudaMemcpyDeviceToDevice,
                            stream_));
  }
  if (world_ > 1) {
    Nccl& n = Nccl::get();
    nccl_check(n.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < world_; ++p) {
      if (p == self) continue;
      const size_t c_s = static_cast<size_t>(sc[static_cast<size_t>(p)]);
      const size_t c_r = static_cast<size_t>(rc[static_cast<size_t>(p)]);
      if (c_s) {
        nccl_check(n.Send(send + so[static_cast<size_t>(p)] * w, c_s * w, ncclFloat32, p, comm_, stream_), "ncclSend");
        bytes += static_cast<double>(c_s * w * 4);
      }
      if (c_r) {
        nccl_check(n.Recv(recv + ro[static_cast<size_t>(p)] * w, c_r * w, ncclFloat32, p, comm_, stream_), "ncclRecv");
      }
    }
    nccl_check(n.GroupEnd(), "ncclGroupEnd");
  }
  if (timing_) {
    SD_CUDA(cudaEventRecord(e1, stream_));
    ev_.emplace_back(e0, e1);
    ev_bytes_.push_back(bytes);
  }
}

// bytes this rank sends to peers in one exchange (kind 0: q|k|v rows, 1: o rows)
double DistEngine::kind_bytes(int kind) const {
  const std::vector<int32_t>& sc = kind == 0 ? plan_.send_cnt : plan_.recv_cnt;
  const int w = kind == 0 ? spec_.qkv_width() : spec_.D;
  double b = 0;
  for (int d = 0; d < world_; ++d) {
    if (d != rank_) b += static_cast<double>(sc[static_cast<size_t>(d)]) * w * 4;
  }
  return b;
}

// the receive side of a producer-fused exchange; under timing, the wait is
// what remains of the exchange once the stores overlapped the producer
void DistEngine::fused_wait(int slot, uint32_t expect, int64_t epoch, double bytes) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timing_) {
    SD_CUDA(cudaEventCreate(&e0));
    SD_CUDA(cudaEventCreate(&e1));
    SD_CUDA(cudaEventRecord(e0, stream_));
  }
  launch_p2p_wait(flags_, slot, expect, world_, epoch, stream_);
  if (timing_) {
    SD_CUDA(cudaEventRecord(e1, stream_));
    ev_.emplace_back(e0, e1);
    ev_bytes_.push_back(bytes);
  }
}

void DistEngine::mark(int phase) {
  if (!ph_on_) return;
  cudaEvent_t e;
  SD_CUDA(cudaEventCreate(&e));
  SD_CUDA(cudaEventRecord(e, stream_));
  ph_.emplace_back(phase, e);
}

void DistEngine::flush_phases() {
  for (size_t i = 0; i < ph_.size(); ++i) {
    SD_CUDA(cudaEventSynchronize(ph_[i].second));
    if (ph_[i].first == 0) {
      ++ph_layers_;
    } else {
      float t = 0;
      SD_CUDA(cudaEventElapsedTime(&t, ph_[i - 1].second, ph_[i].second));
      ph_ms_[ph_[i].first] += t;
    }
  }
  for (auto& p : ph_) cudaEventDestroy(p.second);
  ph_.clear();
}

void DistEngine::read_timing(double* ms, double* bytes, bool reset) {
  if (phases_) flush_phases();
  for (size_t i = 0; i < ev_.size(); ++i) {
    SD_CUDA(cudaEventSynchronize(ev_[i].second));
    float t = 0;
    SD_CUDA(cudaEventElapsedTime(&t, ev_[i].first, ev_[i].second));
    x_ms_ += t;
    x_bytes_ += ev_bytes_[i];
    cudaEventDestroy(ev_[i].first);
    cudaEventDestroy(ev_[i].second);
  }
  ev_.clear();
  ev_bytes_.clear();
  if (ms) *ms = x_ms_;
  if (bytes) *bytes = x_bytes_;
  if (reset) x_ms_ = x_bytes_ = 0;
}

// one decode step with the home tokens already in tok_ (home order)
void DistEngine::run_step() {
  const Spec& s = spec_;
  const int D = s.D, F = s.F, qkvw = s.qkv_width(), kvw = s.kv_width();
  const int nh = static_cast<int>(plan_.home_rows.size());
  const int ns = static_cast<int>(plan_.shard_rows.size());
  // kind::f16 homes keep 16-bit copies of the GEMM A operands (bf16 or fp16)
  const bool bf = w_ && (w_->mode() == SD_DENSE_BF16 || w_->mode() == SD_DENSE_F16);
  const int f16 = w_ && w_->mode() == SD_DENSE_F16 ? 1 : 0;
  if (nh) launch_embed(nh, D, tok_, w_->embedding(), x_, D, bf ? xb_ : nullptr, f16, stream_);
  const bool fused = p2p_ && fused_;
  const bool route_qkv = fused && nh && w_->mode() != SD_DENSE_EXACT_F32;  // exact mode: scatter kernel
  const int32_t* tbl = static_cast<const int32_t*>(route_.p);
  uint32_t to_shards = 0, from_homes = 0, to_homes = 0, from_shards = 0;
  for (int d = 0; d < world_; ++d) {
    if (d == rank_) continue;
    if (plan_.send_cnt[static_cast<size_t>(d)] > 0) to_shards |= 1u << d, from_shards |= 1u << d;
    if (plan_.recv_cnt[static_cast<size_t>(d)] > 0) from_homes |= 1u << d, to_homes |= 1u << d;
  }
  for (int l = 0; l < s.L; ++l) {
    ph_on_ = phases_ && l % 8 == 0;
    mark(0);
    if (route_qkv) {
      // project_qkv with the exchange in its epilogue: every home row lands in
      // its shard's receive buffer; the last CTA publishes the epoch
      RowRoute r{};
      r.rank = tbl;
      r.row = tbl + nh;
      r.ld = qkvw;
      r.rows = (p2p_cap_ + 127) / 128 * 128;  // every rank's rx_qkv_ (p2p_setup)
      for (int d = 0; d < world_; ++d) {
        r.base[d] = peer_qkv_[d];
        r.flag[d] = peer_flags_[d];
      }
      r.done = gemm_done_;
      r.epoch = ++epoch_;
      r.notify = to_shards;
      r.slot = 0;
      r.self = rank_;
      GemmArgs ga = w_->gemm_args(l, 0, nh, x_, D, xb_, D, nullptr, qkvw, nullptr, 0, kEpiNone, nullptr, 0);
      ga.route = &r;
      launch_gemm_sm100(ga, stream_);
      mark(1);
      fused_wait(0, from_homes, r.epoch, kind_bytes(0));
      mark(2);
    } else if (nh) {
      w_->linear(l, 0, nh, x_, D, xb_, D, qkv_h_, qkvw, nullptr, 0, kEpiNone, nullptr, 0, stream_);
      mark(1);
    }
    if (fused && !route_qkv) {  // nothing to send (or exact mode): the same flags / epochs
      if (nh) {
        exchange_p2p(0);
      } else {
        launch_p2p_wait(flags_, 0, from_homes, world_, ++epoch_, stream_);
      }
    }
    float* qkv_s = p2p_ ? rx_qkv_ : qkv_s_;
    float* o_h = p2p_ ? rx_o_ : o_h_;
    // this worker's head slice of a shard row: [q | k | v] (full width when by-sequence)
    const int G = s.H / s.Hkv;
    const int hc = plan_.head_count[static_cast<size_t>(rank_)];
    const int sq = hc * G * s.hd, sk = hc * s.hd, srow = p2p_ ? sq + 2 * sk : qkvw;
    if (fused) {
      // (sent above)
    } else if (p2p_) {
      exchange_p2p(0);
      mark(2);
    } else {
      exchange(qkv_h_, plan_.send_cnt, plan_.send_off, qkv_s, plan_.recv_cnt, plan_.recv_off, qkvw);
    }
    ORoute orr{};
    if (fused) {  // attention rows straight into their home rank's buffer
      orr.rank = tbl + 2 * nh;
      orr.row = tbl + 2 * nh + ns;
      orr.ld = D;
      for (int d = 0; d < world_; ++d) {
        // a kind::f16 home takes its W_o operand straight from the attention
        if (peer_mode_[d] == SD_DENSE_BF16 || peer_mode_[d] == SD_DENSE_F16) {
          orr.bbase[d] = peer_ob_[d];
          if (peer_mode_[d] == SD_DENSE_F16) orr.f16_mask |= 1u << d;
        } else {
          orr.base[d] = peer_o_[d];
        }
        orr.flag[d] = peer_flags_[d];
      }
      orr.bld = D;
      orr.done = attn_done_;
      orr.epoch = ++epoch_;
      orr.notify = to_homes;
      orr.slot = 1;
      orr.self = rank_;
    }
    if (ns) {
      for (int i = 0; i < ns; ++i) {
        pos_[static_cast<size_t>(i)] = static_cast<uint32_t>(kv_->stored(plan_.shard_seqs[static_cast<size_t>(i)], l));
      }
      kv_->append(l, ns, plan_.shard_seqs.data(), pos_.data(), qkv_s + sq, srow, qkv_s + sq + sk, srow, stream_);
      mark(3);
      kv_->attend(l, ns, plan_.shard_seqs.data(), qkv_s, srow, o_s_, p2p_ ? sq : D, stream_, 0, nullptr, 0,
                  fused ? &orr : nullptr);
      mark(4);
    }
    if (fused) {
      fused_wait(1, from_shards, orr.epoch, kind_bytes(1));
      mark(5);
    } else if (p2p_) {
      exchange_p2p(1);
      mark(5);
    } else {
      exchange(o_s_, plan_.recv_cnt, plan_.recv_off, o_h, plan_.send_cnt, plan_.send_off, D);
    }
    if (nh) {
      act16* ob = fused && bf ? rx_ob_ : ob_;  // fused: the attention wrote it
      if (bf && !fused) launch_to_16(nh, D, o_h, D, ob_, D, f16, stream_);
      mark(6);
      w_->linear(l, 4, nh, o_h, D, ob, D, y_, D, bf ? yb_ : nullptr, D, kEpiResidual, x_, D, stream_);
      mark(7);
      w_->linear(l, 5, nh, y_, D, yb_, D, bf ? nullptr : h_, F, bf ? hb_ : nullptr, F, kEpiSilu, nullptr, 0, stream_);
      mark(8);
      w_->linear(l, 6, nh, h_, F, hb_, F, x_, D, bf ? xb_ : nullptr, D, kEpiResidual, y_, D, stream_);
      mark(9);
    }
  }
  if (nh) {
    if (w_->mode() != SD_DENSE_EXACT_F32 && tuning().fused_argmax) {
      // argmax_token in the head GEMM's epilogue: no logits round trip
      GemmArgs ga = w_->gemm_args(0, 7, nh, x_, D, xb_, D, nullptr, s.V, nullptr, 0, kEpiNone, nullptr, 0);
      ga.amax = amax_;
      launch_gemm_sm100(ga, stream_);
      launch_argmax_keys(nh, amax_, tok_, stream_);
    } else {
      w_->linear(0, 7, nh, x_, D, xb_, D, logits_, s.V, nullptr, 0, kEpiNone, nullptr, 0, stream_);
      launch_argmax(nh, s.V, logits_, s.V, tok_, stream_);
    }
  }
}

// validate_batch (core.cpp:37-54): a repeated sequence id is a ConfigError
// before anything is planned or appended
static void check_unique(int B, const uint64_t* seqs) {
  if (B == 0) fail(SD_ERR_CONFIG, "project_qkv: empty batch");
  std::unordered_set<uint64_t> seen;
  for (int i = 0; i < B; ++i) {
    if (!seen.insert(seqs[i]).second) {
      fail(SD_ERR_CONFIG, "token batch: duplicate sequence id " + std::to_string(seqs[i]));
    }
  }
}

void DistEngine::compute(int B, const uint64_t* seqs, const int32_t* tokens, int32_t* next, float* final_x) {
  check_unique(B, seqs);
  DeviceGuard dg(device_);
  ensure(B);
  plan_for(B, seqs);
  pos_.resize(static_cast<size_t>(B));
  const int nh = static_cast<int>(plan_.home_rows.size());
  host_tok_.resize(static_cast<size_t>(nh));
  for (int i = 0; i < nh; ++i) {
    const int32_t t = tokens[plan_.home_rows[static_cast<size_t>(i)]];
    if (t < 0 || t >= spec_.V) fail(SD_ERR_CONFIG, "token out of the vocabulary");
    host_tok_[static_cast<size_t>(i)] = t;
  }
  if (nh) SD_CUDA(cudaMemcpyAsync(tok_, host_tok_.data(), static_cast<size_t>(nh) * 4, cudaMemcpyHostToDevice, stream_));
  run_step();
  // every rank returns the whole batch's next tokens: a row's home can move
  // between steps (balanced homes follow the batch), so each rank's caller
  // keeps every sequence's last token. Homes write their rows into a zeroed
  // batch vector, summed across ranks (B int32 per step).
  if (world_ > 1 && p2p_) {
    // peer stores of the home rows' tokens into every rank's batch vector
    // (double-buffered by step parity: a rank can be at most one step ahead)
    const int64_t ep = ++tok_epoch_;
    const int half = static_cast<int>(ep & 1) * tok_rows_;
    P2PTokens a{};
    a.idx = home_idx_;
    a.src = tok_;
    a.n = nh;
    a.world = world_;
    a.self = rank_;
    a.slot = kTokSlot;
    a.epoch = ep;
    uint32_t others = 0;
    for (int d = 0; d < world_; ++d) {
      a.dst[d] = peer_tok_[d] + half;
      a.flag[d] = peer_flags_[d];
      if (d != rank_) others |= 1u << d;
    }
    a.notify = others;
    launch_p2p_tokens(a, stream_);
    launch_p2p_wait(flags_, kTokSlot, others, world_, ep, stream_);
    SD_CUDA(cudaMemcpyAsync(next, rx_tok_ + half, static_cast<size_t>(B) * 4, cudaMemcpyDeviceToHost, stream_));
  } else if (world_ > 1) {
    SD_CUDA(cudaMemsetAsync(all_tok_, 0, static_cast<size_t>(B) * 4, stream_));
    launch_scatter_i32(nh, home_idx_, tok_, all_tok_, stream_);
    nccl_check(Nccl::get().AllReduce(all_tok_, all_tok_, static_cast<size_t>(B), ncclInt32, ncclSum, comm_, stream_),
               "ncclAllReduce");
    SD_CUDA(cudaMemcpyAsync(next, all_tok_, static_cast<size_t>(B) * 4, cudaMemcpyDeviceToHost, stream_));
  } else if (nh) {
    SD_CUDA(cudaMemcpyAsync(host_tok_.data(), tok_, static_cast<size_t>(nh) * 4, cudaMemcpyDeviceToHost, stream_));
  }
  std::vector<float> fx;
  if (nh && final_x) {
    fx.resize(static_cast<size_t>(nh) * spec_.D);
    SD_CUDA(cudaMemcpyAsync(fx.data(), x_, fx.size() * 4, cudaMemcpyDeviceToHost, stream_));
  }
  SD_CUDA(cudaStreamSynchronize(stream_));
  for (int i = 0; i < nh; ++i) {
    const int row = plan_.home_rows[static_cast<size_t>(i)];
    if (world_ == 1) next[row] = host_tok_[static_cast<size_t>(i)];
    if (final_x) {
      std::memcpy(final_x + static_cast<size_t>(row) * spec_.D, fx.data() + static_cast<size_t>(i) * spec_.D,
                  static_cast<size_t>(spec_.D) * 4);
    }
  }
}

double DistEngine::bench(int B, const uint64_t* seqs, const int32_t* tokens, int steps) {
  check_unique(B, seqs);
  DeviceGuard dg(device_);
  ensure(B);
  plan_for(B, seqs);
  pos_.resize(static_cast<size_t>(B));
  const int nh = static_cast<int>(plan_.home_rows.size());
  host_tok_.resize(static_cast<size_t>(nh));
  for (int i = 0; i < nh; ++i) host_tok_[static_cast<size_t>(i)] = tokens[plan_.home_rows[static_cast<size_t>(i)]];
  if (nh) SD_CUDA(cudaMemcpyAsync(tok_, host_tok_.data(), static_cast<size_t>(nh) * 4, cudaMemcpyHostToDevice, stream_));
  cudaEvent_t e0, e1;
  SD_CUDA(cudaEventCreate(&e0));
  SD_CUDA(cudaEventCreate(&e1));
  SD_CUDA(cudaStreamSynchronize(stream_));
  SD_CUDA(cudaEventRecord(e0, stream_));
  for (int i = 0; i < steps; ++i) run_step();
  SD_CUDA(cudaEventRecord(e1, stream_));
  SD_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  SD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}

// DROP_SEQ (workers.cpp:482-501): routed to worker_for(seq, 0) under
// by-sequence sharding, to every link otherwise. Each rank drops the retiring
// sequences it stores: by-sequence mix64(seq) % world == rank; by-head every
// rank holds every sequence; hybrid the ranks of sequence group
// mix64(seq) % SG (worker w = hg * SG + sg).
bool DistEngine::holds(uint64_t seq) const {
  if (mode_ == SD_SHARD_BY_HEAD) return true;
  if (mode_ == SD_SHARD_HYBRID) {
    const int hg = std::gcd(world_, spec_.Hkv), sg = world_ / hg;
    return sg == 1 || static_cast<int>(mix64(seq) % static_cast<uint64_t>(sg)) == rank_ % sg;
  }
  return shard_of(seq, world_) == rank_;
}

void DistEngine::retire(int n, const uint64_t* seqs) {
  for (int i = 0; i < n; ++i) {
    if (holds(seqs[i])) kv_->drop(seqs[i]);
  }
}

}  // namespace sd
