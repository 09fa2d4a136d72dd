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

void DistEngine::free_group(Group& G) {
  for (void* p : {static_cast<void*>(G.x), static_cast<void*>(G.qkv_h), static_cast<void*>(G.qkv_s),
                  static_cast<void*>(G.o_s), static_cast<void*>(G.o_h), static_cast<void*>(G.y),
                  static_cast<void*>(G.h), static_cast<void*>(G.logits), static_cast<void*>(G.xb),
                  static_cast<void*>(G.ob), static_cast<void*>(G.yb), static_cast<void*>(G.hb),
                  static_cast<void*>(G.tok), static_cast<void*>(G.home_idx), static_cast<void*>(G.amax)}) {
    if (p) cudaFree(p);
  }
  G.x = G.qkv_h = G.qkv_s = G.o_s = G.o_h = G.y = G.h = G.logits = nullptr;
  G.xb = G.ob = G.yb = G.hb = nullptr;
  G.tok = G.home_idx = nullptr;
  G.amax = nullptr;
  G.cap = 0;
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
    static const char* names[] = {"", "qkv", "recv_qkv", "append", "attend", "recv_o", "to_16", "w_o", "mlp_in", "mlp_out"};
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
                  static_cast<void*>(done_), static_cast<void*>(gemm_done_), static_cast<void*>(attn_done_),
                  static_cast<void*>(rx_ob_), static_cast<void*>(rx_tok_), static_cast<void*>(all_tok_)}) {
    if (p) cudaFree(p);
  }
  if (comm_) Nccl::get().CommDestroy(comm_);
  for (Group& G : groups_) free_group(G);
  for (auto& e : ev_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  cudaStreamDestroy(stream_);
}

void DistEngine::set_pipeline(bool on) {
  if (on && world_ > 1 && !p2p_) {
    fail(SD_ERR_CONFIG, "two mini-batches across ranks need the peer exchange (sd_dist_p2p_connect)");
  }
  pipelined_ = on;
  plan_key_.clear();
}

void DistEngine::ensure(int B) {
  if (B <= cap_) return;
  DeviceGuard dg(device_);
  SD_CUDA(cudaStreamSynchronize(stream_));
  if (all_tok_) cudaFree(all_tok_);
  all_tok_ = nullptr;
  const size_t bp = (static_cast<size_t>(B) + 127) / 128 * 128;
  const Spec& s = spec_;
  auto zalloc = [&](auto** p, size_t bytes) {
    SD_CUDA(cudaMalloc(reinterpret_cast<void**>(p), bytes));
    SD_CUDA(cudaMemset(*p, 0, bytes));
  };
  for (Group& G : groups_) {  // either mini-batch may hold the whole batch (merged)
    free_group(G);
    zalloc(&G.x, bp * s.D * 4);
    zalloc(&G.qkv_h, bp * s.qkv_width() * 4);
    zalloc(&G.qkv_s, bp * s.qkv_width() * 4);
    zalloc(&G.o_s, bp * s.D * 4);
    zalloc(&G.o_h, bp * s.D * 4);
    zalloc(&G.y, bp * s.D * 4);
    zalloc(&G.h, bp * s.F * 4);
    zalloc(&G.logits, bp * s.V * 4);
    zalloc(&G.xb, bp * s.D * 2);
    zalloc(&G.ob, bp * s.D * 2);
    zalloc(&G.yb, bp * s.D * 2);
    zalloc(&G.hb, bp * s.F * 2);
    zalloc(&G.tok, bp * 4);
    zalloc(&G.home_idx, bp * 4);
    zalloc(&G.amax, bp * 8);
    G.cap = B;
  }
  zalloc(&all_tok_, bp * 4);
  SD_CUDA(cudaDeviceSynchronize());  // legacy-stream memsets before non-blocking-stream use
  cap_ = B;
}

// Mini-batches (workers.cpp:405-420) and each one's row plan. Every rank
// derives the same groups and plans from the batch.
void DistEngine::plan_for(int B, const uint64_t* seqs) {
  if (plan_key_.size() == static_cast<size_t>(B) && std::equal(plan_key_.begin(), plan_key_.end(), seqs)) return;
  if (mode_ != SD_SHARD_BY_SEQUENCE && !p2p_) {
    fail(SD_ERR_CONFIG, "by-head / hybrid sharding needs the peer exchange (sd_dist_p2p_connect)");
  }
  if (world_ > 1 && !comm_ && !p2p_) {
    fail(SD_ERR_CONFIG, "a distributed engine without an NCCL id needs the peer exchange (sd_dist_p2p_connect)");
  }
  for (Group& G : groups_) {
    G.rows.clear();
    G.seqs.clear();
  }
  if (pipelined_) {
    for (int b = 0; b < B; ++b) groups_[seqs[b] % 2].rows.push_back(b);
  }
  if (!pipelined_ || groups_[0].rows.empty() || groups_[1].rows.empty()) {
    groups_[0].rows.resize(static_cast<size_t>(B));
    std::iota(groups_[0].rows.begin(), groups_[0].rows.end(), 0);
    groups_[1].rows.clear();
  }
  ngroups_ = groups_[1].rows.empty() ? 1 : 2;
  home_set_.clear();
  std::vector<int32_t> hidx;
  for (int g = 0; g < ngroups_; ++g) {
    Group& G = groups_[g];
    for (int32_t r : G.rows) G.seqs.push_back(seqs[r]);
    const int n = static_cast<int>(G.rows.size());
    make_plan(world_, rank_, s_ranks_, n, G.seqs.data(), G.plan, mode_ | home_flags_, spec_.Hkv);
    hidx.clear();
    for (int32_t i : G.plan.home_rows) {
      home_set_.insert(G.seqs[static_cast<size_t>(i)]);
      hidx.push_back(G.rows[static_cast<size_t>(i)]);
    }
    if (!hidx.empty()) {
      SD_CUDA(cudaMemcpyAsync(G.home_idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice, stream_));
      SD_CUDA(cudaStreamSynchronize(stream_));  // hidx is reused by the next group
    }
    G.pos.resize(static_cast<size_t>(n));
    G.to_shards = G.from_homes = G.to_homes = G.from_shards = 0;
    for (int d = 0; d < world_; ++d) {
      if (d == rank_) continue;
      if (G.plan.send_cnt[static_cast<size_t>(d)] > 0) G.to_shards |= 1u << d, G.from_shards |= 1u << d;
      if (G.plan.recv_cnt[static_cast<size_t>(d)] > 0) G.from_homes |= 1u << d, G.to_homes |= 1u << d;
    }
    if (p2p_) {
      // where this rank's rows land in each peer's receive region of this
      // mini-batch (every rank derives every plan from the same batch)
      G.peer_qkv_off.assign(static_cast<size_t>(world_), 0);
      G.peer_o_off.assign(static_cast<size_t>(world_), 0);
      DistPlan q;
      for (int d = 0; d < world_; ++d) {
        make_plan(world_, d, s_ranks_, n, G.seqs.data(), q, mode_ | home_flags_, spec_.Hkv);
        G.peer_qkv_off[static_cast<size_t>(d)] = q.recv_off[static_cast<size_t>(rank_)];
        G.peer_o_off[static_cast<size_t>(d)] = q.send_off[static_cast<size_t>(rank_)];
        if (static_cast<int>(q.home_rows.size()) > p2p_cap_ || static_cast<int>(q.shard_rows.size()) > p2p_cap_) {
          fail(SD_ERR_CAPACITY, "peer exchange: batch exceeds the p2p_setup row capacity");
        }
      }
      if (fused_) build_routes(G);
    }
  }
  plan_key_.assign(seqs, seqs + B);
}

// device tables of the fused exchange: home row -> (shard rank, row in its
// receive region) and shard row -> (home rank, row in its receive region)
void DistEngine::build_routes(Group& G) {
  const DistPlan& P = G.plan;
  const size_t nh = P.home_rows.size(), ns = P.shard_rows.size();
  std::vector<int32_t> t(2 * nh + 2 * ns + 1, 0);
  for (int d = 0; d < world_; ++d) {
    const size_t u = static_cast<size_t>(d);
    for (int j = 0; j < P.send_cnt[u]; ++j) {
      const size_t i = static_cast<size_t>(P.send_off[u] + j);
      t[i] = d;
      t[nh + i] = G.peer_qkv_off[u] + j;
    }
    for (int j = 0; j < P.recv_cnt[u]; ++j) {
      const size_t i = static_cast<size_t>(P.recv_off[u] + j);
      t[2 * nh + i] = d;
      t[2 * nh + ns + i] = G.peer_o_off[u] + j;
    }
  }
  G.route.get(t.size() * 4);
  SD_CUDA(cudaMemcpy(G.route.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
}

void DistEngine::p2p_setup(int max_rows, void* handles_out) {
  if (world_ > kMaxWorld) fail(SD_ERR_CONFIG, "peer exchange supports at most 8 ranks");
  if (max_rows < 1) fail(SD_ERR_CONFIG, "p2p_setup: max_rows must be positive");
  DeviceGuard dg(device_);
  SD_CUDA(cudaStreamSynchronize(stream_));
  for (void* p : {static_cast<void*>(rx_qkv_), static_cast<void*>(rx_o_), static_cast<void*>(flags_),
                  static_cast<void*>(done_), static_cast<void*>(gemm_done_), static_cast<void*>(attn_done_),
                  static_cast<void*>(rx_ob_), static_cast<void*>(rx_tok_)}) {
    if (p) cudaFree(p);
  }
  const size_t rows = (static_cast<size_t>(max_rows) + 127) / 128 * 128;  // per mini-batch region
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_qkv_), 2 * rows * spec_.qkv_width() * 4));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_o_), 2 * rows * spec_.D * 4));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_ob_), 2 * rows * spec_.D * 2));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&rx_tok_), 2 * rows * sizeof(int32_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&flags_), kFlagSlots * kMaxWorld * sizeof(int64_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&done_), sizeof(int32_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&gemm_done_), sizeof(int32_t)));
  SD_CUDA(cudaMalloc(reinterpret_cast<void**>(&attn_done_), sizeof(int32_t)));
  SD_CUDA(cudaMemset(gemm_done_, 0, sizeof(int32_t)));
  SD_CUDA(cudaMemset(attn_done_, 0, sizeof(int32_t)));
  SD_CUDA(cudaMemset(rx_qkv_, 0, 2 * rows * spec_.qkv_width() * 4));
  SD_CUDA(cudaMemset(rx_o_, 0, 2 * rows * spec_.D * 4));
  SD_CUDA(cudaMemset(rx_ob_, 0, 2 * rows * spec_.D * 2));
  SD_CUDA(cudaMemset(flags_, 0, kFlagSlots * kMaxWorld * sizeof(int64_t)));
  SD_CUDA(cudaMemset(rx_tok_, 0, 2 * rows * sizeof(int32_t)));
  SD_CUDA(cudaMemset(done_, 0, sizeof(int32_t)));
  SD_CUDA(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h[kIpcHandles];
  SD_CUDA(cudaIpcGetMemHandle(&h[0], rx_qkv_));
  SD_CUDA(cudaIpcGetMemHandle(&h[1], rx_o_));
  SD_CUDA(cudaIpcGetMemHandle(&h[2], flags_));
  SD_CUDA(cudaIpcGetMemHandle(&h[3], rx_ob_));
  SD_CUDA(cudaIpcGetMemHandle(&h[4], rx_tok_));
  std::memset(handles_out, 0, kIpcBytes);
  std::memcpy(handles_out, h, sizeof(h));
  const int32_t mode = w_ ? w_->mode() : -1;
  std::memcpy(static_cast<uint8_t*>(handles_out) + sizeof(h), &mode, sizeof(mode));
  p2p_cap_ = max_rows;
  rx_rows_ = static_cast<int>(rows);
  tok_rows_ = static_cast<int>(rows);
  steps_run_ = 0;
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

// the scatter kernel's send of one exchange of mini-batch g (no wait): kind
// 0 home rows (full q|k|v width) -> each worker's head slice packed as
// [q slice | k slice | v slice]; kind 1 shard rows (this worker's o slice)
// -> the home rows' o columns. Publishes `epoch` to every destination.
void DistEngine::scatter_p2p(int g, int kind, int64_t epoch) {
  Group& G = groups_[g];
  const DistPlan& P = G.plan;
  const int hd = spec_.hd, Gq = spec_.H / spec_.Hkv, D = spec_.D, kvw = spec_.kv_width();
  const int my_hc = P.head_count[static_cast<size_t>(rank_)], my_h0 = P.head_start[static_cast<size_t>(rank_)];
  P2PScatter a{};
  a.world = world_;
  a.self = rank_;
  a.slot = slot(kind, g);
  a.epoch = epoch;
  a.done = done_;
  const std::vector<int32_t>& sc = kind == 0 ? P.send_cnt : P.recv_cnt;
  const std::vector<int32_t>& so = kind == 0 ? P.send_off : P.recv_off;
  a.src = kind == 0 ? G.qkv_h : G.o_s;
  a.src_stride = kind == 0 ? spec_.qkv_width() : static_cast<int64_t>(my_hc) * Gq * hd;
  const size_t region = static_cast<size_t>(g) * rx_rows_;
  for (int d = 0; d < world_; ++d) {
    const size_t u = static_cast<size_t>(d);
    const int h0 = P.head_start[u], hc = P.head_count[u];
    a.cnt[d] = sc[u];
    a.src_off[d] = so[u];
    a.dst_off[d] = kind == 0 ? G.peer_qkv_off[u] : G.peer_o_off[u];
    a.dst[d] = kind == 0 ? peer_qkv_[d] + region * spec_.qkv_width() : peer_o_[d] + region * D;
    a.flag[d] = peer_flags_[d];
    if (kind == 0) {
      const int qw = hc * Gq * hd, kw = hc * hd;
      a.dst_stride[d] = qw + 2 * kw;
      a.nseg[d] = 3;
      a.seg_src[d][0] = h0 * Gq * hd, a.seg_dst[d][0] = 0, a.seg_n[d][0] = qw;
      a.seg_src[d][1] = D + h0 * hd, a.seg_dst[d][1] = qw, a.seg_n[d][1] = kw;
      a.seg_src[d][2] = D + kvw + h0 * hd, a.seg_dst[d][2] = qw + kw, a.seg_n[d][2] = kw;
    } else {
      a.dst_stride[d] = D;
      a.nseg[d] = 1;
      a.seg_src[d][0] = 0, a.seg_dst[d][0] = my_h0 * Gq * hd, a.seg_n[d][0] = my_hc * Gq * hd;
    }
    if (d != rank_ && sc[u] > 0) a.notify |= 1u << d;
  }
  launch_p2p_scatter(a, stream_);
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
double DistEngine::kind_bytes(const Group& G, int kind) const {
  const std::vector<int32_t>& sc = kind == 0 ? G.plan.send_cnt : G.plan.recv_cnt;
  const int w = kind == 0 ? spec_.qkv_width() : spec_.D;
  double b = 0;
  for (int d = 0; d < world_; ++d) {
    if (d != rank_) b += static_cast<double>(sc[static_cast<size_t>(d)]) * w * 4;
  }
  return b;
}

// the receive side of a peer exchange; under timing, the wait is what
// remains of the exchange once the stores overlapped the producers
void DistEngine::timed_wait(int sl, uint32_t expect, int64_t epoch, double bytes) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timing_) {
    SD_CUDA(cudaEventCreate(&e0));
    SD_CUDA(cudaEventCreate(&e1));
    SD_CUDA(cudaEventRecord(e0, stream_));
  }
  launch_p2p_wait(flags_, sl, expect, world_, epoch, stream_);
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

// project_qkv of mini-batch g's home rows for layer l, and send_layer
// (workers.cpp:324-351): the routed GEMM stores every row into its shard's
// receive region and publishes the epoch; otherwise the scatter kernel
// sends (peer exchange) or shard_part's grouped send/recv does (NCCL).
void DistEngine::layer_in(int g, int l) {
  Group& G = groups_[g];
  const Spec& s = spec_;
  const int D = s.D, qkvw = s.qkv_width();
  const int nh = static_cast<int>(G.plan.home_rows.size());
  mark(0);
  if (!nh) return;
  if (p2p_ && fused_ && w_->mode() != SD_DENSE_EXACT_F32) {
    const int32_t* tbl = static_cast<const int32_t*>(G.route.p);
    RowRoute r{};
    r.rank = tbl;
    r.row = tbl + nh;
    r.ld = qkvw;
    r.rows = rx_rows_;  // one mini-batch region of every rank's rx_qkv_ (p2p_setup)
    for (int d = 0; d < world_; ++d) {
      r.base[d] = peer_qkv_[d] + static_cast<size_t>(g) * rx_rows_ * qkvw;
      r.flag[d] = peer_flags_[d];
    }
    r.done = gemm_done_;
    r.epoch = epoch_of(l);
    r.notify = G.to_shards;
    r.slot = slot(0, g);
    r.self = rank_;
    GemmArgs ga = w_->gemm_args(l, 0, nh, G.x, D, G.xb, D, nullptr, qkvw, nullptr, 0, kEpiNone, nullptr, 0);
    ga.route = &r;
    launch_gemm_sm100(ga, stream_);
  } else {
    w_->linear(l, 0, nh, G.x, D, G.xb, D, G.qkv_h, qkvw, nullptr, 0, kEpiNone, nullptr, 0, stream_);
    if (p2p_) scatter_p2p(g, 0, epoch_of(l));
  }
  mark(1);
}

// this shard's part of layer l for mini-batch g: receive its Q/K/V rows,
// append_request + attend (the R-worker's QKV handler, workers.cpp:110-111),
// send the attention rows back to their homes
void DistEngine::shard_part(int g, int l) {
  Group& G = groups_[g];
  const Spec& s = spec_;
  const int D = s.D, qkvw = s.qkv_width();
  const DistPlan& P = G.plan;
  const int ns = static_cast<int>(P.shard_rows.size());
  const size_t region = static_cast<size_t>(g) * rx_rows_;
  float* qkv_s = p2p_ ? rx_qkv_ + region * qkvw : G.qkv_s;
  if (p2p_) {
    timed_wait(slot(0, g), G.from_homes, epoch_of(l), kind_bytes(G, 0));
  } else {
    exchange(G.qkv_h, P.send_cnt, P.send_off, qkv_s, P.recv_cnt, P.recv_off, qkvw);
  }
  mark(2);
  // this worker's head slice of a shard row: [q | k | v] (full width when by-sequence)
  const int Gq = s.H / s.Hkv;
  const int hc = P.head_count[static_cast<size_t>(rank_)];
  const int sq = hc * Gq * s.hd, sk = hc * s.hd, srow = p2p_ ? sq + 2 * sk : qkvw;
  const bool fused = p2p_ && fused_;
  ORoute orr{};
  if (fused) {  // attention rows straight into their home rank's region
    const int nh = static_cast<int>(P.home_rows.size());
    const int32_t* tbl = static_cast<const int32_t*>(G.route.p);
    orr.rank = tbl + 2 * nh;
    orr.row = tbl + 2 * nh + ns;
    orr.ld = D;
    for (int d = 0; d < world_; ++d) {
      // a kind::f16 home takes its W_o operand straight from the attention
      if (peer_mode_[d] == SD_DENSE_BF16 || peer_mode_[d] == SD_DENSE_F16) {
        orr.bbase[d] = peer_ob_[d] + region * D;
        if (peer_mode_[d] == SD_DENSE_F16) orr.f16_mask |= 1u << d;
      } else {
        orr.base[d] = peer_o_[d] + region * D;
      }
      orr.flag[d] = peer_flags_[d];
    }
    orr.bld = D;
    orr.done = attn_done_;
    orr.epoch = epoch_of(l);
    orr.notify = G.to_homes;
    orr.slot = slot(1, g);
    orr.self = rank_;
  }
  if (ns) {
    for (int i = 0; i < ns; ++i) {
      G.pos[static_cast<size_t>(i)] = static_cast<uint32_t>(kv_->stored(P.shard_seqs[static_cast<size_t>(i)], l));
    }
    kv_->append(l, ns, P.shard_seqs.data(), G.pos.data(), qkv_s + sq, srow, qkv_s + sq + sk, srow, stream_);
    mark(3);
    kv_->attend(l, ns, P.shard_seqs.data(), qkv_s, srow, G.o_s, p2p_ ? sq : D, stream_, g, nullptr, 0,
                fused ? &orr : nullptr);
    if (p2p_ && !fused) scatter_p2p(g, 1, epoch_of(l));
  }
  mark(4);
}

// receive_layer (workers.cpp:353-391) + finish_block (dense.cpp:51-70) of
// mini-batch g's home rows
void DistEngine::layer_out(int g, int l) {
  Group& G = groups_[g];
  const Spec& s = spec_;
  const int D = s.D, F = s.F;
  const DistPlan& P = G.plan;
  const int nh = static_cast<int>(P.home_rows.size());
  const size_t region = static_cast<size_t>(g) * rx_rows_;
  float* o_h = p2p_ ? rx_o_ + region * D : G.o_h;
  if (p2p_) {
    timed_wait(slot(1, g), G.from_shards, epoch_of(l), kind_bytes(G, 1));
  } else {
    exchange(G.o_s, P.recv_cnt, P.recv_off, o_h, P.send_cnt, P.send_off, D);
  }
  mark(5);
  if (!nh) return;
  // kind::f16 homes keep 16-bit copies of the GEMM A operands (bf16 or fp16)
  const bool bf = w_->mode() == SD_DENSE_BF16 || w_->mode() == SD_DENSE_F16;
  const int f16 = w_->mode() == SD_DENSE_F16 ? 1 : 0;
  const bool fused = p2p_ && fused_;
  act16* ob = fused && bf ? rx_ob_ + region * D : G.ob;  // fused: the attention wrote it
  if (bf && !fused) launch_to_16(nh, D, o_h, D, G.ob, D, f16, stream_);
  mark(6);
  w_->linear(l, 4, nh, o_h, D, ob, D, G.y, D, bf ? G.yb : nullptr, D, kEpiResidual, G.x, D, stream_);
  mark(7);
  w_->linear(l, 5, nh, G.y, D, G.yb, D, bf ? nullptr : G.h, F, bf ? G.hb : nullptr, F, kEpiSilu, nullptr, 0, stream_);
  mark(8);
  w_->linear(l, 6, nh, G.h, F, G.hb, F, G.x, D, bf ? G.xb : nullptr, D, kEpiResidual, G.y, D, stream_);
  mark(9);
}

// output_logits + argmax_token (dense.cpp:72-88) of mini-batch g's home rows
void DistEngine::head(int g) {
  Group& G = groups_[g];
  const Spec& s = spec_;
  const int D = s.D;
  const int nh = static_cast<int>(G.plan.home_rows.size());
  if (!nh) return;
  if (w_->mode() != SD_DENSE_EXACT_F32 && tuning().fused_argmax) {
    // argmax_token in the head GEMM's epilogue: no logits round trip
    GemmArgs ga = w_->gemm_args(0, 7, nh, G.x, D, G.xb, D, nullptr, s.V, nullptr, 0, kEpiNone, nullptr, 0);
    ga.amax = G.amax;
    launch_gemm_sm100(ga, stream_);
    launch_argmax_keys(nh, G.amax, G.tok, stream_);
  } else {
    w_->linear(0, 7, nh, G.x, D, G.xb, D, G.logits, s.V, nullptr, 0, kEpiNone, nullptr, 0, stream_);
    launch_argmax(nh, s.V, G.logits, s.V, G.tok, stream_);
  }
}

// One decode step with the home tokens already in each mini-batch's tok, in
// the reference's order (DistributedComputation::compute, workers.cpp:399-452):
// dense_in + send of every mini-batch, then per layer and mini-batch
// receive + dense_out + dense_in + send; each rank runs its shard's part of
// a mini-batch right before that mini-batch's receive.
void DistEngine::run_step() {
  const Spec& s = spec_;
  const int D = s.D;
  ++steps_run_;
  const bool bf = w_ && (w_->mode() == SD_DENSE_BF16 || w_->mode() == SD_DENSE_F16);
  const int f16 = w_ && w_->mode() == SD_DENSE_F16 ? 1 : 0;
  for (int g = 0; g < ngroups_; ++g) {
    Group& G = groups_[g];
    const int nh = static_cast<int>(G.plan.home_rows.size());
    if (nh) launch_embed(nh, D, G.tok, w_->embedding(), G.x, D, bf ? G.xb : nullptr, f16, stream_);
    ph_on_ = phases_;
    layer_in(g, 0);
  }
  for (int l = 0; l < s.L; ++l) {
    ph_on_ = phases_ && l % 8 == 0;
    for (int g = 0; g < ngroups_; ++g) {
      shard_part(g, l);
      layer_out(g, l);
      if (l + 1 < s.L) layer_in(g, l + 1);
    }
  }
  ph_on_ = false;
  for (int g = 0; g < ngroups_; ++g) head(g);
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
  for (int i = 0; i < B; ++i) {
    if (tokens[i] < 0 || tokens[i] >= spec_.V) fail(SD_ERR_CONFIG, "token out of the vocabulary");
  }
  DeviceGuard dg(device_);
  ensure(B);
  plan_for(B, seqs);
  for (int g = 0; g < ngroups_; ++g) {
    Group& G = groups_[g];
    const int nh = static_cast<int>(G.plan.home_rows.size());
    G.host_tok.resize(static_cast<size_t>(nh));
    for (int i = 0; i < nh; ++i) {
      G.host_tok[static_cast<size_t>(i)] = tokens[G.rows[static_cast<size_t>(G.plan.home_rows[static_cast<size_t>(i)])]];
    }
    if (nh) SD_CUDA(cudaMemcpyAsync(G.tok, G.host_tok.data(), static_cast<size_t>(nh) * 4, cudaMemcpyHostToDevice, stream_));
  }
  run_step();
  // every rank returns the whole batch's next tokens: a row's home can move
  // between steps (balanced homes follow the batch), so each rank's caller
  // keeps every sequence's last token
  if (world_ > 1 && p2p_) {
    // peer stores of the home rows' tokens into every rank's batch vector
    // (double-buffered by step parity: a rank can be at most one step ahead)
    const int64_t ep = ++tok_epoch_;
    const int half = static_cast<int>(ep & 1) * tok_rows_;
    P2PTokens a{};
    for (int g = 0; g < ngroups_; ++g) {
      a.idx[g] = groups_[g].home_idx;
      a.src[g] = groups_[g].tok;
      a.n[g] = static_cast<int>(groups_[g].plan.home_rows.size());
    }
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
    // homes write their rows into a zeroed batch vector, summed across ranks
    SD_CUDA(cudaMemsetAsync(all_tok_, 0, static_cast<size_t>(B) * 4, stream_));
    for (int g = 0; g < ngroups_; ++g) {
      launch_scatter_i32(static_cast<int>(groups_[g].plan.home_rows.size()), groups_[g].home_idx, groups_[g].tok,
                         all_tok_, stream_);
    }
    nccl_check(Nccl::get().AllReduce(all_tok_, all_tok_, static_cast<size_t>(B), ncclInt32, ncclSum, comm_, stream_),
               "ncclAllReduce");
    SD_CUDA(cudaMemcpyAsync(next, all_tok_, static_cast<size_t>(B) * 4, cudaMemcpyDeviceToHost, stream_));
  } else {
    for (int g = 0; g < ngroups_; ++g) {
      Group& G = groups_[g];
      const int nh = static_cast<int>(G.plan.home_rows.size());
      if (nh) SD_CUDA(cudaMemcpyAsync(G.host_tok.data(), G.tok, static_cast<size_t>(nh) * 4, cudaMemcpyDeviceToHost, stream_));
    }
  }
  std::vector<float> fx[2];
  for (int g = 0; g < ngroups_ && final_x; ++g) {
    Group& G = groups_[g];
    fx[g].resize(G.plan.home_rows.size() * static_cast<size_t>(spec_.D));
    if (!fx[g].empty()) SD_CUDA(cudaMemcpyAsync(fx[g].data(), G.x, fx[g].size() * 4, cudaMemcpyDeviceToHost, stream_));
  }
  SD_CUDA(cudaStreamSynchronize(stream_));
  for (int g = 0; g < ngroups_; ++g) {
    Group& G = groups_[g];
    for (size_t i = 0; i < G.plan.home_rows.size(); ++i) {
      const int row = G.rows[static_cast<size_t>(G.plan.home_rows[i])];
      if (world_ == 1) next[row] = G.host_tok[i];
      if (final_x) {
        std::memcpy(final_x + static_cast<size_t>(row) * spec_.D, fx[g].data() + i * spec_.D,
                    static_cast<size_t>(spec_.D) * 4);
      }
    }
  }
}

double DistEngine::bench(int B, const uint64_t* seqs, const int32_t* tokens, int steps) {
  check_unique(B, seqs);
  DeviceGuard dg(device_);
  ensure(B);
  plan_for(B, seqs);
  for (int g = 0; g < ngroups_; ++g) {
    Group& G = groups_[g];
    const int nh = static_cast<int>(G.plan.home_rows.size());
    G.host_tok.resize(static_cast<size_t>(nh));
    for (int i = 0; i < nh; ++i) {
      G.host_tok[static_cast<size_t>(i)] = tokens[G.rows[static_cast<size_t>(G.plan.home_rows[static_cast<size_t>(i)])]];
    }
    if (nh) SD_CUDA(cudaMemcpyAsync(G.tok, G.host_tok.data(), static_cast<size_t>(nh) * 4, cudaMemcpyHostToDevice, stream_));
  }
  cudaEvent_t e0, e1;
  SD_CUDA(cudaEventCreate(&e0));
  SD_CUDA(cudaEventCreate(&e1));
  SD_CUDA(cudaStreamSynchronize(stream_));
  SD_CUDA(cudaEventRecord(e0, stream_));
  for (int i = 0; i < steps; ++i) run_step();  // tokens fed back on device
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
