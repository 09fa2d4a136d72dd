// KvStore host logic: reference-exact validation (attention.cpp:139-305),
// slot / page-group allocation, balanced split planning and kernel launch.
#include "kv_store.h"

#include "dense_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

namespace sd {

namespace {

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }


}  // namespace

KvStore::KvStore(const Spec& spec, int head_start, int head_count, int64_t capacity_tokens,
                 int fmt, int device, const sd_kv_options* opts)
    : spec_(spec), head_start_(head_start), head_count_(head_count), cap_(capacity_tokens),
      device_(device) {
  // attention.cpp:66-72 (head range over kv heads under the GQA extension)
  if (head_start < 0 || head_count < 1 || head_start + head_count > spec.Hkv) {
    fail(SD_ERR_CONFIG, "shard head range outside the model's heads");
  }
  if (capacity_tokens < 1) fail(SD_ERR_CONFIG, "shard capacity must be >= 1");
  if (fmt < SD_KV_SINGLE || fmt > SD_KV_INT4) fail(SD_ERR_CONFIG, "unknown kv storage format");
  if (fmt == SD_KV_INT4 && spec.hd % 2) fail(SD_ERR_CONFIG, "int4 kv storage needs an even head_dim");
  G_ = spec.H / spec.Hkv;
  DeviceGuard dg(device);
  SD_CUDA(cudaDeviceGetAttribute(&nsm_, cudaDevAttrMultiProcessorCount, device));

  sd_kv_options o{};
  if (opts) o = *opts;
  max_seqs_ = o.max_sequences > 0 ? o.max_sequences
                                   : static_cast<int>(std::min<int64_t>(capacity_tokens, 4096));
  max_len_ = o.max_seq_len > 0 ? o.max_seq_len
                               : static_cast<int>(std::min<int64_t>(capacity_tokens, 32768));
  int P = o.page_positions > 0 ? o.page_positions : 16;
  if (P & (P - 1)) fail(SD_ERR_CONFIG, "page_positions must be a power of two");
  const int max_pages = static_cast<int>((max_len_ + P - 1) / P);
  const int64_t want_groups = o.pool_pages > 0
                                  ? o.pool_pages
                                  : (capacity_tokens + P - 1) / P + static_cast<int64_t>(max_seqs_);
  if (want_groups > (1LL << 31) - 1) fail(SD_ERR_CONFIG, "KV pool too large");
  pool_groups_ = static_cast<int>(want_groups);

  KvGeom& g = geom_;
  g.fmt = fmt;
  g.hc = head_count;
  g.hd = spec.hd;
  g.width = head_count * spec.hd;
  g.P = P;
  g.log2P = 0;
  while ((1 << g.log2P) < P) ++g.log2P;
  g.max_pages = max_pages;
  g.pos_bytes = kv_row_bytes(fmt, g.width);
  const int64_t lane_bytes = round_up(static_cast<int64_t>(P) * g.pos_bytes, 128);
  g.v_off = lane_bytes;
  int64_t lb = 2 * lane_bytes;
  if (kv_quantized(fmt)) {
    const int64_t sb = round_up(static_cast<int64_t>(P) * head_count * 4, 128);
    g.ks_off = lb;
    g.vs_off = lb + sb;
    lb += 2 * sb;
  } else {
    g.ks_off = g.vs_off = 0;
  }
  // Layer-major pool: [layer][page group][region]. A sequence's pages are
  // allocated in order, so one layer's K/V of a sequence is one contiguous
  // stream for the attention (bulk copies walking 64-KB regions back to back
  // read 7.0-7.4 TB/s, at a 2-MB stride 6.5-6.8: tools/bulk_bw.cu).
  const int64_t rbytes = round_up(lb, 128);
  g.group_bytes = rbytes;
  g.layer_bytes = rbytes * static_cast<int64_t>(pool_groups_);

  const size_t pool_bytes = static_cast<size_t>(rbytes) * spec.L * static_cast<size_t>(pool_groups_);
  void* pool = nullptr;
  cudaError_t e = cudaMalloc(&pool, pool_bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(SD_ERR_CAPACITY, "cannot allocate KV pool of " + std::to_string(pool_bytes) +
                              " bytes on device " + std::to_string(device) + ": " +
                              cudaGetErrorString(e));
  }
  g.pool = static_cast<uint8_t*>(pool);
  const size_t pt_bytes = static_cast<size_t>(max_seqs_) * max_pages * sizeof(int32_t);
  SD_CUDA(cudaMalloc(&g.page_table, pt_bytes));
  SD_CUDA(cudaMemset(g.page_table, 0, pt_bytes));

  len_.assign(static_cast<size_t>(max_seqs_) * spec.L, 0);
  pages_.assign(static_cast<size_t>(max_seqs_) * max_pages, -1);
  npages_.assign(static_cast<size_t>(max_seqs_), 0);
  free_slots_.resize(static_cast<size_t>(max_seqs_));
  for (int i = 0; i < max_seqs_; ++i) free_slots_[static_cast<size_t>(i)] = max_seqs_ - 1 - i;
  free_groups_.resize(static_cast<size_t>(pool_groups_));
  for (int i = 0; i < pool_groups_; ++i) free_groups_[static_cast<size_t>(i)] = pool_groups_ - 1 - i;

  // pipeline geometry for the attention kernel: T positions per stage,
  // 2*T*pos_bytes <= 32 KB, as many stages as fit ~200 KB of shared memory
  T_ = 1;
  while (T_ * 2 <= P && 2 * (T_ * 2) * g.pos_bytes <= 64 * 1024) T_ *= 2;
  int region = 0, sregion = 0;
  nstages_ = tuning().attn_max_stages > 1 ? tuning().attn_max_stages : 8;
  while (nstages_ > 2 && attention_smem_bytes(g, T_, nstages_, G_, &region, &sregion) > 210 * 1024) {
    --nstages_;
  }
  attn_smem_ = attention_smem_bytes(g, T_, nstages_, G_, &stage_region_, &sc_region_);
  use_mma_ = attention_mma_supported(g, G_) && tuning().attn_mma != 0;
  if (use_mma_) {
    T_ = 16;
    attn_smem_ = attention_mma_smem(g, &stage_region_, &sc_region_, &nstages_);
  }

  ring_.resize(8);
  for (Blob& b : ring_) SD_CUDA(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming));
  // the page-table memset (legacy stream) must land before any append on a
  // caller's non-blocking stream writes page-table entries
  SD_CUDA(cudaDeviceSynchronize());
  for (Plan& P : plans_) SD_CUDA(cudaEventCreateWithFlags(&P.blob.done, cudaEventDisableTiming));
}

KvStore::~KvStore() {
  DeviceGuard dg(device_);
  cudaDeviceSynchronize();
  for (Blob& b : ring_) cudaEventDestroy(b.done);
  for (Plan& P : plans_) cudaEventDestroy(P.blob.done);
  for (auto& pr : ev_pending_) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  for (cudaEvent_t ev : ev_pool_) cudaEventDestroy(ev);
  cudaFree(geom_.pool);
  cudaFree(geom_.page_table);
}

int KvStore::stored(uint64_t seq, int layer) const {
  auto it = slot_of_.find(seq);
  if (it == slot_of_.end() || layer < 0 || layer >= spec_.L) return 0;
  return len_[static_cast<size_t>(it->second) * spec_.L + layer];
}

int64_t KvStore::bytes_per_token() const {  // attention.cpp:296-305
  const int64_t w = geom_.width;
  switch (geom_.fmt) {
    case SD_KV_SINGLE: return 2 * w * 4;
    case SD_KV_HALF: return 2 * w * 2;
    case SD_KV_INT4: return 2 * (w / 2 + static_cast<int64_t>(head_count_) * 4);
    default: return 2 * (w + static_cast<int64_t>(head_count_) * 4);
  }
}

KvStore::Blob& KvStore::next_blob() {
  Blob& b = ring_[ring_next_];
  ring_next_ = (ring_next_ + 1) % ring_.size();
  SD_CUDA(cudaEventSynchronize(b.done));  // previous use of this entry finished
  return b;
}

void KvStore::upload(Blob& b, size_t bytes, cudaStream_t s) {
  b.dev.get(bytes);
  SD_CUDA(cudaMemcpyAsync(b.dev.p, b.host.p, bytes, cudaMemcpyHostToDevice, s));
}

int KvStore::slot_for_new(uint64_t seq) {
  if (free_slots_.empty()) {
    fail(SD_ERR_CAPACITY, "capacity exceeded: all " + std::to_string(max_seqs_) +
                              " sequence slots of the shard are live (sd_kv_options.max_sequences)");
  }
  const int slot = free_slots_.back();
  free_slots_.pop_back();
  slot_of_.emplace(seq, slot);
  return slot;
}

void KvStore::release_slot(int slot) {
  const size_t L = static_cast<size_t>(spec_.L);
  int64_t removed = 0;
  for (size_t l = 0; l < L; ++l) {
    removed += len_[slot * L + l];
    len_[slot * L + l] = 0;
  }
  total_ -= removed;
  const size_t mp = static_cast<size_t>(geom_.max_pages);
  for (int p = 0; p < npages_[static_cast<size_t>(slot)]; ++p) {
    int32_t& gid = pages_[slot * mp + static_cast<size_t>(p)];
    if (gid >= 0) free_groups_.push_back(gid);
    gid = -1;
  }
  npages_[static_cast<size_t>(slot)] = 0;
  free_slots_.push_back(slot);
}

int KvStore::alloc_group() {
  if (free_groups_.empty()) {
    fail(SD_ERR_CAPACITY, "capacity exceeded: physical KV pool exhausted (" +
                              std::to_string(pool_groups_) + " page groups of " +
                              std::to_string(geom_.P) + " positions)");
  }
  const int g = free_groups_.back();
  free_groups_.pop_back();
  return g;
}

// --------------------------------------------------------------- append ---
void KvStore::append(int layer, int n, const uint64_t* seqs, const uint32_t* positions,
                     const float* k_dev, int64_t k_stride, const float* v_dev, int64_t v_stride,
                     cudaStream_t s) {
  DeviceGuard dg(device_);
  const int L = spec_.L;
  // validation pass against the pre-call state (attention.cpp:174-195)
  if (total_ + static_cast<int64_t>(n) > cap_ * L) {
    fail(SD_ERR_CAPACITY, "capacity exceeded: batch of " + std::to_string(n) +
                              " does not fit (shard at " + std::to_string(token_count()) + "/" +
                              std::to_string(cap_) + " tokens)");
  }
  if (layer < 0 || layer >= L) fail(SD_ERR_PROTOCOL, "append: layer index out of range");
  // Lockstep fast path: the sequences and positions of the previous call at
  // another layer (the next layer of one decode step) with every target page
  // already open. The reference checks still run per item; only the slot
  // lookups and the descriptor upload are reused.
  Fast* fm = const_cast<Fast*>(fast_match(n, seqs));
  if (fm && layer != fm->layer && n > 0 && total_ + n <= cap_ * L &&
      std::memcmp(positions, fm->pos.data(), static_cast<size_t>(n) * 4) == 0) {
    Fast& f = *fm;
    bool ok = true;
    for (int i = 0; i < n && ok; ++i) {
      ok = static_cast<uint32_t>(len_[static_cast<size_t>(f.slots[static_cast<size_t>(i)]) * L + layer]) ==
           positions[i];
    }
    if (ok) {
      for (int i = 0; i < n; ++i) len_[static_cast<size_t>(f.slots[static_cast<size_t>(i)]) * L + layer] += 1;
      total_ += n;
      AppendArgs a{};
      a.g = geom_;
      a.layer = layer;
      a.n = n;
      const int32_t* d = static_cast<const int32_t*>(f.blob->dev.p);
      a.slot = d;
      a.pos = d + n;
      a.group = d + 2 * n;
      a.upd = d + 3 * n;
      a.nupd = 0;
      a.k = k_dev;
      a.v = v_dev;
      a.k_stride = k_stride;
      a.v_stride = v_stride;
      launch_append(a, s);
      SD_CUDA(cudaEventRecord(f.blob->done, s));
      f.layer = layer;
      f.used = ++fast_clock_;
      return;
    }
  }
  for (int i = 0; i < n; ++i) {
    auto it = slot_of_.find(seqs[i]);
    const uint32_t st = it == slot_of_.end()
                            ? 0u
                            : static_cast<uint32_t>(len_[static_cast<size_t>(it->second) * L + layer]);
    if (it == slot_of_.end() && positions[i] != 0) {
      fail(SD_ERR_UNKNOWN_SEQ, "unknown sequence " + std::to_string(seqs[i]));
    }
    if (positions[i] != st) {
      fail(SD_ERR_PROTOCOL, "append: position mismatch for sequence " + std::to_string(seqs[i]));
    }
  }
  // sequential commit (KvShard::append per item, attention.cpp:139-170);
  // an exception stops the loop with the earlier items already stored.
  Blob& b = next_blob();
  for (Fast& f : fast_) {
    if (f.blob == &b) f.valid = false;  // its descriptor is about to be overwritten
  }
  const size_t need = static_cast<size_t>(n) * 3 * 4 + static_cast<size_t>(n) * 2 * 4 + 64;
  int32_t* h = static_cast<int32_t*>(b.host.get(need));
  b.dev.get(need);  // upper bound (nupd <= n): no reallocation when a step opens pages
  int32_t* h_slot = h;
  int32_t* h_pos = h + n;
  int32_t* h_grp = h + 2 * n;
  int32_t* h_upd = h + 3 * n;
  int nupd = 0;
  int done = 0;
  int err_code = 0;
  std::string err_msg;
  const size_t mp = static_cast<size_t>(geom_.max_pages);
  try {
    for (int i = 0; i < n; ++i) {
      if (total_ + 1 > cap_ * L) {
        fail(SD_ERR_CAPACITY, "capacity exceeded: shard holds " + std::to_string(token_count()) +
                                  " of " + std::to_string(cap_) + " tokens");
      }
      auto it = slot_of_.find(seqs[i]);
      int slot;
      if (it == slot_of_.end()) {
        if (positions[i] != 0) {
          fail(SD_ERR_UNKNOWN_SEQ, "unknown sequence " + std::to_string(seqs[i]) +
                                       " (non-zero position without prior tokens)");
        }
        slot = slot_for_new(seqs[i]);
      } else {
        slot = it->second;
      }
      int32_t& len = len_[static_cast<size_t>(slot) * L + layer];
      if (static_cast<uint32_t>(len) != positions[i]) {
        fail(SD_ERR_PROTOCOL, "append: position " + std::to_string(positions[i]) +
                                  " does not match stored length " + std::to_string(len));
      }
      if (len >= max_len_) {
        fail(SD_ERR_CAPACITY, "capacity exceeded: sequence " + std::to_string(seqs[i]) +
                                  " reached max_seq_len " + std::to_string(max_len_));
      }
      const int page = len >> geom_.log2P;
      int32_t& gid = pages_[static_cast<size_t>(slot) * mp + static_cast<size_t>(page)];
      if (gid < 0) {
        gid = alloc_group();
        npages_[static_cast<size_t>(slot)] = std::max(npages_[static_cast<size_t>(slot)], page + 1);
        h_upd[2 * nupd] = static_cast<int32_t>(static_cast<size_t>(slot) * mp + page);
        h_upd[2 * nupd + 1] = gid;
        ++nupd;
      }
      h_slot[i] = slot;
      h_pos[i] = len;
      h_grp[i] = gid;
      len += 1;
      total_ += 1;
      done = i + 1;
    }
  } catch (const Error& e) {
    err_code = e.code;
    err_msg = e.what();
  }
  // compact (slot, pos, grp, upd) contiguous for the committed prefix
  const size_t bytes = static_cast<size_t>(3 * n + 2 * nupd) * 4;
  upload(b, bytes, s);
  AppendArgs a{};
  a.g = geom_;
  a.layer = layer;
  a.n = done;
  const int32_t* d = static_cast<const int32_t*>(b.dev.p);
  a.slot = d;
  a.pos = d + n;
  a.group = d + 2 * n;
  a.upd = d + 3 * n;
  a.nupd = nupd;
  a.k = k_dev;
  a.v = v_dev;
  a.k_stride = k_stride;
  a.v_stride = v_stride;
  launch_append(a, s);
  SD_CUDA(cudaEventRecord(b.done, s));
  if (err_code) fail(err_code, err_msg);
  // remember the call for the lockstep fast path of the next layers (replace
  // an entry for the same sequences, else the least recently used one)
  Fast* f = const_cast<Fast*>(fast_match(n, seqs));
  if (!f) f = fast_[0].used <= fast_[1].used ? &fast_[0] : &fast_[1];
  f->valid = true;
  f->n = n;
  f->layer = layer;
  f->used = ++fast_clock_;
  f->seqs.assign(seqs, seqs + n);
  f->pos.assign(positions, positions + n);
  f->slots.assign(h_slot, h_slot + n);
  f->blob = &b;
}

bool KvStore::stage_fused_append(int layer, int n, const uint64_t* seqs, const uint32_t* positions,
                                 KvAppendOut* out) {
  const int L = spec_.L;
  if (geom_.fmt != SD_KV_HALF || layer < 0 || layer >= L || n <= 0 || total_ + n > cap_ * L) return false;
  Fast* fm = const_cast<Fast*>(fast_match(n, seqs));
  if (!fm || layer == fm->layer || std::memcmp(positions, fm->pos.data(), static_cast<size_t>(n) * 4) != 0) {
    return false;
  }
  for (int i = 0; i < n; ++i) {  // the reference's per-item checks (attention.cpp:174-195)
    if (static_cast<uint32_t>(len_[static_cast<size_t>(fm->slots[static_cast<size_t>(i)]) * L + layer]) !=
        positions[i]) {
      return false;
    }
  }
  for (int i = 0; i < n; ++i) len_[static_cast<size_t>(fm->slots[static_cast<size_t>(i)]) * L + layer] += 1;
  total_ += n;
  fused_prev_layer_ = fm->layer;
  const int32_t* d = static_cast<const int32_t*>(fm->blob->dev.p);
  out->layer_base = geom_.pool + static_cast<int64_t>(layer) * geom_.layer_bytes;
  out->group_bytes = geom_.group_bytes;
  out->v_off = geom_.v_off;
  out->pos_bytes = geom_.pos_bytes;
  out->pmask = geom_.P - 1;
  out->pos = d + n;
  out->group = d + 2 * n;
  fm->layer = layer;
  fm->used = ++fast_clock_;
  fused_pending_ = fm;
  return true;
}

void KvStore::abort_fused_append() {
  Fast* fm = fused_pending_;
  if (!fm) return;
  const int L = spec_.L, layer = fm->layer;
  for (int i = 0; i < fm->n; ++i) len_[static_cast<size_t>(fm->slots[static_cast<size_t>(i)]) * L + layer] -= 1;
  total_ -= fm->n;
  fm->layer = fused_prev_layer_;
  fused_pending_ = nullptr;
}

void KvStore::end_fused_append(cudaStream_t s) {
  if (!fused_pending_) return;
  SD_CUDA(cudaEventRecord(fused_pending_->blob->done, s));
  fused_pending_ = nullptr;
}

const KvStore::Fast* KvStore::fast_match(int n, const uint64_t* seqs) const {
  for (const Fast& f : fast_) {
    if (f.valid && f.n == n && n > 0 && std::memcmp(seqs, f.seqs.data(), static_cast<size_t>(n) * 8) == 0) {
      return &f;
    }
  }
  return nullptr;
}

// --------------------------------------------------------------- attend ---
void KvStore::attend(int layer, int n, const uint64_t* seqs, const float* q_dev,
                     int64_t q_stride, float* o_dev, int64_t o_stride, cudaStream_t s, int slot,
                     act16* ob, int64_t ob_stride, const ORoute* oroute, int ob_f16) {
  if (oroute && !use_mma_) fail(SD_ERR_INTERNAL, "routed attention output needs the tensor-core path");
  DeviceGuard dg(device_);
  const int L = spec_.L;
  if (layer < 0 || layer >= L) fail(SD_ERR_PROTOCOL, "attend: layer index out of range");
  if (slot < 0 || slot >= kPlanSlots) fail(SD_ERR_INTERNAL, "attend: bad plan slot");
  Plan& P = plans_[slot];
  std::vector<int32_t> slots(static_cast<size_t>(n)), lens(static_cast<size_t>(n));
  const Fast* fm = fast_match(n, seqs);  // slots already resolved by this step's append
  for (int i = 0; i < n; ++i) {
    int slot;
    if (fm) {
      slot = fm->slots[static_cast<size_t>(i)];
    } else {
      auto it = slot_of_.find(seqs[i]);
      if (it == slot_of_.end()) {
        fail(SD_ERR_UNKNOWN_SEQ, "attend: unknown sequence " + std::to_string(seqs[i]));
      }
      slot = it->second;
    }
    const int len = len_[static_cast<size_t>(slot) * L + layer];
    if (len < 1) fail(SD_ERR_LOGIC, "attend: sequence has an empty cache");
    slots[static_cast<size_t>(i)] = slot;
    lens[static_cast<size_t>(i)] = len;
  }
  if (n == 0) return;
  const int sms = grid_limit_ > 0 && grid_limit_ < nsm_ ? grid_limit_ : nsm_;
  if (slots != P.slots || lens != P.lens || sms != P.sms) {
    // ---- balanced split planning
    SD_CUDA(cudaEventSynchronize(P.blob.done));
    int64_t total = 0;
    for (int32_t x : lens) total += x;
    const int64_t min_per_cta = std::max<int64_t>(T_, 64);
    int grid = static_cast<int>(std::min<int64_t>(sms, (total + min_per_cta - 1) / min_per_cta));
    grid = std::max(grid, 1);
    const int64_t per = round_up((total + grid - 1) / grid, T_);
    std::vector<Piece> pieces;
    std::vector<int32_t> cta_begin(static_cast<size_t>(grid) + 1, 0);
    pieces.reserve(static_cast<size_t>(n) + static_cast<size_t>(grid) + 4);
    int item = 0, p = 0;
    int64_t gpos = 0;
    for (int c = 0; c < grid; ++c) {
      cta_begin[static_cast<size_t>(c)] = static_cast<int32_t>(pieces.size());
      const int64_t end = std::min<int64_t>(total, static_cast<int64_t>(c + 1) * per);
      while (gpos < end && item < n) {
        const int li = lens[static_cast<size_t>(item)];
        int64_t pe = p + std::min<int64_t>(li - p, end - gpos);
        if (pe < li) {
          pe = std::max<int64_t>(p + T_, pe / T_ * T_);
          pe = std::min<int64_t>(pe, li);
        }
        pieces.push_back(Piece{item, p, static_cast<int32_t>(pe), 0});
        gpos += pe - p;
        p = static_cast<int>(pe);
        if (p >= li) {
          ++item;
          p = 0;
        }
      }
    }
    cta_begin[static_cast<size_t>(grid)] = static_cast<int32_t>(pieces.size());
    // flags + combine list
    std::vector<int4> comb;
    for (size_t i = 0; i < pieces.size();) {
      size_t j = i;
      while (j < pieces.size() && pieces[j].item == pieces[i].item) ++j;
      if (j - i == 1) {
        pieces[i].flags = 1;
      } else {
        for (size_t k = i; k < j; ++k) pieces[k].flags = static_cast<int32_t>(comb.size()) << 1;
        comb.push_back(make_int4(pieces[i].item, static_cast<int>(i), static_cast<int>(j - i), 0));
      }
      i = j;
    }
    // descriptor and partial buffers sized for the worst case of this batch,
    // so context growth never reallocates them: every item ends one piece and
    // every CTA boundary adds at most two (the T-aligned cut inside an item
    // plus the sub-T remainder up to the boundary)
    const size_t max_pieces = static_cast<size_t>(n) + 2 * static_cast<size_t>(grid) + 1;
    if (pieces.size() > max_pieces) fail(SD_ERR_INTERNAL, "attend: split plan exceeds its piece bound");
    const size_t bound = static_cast<size_t>(round_up(static_cast<int64_t>(n) * 4, 16)) +
                         static_cast<size_t>(round_up(static_cast<int64_t>(max_pieces * sizeof(Piece)), 16)) +
                         static_cast<size_t>(round_up(static_cast<int64_t>(grid + 2) * 4, 16)) +
                         static_cast<size_t>(n) * sizeof(int4) + 16;
    P.blob.host.get(bound);
    P.blob.dev.get(bound);
    P.off_slot = 0;
    P.off_pieces = round_up(static_cast<int64_t>(n) * 4, 16);
    P.off_cta = P.off_pieces + round_up(static_cast<int64_t>(pieces.size()) * sizeof(Piece), 16);
    P.off_comb = P.off_cta + round_up(static_cast<int64_t>(cta_begin.size()) * 4, 16);
    const size_t bytes = P.off_comb + comb.size() * sizeof(int4) + 16;
    uint8_t* hb = static_cast<uint8_t*>(P.blob.host.get(bytes));
    std::memcpy(hb + P.off_slot, slots.data(), slots.size() * 4);
    std::memcpy(hb + P.off_pieces, pieces.data(), pieces.size() * sizeof(Piece));
    std::memcpy(hb + P.off_cta, cta_begin.data(), cta_begin.size() * 4);
    if (!comb.empty()) std::memcpy(hb + P.off_comb, comb.data(), comb.size() * sizeof(int4));
    P.blob.dev.get(bytes);
    SD_CUDA(cudaMemcpyAsync(P.blob.dev.p, hb, bytes, cudaMemcpyHostToDevice, s));
    P.npieces = static_cast<int>(pieces.size());
    P.grid = grid;
    P.sms = sms;
    P.ncombine = static_cast<int>(comb.size());
    P.positions = total;
    P.slots = slots;
    P.lens = lens;
    const size_t pa = max_pieces * q_width() * sizeof(float);
    const size_t pm = max_pieces * spec_.H / spec_.Hkv * head_count_ * 2 * sizeof(float);
    const size_t pc = static_cast<size_t>(n) * static_cast<size_t>(geom_.hc) * sizeof(int32_t);
    if (pa > P.part_acc.bytes || pm > P.part_ml.bytes || pc > P.comb_cnt.bytes) {
      SD_CUDA(cudaStreamSynchronize(s));
      P.part_acc.get(pa);
      P.part_ml.get(pm);
      P.comb_cnt.get(pc);
      // arrival counters start at zero; the fused combine leaves them zero
      SD_CUDA(cudaMemsetAsync(P.comb_cnt.p, 0, P.comb_cnt.bytes, s));
    }
  }
  launch_attention_plan(P, layer, q_dev, q_stride, o_dev, o_stride, ob, ob_stride, s, oroute, ob_f16);
}

void KvStore::launch_attention_plan(Plan& P, int layer, const float* q, int64_t qs, float* o,
                                    int64_t os, act16* ob, int64_t obs, cudaStream_t s,
                                    const ORoute* oroute, int ob_f16) {
  const uint8_t* base = static_cast<const uint8_t*>(P.blob.dev.p);
  AttnArgs a{};
  a.g = geom_;
  a.layer = layer;
  a.item_slot = reinterpret_cast<const int32_t*>(base + P.off_slot);
  a.pieces = reinterpret_cast<const Piece*>(base + P.off_pieces);
  a.cta_begin = reinterpret_cast<const int32_t*>(base + P.off_cta);
  a.q = q;
  a.o = o;
  a.q_stride = qs;
  a.o_stride = os;
  a.part_acc = static_cast<float*>(P.part_acc.p);
  a.part_ml = static_cast<float*>(P.part_ml.p);
  a.qscale = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(spec_.hd)));
  a.G = G_;
  a.T = T_;
  a.nstages = nstages_;
  a.stage_region = stage_region_;
  a.sc_region = sc_region_;
  // the tensor-core kernel fuses the combine and the 16-bit copy of o
  const bool fused = use_mma_;
  a.comb = reinterpret_cast<const int4*>(base + P.off_comb);
  a.comb_cnt = fused ? static_cast<int32_t*>(P.comb_cnt.p) : nullptr;
  a.ob = fused ? ob : nullptr;
  a.ob_stride = obs;
  a.ob_f16 = ob_f16;
  a.l2pf = l2pf_;
  a.l2pf_bytes = use_mma_ ? l2pf_bytes_ : 0;
  l2pf_ = nullptr;  // one launch
  l2pf_bytes_ = 0;
  if (oroute) {
    if (!fused) fail(SD_ERR_INTERNAL, "routed attention output needs the fused combine");
    a.routed = 1;
    a.oroute = *oroute;
  }

  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool timed = timing_ && layer % timing_every_ == 0;
  if (timed) {
    auto take = [&]() {
      if (ev_pool_.empty()) {
        cudaEvent_t ev;
        SD_CUDA(cudaEventCreate(&ev));
        return ev;
      }
      cudaEvent_t ev = ev_pool_.back();
      ev_pool_.pop_back();
      return ev;
    };
    e0 = take();
    e1 = take();
    SD_CUDA(cudaEventRecord(e0, s));
  }
  if (use_mma_) {
    launch_attention_mma(a, P.grid, attn_smem_, s);
  } else if (!launch_attention(a, P.grid, attn_smem_, s)) {
    launch_attention_generic(a, P.npieces, s);
  }
  if (timed) {
    SD_CUDA(cudaEventRecord(e1, s));
    ev_pending_.emplace_back(e0, e1);
    double bytes = static_cast<double>(P.positions) * 2 * geom_.pos_bytes;
    if (kv_quantized(geom_.fmt)) bytes += static_cast<double>(P.positions) * 2 * geom_.hc * 4;
    bytes += static_cast<double>(P.slots.size()) * q_width() * 4 * 2;  // q in, o out
    ev_bytes_.push_back(bytes);
  }
  if (fused) {
    SD_CUDA(cudaEventRecord(P.blob.done, s));
    return;
  }
  CombineArgs c{};
  c.items = reinterpret_cast<const int4*>(base + P.off_comb);
  c.m = P.ncombine;
  c.part_acc = a.part_acc;
  c.part_ml = a.part_ml;
  c.o = o;
  c.o_stride = os;
  c.Hq = head_count_ * G_;
  c.hd = spec_.hd;
  launch_combine(c, s);
  if (ob) launch_to_16(static_cast<int>(P.slots.size()), q_width(), o, os, ob, obs, ob_f16, s);
  SD_CUDA(cudaEventRecord(P.blob.done, s));
}

// ----------------------------------------------------------------- drop ---
void KvStore::drop(uint64_t seq) {
  auto it = slot_of_.find(seq);
  if (it == slot_of_.end()) {
    warnings_ += 1;
    return;
  }
  const int slot = it->second;
  slot_of_.erase(it);
  release_slot(slot);
  for (Plan& P : plans_) {  // slot reuse invalidates the cached plans
    P.slots.clear();
    P.lens.clear();
  }
  for (Fast& f : fast_) f.valid = false;
}

// --------------------------------------------------------------- export ---
int64_t KvStore::export_lane(uint64_t seq, int layer, int which, void* host, size_t host_bytes,
                             float* scales, size_t scales_count) {
  DeviceGuard dg(device_);
  auto it = slot_of_.find(seq);
  if (it == slot_of_.end()) fail(SD_ERR_UNKNOWN_SEQ, "export: unknown sequence");
  if (layer < 0 || layer >= spec_.L) fail(SD_ERR_PROTOCOL, "export: layer index out of range");
  const int slot = it->second;
  const int len = len_[static_cast<size_t>(slot) * spec_.L + layer];
  const int64_t bytes = static_cast<int64_t>(len) * geom_.pos_bytes;
  SD_CUDA(cudaDeviceSynchronize());
  const size_t mp = static_cast<size_t>(geom_.max_pages);
  if (host && static_cast<size_t>(bytes) <= host_bytes) {
    for (int p0 = 0; p0 < len; p0 += geom_.P) {
      const int cnt = std::min(geom_.P, len - p0);
      const int gid = pages_[static_cast<size_t>(slot) * mp + static_cast<size_t>(p0 >> geom_.log2P)];
      const uint8_t* src = geom_.pool + static_cast<int64_t>(gid) * geom_.group_bytes +
                           static_cast<int64_t>(layer) * geom_.layer_bytes + (which ? geom_.v_off : 0);
      SD_CUDA(cudaMemcpy(static_cast<uint8_t*>(host) + static_cast<int64_t>(p0) * geom_.pos_bytes, src,
                         static_cast<size_t>(cnt) * geom_.pos_bytes, cudaMemcpyDeviceToHost));
    }
    // the pool holds offset-binary codes (q + 128, nibbles q + 8): give the
    // reference's two's-complement bytes back
    if (kv_quantized(geom_.fmt)) {
      const uint8_t flip = geom_.fmt == SD_KV_INT8 ? 0x80 : 0x88;
      uint8_t* h = static_cast<uint8_t*>(host);
      for (int64_t i = 0; i < bytes; ++i) h[i] ^= flip;
    }
  }
  if (scales && kv_quantized(geom_.fmt) &&
      static_cast<size_t>(len) * head_count_ <= scales_count) {
    for (int p0 = 0; p0 < len; p0 += geom_.P) {
      const int cnt = std::min(geom_.P, len - p0);
      const int gid = pages_[static_cast<size_t>(slot) * mp + static_cast<size_t>(p0 >> geom_.log2P)];
      const uint8_t* src = geom_.pool + static_cast<int64_t>(gid) * geom_.group_bytes +
                           static_cast<int64_t>(layer) * geom_.layer_bytes +
                           (which ? geom_.vs_off : geom_.ks_off);
      SD_CUDA(cudaMemcpy(scales + static_cast<int64_t>(p0) * head_count_, src,
                         static_cast<size_t>(cnt) * head_count_ * 4, cudaMemcpyDeviceToHost));
    }
  }
  return bytes;
}

// -------------------------------------------------------------- prefill ---
void KvStore::prefill_synthetic(int n, const uint64_t* seqs, int length, uint64_t salt,
                                cudaStream_t s) {
  DeviceGuard dg(device_);
  const int L = spec_.L;
  if (length < 1 || n < 1) return;
  if (total_ + static_cast<int64_t>(n) * length * L > cap_ * L) {
    fail(SD_ERR_CAPACITY, "capacity exceeded: prefill of " + std::to_string(n) + " x " +
                              std::to_string(length) + " tokens does not fit");
  }
  if (length > max_len_) fail(SD_ERR_CAPACITY, "prefill length exceeds max_seq_len");
  for (int i = 0; i < n; ++i) {
    if (slot_of_.count(seqs[i])) fail(SD_ERR_PROTOCOL, "prefill: sequence already present");
  }
  const int npg = (length + geom_.P - 1) / geom_.P;
  std::vector<int32_t> upd, slots;
  const size_t mp = static_cast<size_t>(geom_.max_pages);
  for (int i = 0; i < n; ++i) {
    const int slot = slot_for_new(seqs[i]);
    slots.push_back(slot);
    for (int l = 0; l < L; ++l) len_[static_cast<size_t>(slot) * L + l] = length;
    total_ += static_cast<int64_t>(length) * L;
    for (int p = 0; p < npg; ++p) {
      const int gid = alloc_group();
      pages_[static_cast<size_t>(slot) * mp + static_cast<size_t>(p)] = gid;
      upd.push_back(static_cast<int32_t>(static_cast<size_t>(slot) * mp + p));
      upd.push_back(gid);
    }
    npages_[static_cast<size_t>(slot)] = npg;
  }
  DevBuf d;
  const size_t ints = (upd.size() + slots.size() + 1) / 2 * 2;  // 8-B aligned sequence ids follow
  d.get(ints * 4 + static_cast<size_t>(n) * 8);
  SD_CUDA(cudaMemcpy(d.p, upd.data(), upd.size() * 4, cudaMemcpyHostToDevice));
  int32_t* dslots = static_cast<int32_t*>(d.p) + upd.size();
  SD_CUDA(cudaMemcpy(dslots, slots.data(), slots.size() * 4, cudaMemcpyHostToDevice));
  uint64_t* dseqs = reinterpret_cast<uint64_t*>(static_cast<int32_t*>(d.p) + ints);
  SD_CUDA(cudaMemcpy(dseqs, seqs, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice));
  AppendArgs a{};
  a.g = geom_;
  a.n = 0;
  a.upd = static_cast<const int32_t*>(d.p);
  a.nupd = static_cast<int>(upd.size() / 2);
  launch_append(a, s);
  launch_prefill_synthetic(geom_, L, dslots, dseqs, n, length, salt, head_start_, spec_.Hkv, s);
  SD_CUDA(cudaStreamSynchronize(s));
  for (Plan& P : plans_) {
    P.slots.clear();
    P.lens.clear();
  }
}

// --------------------------------------------------------------- timing ---
void KvStore::set_timing(int every) {
  timing_ = every > 0;
  timing_every_ = every > 0 ? every : 1;
}

void KvStore::read_timing(double* ms, int64_t* launches, double* bytes, bool reset) {
  DeviceGuard dg(device_);
  for (size_t i = 0; i < ev_pending_.size(); ++i) {
    auto& pr = ev_pending_[i];
    SD_CUDA(cudaEventSynchronize(pr.second));
    float t = 0;
    SD_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second));
    t_ms_ += t;
    t_bytes_ += ev_bytes_[i];
    t_launches_ += 1;
    ev_pool_.push_back(pr.first);
    ev_pool_.push_back(pr.second);
  }
  ev_pending_.clear();
  ev_bytes_.clear();
  if (ms) *ms = t_ms_;
  if (launches) *launches = t_launches_;
  if (bytes) *bytes = t_bytes_;
  if (reset) {
    t_ms_ = 0;
    t_bytes_ = 0;
    t_launches_ = 0;
  }
}

}  // namespace sd
