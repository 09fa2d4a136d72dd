// R-Part device interfaces: KV append (K1), split-K decode attention (K2),
// split combine (K3). See DESIGN.md "R-Part kernels".
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "sd_common.h"

namespace sd {

// Geometry of the paged KV pool.
// A page group holds P consecutive positions of one sequence for every
// layer (one region per layer, the pool layer-major); a region is
//   [K rows P x pos_bytes][V rows P x pos_bytes][K scales P x hc f32][V scales P x hc f32]
// where a row is one position's [head][d] vector in the storage format, i.e.
// the reference's per-(seq, layer) lane order (attention.cpp:117-118).
struct KvGeom {
  uint8_t* pool;
  int32_t* page_table;  // [max_sequences][max_pages] page-group ids
  int32_t max_pages;
  int32_t P;            // positions per page group (power of two)
  int32_t log2P;
  int32_t fmt;          // SD_KV_*
  int32_t hc;           // kv heads in the shard
  int32_t hd;           // head dim
  int32_t width;        // hc * hd
  int32_t pos_bytes;    // width * elem bytes
  // a (page group, layer) region (128-B aligned) is at
  // pool + group * group_bytes + layer * layer_bytes; the pool is layer-major
  // (group_bytes = region, layer_bytes = region * pool groups)
  int64_t layer_bytes;  // stride between layers
  int64_t group_bytes;  // stride between page groups
  int64_t v_off, ks_off, vs_off;  // offsets inside a region
};

struct AppendArgs {
  KvGeom g;
  int32_t layer;
  int32_t n;
  const int32_t* slot;   // [n]
  const int32_t* pos;    // [n]
  const int32_t* group;  // [n] physical page group of the written position
  const int32_t* upd;    // [nupd][2] (page-table index, group)
  int32_t nupd;
  const float* k;        // [n][width]
  const float* v;        // [n][width]
  int64_t k_stride, v_stride;  // row strides in floats
};

// One contiguous piece of one item's positions, processed by one CTA.
struct Piece {
  // flags & 1: the item has a single piece (write o directly); otherwise
  // flags >> 1 is the item's index in the combine list
  int32_t item, p0, p1, flags;
};

// Multi-GPU exchange fused into the attention (tensor-core path): the o row of
// item i (fp32, and bf16 when bbase is set) goes to base[rank[i]] + row[i] * ld
// on the sequence's home rank; the last CTA publishes flag[d][slot * 8 + self]
// = epoch (release, system scope) for every d in `notify`.
struct ORoute {
  const int32_t* rank;
  const int32_t* row;
  float* base[8];
  act16* bbase[8];      // 16-bit copy (the home's W_o operand) instead of fp32
  uint32_t f16_mask;    // destinations whose 16-bit copy is fp16 (else bf16)
  int64_t ld, bld;
  int64_t* flag[8];
  int32_t* done;
  int64_t epoch;
  uint32_t notify;
  int slot, self;
};

struct AttnArgs {
  KvGeom g;
  int32_t layer;
  const int32_t* item_slot;   // [n]
  const Piece* pieces;        // [npieces], item-contiguous
  const int32_t* cta_begin;   // [grid + 1] piece ranges per CTA
  const float* q;             // [n][q_stride] row-major
  float* o;                   // [n][o_stride]
  int64_t q_stride, o_stride;
  float* part_acc;            // [npieces][Hq * hd]
  float* part_ml;             // [npieces][Hq][2]
  float qscale;               // log2(e) / sqrt(hd)
  int32_t G;                  // q heads per kv head
  int32_t T;                  // positions per pipeline stage
  int32_t nstages;
  int32_t stage_region;       // bytes of one K (or V) stage region (128-B aligned)
  int32_t sc_region;          // bytes of one int8 / int4 scale region per stage (0: scales read from L2)
  // fused combine (kv_mma.cu): the last piece of a split item to finish, per
  // kv head, merges the item's partials in piece order (the combine_kernel
  // arithmetic) and resets its counter
  const int4* comb;           // [ncombine] (item, first piece, piece count, -)
  int32_t* comb_cnt;          // [ncombine][hc] arrival counters, zero between launches
  act16* ob;          // optional 16-bit copy of o (the W_o GEMM operand)
  int64_t ob_stride;
  int ob_f16;                 // the copy is fp16 (else bf16)
  int routed;                 // o rows go to the home ranks (oroute), o/ob unused
  ORoute oroute;
  const uint8_t* l2pf;        // optional: bytes to prefetch into L2 at the end (the next GEMM's weights)
  int64_t l2pf_bytes;
  int32_t iv_flush;           // kv_mma.cu IV: stages between forced flushes (set at launch)
};

// Static shape of the fast attention kernel for a geometry (kv_kernels.cu).
struct AttnConfig {
  bool supported;
  int lpr, epl, maxh, rg;
  int cw;  // consumer warps per CTA (8, or 10 for 40-head shards)
};
AttnConfig choose_attn_config(const KvGeom& g, int G);

struct CombineArgs {
  const int4* items;  // [m] (item, first piece, piece count, -)
  int32_t m;
  const float* part_acc;
  const float* part_ml;
  float* o;
  int64_t o_stride;
  int32_t Hq, hd;
};

// launchers (kv_kernels.cu)
void launch_append(const AppendArgs& a, cudaStream_t s);
// returns false if the fast path does not support the shape (caller uses generic)
bool launch_attention(const AttnArgs& a, int grid, size_t smem, cudaStream_t s);
void launch_attention_generic(const AttnArgs& a, int npieces, cudaStream_t s);
void launch_combine(const CombineArgs& a, cudaStream_t s);
void launch_prefill_synthetic(const KvGeom& g, int num_layers, const int32_t* slots, const uint64_t* seq_ids,
                              int n, int length, uint64_t salt, int h0, int kv_heads_total, cudaStream_t s);
int attention_consumer_warps();
// tensor-core GQA path (kv_mma.cu): fp16 KV, hd 128, 8 kv heads per shard, G in {2, 4, 8}
bool attention_mma_supported(const KvGeom& g, int G);
int attention_mma_rows_per_slot(const KvGeom& g);  // positions per bulk copy (2 or 4)
size_t attention_mma_smem(const KvGeom& g, int* stage_region, int* sc_region, int* nstages);
void launch_attention_mma(const AttnArgs& a, int grid, size_t smem, cudaStream_t s);
size_t attention_smem_bytes(const KvGeom& g, int T, int nstages, int G, int* stage_region,
                            int* sc_region);

}  // namespace sd
