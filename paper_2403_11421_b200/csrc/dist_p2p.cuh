// Peer-memory exchange kernels (dist_p2p.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace sd {

constexpr int kMaxWorld = 8;

// One exchange: for every destination rank d, rows [src_off[d], +cnt[d]) of
// `src` go to rows [dst_off[d], +cnt[d]) of rank d's buffer dst[d] (a peer
// mapping, or this rank's own buffer for d == self). A row's payload is up
// to three column segments (src column, dst column, width; multiples of 4
// floats): the full Q/K/V row under by-sequence sharding, a worker's head
// slices [q | k | v] under by-head / hybrid, an o slice on the way back.
// Then flag[d][slot][self] = epoch for every d in `notify`.
struct P2PScatter {
  const float* src;
  int64_t src_stride;  // floats
  int world, self, slot;
  int64_t epoch;
  uint32_t notify;
  int32_t cnt[kMaxWorld], src_off[kMaxWorld], dst_off[kMaxWorld];
  int64_t dst_stride[kMaxWorld];
  int32_t nseg[kMaxWorld];
  int32_t seg_src[kMaxWorld][3], seg_dst[kMaxWorld][3], seg_n[kMaxWorld][3];
  float* dst[kMaxWorld];
  int64_t* flag[kMaxWorld];  // each rank's flag array [2 slots][kMaxWorld sources]
  int32_t* done;             // block-arrival counter (this rank), zero between launches
};

void launch_p2p_scatter(const P2PScatter& a, cudaStream_t s);
// dst[idx[i]] = src[i] for i < n (a rank's next tokens into the batch vector)
void launch_scatter_i32(int n, const int32_t* idx, const int32_t* src, int32_t* dst, cudaStream_t s);
// The next-token gather of a distributed step over peer memory: every rank
// stores its home rows' tokens at their batch rows into every rank's token
// buffer (dst[d] + idx[j][i] = src[j][i] for each mini-batch j), then
// publishes flag[d][slot][self] = epoch for every d in `notify` (one block;
// B int32 per step).
struct P2PTokens {
  const int32_t* idx[2];
  const int32_t* src[2];
  int n[2];
  int world, self, slot;
  int64_t epoch;
  uint32_t notify;
  int32_t* dst[kMaxWorld];
  int64_t* flag[kMaxWorld];
};
void launch_p2p_tokens(const P2PTokens& a, cudaStream_t s);
// wait until flags[slot][src] >= epoch for every src bit in `expect`
void launch_p2p_wait(const int64_t* flags, int slot, uint32_t expect, int world, int64_t epoch, cudaStream_t s);

}  // namespace sd
