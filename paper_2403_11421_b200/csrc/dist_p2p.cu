// Peer-memory exchange for DistEngine (dist.h): the per-layer scatter of
// Q/K/V rows to their R-shards and the gather of attention outputs back
// (send_layer / receive_layer, workers.cpp:324-391) as direct NVLink stores
// into the destination rank's receive buffer (CUDA IPC mapping), signalled
// by a per-(exchange, source) epoch flag in the destination's memory.
#include <cstdint>

#include "dist_p2p.cuh"
#include "pdl.cuh"
#include "sd_common.h"

namespace sd {

namespace {

__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// grid-stride over (destination, row, 16-B chunk of the row's segments)
__global__ void p2p_scatter_kernel(const P2PScatter a) {
  pdl_trigger();
  pdl_wait();
  int64_t total = 0;
  int vrow[kMaxWorld];
  for (int d = 0; d < a.world; ++d) {
    vrow[d] = 0;
    for (int q = 0; q < a.nseg[d]; ++q) vrow[d] += a.seg_n[d][q] / 4;
    total += static_cast<int64_t>(a.cnt[d]) * vrow[d];
  }
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = i;
    int d = 0;
    while (rem >= static_cast<int64_t>(a.cnt[d]) * vrow[d]) {
      rem -= static_cast<int64_t>(a.cnt[d]) * vrow[d];
      ++d;
    }
    const int64_t r = rem / vrow[d];
    int c = static_cast<int>(rem - r * vrow[d]);
    int q = 0;
    while (c >= a.seg_n[d][q] / 4) {
      c -= a.seg_n[d][q] / 4;
      ++q;
    }
    const float4 v =
        reinterpret_cast<const float4*>(a.src + (a.src_off[d] + r) * a.src_stride + a.seg_src[d][q])[c];
    reinterpret_cast<float4*>(a.dst[d] + (a.dst_off[d] + r) * a.dst_stride[d] + a.seg_dst[d][q])[c] = v;
  }
  // last block publishes: all of this rank's stores to every peer are
  // visible system-wide before the epoch flag
  __threadfence_system();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = atomicAdd(a.done, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (last) {
    __threadfence_system();
    if (threadIdx.x < a.world && (a.notify >> threadIdx.x & 1)) {
      st_release_sys(a.flag[threadIdx.x] + a.slot * kMaxWorld + a.self, a.epoch);
    }
    if (threadIdx.x == 0) *a.done = 0;
  }
}

// spin until every expected source has published this epoch; bounded so a
// lost peer traps instead of hanging the GPU
__global__ void p2p_wait_kernel(const int64_t* flags, int slot, uint32_t expect, int world, int64_t epoch) {
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x;
  if (t >= world || !(expect >> t & 1)) return;
  const int64_t* f = flags + slot * kMaxWorld + t;
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < epoch) {
    if (clock64() - t0 > 40'000'000'000LL) __trap();  // ~20 s
    __nanosleep(64);
  }
}

__global__ void p2p_tokens_kernel(const P2PTokens a) {
  pdl_trigger();
  pdl_wait();
  for (int j = 0; j < 2; ++j) {
    for (int i = threadIdx.x; i < a.n[j]; i += blockDim.x) {
      const int32_t t = a.src[j][i], r = a.idx[j][i];
      for (int d = 0; d < a.world; ++d) a.dst[d][r] = t;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < a.world && (a.notify >> threadIdx.x & 1)) {
    st_release_sys(a.flag[threadIdx.x] + a.slot * kMaxWorld + a.self, a.epoch);
  }
}

}  // namespace

void launch_p2p_tokens(const P2PTokens& a, cudaStream_t s) {
  SD_CUDA(launch_pdl(p2p_tokens_kernel, dim3(1), dim3(1024), 0, s, 1, a));
  SD_CUDA(cudaGetLastError());
  count_launch();
}

void launch_p2p_scatter(const P2PScatter& a, cudaStream_t s) {
  int64_t work = 0;
  for (int d = 0; d < a.world; ++d) {
    int w = 0;
    for (int q = 0; q < a.nseg[d]; ++q) {
      if (a.seg_n[d][q] % 4 || a.seg_src[d][q] % 4 || a.seg_dst[d][q] % 4) {
        fail(SD_ERR_CONFIG, "peer exchange: row segments must be multiples of 4 floats");
      }
      w += a.seg_n[d][q] / 4;
    }
    work += static_cast<int64_t>(a.cnt[d]) * w;
  }
  int grid = static_cast<int>(std::min<int64_t>(264, (work + 255) / 256));
  if (grid < 1) grid = 1;
  SD_CUDA(launch_pdl(p2p_scatter_kernel, dim3(grid), dim3(256), 0, s, 1, a));
  SD_CUDA(cudaGetLastError());
  count_launch();
}

__global__ void scatter_i32_kernel(int n, const int32_t* idx, const int32_t* src, int32_t* dst) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
  pdl_trigger();
}

void launch_scatter_i32(int n, const int32_t* idx, const int32_t* src, int32_t* dst, cudaStream_t s) {
  if (n <= 0) return;
  SD_CUDA(launch_pdl(scatter_i32_kernel, dim3((n + 255) / 256), dim3(256), 0, s, 1, n, idx, src, dst));
  SD_CUDA(cudaGetLastError());
  count_launch();
}

void launch_p2p_wait(const int64_t* flags, int slot, uint32_t expect, int world, int64_t epoch, cudaStream_t s) {
  if (!expect) return;
  SD_CUDA(launch_pdl(p2p_wait_kernel, dim3(1), dim3(32), 0, s, 1, flags, slot, expect, world, epoch));
  SD_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace sd
