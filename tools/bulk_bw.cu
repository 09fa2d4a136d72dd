// Streaming ceiling of the attention producer's copy pattern (standalone):
// one CTA per SM, a producer warp whose lanes issue cp.async.bulk copies into
// a ring of stages completed on mbarriers, consumer warps that only release
// the stages. A stage is two 32-KB halves (the K and V rows of 16 positions,
// 2 KB each) fetched as 4-KB copies; consecutive stages walk page groups of
// `group` bytes (one layer's 64-KB region inside each) — the C5 KV layout.
// Prints GB/s for a few ring depths and group strides, and for a contiguous
// walk, to separate the copy mechanism from the attention's consumer work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk_bw tools/bulk_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}

constexpr int kCons = 8;

__global__ void __launch_bounds__((kCons + 1) * 32, 1)
    stream(const uint8_t* __restrict__ src, int64_t per_cta_stages, int64_t group, int nst, int copy) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + nst;
  uint8_t* ring = smem + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], kCons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  constexpr uint32_t kStage = 64 * 1024;
  if (warp == kCons) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int s = 0;
    uint32_t ph = 0;
    for (int64_t j = 0; j < per_cta_stages; ++j) {
      const int64_t idx = static_cast<int64_t>(blockIdx.x) * per_cta_stages + j;
      const uint8_t* base = src + idx * group;
      if (lane == 0) {
        bar_wait(&empty[s], ph ^ 1);
        bar_expect(&full[s], kStage);
      }
      __syncwarp();
      const int ncopy = static_cast<int>(kStage / copy);
      if (lane < ncopy) bulk(ring + s * kStage + lane * copy, base + lane * copy, copy, &full[s], pol);
      if (++s == nst) {
        s = 0;
        ph ^= 1;
      }
    }
    return;
  }
  int s = 0;
  uint32_t ph = 0;
  for (int64_t j = 0; j < per_cta_stages; ++j) {
    bar_wait(&full[s], ph);
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[s]);
    if (++s == nst) {
      s = 0;
      ph ^= 1;
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 16ull << 30;
  uint8_t* p;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
  cudaMemset(p, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int64_t group : {64LL * 1024, 2LL * 1024 * 1024}) {
    for (int copy : {4096, 8192, 16384}) {
      for (int nst : {2, 3}) {
        const size_t smem = 1024 + static_cast<size_t>(nst) * 64 * 1024;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        const int64_t total_stages = static_cast<int64_t>((bytes - 64 * 1024) / group);
        const int64_t per = total_stages / sms;
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
          cudaEventRecord(e0);
          stream<<<sms, (kCons + 1) * 32, smem>>>(p, per, group, nst, copy);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = ms < best ? ms : best;
        }
        const double moved = static_cast<double>(per) * sms * 64 * 1024;
        printf("{\"kernel\": \"bulk\", \"copy\": %d, \"group_stride\": %lld, \"stages\": %d, \"GBps\": %.0f, \"err\": \"%s\"}\n",
               copy, static_cast<long long>(group), nst, moved / (best * 1e6), cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
