// Streaming ceiling of a tensor-map (TMA) producer over the C5 fp16 KV layout
// (standalone probe): one page group of one layer = K rows then V rows, 16
// positions x 8 heads x 128 fp16 each (32 KB per half). A 5-D tensor map
// (d 64 | position 16 | d-half 2 | head 8 | half-group) with 128-B swizzle
// brings one half (K or V) of a stage per copy, laid out [head][half][pos]
// [128 B] in shared memory (the swizzle row is the position, so ldmatrix over
// 8 positions is conflict-free). Compared with 16 bulk copies of 4 KB.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_pool_bw tools/tma_pool_bw.cu -lcuda
#include <cuda.h>
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
__device__ __forceinline__ void tma5(void* dst, const CUtensorMap* m, uint64_t* bar, int c4, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(0), "r"(0), "r"(0), "r"(0), "r"(c4), "l"(pol)
      : "memory");
}

constexpr int kCons = 8;

__global__ void __launch_bounds__((kCons + 1) * 32, 1)
    stream(const __grid_constant__ CUtensorMap map, int64_t per_cta_stages, int nst) {
  extern __shared__ __align__(1024) uint8_t smem[];
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
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      uint32_t ph = 0;
      for (int64_t j = 0; j < per_cta_stages; ++j) {
        const int64_t grp = static_cast<int64_t>(blockIdx.x) * per_cta_stages + j;
        bar_wait(&empty[s], ph ^ 1);
        bar_expect(&full[s], kStage);
        tma5(ring + s * kStage, &map, &full[s], static_cast<int>(2 * grp), pol);
        tma5(ring + s * kStage + kStage / 2, &map, &full[s], static_cast<int>(2 * grp + 1), pol);
        if (++s == nst) {
          s = 0;
          ph ^= 1;
        }
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
  const int64_t halves = static_cast<int64_t>(bytes / (32 * 1024));
  CUtensorMap map;
  cuuint64_t dims[5] = {64, 16, 2, 8, static_cast<cuuint64_t>(halves)};
  cuuint64_t strides[4] = {2048, 128, 256, 32 * 1024};  // bytes, dims 1..4
  cuuint32_t box[5] = {64, 16, 2, 8, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, p, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("{\"error\": \"encode %d\"}\n", static_cast<int>(r));
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int nst : {2, 3}) {
    const size_t smem = 1024 + static_cast<size_t>(nst) * 64 * 1024;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const int64_t per = (halves / 2) / sms;
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      stream<<<sms, (kCons + 1) * 32, smem>>>(map, per, nst);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double moved = static_cast<double>(per) * sms * 64 * 1024;
    printf("{\"kernel\": \"tma5d\", \"stages\": %d, \"GBps\": %.0f, \"err\": \"%s\"}\n", nst, moved / (best * 1e6),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
