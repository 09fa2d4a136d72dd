// TMA ingress microbenchmark (standalone; not part of the library).
// Each CTA streams 2 x 16 KB tensor-map boxes (128-B swizzle, 128 rows) per
// stage through a STAGES-deep smem ring from an L2-resident bf16 matrix; a
// consumer thread only releases slots. Reports bytes landed in smem per SM
// per clock and in aggregate, for several grid sizes, without and with a
// 2-CTA cluster that multicasts each box half (halving L2 reads per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tools/tma_bw.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int ROWS = 8192, COLS = 2048;  // 32 MB bf16: L2-resident
constexpr int MAX_STAGES = 12, STAGE = 32 * 1024;  // stage = nbox boxes of (256 / nbox) rows x 128 B

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(b)),
               "r"(ph)
               : "memory");
}

__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap map, int iters, int cs,
                                                    int STAGES, int nbox, long long* cycles) {
  const int BOX_ROWS = 256 / nbox;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[MAX_STAGES], empty[MAX_STAGES];
  uint32_t rank = 0;
  if (cs > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(cs));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (cs > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const long long t0 = clock64();
  const int cluster = blockIdx.x / cs;
  if (threadIdx.x == 0) {  // producer
    uint32_t ph = 0;
    int s = 0;
    for (int i = 0; i < iters; ++i) {
      wait(&empty[s], ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(STAGE) : "memory");
      const int row = (cluster * 256 + (i / 32) * 512) % ROWS;
      const int col = (i % 32) * 64;
      for (int b = 0; b < nbox; ++b) {
        uint8_t* dst = ring + s * STAGE + b * BOX_ROWS * 128;
        if (cs > 1) {  // each rank loads BOX_ROWS/cs rows of the box and multicasts
          const int sub = BOX_ROWS / cs;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
              "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(dst + rank * sub * 128)),
              "l"(&map), "r"(su32(&full[s])), "r"(col), "r"(row + b * BOX_ROWS + rank * sub),
              "h"(static_cast<uint16_t>((1 << cs) - 1))
              : "memory");
        } else {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
              "[%2];" ::"r"(su32(dst)),
              "l"(&map), "r"(su32(&full[s])), "r"(col), "r"(row + b * BOX_ROWS)
              : "memory");
        }
      }
      if (++s == STAGES) {
        s = 0;
        ph ^= 1;
      }
    }
    for (int i = 0; i < STAGES; ++i) {  // drain
      wait(&empty[s], ph ^ 1);
      if (++s == STAGES) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {  // consumer: release each slot in every cluster CTA
    uint32_t ph = 0;
    int s = 0;
    for (int i = 0; i < iters; ++i) {
      wait(&full[s], ph);
      for (int r = 0; r < cs; ++r) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&empty[s])), "r"(r));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
      if (++s == STAGES) {
        s = 0;
        ph ^= 1;
      }
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (cs > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  void* buf;
  cudaMalloc(&buf, static_cast<size_t>(ROWS) * COLS * 2);
  cudaMemset(buf, 0, static_cast<size_t>(ROWS) * COLS * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  long long* cyc;
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  const int iters = 2048;
  const int cs = 1, grid = 148;
  for (int nbox : {1, 2, 4, 8}) {
    for (int stages : {2, 3, 4, 6}) {
      const int smem = stages * STAGE + 1024;
      cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      CUtensorMap map;
      cuuint64_t dims[2] = {COLS, ROWS};
      cuuint64_t strides[1] = {COLS * 2};
      cuuint32_t box[2] = {64, static_cast<cuuint32_t>(256 / nbox)};
      cuuint32_t es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        tma_stream<<<grid, 64, smem>>>(map, iters, cs, stages, nbox, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      long long c[1024];
      cudaMemcpy(c, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = c[i] > mx ? c[i] : mx;
      const double bytes_per_sm = static_cast<double>(iters) * STAGE;
      const double bpc = bytes_per_sm / mx;
      printf("{\"box_rows\": %d, \"stages\": %d, \"err\": \"%s\", \"B_per_clk_per_sm\": %.1f, \"agg_TBs\": %.2f, "
             "\"implied_latency_clk\": %.0f}\n",
             256 / nbox, stages, cudaGetErrorString(cudaGetLastError()), bpc, bytes_per_sm * grid / (ms * 1e9),
             stages * STAGE / bpc);
    }
  }
  return 0;
}
