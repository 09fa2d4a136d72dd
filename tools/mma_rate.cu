// tcgen05.mma issue-rate microbenchmark (standalone; not part of the library).
// One CTA (or CTA pair) per SM issues `iters` bf16 MMAs of M x N x 16 from
// zeroed shared memory into TMEM back to back, with one commit at the end.
// Prints MACs/clk/SM and TFLOP/s for each (pair, N).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return static_cast<uint64_t>((a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <bool PAIR>
__global__ void __launch_bounds__(128, 1) mma_loop(int n, int iters, long long* cycles, int commit_every, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, dummy, ring[8], fullb[8];
  __shared__ uint32_t tslot;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&dummy)), "r"(mode == 1 ? (1 << 19) : 1));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&ring[i])));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&fullb[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                         (static_cast<uint32_t>((PAIR ? 256 : 128) >> 4) << 24);
  long long t0 = clock64();
  const int S = commit_every > 0 ? commit_every : 6;  // ring depth for modes 6/7
  if ((mode == 6 || mode == 7) && threadIdx.x == 32) {
    // producer: wait slot released (commit), then arrive "full"
    uint32_t ph = 0;
    int st = 0;
    for (int kb = 0; kb < iters / 4; ++kb) {
      if (mode == 6) {
        asm volatile("{\n.reg .pred p;\nW1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}\n" ::"r"(su32(&ring[st])), "r"(ph ^ 1) : "memory");
      } else {
        asm volatile("{\n.reg .pred p;\nW2: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(su32(&ring[st])), "r"(ph ^ 1) : "memory");
      }
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&fullb[st])) : "memory");
      if (++st == S) { st = 0; ph ^= 1; }
    }
  }
  if ((mode == 6 || mode == 7) && threadIdx.x == 0) {
    const uint64_t da = desc(su32(base)), db = desc(su32(base + 32 * 1024));
    uint32_t ph = 0;
    int st = 0;
    for (int kb = 0; kb < iters / 4; ++kb) {
      if (mode == 6) {
        asm volatile("{\n.reg .pred p;\nW3: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W3;\n}\n" ::"r"(su32(&fullb[st])), "r"(ph) : "memory");
      } else {
        asm volatile("{\n.reg .pred p;\nW4: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W4;\n}\n" ::"r"(su32(&fullb[st])), "r"(ph) : "memory");
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&ring[st])) : "memory");
      if (++st == S) { st = 0; ph ^= 1; }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  } else if (mode != 6 && mode != 7 && threadIdx.x == 0 && rank == 0) {
    const uint64_t da = desc(su32(base)), db = desc(su32(base + 32 * 1024));
    if (mode == 5) {  // GEMM issuer shape: 4 unrolled MMAs + one commit per k-block, rotating slots
      for (int kb = 0; kb < iters / 4; ++kb) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (PAIR) {
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                         "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(1));
          } else {
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                         "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(1));
          }
        }
        if (commit_every) {
          if (PAIR) {
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&ring[kb & 7])), "h"((uint16_t)3) : "memory");
          } else {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&ring[kb & 7])) : "memory");
          }
        }
      }
    } else
    for (int i = 0; i < iters; ++i) {
      const uint64_t k = 2 * (i & 3);
      if (PAIR) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da + k), "l"(db + k), "r"(idesc), "r"(1));
      } else {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da + k), "l"(db + k), "r"(idesc), "r"(1));
      }
      if (commit_every && (i % commit_every) == commit_every - 1) {
        uint64_t* target = mode == 3 ? &ring[(i / commit_every) & 7] : &dummy;
        if (PAIR) {
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(target)), "h"((uint16_t)3) : "memory");
        } else if (mode == 4) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(target) : "memory");
        } else {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(target)) : "memory");
        }
      }
    }
    if (PAIR) {
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)), "h"((uint16_t)3) : "memory");
    } else {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (PAIR) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    } else {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(long long));
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(mma_loop<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_loop<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  for (int mode : {6, 7}) {
  for (int ce : {2, 4, 6, 8}) {
  for (int pair = 0; pair < 2; ++pair) {
    for (int n : {128, 256}) {
      if ((mode == 4 || mode >= 6) && pair) continue;
      if (pair && n % 16) continue;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(pair ? (sms / 2) * 2 : sms);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = pair ? 2 : 1;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (pair) {
          cudaLaunchKernelEx(&cfg, mma_loop<true>, n, iters, cyc, ce, mode);
        } else {
          cudaLaunchKernelEx(&cfg, mma_loop<false>, n, iters, cyc, ce, mode);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      cudaError_t err = cudaGetLastError();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      long long c0 = 0;
      cudaMemcpy(&c0, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
      const double m = pair ? 256 : 128;
      const double macs_per_sm = (pair ? m / 2 : m) * n * 16.0 * iters;
      const double ctas = pair ? (sms / 2) * 2 : sms;
      printf("{\"mode\": %d, \"commit_every\": %d, \"pair\": %d, \"N\": %d, \"err\": \"%s\", \"ms\": %.3f, \"cyc\": %lld, \"mac_per_clk_sm\": %.0f, \"tflops\": %.0f, \"clk_ghz\": %.3f}\n",
             mode, ce, pair, n, cudaGetErrorString(err), ms, c0, macs_per_sm / c0, 2 * macs_per_sm * ctas / (ms * 1e-3) / 1e12,
             c0 / (ms * 1e6));
    }
  }
  }
  }
  return 0;
}
