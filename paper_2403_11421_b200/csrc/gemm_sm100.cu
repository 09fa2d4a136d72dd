// S-Part GEMM for sm_100a: C[M][N] = A[M][K] . B[N][K]^T on 5th-generation
// tensor cores. Persistent, warp-specialized, clustered:
//   warp 0  TMA producer: 2-D tensor-map loads (128-B swizzle) into a
//           STAGES-deep shared-memory ring. A (activations) is per CTA; the B
//           tile (weights) is split into CS slices, each CTA of a CS-CTA
//           cluster loads one slice and multicasts it to the whole cluster,
//           so a weight tile crosses L2 once per cluster instead of once per
//           M-block (decode batches make M small and L2 bandwidth the limit).
//   warp 1  MMA issuer: one elected lane issues tcgen05.mma (kind::f16 for
//           bf16 operands, kind::tf32 for fp32) into one of two TMEM
//           accumulators (128 lanes x BN fp32 columns) and releases the smem
//           slot in every cluster CTA with a multicast tcgen05.commit.
//   warps 2-5 epilogue: tcgen05.ld the accumulator, fuse the finish_block
//           epilogues (residual add, SiLU; dense.cpp:51-70), transpose through
//           shared memory and write coalesced fp32 and/or bf16 rows.
// Accumulation is fp32 in TMEM; results match the fp32 reference within
// the operand rounding (bf16 2^-9, tf32 2^-11 relative per product).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <functional>
#include <mutex>
#include <unordered_map>

#include "dense_kernels.cuh"
#include "sd_common.h"

namespace sd {

namespace {

constexpr int BM = 128;
constexpr int BK_BYTES = 128;              // one 128-B swizzle row per operand row
constexpr int A_STAGE = BM * BK_BYTES;     // 16 KB
constexpr int kThreads = 192;
constexpr int EPI_TILE = 32 * 33;          // floats per epilogue warp transpose tile

template <int BN>
struct Cfg {
  static constexpr int B_STAGE = BN * BK_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int TMEM_COLS = 2 * BN;  // two accumulators
  static constexpr size_t SMEM = 1024 + STAGES * (A_STAGE + B_STAGE) + 256 + 4 * EPI_TILE * 4;
};

struct Params {
  int M, N, K;
  int mb, nb, kb;  // blocks along M, N, K
  int cs;          // cluster size along M (1, 2, 4)
  float* C;
  int64_t ldc;
  __nv_bfloat16* Cb;
  int64_t ldcb;
  int epi;
  const float* res;
  int64_t ldr;
  uint32_t idesc;
  int kind;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// same smem offset / mbarrier offset in every CTA of `mask`
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major operand tile, 128-B swizzle,
// 8-row (1024 B) swizzle atoms stacked along M/N (SBO = 1024 B), version 1.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, const Params p) {
  using C_ = Cfg<BN>;
  constexpr int STAGES = C_::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint8_t* tail = sB + STAGES * C_::B_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* epi_smem = reinterpret_cast<float*>(tail + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cs = p.cs;
  const int rank = cs > 1 ? static_cast<int>(cluster_rank()) : 0;
  const uint16_t mask = static_cast<uint16_t>((1u << cs) - 1u);
  const int cluster = blockIdx.x / cs, nclusters = gridDim.x / cs;
  const int mgroups = p.mb / cs;
  const int items = mgroups * p.nb;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], cs);  // one release per cluster CTA
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C_::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();  // peers' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const int kelems = p.kind == 2 ? 32 : 64;
      const int slice = BN / cs;
      for (int it = cluster; it < items; it += nclusters) {
        const int m0 = ((it % mgroups) * cs + rank) * BM, n0 = (it / mgroups) * BN;
        for (int kb = 0; kb < p.kb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);  // every cluster CTA released slot s
          mbar_expect_tx(&full[s], A_STAGE + C_::B_STAGE);
          tma_load_2d(sA + s * A_STAGE, &tma_a, &full[s], kb * kelems, m0);
          if (cs > 1) {
            tma_load_2d_mc(sB + s * C_::B_STAGE + rank * slice * BK_BYTES, &tma_b, &full[s], kb * kelems,
                           n0 + rank * slice, mask);
          } else {
            tma_load_2d(sB + s * C_::B_STAGE, &tma_b, &full[s], kb * kelems, n0);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      // tail: wait until every in-flight slot has been released by all
      // cluster CTAs, so no remote arrive targets an exited CTA
      for (int i = 0; i < STAGES; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int it = cluster; it < items; it += nclusters, ++local) {
        const int acc = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + acc * BN;
        for (int kb = 0; kb < p.kb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t da = make_desc(smem_u32(sA + s * A_STAGE));
          const uint64_t db = make_desc(smem_u32(sB + s * C_::B_STAGE));
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 x 32 B along the 128-B swizzle row
            const uint32_t accum = (kb | k) != 0;
            if (p.kind == 2) {
              mma_tf32(dcol, da + 2 * k, db + 2 * k, p.idesc, accum);
            } else {
              mma_f16(dcol, da + 2 * k, db + 2 * k, p.idesc, accum);
            }
          }
          if (cs > 1) {
            tc_commit_mc(&empty[s], mask);  // release slot s in every cluster CTA
          } else {
            tc_commit(&empty[s]);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    float* tile = epi_smem + (warp - 2) * EPI_TILE;
    int local = 0;
    for (int it = cluster; it < items; it += nclusters, ++local) {
      const int acc = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      const int m0 = ((it % mgroups) * cs + rank) * BM, n0 = (it / mgroups) * BN;
      mbar_wait(&tfull[acc], use & 1);
      __syncwarp();  // lanes leave the try_wait spin independently; .sync.aligned needs convergence
      tc_fence_after();
      const int row0 = m0 + q * 32;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int col0 = n0 + c * 32;
        if (col0 >= p.N) break;  // warp-uniform
        float v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 32, v);
        // lane = row (q*32 + lane) of the tile; transpose through smem
#pragma unroll
        for (int i = 0; i < 32; ++i) tile[lane * 33 + i] = v[i];
        __syncwarp();
        const int col = col0 + lane;
        if (col < p.N) {
          for (int r = 0; r < 32; ++r) {
            const int row = row0 + r;
            if (row >= p.M) break;
            float x = tile[r * 33 + lane];
            if (p.epi == kEpiResidual) {
              x = x + p.res[static_cast<int64_t>(row) * p.ldr + col];
            } else if (p.epi == kEpiSilu) {
              x = x / (1.0f + expf(-x));
            }
            if (p.C) p.C[static_cast<int64_t>(row) * p.ldc + col] = x;
            if (p.Cb) p.Cb[static_cast<int64_t>(row) * p.ldcb + col] = __float2bfloat16_rn(x);
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C_::TMEM_COLS));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
  });
  if (!fn) fail(SD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap encode_map(const void* base, int rows, int cols, int64_t ld, int kind, int box_rows);

// Tensor maps only encode (address, extents, strides, box), so they are
// cached: the weights' maps never change and the activations' maps repeat
// every layer and step.
CUtensorMap make_map(const void* base, int rows, int cols, int64_t ld, int kind, int box_rows) {
  struct Key {
    const void* b;
    int r, c, k, box;
    int64_t ld;
    bool operator==(const Key& o) const {
      return b == o.b && r == o.r && c == o.c && k == o.k && box == o.box && ld == o.ld;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      size_t h = std::hash<const void*>()(k.b);
      for (int64_t v : {static_cast<int64_t>(k.r), static_cast<int64_t>(k.c), static_cast<int64_t>(k.k),
                        static_cast<int64_t>(k.box), k.ld}) {
        h = h * 1000003u ^ std::hash<int64_t>()(v);
      }
      return h;
    }
  };
  static std::unordered_map<Key, CUtensorMap, Hash> cache;
  static std::mutex mu;
  const Key key{base, rows, cols, kind, box_rows, ld};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 4096) cache.clear();
  const CUtensorMap m = encode_map(base, rows, cols, ld, kind, box_rows);
  cache.emplace(key, m);
  return m;
}

CUtensorMap encode_map(const void* base, int rows, int cols, int64_t ld, int kind, int box_rows) {
  CUtensorMap m;
  const int es = kind == 2 ? 4 : 2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * es};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK_BYTES / es), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = get_encode()(&m, kind == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SD_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN>
void launch(const GemmArgs& g, int cs, cudaStream_t s) {
  using C_ = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    SD_CUDA(cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(C_::SMEM)));
    SD_CUDA(cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_set = true;
  }
  const CUtensorMap ta = make_map(g.A, g.M, g.K, g.lda, g.kind, BM);
  const CUtensorMap tb = make_map(g.B, g.N, g.K, g.ldb, g.kind, BN / cs);
  Params p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.mb = (g.M + BM - 1) / BM;
  p.nb = (g.N + BN - 1) / BN;
  p.kb = g.K / (BK_BYTES / (g.kind == 2 ? 4 : 2));
  p.cs = cs;
  p.C = g.C;
  p.ldc = g.ldc;
  p.Cb = g.Cb;
  p.ldcb = g.ldcb;
  p.epi = g.epi;
  p.res = g.res;
  p.ldr = g.ldr;
  p.kind = g.kind;
  const uint32_t fmt = g.kind == 2 ? 2u : 1u;  // TF32 : BF16
  p.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
            (static_cast<uint32_t>(BM >> 4) << 24);
  const int items = (p.mb / cs) * p.nb;
  const int budget = g.max_ctas > 0 && g.max_ctas < num_sms() ? g.max_ctas : num_sms();
  const int max_clusters = budget / cs > 0 ? budget / cs : 1;
  const int clusters = items < max_clusters ? items : max_clusters;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * cs));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C_::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SD_CUDA(cudaLaunchKernelEx(&cfg, gemm_kernel<BN>, ta, tb, p));
  count_launch();
}

}  // namespace

bool gemm_sm100_supported(const GemmArgs& g) {
  const int es = g.kind == 2 ? 4 : 2;
  if (g.kind != 1 && g.kind != 2) return false;
  if (g.M < 1 || g.N < 1 || g.K < 1) return false;
  if ((g.lda * es) % 16 || (g.ldb * es) % 16) return false;
  if (reinterpret_cast<uintptr_t>(g.A) % 16 || reinterpret_cast<uintptr_t>(g.B) % 16) return false;
  if (g.K % (BK_BYTES / es) != 0) return false;  // whole k-blocks
  return true;
}

// Tile shape and cluster size (measured at decode batches, tools/bench_gemm.py):
// 256-wide tiles with a 2-CTA cluster sharing each weight tile by multicast;
// 128-wide tiles without a cluster when 256-wide tiles would leave more than
// half of the SMs idle (the N = D GEMMs at M = 512).
void launch_gemm_sm100(const GemmArgs& g, cudaStream_t s) {
  const int mb = (g.M + BM - 1) / BM;
  static const int force_cs = getenv("SD_GEMM_CS") ? atoi(getenv("SD_GEMM_CS")) : 0;
  static const int force_bn = getenv("SD_GEMM_BN") ? atoi(getenv("SD_GEMM_BN")) : 0;
  const int tiles256 = mb * ((g.N + 255) / 256);
  const int sms = g.max_ctas > 0 && g.max_ctas < num_sms() ? g.max_ctas : num_sms();
  int bn = tiles256 * 2 <= sms ? 128 : 256;
  int cs = (bn == 256 && mb % 2 == 0) ? 2 : 1;
  if (force_cs > 0 && mb % force_cs == 0) cs = force_cs;
  if (force_bn == 128 || force_bn == 256) bn = force_bn;
  if (bn == 128) {
    launch<128>(g, cs, s);
  } else {
    launch<256>(g, cs, s);
  }
}

}  // namespace sd
