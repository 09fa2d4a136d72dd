// S-Part GEMM for sm_100a: C[M][N] = A[M][K] . B[N][K]^T on 5th-generation
// tensor cores. Persistent, warp-specialized, clustered:
//   warp 0  TMA producer: 2-D tensor-map loads (128-B swizzle) into a
//           STAGES-deep shared-memory ring. A (activations) is per CTA; the B
//           tile (weights) is split into CS slices, each CTA of a CS-CTA
//           cluster loads one slice and multicasts it to the whole cluster,
//           so a weight tile crosses L2 once per cluster instead of once per
//           M-block (decode batches make M small and L2 bandwidth the limit).
//   warp 1  MMA issuer: one elected lane issues tcgen05.mma (kind::f16 for
//           bf16 or fp16 operands, kind::tf32 for fp32) into one of two TMEM
//           accumulators (128 lanes x BN fp32 columns) and releases the smem
//           slot in every cluster CTA with a multicast tcgen05.commit.
//   warps 2-5 epilogue: tcgen05.ld the accumulator, fuse the finish_block
//           epilogues (residual add, SiLU; dense.cpp:51-70), transpose through
//           shared memory and write coalesced fp32 and/or 16-bit rows.
// Accumulation is fp32 in TMEM; results match the fp32 reference within
// the operand rounding (bf16 2^-9, fp16 2^-11 RNE, tf32 2^-11 truncated,
// relative per operand).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <functional>
#include <mutex>
#include <unordered_map>

#include "dense_kernels.cuh"
#include "pdl.cuh"
#include "sd_common.h"

namespace sd {

namespace {

constexpr int BM = 128;
constexpr int BK_BYTES = 128;              // one 128-B swizzle row per operand row
constexpr int kThreads = 192;

struct Params {
  int M, N, K;
  int mb, nb, kb;  // blocks along M, N, K
  int cs;          // cluster size along M (1, 2, 4)
  float* C;
  int64_t ldc;
  uint16_t* Cb;  // 16-bit copy of C (the next GEMM's A operand): bf16, or fp16 when f16
  int64_t ldcb;
  int epi;
  const float* res;
  int64_t ldr;
  uint32_t idesc;
  int kind;
  int f16;   // kind::f16 operands are fp16 (else bf16); Cb is written in the same format
  int bn;    // tile width along N (<= BN; a multiple of 16 in PAIR mode)
  int vec;   // outputs / residual 16-B aligned: vector epilogue
  int tma_out;  // outputs written by TMA tensor stores
  int routed;      // C rows go to route.base[route.rank[m]] (fused multi-GPU exchange)
  int route_tma;   // contiguous 32-row slabs leave as tensor stores (RouteMaps), other rows as bulk copies
  RowRoute route;
  unsigned long long* amax;  // fused argmax keys per row (GemmArgs::amax)
  int kvapp;                 // K/V columns go to the KV pages (kva)
  KvAppendOut kva;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
// same smem offset / mbarrier offset in every CTA of `mask`
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// ---- elected forms: the producer and MMA warps run their loops warp-wide
// (uniform control flow keeps descriptors and coordinates in uniform
// registers) and let one elected lane issue each instruction
#define SD_ELECT "elect.sync _|e, 0xffffffff;\n"
__device__ __forceinline__ void e_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n.reg .pred e;\n" SD_ELECT "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void e_tma_load(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "{\n.reg .pred e;\n" SD_ELECT
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n}\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void e_tma_load_mc(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                              uint16_t mask) {
  asm volatile(
      "{\n.reg .pred e;\n" SD_ELECT
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;\n}\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void e_tma_load_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "{\n.reg .pred e;\n" SD_ELECT
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
template <int KIND, bool PAIR>
__device__ __forceinline__ void e_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (PAIR) {
    if (KIND == 2) {
      asm volatile("{\n.reg .pred e, p;\n" SD_ELECT
                   "setp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                   "l"(a), "l"(b), "r"(idesc), "r"(acc));
    } else {
      asm volatile("{\n.reg .pred e, p;\n" SD_ELECT
                   "setp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                   "l"(a), "l"(b), "r"(idesc), "r"(acc));
    }
  } else if (KIND == 2) {
    asm volatile("{\n.reg .pred e, p;\n" SD_ELECT
                 "setp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile("{\n.reg .pred e, p;\n" SD_ELECT
                 "setp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}
// commit: arrive (once) on `bar` in every CTA of `mask` when the issued MMAs complete
template <bool PAIR>
__device__ __forceinline__ void e_commit(uint64_t* bar, uint16_t mask) {
  if (PAIR) {
    asm volatile("{\n.reg .pred e;\n" SD_ELECT
                 "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                 "%1;\n}\n" ::"r"(smem_u32(bar)),
                 "h"(mask)
                 : "memory");
  } else if (mask != 1) {
    asm volatile("{\n.reg .pred e;\n" SD_ELECT
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                 "%1;\n}\n" ::"r"(smem_u32(bar)),
                 "h"(mask)
                 : "memory");
  } else {
    asm volatile("{\n.reg .pred e;\n" SD_ELECT
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
  }
}

// ---- CTA-pair (cta_group::2) forms
// shared::cluster address of the same variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// TMA load into this CTA's smem whose completion bytes count on the pair
// leader's mbarrier (`bar_cluster` from mapa)
// arrive on the same-offset mbarrier of both pair CTAs once the issued MMAs complete
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
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


__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// contiguous smem -> global bulk copy (any mapped global address, peers included)
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void sts128(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
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

// Stage geometry. A stage holds ATOMS 128-B swizzle atoms along K per
// operand (ATOMS x 4 MMAs per barrier handshake: the MMA thread's
// wait/fence/issue costs ~430 cycles per handshake, more than four 256 x 128
// MMAs take; tools/mma_rate.cu). PAIR: a CTA pair computes a 256 x bn tile
// with cta_group::2 MMAs, each CTA staging its own 128 A rows and half of
// the B tile.
template <int BN, bool PAIR, int ATOMS>
struct Cfg {
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;  // B rows staged per CTA (max)
  static constexpr int A_ATOM = BM * BK_BYTES;
  static constexpr int B_ATOM = B_ROWS * BK_BYTES;
  static constexpr int A_ST = ATOMS * A_ATOM;
  static constexpr int B_ST = ATOMS * B_ATOM;
  static constexpr int STAGES = (196 * 1024 / (A_ST + B_ST)) > 8 ? 8 : (196 * 1024 / (A_ST + B_ST));
  // two accumulators, allocated in a power-of-two column count
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  // epilogue staging for TMA stores: per epilogue warp, two buffers of
  // 32 rows x 16 columns in fp32 (2 KB, 64-B swizzle) and 16-bit (1 KB, 32-B swizzle)
  static constexpr int OUT_F32 = 32 * 16 * 4, OUT_BF16 = 32 * 16 * 2;
  static constexpr int OUT_WARP = 2 * (OUT_F32 + OUT_BF16);
  static constexpr size_t SMEM = 1024 + STAGES * (A_ST + B_ST) + 4 * OUT_WARP + 256;
};

// fp32 tensor maps (64-B swizzle, 16-column x 32-row boxes) of a routed
// GEMM's destination buffers, one per rank
struct RouteMaps {
  CUtensorMap m[8];
};

template <int BN, bool PAIR, int ATOMS, int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_cb, const Params p,
                const __grid_constant__ RouteMaps rmaps) {
  using C_ = Cfg<BN, PAIR, ATOMS>;
  constexpr int STAGES = C_::STAGES;
  constexpr int KELEMS = BK_BYTES / (KIND == 2 ? 4 : 2);  // elements per atom row
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C_::A_ST;
  uint8_t* sOut = sB + STAGES * C_::B_ST;  // 1024-aligned: stage sizes are multiples of 1 KB
  uint8_t* tail = sOut + 4 * C_::OUT_WARP;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cs = PAIR ? 2 : p.cs;
  const int rank = cs > 1 ? static_cast<int>(cluster_rank()) : 0;
  const bool leader = rank == 0;
  const uint16_t mask = static_cast<uint16_t>((1u << cs) - 1u);
  const int cluster = blockIdx.x / cs, nclusters = gridDim.x / cs;
  // PAIR: a cluster item is a 256-row M block (rank r owns rows r*128..);
  // otherwise cs consecutive 128-row M blocks sharing one B tile (multicast)
  const int mgroups = PAIR ? (p.mb + 1) / 2 : p.mb / cs;
  const int items = mgroups * p.nb;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PAIR ? 1 : cs);  // PAIR: one multicast commit from the leader
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 8 : 4);  // PAIR: both CTAs' epilogue warps release the leader
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C_::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C_::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  pdl_trigger();
  __syncthreads();
  if (cs > 1) cluster_sync();  // peers' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // A operand / residual of the previous kernel from here on

  // first row of this CTA's block 0 (block b adds b * cs * BM)
  auto m_origin = [&](int it) { return ((it % mgroups) * cs + rank) * BM; };

  if (warp == 0) {
    // ------------------------------------------------------- TMA producer
    {
      int s = 0;
      uint32_t ph = 0;
      const int slice = PAIR ? p.bn / 2 : BN / cs;
      const uint32_t bytes = static_cast<uint32_t>(ATOMS * (C_::A_ATOM + (PAIR ? slice : BN) * BK_BYTES)) *
                             (PAIR ? 2u : 1u);  // PAIR: both CTAs' bytes land on the leader's barrier
      const uint32_t full0 = PAIR ? mapa(&full[0], 0) : smem_u32(&full[0]);
      for (int it = cluster; it < items; it += nclusters) {
        const int m0 = m_origin(it), n0 = (it / mgroups) * p.bn;
        for (int kb = 0; kb < p.kb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);  // slot s released (by every cluster CTA / the pair leader)
          if (!PAIR || leader) e_expect_tx(&full[s], bytes);
          const uint32_t fb = full0 + s * static_cast<uint32_t>(sizeof(uint64_t));
#pragma unroll
          for (int a = 0; a < ATOMS; ++a) {
            const int kc = (kb * ATOMS + a) * KELEMS;
            uint8_t* dA = sA + s * C_::A_ST + a * C_::A_ATOM;
            uint8_t* dB = sB + s * C_::B_ST + a * C_::B_ATOM;
            if (PAIR) {
              e_tma_load_pair(dA, &tma_a, fb, kc, m0);
              e_tma_load_pair(dB, &tma_b, fb, kc, n0 + rank * slice);
            } else {
              e_tma_load(dA, &tma_a, fb, kc, m0);
              if (cs > 1) {
                e_tma_load_mc(dB + rank * slice * BK_BYTES, &tma_b, fb, kc, n0 + rank * slice, mask);
              } else {
                e_tma_load(dB, &tma_b, fb, kc, n0);
              }
            }
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      // tail: wait until every in-flight slot has been released, so no
      // remote arrive targets an exited CTA
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
    if (!PAIR || leader) {
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      const uint64_t da0 = make_desc(smem_u32(sA)), db0 = make_desc(smem_u32(sB));
      const uint16_t cmask = PAIR ? static_cast<uint16_t>(3) : mask;
      for (int it = cluster; it < items; it += nclusters, ++local) {
        // two accumulator slots alternate across this CTA's items
        const int acc = local & 1;
        mbar_wait(&tempty[acc], (static_cast<uint32_t>(local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + acc * BN;
        for (int kb = 0; kb < p.kb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          // descriptor start addresses advance in 16-B units
          const uint64_t da = da0 + static_cast<uint64_t>(s * (C_::A_ST >> 4));
          const uint64_t db = db0 + static_cast<uint64_t>(s * (C_::B_ST >> 4));
#pragma unroll
          for (int a = 0; a < ATOMS; ++a) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 x 32 B along the 128-B swizzle row
              e_mma<KIND, PAIR>(dcol, da + a * (C_::A_ATOM >> 4) + 2 * k, db + a * (C_::B_ATOM >> 4) + 2 * k,
                                p.idesc, (kb | a | k) != 0);
            }
          }
          e_commit<PAIR>(&empty[s], cmask);  // release slot s (both pair CTAs / every cluster CTA)
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        e_commit<PAIR>(&tfull[acc], PAIR ? static_cast<uint16_t>(3) : static_cast<uint16_t>(1));
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue
    // tcgen05.ld 32x32b gives each lane one row and 32 consecutive columns:
    // with aligned outputs the lane writes them straight from registers as
    // 16-B vectors (8 per fp32 chunk, 4 per bf16 chunk), no smem transpose.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t tempty_leader0 = PAIR ? mapa(&tempty[0], 0) : 0;
    int local = 0;
    if (p.tma_out) {
      // TMA-store epilogue: 16-column chunks staged in swizzled smem (two
      // buffers per warp) and written by one bulk tensor store per output;
      // the tensor maps clip rows >= M and columns >= N
      uint8_t* myout = sOut + (warp - 2) * C_::OUT_WARP;
      int nchunk = 0;
      for (int it = cluster; it < items; it += nclusters, ++local) {
        const int acc = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        const int m0 = m_origin(it), n0 = (it / mgroups) * p.bn;
        const int nend = n0 + p.bn < p.N ? n0 + p.bn : p.N;
        mbar_wait(&tfull[acc], use & 1);
        __syncwarp();
        tc_fence_after();
        const int rowb = m0 + q * 32;
        const int64_t row = rowb + lane;
        const bool rin = row < p.M;
        // fused append: this row's K row in its KV page (V at + v_off)
        uint8_t* krow = nullptr;
        if (p.kvapp && rin) {
          krow = p.kva.layer_base + static_cast<int64_t>(p.kva.group[row]) * p.kva.group_bytes +
                 static_cast<int64_t>(p.kva.pos[row] & p.kva.pmask) * p.kva.pos_bytes;
        }
#pragma unroll 1
        for (int c = 0; c < (p.bn + 15) / 16; ++c) {
          const int col0 = n0 + c * 16;
          if (col0 >= nend) break;  // warp-uniform
          float v[16];
          tmem_ld16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 16, v);
          if (p.kvapp && col0 >= p.kva.col_k && col0 < p.kva.col_k + 2 * p.kva.width) {  // warp-uniform
            if (krow) {
              const bool isv = col0 >= p.kva.col_k + p.kva.width;
              const int e0 = col0 - p.kva.col_k - (isv ? p.kva.width : 0);
              uint32_t w[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const __half2 h = __floats2half2_rn(v[2 * e], v[2 * e + 1]);
                w[e] = *reinterpret_cast<const uint32_t*>(&h);
              }
              uint4* d = reinterpret_cast<uint4*>(krow + (isv ? p.kva.v_off : 0) + static_cast<int64_t>(e0) * 2);
              d[0] = make_uint4(w[0], w[1], w[2], w[3]);
              d[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
            continue;
          }
          if (p.epi == kEpiResidual) {
            if (rin && p.vec && col0 + 16 <= p.N) {
              const float4* r4 = reinterpret_cast<const float4*>(p.res + row * p.ldr + col0);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float4 t = r4[k];
                v[4 * k] = v[4 * k] + t.x;
                v[4 * k + 1] = v[4 * k + 1] + t.y;
                v[4 * k + 2] = v[4 * k + 2] + t.z;
                v[4 * k + 3] = v[4 * k + 3] + t.w;
              }
            } else {
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                if (rin && col0 + k < p.N) v[k] = v[k] + p.res[row * p.ldr + col0 + k];
              }
            }
          } else if (p.epi == kEpiSilu) {
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = v[k] / (1.0f + expf(-v[k]));
          }
          uint8_t* bf = myout + (nchunk & 1) * (C_::OUT_F32 + C_::OUT_BF16);
          uint8_t* bb = bf + C_::OUT_F32;
          ++nchunk;
          if (lane == 0) bulk_wait_read<1>();  // this buffer's store (two chunks ago) has read it
          __syncwarp();
          if (p.C) {  // row = lane, 64 B = four 16-B chunks, 64-B swizzle
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              sts128(bf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4), __float_as_uint(v[4 * j]),
                     __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            }
          }
          if (p.Cb) {  // 32 B = two 16-B chunks, 32-B swizzle
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) w[e] = pack16x2(v[2 * e], v[2 * e + 1], p.f16);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              sts128(bb + lane * 32 + ((j ^ ((lane >> 2) & 1)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2],
                     w[4 * j + 3]);
            }
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (p.C) tma_store_2d(&tma_c, bf, col0, rowb);
            if (p.Cb) tma_store_2d(&tma_cb, bb, col0, rowb);
            bulk_commit();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) {
            mbar_arrive_cluster(tempty_leader0 + acc * static_cast<uint32_t>(sizeof(uint64_t)));
          } else {
            mbar_arrive(&tempty[acc]);
          }
        }
      }
      if (lane == 0) bulk_wait_all();  // stores complete before the CTA retires
    } else
    for (int it = cluster; it < items; it += nclusters, ++local) {
      const int acc = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      const int m0 = m_origin(it), n0 = (it / mgroups) * p.bn;
      const int nend = n0 + p.bn < p.N ? n0 + p.bn : p.N;
      mbar_wait(&tfull[acc], use & 1);
      __syncwarp();  // lanes leave the try_wait spin independently; .sync.aligned needs convergence
      tc_fence_after();
      const int64_t row = m0 + q * 32 + lane;
      const bool rowok = row < p.M;
      // routed rows (peer memory over NVLink): each lane's destination row,
      // resolved once per tile
      float* rrow = p.routed && rowok ? p.route.base[p.route.rank[row]] + p.route.row[row] * p.route.ld : nullptr;
      // a warp slab whose 32 rows land on consecutive rows of one buffer (the
      // common case: home rows are grouped by destination) leaves as TMA
      // tensor stores, 16 columns x 32 rows per store
      bool slab = false;
      int slab_rank = 0, slab_row = 0;
      if (p.routed) {
        const int rk = rowok ? p.route.rank[row] : -1, rw = rowok ? p.route.row[row] : -1;
        slab_rank = __shfl_sync(0xffffffffu, rk, 0);
        slab_row = __shfl_sync(0xffffffffu, rw, 0);
        slab = p.route_tma && __all_sync(0xffffffffu, rk >= 0 && rk == slab_rank && rw == slab_row + lane) != 0;
        bulk_wait_read<0>();  // no copy of the previous tile still reads this warp's staging
        __syncwarp();
      }
      int nchunk = 0;
      unsigned long long best = 0;  // fused argmax: this row's best key in the tile
#pragma unroll 1
      for (int c = 0; c < (p.bn + 31) / 32; ++c) {
        const int col0 = n0 + c * 32;
        if (col0 >= nend) break;  // warp-uniform
        float v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 32, v);
        if (p.amax) {
          // key = order-preserving bits of the value (NaN never wins, -0 is
          // +0) above the inverted column, so the largest key is the first
          // maximum (argmax_token, dense.cpp:80-88)
          if (rowok) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const float x = v[k];
              if (col0 + k < nend && x == x) {
                const uint32_t b = x == 0.0f ? 0u : __float_as_uint(x);
                const uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
                const unsigned long long key =
                    (static_cast<unsigned long long>(ord) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(col0 + k));
                best = key > best ? key : best;
              }
            }
          }
          continue;
        }
        if (p.routed) {
          // remote NVLink writes are packetised per contiguous run: a warp
          // slab bound for 32 consecutive rows of one buffer leaves as tensor
          // stores, any other row as one bulk copy of its 32 columns
          // (kEpiNone; host-checked)
          float* st = reinterpret_cast<float*>(sOut + (warp - 2) * C_::OUT_WARP);
          const int ncols = nend - col0 < 32 ? nend - col0 : 32;  // multiple of 16
          if (slab) {
            uint8_t* myout = sOut + (warp - 2) * C_::OUT_WARP;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h * 16 >= ncols) break;  // warp-uniform
              uint8_t* bf = myout + (nchunk & 1) * (C_::OUT_F32 + C_::OUT_BF16);
              ++nchunk;
              if (lane == 0) bulk_wait_read<1>();  // this buffer's store (two chunks ago) has read it
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 4; ++j) {  // row = lane, 64 B, 64-B swizzle
                sts128(bf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4), __float_as_uint(v[h * 16 + 4 * j]),
                       __float_as_uint(v[h * 16 + 4 * j + 1]), __float_as_uint(v[h * 16 + 4 * j + 2]),
                       __float_as_uint(v[h * 16 + 4 * j + 3]));
              }
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&rmaps.m[slab_rank], bf, col0 + h * 16, slab_row);
                bulk_commit();
              }
            }
            continue;
          }
          // each lane stages its own row (144-B stride, conflict-free) and
          // hands it to the bulk-copy engine: one async smem->peer copy per
          // row, no LSU slots held while the NVLink writes drain
          float* mine = st + lane * 36;
          bulk_wait_read<0>();  // this lane's previous copy has read its row
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            sts128(mine + 4 * k, __float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                   __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3]));
          }
          if (rrow) {
            fence_async_smem();
            bulk_s2g(rrow + col0, mine, static_cast<uint32_t>(ncols) * 4u);
            bulk_commit();
          }
          __syncwarp();  // reconverge before the next .sync.aligned tcgen05.ld
          continue;
        }
        if (!rowok) continue;
        const int ncols = nend - col0 < 32 ? nend - col0 : 32;
        if (p.vec && ncols == 32) {
          if (p.epi == kEpiResidual) {
            const float4* r4 = reinterpret_cast<const float4*>(p.res + row * p.ldr + col0);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 t = r4[k];
              v[4 * k] = v[4 * k] + t.x;
              v[4 * k + 1] = v[4 * k + 1] + t.y;
              v[4 * k + 2] = v[4 * k + 2] + t.z;
              v[4 * k + 3] = v[4 * k + 3] + t.w;
            }
          } else if (p.epi == kEpiSilu) {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = v[k] / (1.0f + expf(-v[k]));
          }
          if (p.C || p.routed) {
            float* crow = p.routed ? p.route.base[p.route.rank[row]] + p.route.row[row] * p.route.ld
                                   : p.C + row * p.ldc;
            float4* c4 = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
            for (int k = 0; k < 8; ++k) c4[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          }
          if (p.Cb) {
            uint4* b4 = reinterpret_cast<uint4*>(p.Cb + row * p.ldcb + col0);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) w[e] = pack16x2(v[8 * k + 2 * e], v[8 * k + 2 * e + 1], p.f16);
              b4[k] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        } else {
#pragma unroll 1
          for (int k = 0; k < ncols; ++k) {
            const int col = col0 + k;
            float x = v[0];
#pragma unroll
            for (int e = 1; e < 32; ++e) x = k == e ? v[e] : x;  // v[k] without local-memory indexing
            if (p.epi == kEpiResidual) {
              x = x + p.res[row * p.ldr + col];
            } else if (p.epi == kEpiSilu) {
              x = x / (1.0f + expf(-x));
            }
            if (p.routed) {
              p.route.base[p.route.rank[row]][p.route.row[row] * p.route.ld + col] = x;
            } else if (p.C) {
              p.C[row * p.ldc + col] = x;
            }
            if (p.Cb) p.Cb[row * p.ldcb + col] = to16(x, p.f16);
          }
        }
      }
      if (p.amax && best) atomicMax(p.amax + row, best);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) {
          mbar_arrive_cluster(tempty_leader0 + acc * static_cast<uint32_t>(sizeof(uint64_t)));
        } else {
          mbar_arrive(&tempty[acc]);
        }
      }
    }
  }

  tc_fence_before();
  if (p.routed) bulk_wait_all();  // this thread's row copies / tensor stores have landed
  __syncthreads();
  if (p.routed && threadIdx.x == 0) {
    // one system-scope fence per CTA: cumulative over the CTA's routed
    // stores, which the barrier ordered before it; then the last CTA
    // publishes this exchange's epoch to every destination
    __threadfence_system();
    if (atomicAdd(p.route.done, 1) == static_cast<int>(gridDim.x) - 1) {
      __threadfence_system();
      for (int d = 0; d < 8; ++d) {
        if (p.route.notify >> d & 1) {
          asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p.route.flag[d] + p.route.slot * 8 + p.route.self),
                       "l"(p.route.epoch)
                       : "memory");
        }
      }
      *p.route.done = 0;
    }
  }
  if (cs > 1) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C_::TMEM_COLS));
    } else {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C_::TMEM_COLS));
    }
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

CUtensorMap encode_map(const void* base, int rows, int cols, int64_t ld, int kind, int box_rows, int swb);

// Tensor maps only encode (address, extents, strides, box), so they are
// cached: the weights' maps never change and the activations' maps repeat
// every layer and step.
CUtensorMap make_map(const void* base, int rows, int cols, int64_t ld, int kind, int box_rows, int swb = 128) {
  struct Key {
    const void* b;
    int r, c, k, box, sw;
    int64_t ld;
    bool operator==(const Key& o) const {
      return b == o.b && r == o.r && c == o.c && k == o.k && box == o.box && sw == o.sw && ld == o.ld;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      size_t h = std::hash<const void*>()(k.b);
      for (int64_t v : {static_cast<int64_t>(k.r), static_cast<int64_t>(k.c), static_cast<int64_t>(k.k),
                        static_cast<int64_t>(k.box), static_cast<int64_t>(k.sw), k.ld}) {
        h = h * 1000003u ^ std::hash<int64_t>()(v);
      }
      return h;
    }
  };
  static std::unordered_map<Key, CUtensorMap, Hash> cache;
  static std::mutex mu;
  const Key key{base, rows, cols, kind, box_rows, swb, ld};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 4096) cache.clear();
  const CUtensorMap m = encode_map(base, rows, cols, ld, kind, box_rows, swb);
  cache.emplace(key, m);
  return m;
}

CUtensorMap encode_map(const void* base, int rows, int cols, int64_t ld, int kind, int box_rows, int swb) {
  CUtensorMap m;
  const int es = kind == 2 ? 4 : 2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * es};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(swb / es), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw =
      swb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (swb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  const CUtensorMapDataType dt = kind == 2   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : kind == 3 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const CUresult r = get_encode()(&m, dt, 2,
                                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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

// Tile choice (measured at decode batches): the S-Part
// GEMMs at M = 512 are neither L2- nor HBM-bandwidth-bound; within a tile the
// operand loads are latency-bound (bytes in flight per SM / load latency: one
// more stage of the same smem is -14% on the bn = 112 GEMMs), and across
// tiles the cost is quantized into waves of CTA pairs. So when M spans at
// least two 128-row blocks, a CTA pair (cta_group::2, 256 x bn tiles) is used
// with the tile width bn (a multiple of 16, 64..256) that minimizes
// waves x (bn + fixed per-tile cost); e.g. N = 14336 -> bn 208 (138 tiles on
// 74 pairs) instead of 256 (112 tiles = 1.5 waves).
int pick_pair_bn(int mgroups, int N, int pairs) {
  int best = 256;
  long best_cost = -1;
  for (int bn = 256; bn >= 64; bn -= 16) {
    const long items = static_cast<long>(mgroups) * ((N + bn - 1) / bn);
    const long waves = (items + pairs - 1) / pairs;
    const long cost = waves * (bn + 32);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

template <int BN, bool PAIR, int ATOMS, int KIND>
void launch(const GemmArgs& g, int cs, int bn, cudaStream_t s) {
  using C_ = Cfg<BN, PAIR, ATOMS>;
  auto* kern = gemm_kernel<BN, PAIR, ATOMS, KIND>;
  static std::once_flag attrs;  // one per instantiation: the attributes are set at its first launch
  std::call_once(attrs, [&] {
    SD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C_::SMEM)));
    SD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  if (PAIR) cs = 2;
  if (!PAIR) bn = BN;
  if (bn < 16 || bn > BN || (PAIR && bn % 16)) fail(SD_ERR_CONFIG, "gemm: bad tile width");
  const int f16 = g.kind == 3 ? 1 : 0;
  const CUtensorMap ta = make_map(g.A, g.M, g.K, g.lda, g.kind, BM);
  // output tensor maps (16-column boxes: fp32 rows 64 B, 16-bit rows 32 B)
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool tma_out = (g.C || g.Cb) && (!g.C || (al16(g.C) && g.ldc % 4 == 0)) &&
                       (!g.Cb || (al16(g.Cb) && g.ldcb % 8 == 0));
  const CUtensorMap tc = tma_out && g.C ? make_map(g.C, g.M, g.N, g.ldc, 2, 32, 64) : ta;
  const CUtensorMap tcb = tma_out && g.Cb ? make_map(g.Cb, g.M, g.N, g.ldcb, f16 ? 3 : 1, 32, 32) : ta;
  const CUtensorMap tb = make_map(g.B, g.N, g.K, g.ldb, g.kind, PAIR ? bn / 2 : BN / cs);
  Params p{};
  RouteMaps rmaps{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.mb = (g.M + BM - 1) / BM;
  p.nb = (g.N + bn - 1) / bn;
  const int kstage = ATOMS * (BK_BYTES / (KIND == 2 ? 4 : 2));
  p.kb = (g.K + kstage - 1) / kstage;  // a partial last stage reads zero-filled columns
  p.cs = cs;
  p.C = g.C;
  p.ldc = g.ldc;
  p.Cb = reinterpret_cast<uint16_t*>(g.Cb);
  p.ldcb = g.ldcb;
  p.epi = g.epi;
  p.res = g.res;
  p.ldr = g.ldr;
  p.kind = KIND;
  p.f16 = f16;
  p.bn = bn;
  p.tma_out = tma_out && !g.route ? 1 : 0;  // routed rows use the smem-staged row stores
  if (g.route) {
    p.routed = 1;
    p.route_tma = g.route->rows > 0 ? 1 : 0;
    p.route = *g.route;
    for (int d = 0; d < 8 && p.route_tma; ++d) {
      if (g.route->base[d]) {
        if (!al16(g.route->base[d])) fail(SD_ERR_CONFIG, "routed GEMM: destination buffers must be 16-B aligned");
        rmaps.m[d] = make_map(g.route->base[d], g.route->rows, g.N, g.route->ld, 2, 32, 64);
      }
    }
    if (g.N % 32 || g.route->ld % 4) fail(SD_ERR_CONFIG, "routed GEMM: N and the row stride must be multiples of 32 / 4");
    if (g.C || g.Cb || g.epi != kEpiNone) fail(SD_ERR_CONFIG, "routed GEMM: plain fp32 rows only");
  }
  p.amax = g.amax;
  if (g.kvapp) {
    if (!p.tma_out || g.kvapp->col_k % 16 || g.kvapp->width % 16 || (g.kvapp->pos_bytes % 16)) {
      fail(SD_ERR_INTERNAL, "fused append: needs the TMA-store epilogue and 16-column-aligned K/V");
    }
    p.kvapp = 1;
    p.kva = *g.kvapp;
  }
  if (g.amax && (g.route || g.C || g.Cb)) fail(SD_ERR_CONFIG, "fused-argmax GEMM: no other output");
  p.vec = (!g.C || (g.ldc % 4 == 0 && al16(g.C))) && (!g.Cb || (g.ldcb % 8 == 0 && al16(g.Cb))) &&
          (g.epi != kEpiResidual || (g.ldr % 4 == 0 && al16(g.res)));
  // instruction descriptor: A/B format (kind::f16: 0 F16, 1 BF16; kind::tf32: 2), fp32 D, N >> 3, M >> 4
  const uint32_t fmt = KIND == 2 ? 2u : (f16 ? 0u : 1u);
  p.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(bn >> 3) << 17) |
            (static_cast<uint32_t>((PAIR ? 2 * BM : BM) >> 4) << 24);
  const int items = (PAIR ? (p.mb + 1) / 2 : p.mb / cs) * p.nb;
  const int budget = g.max_ctas > 0 && g.max_ctas < num_sms() ? g.max_ctas : num_sms();
  const int max_clusters = budget / cs > 0 ? budget / cs : 1;
  const int clusters = items < max_clusters ? items : max_clusters;
  SD_CUDA(launch_pdl(kern, dim3(static_cast<unsigned>(clusters * cs)), dim3(kThreads), C_::SMEM, s,
                     static_cast<unsigned>(cs), ta, tb, tc, tcb, p, rmaps));
  count_launch();
}

template <int KIND>
void dispatch(const GemmArgs& g, cudaStream_t s) {
  const Tuning& t = tuning();
  const int mb = (g.M + BM - 1) / BM;
  const int sms = g.max_ctas > 0 && g.max_ctas < num_sms() ? g.max_ctas : num_sms();
  if (t.gemm_pair && mb >= 2 && sms >= 2) {
    int bn = pick_pair_bn((mb + 1) / 2, g.N, sms / 2);
    if (t.gemm_bn >= 64 && t.gemm_bn <= 256 && t.gemm_bn % 16 == 0) bn = t.gemm_bn;
    // The stage ring is sized for the widest tile of the instantiation, so
    // the tile width picks the instantiation: one swizzle atom per stage and
    // a B stage no wider than needed gives the most stages in the same smem
    // (bn <= 128: 8, <= 192: 7, else 6; the loads are latency-bound, so more,
    // smaller stages keep more of them in flight). Measured at M = 512 with
    // the weights streamed from HBM: QKV 25.1 -> 22.5 us, MLP-in 50.5 -> 48.2,
    // MLP-out 58.8 -> 50.1, W_o 20.8 -> 18.2 against two-atom stages of the
    // 256-wide instantiation (3 stages).
    if (bn <= 128) {
      launch<128, true, 1, KIND>(g, 2, bn, s);
    } else if (bn <= 192) {
      launch<192, true, 1, KIND>(g, 2, bn, s);
    } else {
      launch<256, true, 1, KIND>(g, 2, bn, s);
    }
    return;
  }
  // one 128-row block (or an SM budget of one): single-CTA tiles, B
  // multicast over a cluster of M blocks when that fills the machine
  const int tiles256 = mb * ((g.N + 255) / 256);
  const int bn = tiles256 * 2 <= sms ? 128 : 256;
  const int cs = (bn == 256 && mb % 2 == 0) ? 2 : 1;
  if (bn == 128) {
    launch<128, false, 2, KIND>(g, cs, 128, s);
  } else {
    launch<256, false, 1, KIND>(g, cs, 256, s);
  }
}

}  // namespace

bool gemm_sm100_supported(const GemmArgs& g) {
  const int es = g.kind == 2 ? 4 : 2;
  if (g.kind < 1 || g.kind > 3) return false;
  if (g.M < 1 || g.N < 1 || g.K < 1) return false;
  if ((g.lda * es) % 16 || (g.ldb * es) % 16) return false;
  if (reinterpret_cast<uintptr_t>(g.A) % 16 || reinterpret_cast<uintptr_t>(g.B) % 16) return false;
  if (g.K % (BK_BYTES / es) != 0) return false;  // whole 128-B atoms
  return true;
}

void launch_gemm_sm100(const GemmArgs& g, cudaStream_t s) {
  if (g.kind == 2) {
    dispatch<2>(g, s);
  } else {
    dispatch<1>(g, s);  // bf16 and fp16 operands: kind::f16
  }
}

}  // namespace sd
