// K2 for grouped-query attention over fp16, int8 or int4 KV (BASELINE
// config 5): the G query heads that share a kv head make the R-Part a thin
// GEMM, so the dot products and the value sum run on tensor cores
// (mma.sync m16n8k16, fp32 accumulate; int8 / int4 scores on m16n8k32
// IMMA, see IM below) instead of CUDA-core FMAs.
//
//   S^T[pos][q] = K[pos][:] . Q^T[:][q]     M = 16 positions, N = 8 (G <= 8 heads), K = hd
//   O^T[d][q]  += V^T[d][pos] . P^T[pos][q]  M = 16 head-dims,  N = 8 heads,         K = 16 pos
//
// K rows are the A operand (ldmatrix), V rows the transposed A operand
// (ldmatrix.trans); Q^T is a register-resident B operand; P^T is built from
// the S^T accumulators with movmatrix.trans. fp16 K/V are exact tensor-core
// operands; q and p are split into fp16 hi + lo parts, so the products carry
// ~22 significant bits — fp32-level agreement with the reference's fp32
// attend (attention.cpp:204-282), not fp16 rounding. With G <= 4 query heads
// per kv head the hi and lo parts share one MMA: hi in N columns [0, G), lo
// in [G, 2G) (an m16n8 tile has 8 columns), summed by one lane shuffle — half
// the MMAs of issuing them separately.
//
// Work split, TMA bulk-copy producer, mbarrier ring and piece/partial
// protocol are those of attn_kernel (kv_kernels.cu); stages hold 16
// positions copied four per bulk copy (int8: two with attn_i8_quad = 0; fp16
// shards of 1-2 kv heads: eight) — the per-SM copy issue rate, not bytes,
// limits row-sized copies — into slots with a 16-B pad;
// MMA row r holds position (r % NS) * RPS + r / NS (NS slots of RPS rows).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "kv_kernels.cuh"
#include "pdl.cuh"
#include "sd_common.h"

namespace sd {

namespace {

// consumer warps per CTA: one per kv head (two per head for int8 KV as
// position classes measured slower: 0.517 vs 0.498 ms per C5 layer)
template <int FMT>
constexpr int consumer_warps() { return 8; }
constexpr int kT = 16;                    // positions per stage
constexpr int kHD = 128;

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
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
// D (+)= A . B, m16n8k16, fp16 in, fp32 accumulate
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo_col, float hi_col) {
  __half2 h = __floats2half2_rn(lo_col, hi_col);
  return *reinterpret_cast<uint32_t*>(&h);
}
// split (x0, x1) into fp16 hi pair + fp16 lo pair (residuals)
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_h2(x0 - hf.x, x1 - hf.y);
}

// four int8 (one 32-bit word, stored q + 128) -> two fp16 pairs holding the
// exact integers: byte u becomes fp16 1024 + u (0x64xx), minus 1152. (Folding the
// 1152 bias out of the MMAs instead — subtracting 1152 x the other operand's
// column sums from the accumulators — saves the HSUB2s but costs ~7 bits of
// the fp32 accumulation at context 2048: 1.3e-4 error, measured; kept out.)
__device__ __forceinline__ uint32_t i8x2_to_h2(uint32_t u, uint32_t sel) {
  const uint32_t biased = __byte_perm(u, 0x64646464u, sel);
  __half2 h = *reinterpret_cast<const __half2*>(&biased);
  h = __hsub2(h, __floats2half2_rn(1152.0f, 1152.0f));
  return *reinterpret_cast<const uint32_t*>(&h);
}
// eight int4 (one word, element 2i in the low nibble, each stored q + 8)
// -> four fp16 pairs holding the exact integers
// q: h[0] = (q0, q4), h[1] = (q1, q5), h[2] = (q2, q6), h[3] = (q3, q7).
// A nibble or'ed under 0x6400 is fp16 1024 + n (low nibble of a half) or
// 1024 + 16 n (high nibble): one LOP3 each, then a subtract or an FMA.
__device__ __forceinline__ void i4x8_to_h2(uint32_t u, uint32_t (&h)[4]) {
  const uint32_t t = u >> 8;
  const uint32_t r[4] = {(u & 0x000F000Fu) | 0x64006400u, (u & 0x00F000F0u) | 0x64006400u,
                         (t & 0x000F000Fu) | 0x64006400u, (t & 0x00F000F0u) | 0x64006400u};
  const __half2 b_lo = __floats2half2_rn(1032.0f, 1032.0f), m_hi = __floats2half2_rn(0.0625f, 0.0625f),
                b_hi = __floats2half2_rn(-72.0f, -72.0f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 x = *reinterpret_cast<const __half2*>(&r[i]);
    const __half2 y = (i & 1) ? __hfma2(x, m_hi, b_hi) : __hsub2(x, b_lo);
    h[i] = *reinterpret_cast<const uint32_t*>(&y);
  }
}
// D (+)= A . B, m16n8k32, A unsigned bytes (offset-binary K codes), B signed
// bytes (a q limb), exact int32 accumulate
__device__ __forceinline__ void imma16832(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// D (+)= A . B, m16n8k16, both unsigned bytes (V codes, p limbs), exact int32 accumulate
__device__ __forceinline__ void imma16816u(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(b));
}
// 16 x 16 byte tile, transposed (sm_100a): lane l receives, for matrix
// columns c = l / 4 and c + 8, the bytes of rows 4 (l % 4) .. 4 (l % 4) + 3 —
// the A fragment of an m16n8k16 byte MMA whose rows are the tile's columns;
// lanes 0-15 give the row addresses (layout probed on the B200)
__device__ __forceinline__ void ldsm_b8_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
// the low byte of x as a signed value
__device__ __forceinline__ int sbyte(int x) { return static_cast<int>(static_cast<int8_t>(x & 0xFF)); }
constexpr int kVPitch = kHD * 2 + 16;
// int8: per-warp scratch = the dequantized V tile, reused at the end of a
// piece as the warp's softmax-state merge slot (32 lanes x 36 floats)
constexpr int kScratch = kT * kVPitch + 256;
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}  // bytes per row of a warp's dequantized V tile

// IM (quantized KV only): the scores on integer tensor cores. K codes are
// exact unsigned bytes (int4: nibbles unpacked to bytes with two LOP3s) and
// q is carried as a 22-bit fixed-point integer per head (scale 2^(22-E),
// E = exponent of the head's max |q|) split into three signed byte limbs:
// three m16n8k32 IMMAs per 32 head dims give the exact int32 dot of each
// limb, the codes' offset (128 / 8 x the limb's column sum) preloaded into
// the accumulators; the limbs recombine in fp32. No per-element conversion
// of K at all, where the fp16 path spends a byte permute and a subtract per
// two values.
//
// IV (int8 / int4 KV, G <= 4): the value product on integer tensor cores
// too. V^T comes straight from the ring as the A operand of u8 x u8 m16n8k16
// IMMAs (transposed byte ldmatrix, no dequantized scratch tile; int4: one AND
// / shift-AND per word splits a byte column into its two head dims); P^T is carried as
// a 23-bit fixed-point integer W = p * vscale * 2^22 / Sb in three byte limbs
// (3G <= 12 B columns: limb-major, 8 per tile). The int32 accumulators live
// across stages: p is taken against a reference max mref that moves only
// when a stage's max passes mref + 1 (so p <= 2), and Sb bounds the warp's V
// scales, so the integers are converted into the fp32 O (offset 128 x the
// limb column sums removed exactly in int32, limbs recombined, rescaled to the
// new mref) only when mref or Sb moves or before 2000 stages could overflow.
// Resolution 2^-22 of Sb per term: ~1e-6 of max|v| against the 2e-5 bar.
template <int G, int FMT, int RPS, bool IM = false, bool IV = false>
__global__ void __launch_bounds__((consumer_warps<FMT>() + 1) * 32, 1) attn_mma_kernel(const AttnArgs a) {
  constexpr bool I8 = FMT == SD_KV_INT8;
  constexpr bool I4 = FMT == SD_KV_INT4;
  constexpr bool QNT = I8 || I4;  // quantized: scales in the stage, V dequantized into scratch
  static_assert(!IM || QNT, "integer scores need quantized KV");
  static_assert(!IV || (QNT && 2 * G <= 8), "integer value product: quantized KV, G <= 4");
  constexpr int kWarps = consumer_warps<FMT>();
  constexpr int kThreads = (kWarps + 1) * 32;
  static_assert(RPS == 2 || RPS == 4 || RPS == 8, "pair, quad or octet slots");
  // hi / lo parts of q and p packed into the N columns of one MMA
  constexpr bool PACK = 2 * G <= 8;
  constexpr int XG = G / 2;  // lane xor between a column's hi and lo holders
  constexpr int NS = kT / RPS;  // slots per K (V) half of a stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int nst = a.nstages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + nst;
  uint8_t* ring = smem + 128 * ((16 * nst + 127) / 128);
  // stage region: kT/2 pair slots of two position rows + a 16-B pad; MMA row m
  // holds position 2m (m < 8) or 2(m-8)+1, i.e. slot m & 7, row m >> 3
  const int ppitch = RPS * a.g.pos_bytes + 16;
  // int8: [K rows][V rows][K scales kT x hc][V scales kT x hc]
  const size_t stage_bytes = static_cast<size_t>(2) * a.stage_region + (QNT ? 2 * a.sc_region : 0);
  const KvGeom& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], g.hc);  // the hc warps of the stage's position class (nst % P == 0: one class per slot)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // rows past a stage's valid count are read (and masked): keep them finite
  for (size_t i = threadIdx.x * 16; i < stage_bytes * nst; i += kThreads * 16) {
    *reinterpret_cast<uint4*>(ring + i) = make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  pdl_trigger();
  __syncthreads();
  // The plan (host-uploaded: a copy in the stream orders before this launch)
  // and the KV of every position but the one this step appends are inputs
  // no kernel still running can change, so the producer streams the first
  // stages before the wait on the previous kernel (the QKV GEMM that writes
  // q and the new position); the consumers wait first.
  if (warp != kWarps) pdl_wait();

  const int cb = a.cta_begin[blockIdx.x], ce = a.cta_begin[blockIdx.x + 1];
  const uint8_t* layer_base = g.pool + static_cast<int64_t>(a.layer) * g.layer_bytes;
  // softmax-state merge slots (P > 1): after the ring (fp16), in the V
  // scratch of each warp (int8)
  uint8_t* scr = ring + nst * stage_bytes;
  auto merge_slot = [&](int wp) {
    return QNT ? reinterpret_cast<float*>(scr + wp * kScratch) + lane * 36
              : reinterpret_cast<float*>(scr) + (wp * 32 + lane) * 36;
  };

  if (warp == kWarps) {
    // producer warp: lane 0 arms the stage barrier, then lanes 0-15 copy the
    // K rows and lanes 16-31 the V rows of the stage in parallel (per-lane
    // issue measured faster than one elected lane issuing all 32 copies)
    const uint64_t pol = evict_first_policy();
    int stage = 0;
    uint32_t phase = 0;
    bool waited = false;
    for (int w = cb; w < ce; ++w) {
      const Piece pc = a.pieces[w];
      const int32_t* pt = g.page_table + static_cast<int64_t>(a.item_slot[pc.item]) * g.max_pages;
      // the page of the next stage is loaded one stage ahead, so its latency
      // overlaps the wait for a free slot (small shards: ~1,000 cycles per stage
      // of producer latency otherwise)
      int32_t pg_next = pc.p0 < pc.p1 ? pt[pc.p0 >> g.log2P] : 0;
      for (int pos = pc.p0; pos < pc.p1; pos += kT) {
        // a stage ending before the piece's last position cannot hold the
        // position being appended (the item's last) nor a page opened for it
        if (!waited && pos + kT >= pc.p1) {
          pdl_wait();
          waited = true;
          pg_next = pt[pos >> g.log2P];  // (re-read after the wait: the appended position's page)
        }
        const int32_t pg = pg_next;
        if (pos + kT < pc.p1) pg_next = pt[(pos + kT) >> g.log2P];
        const int cnt = min(kT, pc.p1 - pos);
        const uint8_t* base = layer_base + static_cast<int64_t>(pg) * g.group_bytes +
                              static_cast<int64_t>(pos & (g.P - 1)) * g.pos_bytes;
        // scale block rounded up to the bulk-copy granule (16 B): stages start
        // 16-aligned in a page group, so the extra scales stay inside its region
        const uint32_t scb = QNT ? (static_cast<uint32_t>(cnt * g.hc * 4) + 15u) & ~15u : 0u;
        if (lane == 0) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], 2u * cnt * g.pos_bytes + 2u * scb);
        }
        __syncwarp();
        {
          // two consecutive positions per copy (the per-SM bulk-copy issue
          // rate, not bytes, limits row-sized copies); each pair slot carries
          // a 16-B pad so the ldmatrix / 32-bit fragment rows are conflict-free
          const int pr = lane & 15;
          if (pr < NS && RPS * pr < cnt) {
            uint8_t* dst = ring + stage * stage_bytes + (lane >= 16 ? a.stage_region : 0) + pr * ppitch;
            const uint32_t nb = static_cast<uint32_t>(min(RPS, cnt - RPS * pr)) * g.pos_bytes;
            bulk_g2s(dst, base + (lane >= 16 ? g.v_off : 0) + RPS * pr * g.pos_bytes, nb, &full[stage], pol);
          }
        }
        if (QNT && (lane == 0 || lane == 16)) {  // the stage's scales (one page group: contiguous)
          const uint8_t* lb = layer_base + static_cast<int64_t>(pg) * g.group_bytes;
          const int off = pos & (g.P - 1);
          uint8_t* dst = ring + stage * stage_bytes + 2 * a.stage_region + (lane ? a.sc_region : 0);
          bulk_g2s(dst, lb + (lane ? g.vs_off : g.ks_off) + off * g.hc * 4, scb, &full[stage], pol);
        }
        if (++stage == nst) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    // the next GEMM's weights into L2 while the consumers drain the last
    // stages (this CTA's slice, in 32-KB requests over the lanes): W_o then
    // reads its B operand from L2 instead of streaming it at the ring's
    // bytes-in-flight limit
    if (a.l2pf_bytes > 0) {
      const int64_t per = ((a.l2pf_bytes + gridDim.x - 1) / gridDim.x + 15) & ~int64_t{15};
      const int64_t b0 = per * blockIdx.x, b1 = min(a.l2pf_bytes, b0 + per);
      for (int64_t o = b0 + static_cast<int64_t>(lane) * 32768; o < b1; o += 32 * 32768) {
        const int64_t left = b1 - o;
        const uint32_t n = static_cast<uint32_t>(left < 32768 ? left : 32768);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.l2pf + o), "r"(n) : "memory");
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumer
  // warp = (kv head, position class): with hc < 8 kv heads per shard the
  // P = 8/hc warps of a head take every P-th stage and merge their softmax
  // states at the end of a piece. fragment coordinates: gq = lane/4, tq = lane%4
  const int P = kWarps / g.hc;
  const int hk = warp % g.hc, cls = warp / g.hc;
  int jst = 0;  // stage sequence number (same order as the producer)
  const int gq = lane >> 2, tq = lane & 3;
  const bool lo_role = PACK && (tq & XG) != 0;  // this lane's columns carry lo parts
  const int Hq = g.hc * G;
  float o[8][4];      // O^T fragments: hd rows 16*mt + {gq, gq+8}, heads {2tq, 2tq+1}
  float m[2], l[2];   // per head 2tq, 2tq+1 (replicated over gq lanes; l partial per lane)
  uint32_t qb[8][2][2];  // Q^T B-fragments: [k-step][b0|b1][hi|lo]
  // IM: q limbs as B fragments [limb][k32-step][b0|b1]; per output column
  // (heads 2tq', 2tq'+1) the accumulator preload and the fixed-point scale
  uint32_t ql[3][4][2];
  int qinit[3][2];
  float qdown[2];
  int stage = 0;
  uint32_t phase = 0;
  // ldmatrix lane address components
  const int lm = lane >> 3, lr = lane & 7;
  // IV: int32 O^T accumulators [B tile][hd tile] (B column c = limb * G + head),
  // per-lane partial column sums of the B fragments, the V scale bound Sb and
  // the fixed-point factor 2^22 / Sb, stages accumulated since the last flush
  constexpr int NT = IV ? (3 * G + 7) / 8 : 1;
  int vacc[NT][8][4];
  uint32_t vcs[NT];
  float sb = 1.0f, fs = 4194288.0f;
  int nacc = 0;
  // this lane's B column gq in tile k holds limb (8k + gq) / G of head gq % G;
  // row 4tq + i of the fragment is MMA row sigma(4tq + i) = 2tq + {0, 1, 8, 9}
  // IM int8: ldmatrix x4 row addresses of the K tile (lanes 0-15: MMA rows
  // 0-15 at k bytes 0-15 of a k-step, lanes 16-31: the same rows at 16-31)
  // (int4: 16-B chunks 2j and 2j + 1 of a row, two k32-steps per LDSM)
  const uint32_t klsm_off = hk * (I4 ? kHD / 2 : kHD) + ((lane & 15) % NS) * ppitch + ((lane & 15) / NS) * g.pos_bytes +
                            (lane >> 4) * 16;
  uint32_t vrow_addr_off = 0;
  if constexpr (IV) {
    const int i = lane & 15;
    const int srow = (i >> 2) * 2 + ((i & 3) < 2 ? (i & 3) : 6 + (i & 3));
    vrow_addr_off = (srow % NS) * ppitch + (srow / NS) * g.pos_bytes;
  }
  // IV: the fp32 O^T lives in the warp's scratch ([element][lane], conflict
  // free) while the int32 sums hold the registers; it is only touched by the
  // (rare) flushes and read back into o at the end of a piece
  auto ivo = [&]() { return reinterpret_cast<float*>(scr + warp * kScratch) + lane; };
  // IV flush: int32 accumulators -> fp32 O (o = (o + W-sum * Sb / 2^22) * c),
  // then cleared. Lanes tq < XG own heads 2tq, 2tq + 1; the other lanes keep 0
  // so the PACK finalize adds nothing from them.
  auto iv_flush = [&](float c0, float c1) {
    if constexpr (IV) {
      int cs[NT][2];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        uint32_t t = vcs[k] + __shfl_xor_sync(0xffffffffu, vcs[k], 1);
        t += __shfl_xor_sync(0xffffffffu, t, 2);  // lanes 4c..4c+3: column c's sum
        cs[k][0] = static_cast<int>(__shfl_sync(0xffffffffu, t, 4 * (2 * tq)));
        cs[k][1] = static_cast<int>(__shfl_sync(0xffffffffu, t, 4 * (2 * tq + 1)));
        vcs[k] = 0u;
      }
      const float kf = sb * (1.0f / 4194288.0f);
      const bool own = tq < XG;
      float* os = ivo();
      const int sl1 = (lane & ~3) | (((G % 8) / 2) + (tq & (XG - 1)));        // limb 1's holder
      const int sl2 = (lane & ~3) | (((2 * G) % 8) / 2 + (tq & (XG - 1)));  // limb 2's holder
      constexpr int T1 = G / 8, T2 = (2 * G) / 8;                           // their tiles
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int d[NT];
#pragma unroll
          for (int k = 0; k < NT; ++k) {
            d[k] = vacc[k][mt][e] - (I8 ? 128 : 8) * cs[k][e & 1];  // exact: the codes are q + 128 (q + 8)
            vacc[k][mt][e] = 0;
          }
          const int d1 = __shfl_sync(0xffffffffu, d[T1], sl1), d2 = __shfl_sync(0xffffffffu, d[T2], sl2);
          const float v = fmaf(static_cast<float>(d2), 65536.0f, fmaf(static_cast<float>(d1), 256.0f, static_cast<float>(d[0])));
          float& x = os[(4 * mt + e) * 32];
          x = own ? (x + v * kf) * ((e & 1) ? c1 : c0) : 0.0f;
        }
      nacc = 0;
    }
  };

  for (int w = cb; w < ce; ++w) {
    const Piece pc = a.pieces[w];
    if constexpr (IM) {
      // B column gq = head gq (< G); k slot i of step s, half h is head dim
      // 32s + 16h + 4tq + i (int8: a lane's 4 K bytes) or 32s + 8tq + 2i + h
      // (int4: low / high nibbles of a lane's K word). PACK (G <= 4): limbs 0
      // and 1 share one MMA (columns [0, G) and [G, 2G)), limb 2 takes a
      // second: two IMMAs per k-step instead of three
      const float* qrow = a.q + static_cast<int64_t>(pc.item) * a.q_stride + static_cast<int64_t>(hk) * G * kHD;
      const bool colv = gq < (PACK ? 2 * G : G);
      const int hcol = PACK && gq >= G ? gq - G : gq;
      float xv[4][2][4];
      float mx = 0.0f;
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int d = I8 ? 32 * s + 16 * h + 4 * tq + i : 32 * s + 8 * tq + 2 * i + h;
            xv[s][h][i] = colv ? qrow[hcol * kHD + d] * a.qscale : 0.0f;
            mx = fmaxf(mx, fabsf(xv[s][h][i]));
          }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      int E = 0;
      if (mx > 0.0f) frexpf(mx, &E);  // mx < 2^E
      E = max(E, -100);               // keeps 2^(22-E) finite for subnormal-sized heads
      const float up = ldexpf(1.0f, 22 - E), down = ldexpf(1.0f, E - 22);
      int cs[3] = {0, 0, 0};
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t pk[3] = {0u, 0u, 0u};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            // |n| < 2^22: balanced base-256 digits n = l0 * 2^16 + l1 * 2^8 + l2
            const int n = __float2int_rn(xv[s][h][i] * up);
            const int l2 = sbyte(n), r = (n - l2) >> 8;
            const int l1 = sbyte(r), l0 = (r - l1) >> 8;
            cs[0] += l0;
            cs[1] += l1;
            cs[2] += l2;
            pk[0] |= static_cast<uint32_t>(l0 & 0xFF) << (8 * i);
            pk[1] |= static_cast<uint32_t>(l1 & 0xFF) << (8 * i);
            pk[2] |= static_cast<uint32_t>(l2 & 0xFF) << (8 * i);
          }
          if constexpr (PACK) {
            ql[0][s][h] = gq < G ? pk[0] : pk[1];  // (columns >= 2G: zero q, zero limbs)
            ql[1][s][h] = gq < G ? pk[2] : 0u;
          } else {
#pragma unroll
            for (int t = 0; t < 3; ++t) ql[t][s][h] = pk[t];
          }
        }
      const int bias = I8 ? 128 : 8;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 1);
        cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], 2);
      }
      if constexpr (PACK) {
        const int ca = gq < G ? cs[0] : cs[1], cb2 = gq < G ? cs[2] : 0;
        cs[0] = ca;
        cs[1] = cb2;
      }
#pragma unroll
      for (int t = 0; t < 3; ++t) {
#pragma unroll
        for (int j = 0; j < 2; ++j) qinit[t][j] = -bias * __shfl_sync(0xffffffffu, cs[t], 4 * ((2 * tq + j) & 7));
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) qdown[j] = __shfl_sync(0xffffffffu, down, 4 * ((2 * tq + j) & 7));
    } else {
      const float* qrow = a.q + static_cast<int64_t>(pc.item) * a.q_stride + static_cast<int64_t>(hk) * G * kHD;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float2 x = make_float2(0.0f, 0.0f);
          // int8 K fragments take 4 contiguous d per lane (a permutation of
          // the dot's k index); Q^T uses the same permutation
          // int4: a word of 8 nibbles feeds k-steps 2j, 2j+1 as pairs (d, d + 4)
          const int d = I8   ? 16 * kk + 4 * tq + 2 * h
                        : I4 ? 32 * (kk >> 1) + 8 * tq + 2 * (kk & 1) + h
                             : 16 * kk + 8 * h + 2 * tq;
          const int hq = PACK && gq >= G ? gq - G : gq;  // PACK: column gq >= G is head gq - G's lo part
          if (hq < G && gq < (PACK ? 2 * G : G)) {
            x = I4 ? make_float2(qrow[hq * kHD + d], qrow[hq * kHD + d + 4])
                   : *reinterpret_cast<const float2*>(qrow + hq * kHD + d);
          }
          split2(x.x * a.qscale, x.y * a.qscale, qb[kk][h][0], qb[kk][h][1]);
          if (PACK && gq >= G) qb[kk][h][0] = qb[kk][h][1];  // the MMA's B column gets the lo part
        }
      }
    }
    if constexpr (!IV) {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[mt][i] = 0.0f;
    }
    m[0] = m[1] = -INFINITY;
    l[0] = l[1] = 0.0f;
    if constexpr (IV) {
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        vcs[k] = 0u;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int i = 0; i < 4; ++i) vacc[k][mt][i] = 0;
      }
      nacc = 0;
      float* os = ivo();
#pragma unroll
      for (int i = 0; i < 32; ++i) os[32 * i] = 0.0f;
    }

    for (int pos = pc.p0; pos < pc.p1; pos += kT, ++jst) {
      if (P > 1 && jst % P != cls) {  // another class's stage (warp-uniform)
        if (++stage == nst) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      const int cnt = min(kT, pc.p1 - pos);
      mbar_wait(&full[stage], phase);
      __syncwarp();
      const uint8_t* st8 = ring + stage * stage_bytes;
      const uint32_t Ks = smem_u32(st8) + hk * kHD * (I8 ? 1 : 2);
      uint32_t Vs = Ks + a.stage_region;
      int vpitch = 0;  // 0: fp16 rows in the ring's pair slots; else the int8 scratch pitch
      float vs0 = 1.0f, vs1 = 1.0f;  // int8: the V scales of MMA rows gq, gq + 8
      // ---- S^T = K . Q^T  (16 positions x 8 heads), hi + lo parts of q; two
      // accumulator chains (even / odd k-steps) halve the dependent HMMA depth
      float s[4] = {0.0f, 0.0f, 0.0f, 0.0f}, s2[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      if constexpr (IM) {
        int dacc[3][4];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          dacc[t][0] = dacc[t][2] = qinit[t][0];
          dacc[t][1] = dacc[t][3] = qinit[t][1];
        }
        uint32_t kw4[4];  // int4: rows gq, gq + 8 of two 16-B chunks
#pragma unroll
        for (int st = 0; st < 4; ++st) {
          uint32_t ka[4];
          if (I8) {
            // the m16n8k32 byte A fragment is the b16 ldmatrix x4 layout read
            // as bytes: one LDSM per k-step instead of four 32-bit loads
            ldsm_x4(smem_u32(st8) + klsm_off + 32 * st, ka);
          } else {
            if ((st & 1) == 0) ldsm_x4(smem_u32(st8) + klsm_off + 16 * st, kw4);
            const uint32_t w0 = kw4[2 * (st & 1)], w1 = kw4[2 * (st & 1) + 1];
            ka[0] = w0 & 0x0F0F0F0Fu;
            ka[1] = w1 & 0x0F0F0F0Fu;
            ka[2] = (w0 >> 4) & 0x0F0F0F0Fu;
            ka[3] = (w1 >> 4) & 0x0F0F0F0Fu;
          }
#pragma unroll
          for (int t = 0; t < (PACK ? 2 : 3); ++t) imma16832(dacc[t], ka, ql[t][st][0], ql[t][st][1]);
        }
        // per-(position, head) K scales: S = kscale * 2^(E-22) * (q_int . k)
        const float* ksc = reinterpret_cast<const float*>(st8 + 2 * a.stage_region);
        const int pos0 = (gq % NS) * RPS + gq / NS, pos1 = ((gq + 8) % NS) * RPS + (gq + 8) / NS;
        const float k0 = ksc[pos0 * g.hc + hk], k1 = ksc[pos1 * g.hc + hk];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          // PACK: limb 1 of this lane's heads sits XG lanes over (columns + G),
          // limb 2 in the second accumulator (lanes tq >= XG: filled below)
          const int l1 = PACK ? __shfl_xor_sync(0xffffffffu, dacc[0][e], XG) : dacc[1][e];
          const int l2 = PACK ? dacc[1][e] : dacc[2][e];
          const float v = fmaf(static_cast<float>(dacc[0][e]), 65536.0f,
                               fmaf(static_cast<float>(l1), 256.0f, static_cast<float>(l2)));
          s[e] = v * (qdown[e & 1] * (e < 2 ? k0 : k1));
        }
        if (PACK) {  // lanes whose columns are past G take the scores of lane tq & (XG - 1)
#pragma unroll
          for (int e = 0; e < 4; ++e) s[e] = __shfl_sync(0xffffffffu, s[e], (lane & ~3) | (tq & (XG - 1)));
        }
      }
      if (QNT) {
        // MMA row r holds position (r % NS) * RPS + r / NS: rows gq and gq+8
        // of this lane are rows gq / NS and (gq + 8) / NS of slot gq % NS
        // (pair slots: conflict-free, slot pitch = 4 mod 32 words; quad slots:
        // rows gq and gq + 4 share banks, 2-way)
        const uint8_t* kb = st8 + hk * (I4 ? kHD / 2 : kHD) + 4 * tq + (gq % NS) * ppitch + (gq / NS) * g.pos_bytes;
        const int krow8 = ((gq + 8) / NS - gq / NS) * g.pos_bytes;  // row gq + 8, same slot
        if (IM) {
          // scores done above on the integer tensor cores
        } else if (I8) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t w0 = *reinterpret_cast<const uint32_t*>(kb + 16 * kk);
            const uint32_t w1 = *reinterpret_cast<const uint32_t*>(kb + krow8 + 16 * kk);
            const uint32_t ka[4] = {i8x2_to_h2(w0, 0x5140), i8x2_to_h2(w1, 0x5140), i8x2_to_h2(w0, 0x5342),
                                    i8x2_to_h2(w1, 0x5342)};
            float(&acc)[4] = (kk & 1) ? s2 : s;
            mma16816(acc, ka, qb[kk][0][0], qb[kk][1][0]);
            if (!PACK) mma16816(acc, ka, qb[kk][0][1], qb[kk][1][1]);
          }
        } else {
          // one word per row and lane covers two k-steps (32 head dims per
          // word column): pairs (q0, q4), (q1, q5) for the even one,
          // (q2, q6), (q3, q7) for the odd one
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t h0[4], h1[4];
            i4x8_to_h2(*reinterpret_cast<const uint32_t*>(kb + 16 * j), h0);
            i4x8_to_h2(*reinterpret_cast<const uint32_t*>(kb + krow8 + 16 * j), h1);
            const uint32_t ka0[4] = {h0[0], h1[0], h0[1], h1[1]}, ka1[4] = {h0[2], h1[2], h0[3], h1[3]};
            mma16816(s, ka0, qb[2 * j][0][0], qb[2 * j][1][0]);
            if (!PACK) mma16816(s, ka0, qb[2 * j][0][1], qb[2 * j][1][1]);
            mma16816(s2, ka1, qb[2 * j + 1][0][0], qb[2 * j + 1][1][0]);
            if (!PACK) mma16816(s2, ka1, qb[2 * j + 1][0][1], qb[2 * j + 1][1][1]);
          }
        }
        if (!IM) {
#pragma unroll
          for (int i = 0; i < 4; ++i) s[i] += s2[i];
          // per-(position, head) K scales: S = scale * (q . k_int)
          const float* ksc = reinterpret_cast<const float*>(st8 + 2 * a.stage_region);
          const int pos0 = (gq % NS) * RPS + gq / NS, pos1 = ((gq + 8) % NS) * RPS + (gq + 8) / NS;
          const float k0 = ksc[pos0 * g.hc + hk], k1 = ksc[pos1 * g.hc + hk];
          s[0] *= k0;
          s[1] *= k0;
          s[2] *= k1;
          s[3] *= k1;
        }
        // V tile of this head -> exact fp16 integers in the warp's scratch
        // lane l converts word l (4 head dims) of every row: conflict-free
        // 32-bit loads (pitch = 4 mod 32 words) and full-wavefront 64-bit stores
        uint8_t* vscr = scr + warp * kScratch;
        if (IV) {
          // the value product reads the codes from the ring itself
        } else if (I8) {
          const uint8_t* vb = st8 + a.stage_region + hk * kHD + 4 * lane;
          uint8_t* vd = vscr + 8 * lane;
#pragma unroll
          for (int m = 0; m < kT; ++m) {  // scratch row m = MMA row m (position pair mapping)
            const int slot = m % NS, sub = m / NS;
            const uint32_t u = *reinterpret_cast<const uint32_t*>(vb + slot * ppitch + sub * g.pos_bytes);
            *reinterpret_cast<uint2*>(vd + m * kVPitch) = make_uint2(i8x2_to_h2(u, 0x5140), i8x2_to_h2(u, 0x5342));
          }
        } else {
          // int4: a row is 16 words; half-warps take alternate rows, lane
          // converts one word (8 head dims) and stores them in d order
          const uint8_t* vb = st8 + a.stage_region + hk * (kHD / 2) + 4 * (lane & 15);
          uint8_t* vd = vscr + 16 * (lane & 15);
          // loads first: the scratch stores may alias the ring for the
          // compiler, which then keeps each row's load behind the previous
          // row's store (0.454 -> 0.421 ms per C5 layer; for int8 the extra
          // 16 registers cost more than the overlap gains)
          uint32_t u[kT / 2];
#pragma unroll
          for (int i = 0; i < kT / 2; ++i) {
            const int m = 2 * i + (lane >> 4);
            u[i] = *reinterpret_cast<const uint32_t*>(vb + (m % NS) * ppitch + (m / NS) * g.pos_bytes);
          }
#pragma unroll
          for (int i = 0; i < kT / 2; ++i) {
            const int m = 2 * i + (lane >> 4);
            uint32_t h[4];
            i4x8_to_h2(u[i], h);
            *reinterpret_cast<uint4*>(vd + m * kVPitch) =
                make_uint4(__byte_perm(h[0], h[1], 0x5410), __byte_perm(h[2], h[3], 0x5410),
                           __byte_perm(h[0], h[1], 0x7632), __byte_perm(h[2], h[3], 0x7632));
          }
        }
        // the V scales too, then the ring slot is free: everything after this
        // reads registers and the warp's scratch, so the producer can refill
        // the slot while the softmax and the value product run
        {
          const float* vsc = reinterpret_cast<const float*>(st8 + 2 * a.stage_region + a.sc_region);
          const int pos0 = (gq % NS) * RPS + gq / NS, pos1 = ((gq + 8) % NS) * RPS + (gq + 8) / NS;
          vs0 = vsc[pos0 * g.hc + hk];
          vs1 = vsc[pos1 * g.hc + hk];
        }
        if (!IV) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          Vs = smem_u32(vscr);
          vpitch = kVPitch;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint32_t ka[4];
          // matrices: (pos 0-7, d 0-7), (pos 8-15, d 0-7), (pos 0-7, d 8-15), (pos 8-15, d 8-15)
          // matrix rows are MMA rows lr (+8): positions 2lr / 2lr+1 -> slot lr
          const int mr = lr + 8 * (lm & 1);  // MMA row: slot mr % NS, row mr / NS of the slot
          ldsm_x4(Ks + (mr % NS) * ppitch + (mr / NS) * g.pos_bytes + (16 * kk + 8 * (lm >> 1)) * 2, ka);
          float(&acc)[4] = (kk & 1) ? s2 : s;
          mma16816(acc, ka, qb[kk][0][0], qb[kk][1][0]);
          if (!PACK) mma16816(acc, ka, qb[kk][0][1], qb[kk][1][1]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] += s2[i];
      }
      if (PACK && !IM) {  // hi + lo columns: every lane of the pair holds the full score
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], XG);
      }
      // s[0], s[1]: (pos gq, heads 2tq, 2tq+1); s[2], s[3]: (pos gq+8, ...)
      // positions of MMA rows gq and gq + 8 (slot-major: row r is position (r % NS) * RPS + r / NS)
      const bool v0 = (gq % NS) * RPS + gq / NS < cnt, v1 = ((gq + 8) % NS) * RPS + (gq + 8) / NS < cnt;
      if (!v0) s[0] = s[1] = -INFINITY;
      if (!v1) s[2] = s[3] = -INFINITY;
      float mx0 = fmaxf(s[0], s[2]), mx1 = fmaxf(s[1], s[3]);
#pragma unroll
      for (int sh = 4; sh < 32; sh <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, sh));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, sh));
      }
      if constexpr (IV) {
        // flush when the stage's max passes mref + 1 (p would exceed 2), a
        // valid row's V scale passes Sb, or the int32 sums could overflow
        // (iv_flush <= 2000 stages: 2000 x 16 rows x 255 x 255 < 2^31)
        const float vl = fmaxf(v0 ? vs0 : 0.0f, v1 ? vs1 : 0.0f);
        if (__any_sync(0xffffffffu, mx0 > m[0] + 1.0f || mx1 > m[1] + 1.0f || vl > sb || nacc == a.iv_flush)) {
          float vm = vl;
#pragma unroll
          for (int sh = 4; sh < 32; sh <<= 1) vm = fmaxf(vm, __shfl_xor_sync(0xffffffffu, vm, sh));
          const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);  // finite: position 0 of a piece is valid
          const float c0 = fast_exp2(m[0] - mn0), c1 = fast_exp2(m[1] - mn1);
          iv_flush(c0, c1);
          l[0] *= c0;
          l[1] *= c1;
          m[0] = mn0;
          m[1] = mn1;
          sb = fmaxf(vm * 1.0625f, 1e-30f);  // a little headroom: fewer flushes, 0.09 bit
          fs = 4194288.0f / sb;               // (2^22 - 16) / Sb: W < 2^23 for p <= 2
        }
        ++nacc;
        const float p0 = fast_exp2(s[0] - m[0]), p1 = fast_exp2(s[1] - m[1]);
        const float p2 = fast_exp2(s[2] - m[0]), p3 = fast_exp2(s[3] - m[1]);
        l[0] += p0 + p2;
        l[1] += p1 + p3;
        // W = rn(p * vscale * fs) in the low 23 bits of the float 2^23 + W
        const float f0 = v0 ? vs0 * fs : 0.0f, f1 = v1 ? vs1 * fs : 0.0f;
        const uint32_t w0 = __float_as_uint(fmaf(p0, f0, 8388608.0f)), w1 = __float_as_uint(fmaf(p1, f0, 8388608.0f));
        const uint32_t w2 = __float_as_uint(fmaf(p2, f1, 8388608.0f)), w3 = __float_as_uint(fmaf(p3, f1, 8388608.0f));
        // transposes of the (limb 0 | limb 1) and (limb 2 | exponent) 16-bit
        // planes: lane (gq, tq) gets head gq % G at MMA rows 2tq, 2tq + 1 (x01)
        // and 2tq + 8, 2tq + 9 (x23)
        const uint32_t lo01 = movm_t(__byte_perm(w0, w1, 0x5410)), lo23 = movm_t(__byte_perm(w2, w3, 0x5410));
        const uint32_t hi01 = movm_t(__byte_perm(w0, w1, 0x7632)), hi23 = movm_t(__byte_perm(w2, w3, 0x7632));
        uint32_t bf[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          const int limb = (8 * k + gq) / G;
          const uint32_t x = limb == 2 ? __byte_perm(hi01, hi23, 0x6420) : __byte_perm(lo01, lo23, limb ? 0x7531 : 0x6420);
          bf[k] = limb <= 2 ? x : 0u;
          vcs[k] = __dp4a(bf[k], 0x01010101u, vcs[k]);
        }
        // ---- O^T(int) += V^T . P^T, V^T codes straight from the ring
        if constexpr (I8) {
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            uint32_t r0, r1;
            ldsm_b8_t(Vs + vrow_addr_off + 16 * mt, r0, r1);
#pragma unroll
            for (int k = 0; k < NT; ++k) imma16816u(vacc[k][mt], r0, r1, bf[k]);
          }
        } else {
          // int4: byte column c of a 16 x 16 tile is head dims (2c, 2c + 1) of
          // 32; its low / high nibbles make the A rows of tiles 2j (dims
          // 32j + 2g, 32j + 2g + 16) and 2j + 1 (the same + 1)
          const uint32_t vb4 = smem_u32(st8) + a.stage_region + hk * (kHD / 2) + vrow_addr_off;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t r0, r1;
            ldsm_b8_t(vb4 + 16 * j, r0, r1);
            const uint32_t a0 = r0 & 0x0F0F0F0Fu, a1 = r1 & 0x0F0F0F0Fu;
            const uint32_t b0 = (r0 >> 4) & 0x0F0F0F0Fu, b1 = (r1 >> 4) & 0x0F0F0F0Fu;
#pragma unroll
            for (int k = 0; k < NT; ++k) {
              imma16816u(vacc[k][2 * j], a0, a1, bf[k]);
              imma16816u(vacc[k][2 * j + 1], b0, b1, bf[k]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == nst) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);  // finite: position 0 of a piece is valid
      const float c0 = fast_exp2(m[0] - mn0), c1 = fast_exp2(m[1] - mn1);
      m[0] = mn0;
      m[1] = mn1;
      const float p0 = fast_exp2(s[0] - mn0), p1 = fast_exp2(s[1] - mn1);
      const float p2 = fast_exp2(s[2] - mn0), p3 = fast_exp2(s[3] - mn1);
      l[0] = fmaf(l[0], c0, p0 + p2);
      l[1] = fmaf(l[1], c1, p1 + p3);
      // the running max rarely moves after the first stages: rescale only
      // when it did in some lane (c = exp2(0) = 1 exactly otherwise)
      if (__any_sync(0xffffffffu, c0 != 1.0f || c1 != 1.0f)) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          o[mt][0] *= c0;
          o[mt][2] *= c0;
          o[mt][1] *= c1;
          o[mt][3] *= c1;
        }
      }
      // ---- P^T B-fragments via transposes of the S^T accumulator layout
      // (int8: the V scale of each position is folded into p)
      uint32_t h01, l01, h23, l23;
      split2(p0 * vs0, p1 * vs0, h01, l01);  // (pos gq, heads 2tq..): rows = pos
      split2(p2 * vs1, p3 * vs1, h23, l23);  // (pos gq+8, ...)
      if (lo_role) {  // PACK: this lane's columns take the lo parts
        h01 = l01;
        h23 = l23;
      }
      const uint32_t bh0 = movm_t(h01), bh1 = movm_t(h23);
      const uint32_t bl0 = PACK ? 0u : movm_t(l01), bl1 = PACK ? 0u : movm_t(l23);
      // ---- O^T += V^T . P^T  (8 tiles of 16 head-dims)
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t va[4];
        // A = V^T: matrices (pos 0-7, d 0-7), (pos 0-7, d 8-15), (pos 8-15, d 0-7), (pos 8-15, d 8-15)
        const int vrow = lr + 8 * (lm >> 1);  // MMA k row (position mapping as for K)
        const uint32_t vaddr = vpitch ? Vs + vrow * vpitch : Vs + (vrow % NS) * ppitch + (vrow / NS) * g.pos_bytes;
        ldsm_x4_t(vaddr + (16 * mt + 8 * (lm & 1)) * 2, va);
        mma16816(o[mt], va, bh0, bh1);
        if (!PACK) mma16816(o[mt], va, bl0, bl1);
      }
      __syncwarp();
      if (!QNT && lane == 0) mbar_arrive(&empty[stage]);  // (int8 / int4 released the slot after their loads)
      if (++stage == nst) {
        stage = 0;
        phase ^= 1;
      }
    }

    // ---- finalize: full row sums, then direct output or partial
    if constexpr (IV) {
      iv_flush(1.0f, 1.0f);  // the integer sums since the last flush, same mref
      const float* os = ivo();
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[mt][e] = os[(4 * mt + e) * 32];
      __syncwarp();  // the scratch becomes the merge slot below
      if constexpr (I4) {
        // back to the standard fragment layout (tile mt = head dims 16 mt ..
        // 16 mt + 15) through the scratch as O^T[dim][column]
        float* t = reinterpret_cast<float*>(scr + warp * kScratch);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int dim = 32 * (mt >> 1) + 2 * gq + 16 * (e >> 1) + (mt & 1);
            t[dim * 8 + 2 * tq + (e & 1)] = o[mt][e];
          }
        __syncwarp();
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) o[mt][e] = t[(16 * mt + gq + 8 * (e >> 1)) * 8 + 2 * tq + (e & 1)];
        __syncwarp();
      }
    }
    if (PACK) {  // O^T columns [G, 2G) hold V . P_lo: add them to the hi columns
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[mt][i] += __shfl_xor_sync(0xffffffffu, o[mt][i], XG);
    }
#pragma unroll
    for (int sh = 4; sh < 32; sh <<= 1) {
      l[0] += __shfl_xor_sync(0xffffffffu, l[0], sh);
      l[1] += __shfl_xor_sync(0xffffffffu, l[1], sh);
    }
    if (P > 1) {
      // merge the P position classes of this head into class 0 (same
      // fragment layout in every warp: elementwise per lane)
      float* mine = merge_slot(warp);
      if (cls > 0) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int i = 0; i < 4; ++i) mine[4 * mt + i] = o[mt][i];
        mine[32] = m[0];
        mine[33] = m[1];
        mine[34] = l[0];
        mine[35] = l[1];
      }
      named_bar(1 + hk, P * 32);
      if (cls == 0) {
        for (int c = 1; c < P; ++c) {
          const float* th = merge_slot(hk + c * g.hc);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float mn = fmaxf(m[j], th[32 + j]);
            const float a0 = m[j] == -INFINITY ? 0.0f : fast_exp2(m[j] - mn);
            const float a1 = th[32 + j] == -INFINITY ? 0.0f : fast_exp2(th[32 + j] - mn);
            l[j] = l[j] * a0 + th[34 + j] * a1;
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
              o[mt][j] = o[mt][j] * a0 + th[4 * mt + j] * a1;
              o[mt][2 + j] = o[mt][2 + j] * a0 + th[4 * mt + 2 + j] * a1;
            }
            m[j] = mn;
          }
        }
      }
      named_bar(1 + hk, P * 32);  // class slots free for the next piece
      if (cls != 0) continue;
    }
    const bool direct = pc.flags & 1;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int hq = 2 * tq + j;
      if (hq >= G) continue;
      const int qh = hk * G + hq;
      if (direct) {
        float* orow;
        act16* brow;
        int f16 = a.ob_f16;  // format of the 16-bit copy (fp16 when set)
        if (a.routed) {
          const int rk = a.oroute.rank[pc.item];
          const int64_t rr = a.oroute.row[pc.item];
          orow = a.oroute.base[rk] ? a.oroute.base[rk] + rr * a.oroute.ld + qh * kHD : nullptr;
          brow = a.oroute.bbase[rk] ? a.oroute.bbase[rk] + rr * a.oroute.bld + qh * kHD : nullptr;
          f16 = static_cast<int>(a.oroute.f16_mask >> rk & 1u);
        } else {
          orow = a.o + static_cast<int64_t>(pc.item) * a.o_stride + qh * kHD;
          brow = a.ob ? a.ob + static_cast<int64_t>(pc.item) * a.ob_stride + qh * kHD : nullptr;
        }
        const float inv = 1.0f / l[j];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const float x0 = o[mt][j] * inv, x1 = o[mt][2 + j] * inv;
          if (orow) {
            orow[16 * mt + gq] = x0;
            orow[16 * mt + gq + 8] = x1;
          }
          if (brow) {
            brow[16 * mt + gq] = to16(x0, f16);
            brow[16 * mt + gq + 8] = to16(x1, f16);
          }
        }
      } else {
        float* pa = a.part_acc + (static_cast<int64_t>(w) * Hq + qh) * kHD;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          pa[16 * mt + gq] = o[mt][j];
          pa[16 * mt + gq + 8] = o[mt][2 + j];
        }
        if (gq == 0) {
          float* pm = a.part_ml + (static_cast<int64_t>(w) * Hq + qh) * 2;
          pm[0] = m[j];
          pm[1] = l[j];
        }
      }
    }
    if (!direct && a.comb_cnt) {
      // last arriver of this (item, kv head) merges the item's partials
      const int ci = pc.flags >> 1;
      __threadfence();
      __syncwarp();
      int last = 0;
      const int4 it = a.comb[ci];
      if (lane == 0) last = atomicAdd(&a.comb_cnt[ci * g.hc + hk], 1) == it.z - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();
        // lane -> (head hq, DPL contiguous head dims); independent 16-B loads
        // per piece, same operation order as combine_kernel
        constexpr int LPH = 32 / G, DPL = kHD / LPH;
        const int hq = lane / LPH, d0 = (lane % LPH) * DPL;
        const int qh = hk * G + hq;
        const float* mlb = a.part_ml + static_cast<int64_t>(it.y) * Hq * 2 + qh * 2;
        const float* accb = a.part_acc + static_cast<int64_t>(it.y) * Hq * kHD + qh * kHD + d0;
        float M = -INFINITY;
        for (int p = 0; p < it.z; ++p) M = fmaxf(M, __ldcg(mlb + static_cast<int64_t>(p) * Hq * 2));
        float L = 0.0f, acc[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] = 0.0f;
#pragma unroll 2
        for (int p = 0; p < it.z; ++p) {
          const float2 ml = __ldcg(reinterpret_cast<const float2*>(mlb + static_cast<int64_t>(p) * Hq * 2));
          const float4* src = reinterpret_cast<const float4*>(accb + static_cast<int64_t>(p) * Hq * kHD);
          float4 t[DPL / 4];
#pragma unroll
          for (int k = 0; k < DPL / 4; ++k) t[k] = __ldcg(src + k);
          const float wgt = fast_exp2(ml.x - M);
          L = fmaf(wgt, ml.y, L);
#pragma unroll
          for (int k = 0; k < DPL / 4; ++k) {
            acc[4 * k] = fmaf(wgt, t[k].x, acc[4 * k]);
            acc[4 * k + 1] = fmaf(wgt, t[k].y, acc[4 * k + 1]);
            acc[4 * k + 2] = fmaf(wgt, t[k].z, acc[4 * k + 2]);
            acc[4 * k + 3] = fmaf(wgt, t[k].w, acc[4 * k + 3]);
          }
        }
        float* orow;
        act16* bro;
        int f16 = a.ob_f16;
        if (a.routed) {
          const int rk = a.oroute.rank[it.x];
          const int64_t rr = a.oroute.row[it.x];
          orow = a.oroute.base[rk] ? a.oroute.base[rk] + rr * a.oroute.ld + qh * kHD + d0 : nullptr;
          bro = a.oroute.bbase[rk] ? a.oroute.bbase[rk] + rr * a.oroute.bld + qh * kHD + d0 : nullptr;
          f16 = static_cast<int>(a.oroute.f16_mask >> rk & 1u);
        } else {
          orow = a.o + static_cast<int64_t>(it.x) * a.o_stride + qh * kHD + d0;
          bro = a.ob ? a.ob + static_cast<int64_t>(it.x) * a.ob_stride + qh * kHD + d0 : nullptr;
        }
#pragma unroll
        for (int k = 0; k < DPL / 4; ++k) {
          const float4 x = make_float4(acc[4 * k] / L, acc[4 * k + 1] / L, acc[4 * k + 2] / L, acc[4 * k + 3] / L);
          if (orow) *reinterpret_cast<float4*>(orow + 4 * k) = x;
          if (bro) {
            act16* brow = bro + 4 * k;
            *reinterpret_cast<uint2*>(brow) = make_uint2(pack16x2(x.x, x.y, f16), pack16x2(x.z, x.w, f16));
          }
        }
        if (lane == 0) a.comb_cnt[ci * g.hc + hk] = 0;  // ready for the next launch
      }
    }
  }
  if (a.routed) {
    // every consumer's routed o stores, ordered by the barrier before one
    // cumulative system-scope fence; then the last CTA publishes the epoch
    named_bar(15, kWarps * 32);  // the consumer warps (the producer has returned)
    if (threadIdx.x == 0) __threadfence_system();
    if (threadIdx.x == 0 && atomicAdd(a.oroute.done, 1) == static_cast<int>(gridDim.x) - 1) {
      __threadfence_system();
      for (int d = 0; d < 8; ++d) {
        if (a.oroute.notify >> d & 1) {
          asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(a.oroute.flag[d] + a.oroute.slot * 8 + a.oroute.self),
                       "l"(a.oroute.epoch)
                       : "memory");
        }
      }
      *a.oroute.done = 0;
    }
  }
}

}  // namespace

// fp16 stages copy four positions per bulk copy (8 KB at 8 kv heads: the
// producer's own pattern streams 7.20 vs 6.98 TB/s with 8-KB over 4-KB
// copies, tools/bulk_bw.cu; the C5 layer 0.630 -> 0.626 ms) at the price of
// 2-way ldmatrix conflicts (rows of a slot share bank groups); int8 keeps
// pair slots, which its 32-bit fragment loads need.
int attention_mma_rows_per_slot(const KvGeom& g) {
  // fp16 shards of 1-2 kv heads have 256-512-B positions: eight per copy
  // (2-4 KB) instead of four, the per-copy issue cost being the limit there
  if (g.fmt == SD_KV_HALF && g.hc <= 2 && tuning().attn_rps8) return 8;
  // quantized shards of <= 2 kv heads (128-256 B int8 positions, half that
  // int4): the ten copies per stage bound them at every width, so eight
  // positions per copy there too
  if (kv_quantized(g.fmt) && g.hc <= 2 && tuning().attn_rps8) return 8;
  // int8: quads. With the value product on integer tensor cores (IV) the
  // consumers keep up and the copy count is the limit: 0.448 -> 0.351 ms per
  // C5 layer with quads (0.975 of the copy peak); with fp16 values (G = 8) quads
  // are neutral at 8 kv heads and faster on smaller shards (hc = 4: 0.40 ->
  // 0.53 of the copy peak, hc = 2: 0.21 -> 0.29). attn_i8_quad = 0: pairs.
  return g.fmt == SD_KV_HALF || g.fmt == SD_KV_INT4 || tuning().attn_i8_quad || g.hc < 8 ? 4 : 2;
}

bool attention_mma_supported(const KvGeom& g, int G) {
  return (g.fmt == SD_KV_HALF || g.fmt == SD_KV_INT8 || g.fmt == SD_KV_INT4) && g.hd == kHD &&
         (g.hc == 8 || g.hc == 4 || g.hc == 2 || g.hc == 1) && (G == 2 || G == 4 || G == 8) && g.P % kT == 0;
}

size_t attention_mma_smem(const KvGeom& g, int* stage_region, int* sc_region, int* nstages) {
  // kT/2 pair slots of two rows + a 16-B pad
  const int rps = attention_mma_rows_per_slot(g);
  *stage_region = (kT / rps) * (rps * g.pos_bytes + 16);
  const bool qnt = kv_quantized(g.fmt);
  *sc_region = qnt ? ((kT * g.hc * 4 + 127) / 128) * 128 : 0;
  const size_t stage = 2 * static_cast<size_t>(*stage_region) + 2 * static_cast<size_t>(*sc_region);
  const int warps = consumer_warps<SD_KV_HALF>();
  const size_t scratch = qnt ? static_cast<size_t>(warps) * kScratch  // V tiles + merge slots
                         : (g.hc < warps ? static_cast<size_t>(warps) * 32 * 36 * 4 : 0);  // merge slots
  // fp16: two 64-KB stages stream faster than three (0.605 vs 0.643 ms per C5
  // layer, tools/bench_rpart.py, round 2); int8 (34-KB stages) is flat from
  // three to five stages and slower at two
  const int dflt = g.fmt == SD_KV_HALF ? 2 : g.fmt == SD_KV_INT8 ? 5 : 8;
  // The ring depth is a multiple of the P = warps / hc position classes, so
  // every fill of a slot is consumed by the same class: a class then waits on
  // a slot's full barrier only after it consumed the slot's previous fill, and
  // the parity wait cannot alias the phase before it (with P > depth a class
  // could see the previous fill's parity and read a stage not yet landed).
  // With P position classes each class needs two slots of its own to overlap
  // a stage's copy with the previous one's math: 1-kv-head-per-warp shards
  // (by-head ShardMap) run 4 stages at hc = 4, measured 0.613 ms against
  // 0.806 with 2 (1.08 vs 0.82 of the copy peak, tools/bench_rpart.py).
  const int P = warps / g.hc;
  int n = tuning().attn_max_stages > 1 ? tuning().attn_max_stages : std::max(dflt, P > 1 ? 2 * P : dflt);
  n = std::max(P, (n + P - 1) / P * P);
  auto bytes = [&](int k) { return static_cast<size_t>(128 * ((16 * k + 127) / 128)) + k * stage + scratch; };
  while (n > std::max(P, 2) && bytes(n) > 215 * 1024) n -= P;
  if (bytes(n) > 227 * 1024) fail(SD_ERR_INTERNAL, "attention_mma: ring does not fit shared memory");
  *nstages = n;
  return bytes(n);
}

template <int G>
void (*pick_mma(bool i8, bool i4, bool quad, bool octet, bool im, bool iv))(const AttnArgs) {
  if (octet) {  // quantized shards of 1-2 kv heads: eight positions per copy
    if constexpr (G <= 4) {
      if (iv && im) return i4 ? attn_mma_kernel<G, SD_KV_INT4, 8, true, true> : attn_mma_kernel<G, SD_KV_INT8, 8, true, true>;
    }
    if (i4) return im ? attn_mma_kernel<G, SD_KV_INT4, 8, true> : attn_mma_kernel<G, SD_KV_INT4, 8>;
    return im ? attn_mma_kernel<G, SD_KV_INT8, 8, true> : attn_mma_kernel<G, SD_KV_INT8, 8>;
  }
  if constexpr (G <= 4) {  // the integer value product (scores on integer tensor cores too)
    if (i4 && iv && im) return attn_mma_kernel<G, SD_KV_INT4, 4, true, true>;
    if (i8 && iv && im) return quad ? attn_mma_kernel<G, SD_KV_INT8, 4, true, true> : attn_mma_kernel<G, SD_KV_INT8, 2, true, true>;
  }
  if (i4) return im ? attn_mma_kernel<G, SD_KV_INT4, 4, true> : attn_mma_kernel<G, SD_KV_INT4, 4>;
  if (i8 && quad) return im ? attn_mma_kernel<G, SD_KV_INT8, 4, true> : attn_mma_kernel<G, SD_KV_INT8, 4>;
  if (i8) return im ? attn_mma_kernel<G, SD_KV_INT8, 2, true> : attn_mma_kernel<G, SD_KV_INT8, 2>;
  return attn_mma_kernel<G, SD_KV_HALF, 4>;
}
template <int G>
void (*pick_mma_half(int rps))(const AttnArgs) {
  return rps == 8 ? attn_mma_kernel<G, SD_KV_HALF, 8> : attn_mma_kernel<G, SD_KV_HALF, 4>;
}

void launch_attention_mma(const AttnArgs& a, int grid, size_t smem, cudaStream_t s) {
  void (*fn)(const AttnArgs) = nullptr;
  const bool i8 = a.g.fmt == SD_KV_INT8, i4 = a.g.fmt == SD_KV_INT4;
  // the slot layout the store was built with (a later attn_i8_quad flip
  // does not change an existing store's stage geometry)
  const bool quad = a.stage_region == (kT / 4) * (4 * a.g.pos_bytes + 16);
  const bool octet = a.stage_region == (kT / 8) * (8 * a.g.pos_bytes + 16);
  const bool im = tuning().attn_imma != 0;
  const bool iv = tuning().attn_ivalue != 0;
  if (!i8 && !i4 && octet) {
    switch (a.G) {
      case 2: fn = pick_mma_half<2>(8); break;
      case 4: fn = pick_mma_half<4>(8); break;
      case 8: fn = pick_mma_half<8>(8); break;
      default: fail(SD_ERR_INTERNAL, "attention_mma: unsupported group size");
    }
  } else {
    switch (a.G) {
      case 2: fn = pick_mma<2>(i8, i4, quad, octet, im, iv); break;
      case 4: fn = pick_mma<4>(i8, i4, quad, octet, im, iv); break;
      case 8: fn = pick_mma<8>(i8, i4, quad, octet, im, iv); break;
      default: fail(SD_ERR_INTERNAL, "attention_mma: unsupported group size");
    }
  }

  // the dynamic-smem opt-in once per instantiation and size
  static std::mutex mu;
  static std::vector<std::pair<void (*)(const AttnArgs), size_t>> set;
  {
    std::lock_guard<std::mutex> lock(mu);
    bool have = false;
    for (auto& e : set) have = have || (e.first == fn && e.second >= smem);
    if (!have) {
      SD_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      set.emplace_back(fn, smem);
    }
  }
  const int threads = (consumer_warps<SD_KV_HALF>() + 1) * 32;
  AttnArgs b = a;
  // attn_ivalue > 1: forced flushes every that many stages (tests reach the
  // overflow guard's path without 32,000-position pieces)
  b.iv_flush = tuning().attn_ivalue > 1 ? std::min(tuning().attn_ivalue, 2000) : 2000;
  SD_CUDA(launch_pdl(fn, dim3(grid), dim3(threads), smem, s, 1, b));
  SD_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace sd
