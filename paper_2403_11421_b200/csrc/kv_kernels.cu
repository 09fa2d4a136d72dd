// R-Part kernels for sm_100a: in-place KV append (K1), split-K flash-decode
// attention streaming the paged KV pool through a TMA bulk-copy / mbarrier
// pipeline (K2), and the deterministic split combine (K3).
//
// Semantics follow KvShard::append_lane / attend (reference
// proj/src/attention.cpp:91-112, 204-282): scores are scaled dot products
// over every stored position including the current token, softmax is taken
// over all of them, all arithmetic is fp32 regardless of the storage format
// (fp32 | fp16 RNE | int8 with per-(position, head) scale).
#include <cuda_fp16.h>

#include <cfloat>
#include <cmath>

#include "kv_kernels.cuh"
#include "pdl.cuh"
#include "sd_common.h"

namespace sd {

namespace {

constexpr int kConsumerWarps = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
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

// TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
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

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Eight consecutive elements of a row as four fp32 pairs (the K2 inner
// loops run on Blackwell's paired FFMA2 / FADD2: two fp32 lanes per issue).
template <int FMT>
struct Fmt;
template <>
struct Fmt<SD_KV_SINGLE> {
  __device__ static __forceinline__ void load8(const uint8_t* p, float2 (&x)[4]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 16);
    x[0] = make_float2(a.x, a.y);
    x[1] = make_float2(a.z, a.w);
    x[2] = make_float2(b.x, b.y);
    x[3] = make_float2(b.z, b.w);
  }
};
template <>
struct Fmt<SD_KV_HALF> {
  __device__ static __forceinline__ void load8(const uint8_t* p, float2 (&x)[4]) {
    const uint4 r = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h;
      *reinterpret_cast<uint32_t*>(&h) = w[i];
      x[i] = __half22float2(h);
    }
  }
};
template <>
struct Fmt<SD_KV_INT8> {
  // int8 -> fp32 without I2F: the pool stores q + 128 (kv_store.h), so
  // byte u becomes the float 2^23 + u (one PRMT into 0x4B0000xx), minus
  // 2^23 + 128 (one FADD2 per pair): exact, equal to (float)q
  __device__ static __forceinline__ float2 cvt2(uint32_t u, uint32_t s0, uint32_t s1) {
    return __fadd2_rn(make_float2(__uint_as_float(__byte_perm(u, 0x4B000000u, s0)),
                                  __uint_as_float(__byte_perm(u, 0x4B000000u, s1))),
                      make_float2(-8388736.0f, -8388736.0f));
  }
  __device__ static __forceinline__ void load8(const uint8_t* p, float2 (&x)[4]) {
    const uint2 r = *reinterpret_cast<const uint2*>(p);
    x[0] = cvt2(r.x, 0x7650, 0x7651);
    x[1] = cvt2(r.x, 0x7652, 0x7653);
    x[2] = cvt2(r.y, 0x7650, 0x7651);
    x[3] = cvt2(r.y, 0x7652, 0x7653);
  }
};
template <>
struct Fmt<SD_KV_INT4> {
  // eight nibbles (element 2i low) holding q + 8 -> fp32: byte i goes under
  // 0x4B0000 (one PRMT); masking keeps 2^23 + lo or 2^23 + 16 hi, and one
  // FFMA2 maps them to lo - 8 and (2^23 + 16 hi) / 16 - (2^19 + 8) = hi - 8,
  // both exact
  __device__ static __forceinline__ void load8(const uint8_t* p, float2 (&x)[4]) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t b = __byte_perm(u, 0x4B000000u, 0x7650 + i);
      x[i] = __ffma2_rn(make_float2(__uint_as_float(b & 0xFFFFFF0Fu), __uint_as_float(b & 0xFFFFFFF0u)),
                        make_float2(1.0f, 0.0625f), make_float2(-8388616.0f, -524296.0f));
    }
  }
};

// --------------------------------------------------------------- K2 ------
// Persistent split-K decode attention. One CTA per SM walks a contiguous,
// balanced range of (item, position) pieces (host-built). Warp
// kConsumerWarps is the producer: one lane streams T-position stages of the
// item's K and V rows (all shard heads, contiguous inside a page group; plus
// the int8 scales) into an nstages-deep shared-memory ring with
// cp.async.bulk + mbarriers. The consumer warps are split into row groups
// of LPR lanes; each lane owns EPL consecutive elements of a head row, so a
// K.q dot is EPL FMAs plus log2(LPR) xor-shuffles. Row group rg owns MAXH kv
// heads (and their G query heads) in one position class. Rows are processed
// in batches of PB positions per head: all K dots of a batch are issued
// before any reduction (ILP), the online softmax rescales once per batch, in
// the log2 domain, fp32 throughout.
// CW consumer warps (8, or 10 for 40-head shards: 40 row groups of 8 lanes,
// one head each, instead of 16 row groups carrying 2-3 heads)
template <int FMT, int LPR, int EPL, int MAXH, int G, int CW = kConsumerWarps>
__global__ void __launch_bounds__((CW + 1) * 32, 1) attn_kernel(const AttnArgs a) {
  constexpr int kConsumerWarps = CW;
  constexpr bool QNT = kv_quantized(FMT);
  constexpr int HD = LPR * EPL;
  constexpr int RGW = 32 / LPR;              // row groups per warp
  constexpr int RG = kConsumerWarps * RGW;   // row groups per CTA
  constexpr int MAXQ = MAXH * G;
  constexpr int PB = 4;                      // positions per batch
  constexpr int NC = EPL / 8;                // 8-element chunks per lane

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + a.nstages;
  uint8_t* ring = smem + 128 * ((16 * a.nstages + 127) / 128);
  const size_t stage_bytes = static_cast<size_t>(2) * a.stage_region + 2 * a.sc_region;
  float* scratch = reinterpret_cast<float*>(ring + stage_bytes * a.nstages);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const KvGeom& g = a.g;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();  // inputs of the previous kernel (q, plan, pool) from here on

  const int cb = a.cta_begin[blockIdx.x];
  const int ce = a.cta_begin[blockIdx.x + 1];
  const uint8_t* layer_base = g.pool + static_cast<int64_t>(a.layer) * g.layer_bytes;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int w = cb; w < ce; ++w) {
        const Piece pc = a.pieces[w];
        const int slot = a.item_slot[pc.item];
        const int32_t* pt = g.page_table + static_cast<int64_t>(slot) * g.max_pages;
        for (int pos = pc.p0; pos < pc.p1; pos += a.T) {
          const int cnt = min(a.T, pc.p1 - pos);
          const int grp = pt[pos >> g.log2P];
          const int off = pos & (g.P - 1);
          const uint8_t* lb = layer_base + static_cast<int64_t>(grp) * g.group_bytes;
          const uint8_t* base = lb + static_cast<int64_t>(off) * g.pos_bytes;
          const uint32_t bytes = static_cast<uint32_t>(cnt) * g.pos_bytes;
          const uint32_t sbytes = a.sc_region ? static_cast<uint32_t>(cnt) * g.hc * 4u : 0u;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], 2 * bytes + 2 * sbytes);
          uint8_t* dst = ring + stage * stage_bytes;
          bulk_g2s(dst, base, bytes, &full[stage], pol);
          bulk_g2s(dst + a.stage_region, base + g.v_off, bytes, &full[stage], pol);
          if (sbytes) {
            const uint8_t* sb = lb + static_cast<int64_t>(off) * g.hc * 4;
            bulk_g2s(dst + 2 * a.stage_region, sb + g.ks_off, sbytes, &full[stage], pol);
            bulk_g2s(dst + 2 * a.stage_region + a.sc_region, sb + g.vs_off, sbytes, &full[stage], pol);
          }
          if (++stage == a.nstages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int rg = warp * RGW + lane / LPR;
  const int li = lane % LPR;
  const int hkv = g.hc;
  int ncls, cls, h0, hstride, nh;
  if (hkv >= RG) {
    ncls = 1;
    cls = 0;
    h0 = rg;
    hstride = RG;
    nh = (hkv - rg + RG - 1) / RG;
  } else {
    ncls = RG / hkv;
    cls = rg / hkv;
    h0 = rg % hkv;
    hstride = hkv;
    nh = cls < ncls ? 1 : 0;
  }
  const int Hq = hkv * G;
  constexpr int row_bytes = kv_row_bytes(FMT, HD);
  const int tstep = ncls * PB;

  float q[MAXQ][EPL], acc[MAXQ][EPL], m[MAXQ], l[MAXQ];
  int stage = 0;
  uint32_t phase = 0;

  for (int w = cb; w < ce; ++w) {
    const Piece pc = a.pieces[w];
    const float* qrow = a.q + static_cast<int64_t>(pc.item) * a.q_stride;
#pragma unroll
    for (int j = 0; j < MAXQ; ++j) {
      const int hh = j / G;
      m[j] = -INFINITY;
      l[j] = 0.0f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[j][i] = 0.0f;
      if (hh < nh) {
        const int qh = (h0 + hh * hstride) * G + (j % G);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const float4* src = reinterpret_cast<const float4*>(qrow + qh * HD + (c * LPR + li) * 8);
          const float4 x0 = src[0], x1 = src[1];
          q[j][8 * c + 0] = x0.x * a.qscale;
          q[j][8 * c + 1] = x0.y * a.qscale;
          q[j][8 * c + 2] = x0.z * a.qscale;
          q[j][8 * c + 3] = x0.w * a.qscale;
          q[j][8 * c + 4] = x1.x * a.qscale;
          q[j][8 * c + 5] = x1.y * a.qscale;
          q[j][8 * c + 6] = x1.z * a.qscale;
          q[j][8 * c + 7] = x1.w * a.qscale;
        }
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) q[j][i] = 0.0f;
      }
    }
    const int slot = a.item_slot[pc.item];
    const int32_t* pt = g.page_table + static_cast<int64_t>(slot) * g.max_pages;

    for (int pos = pc.p0; pos < pc.p1; pos += a.T) {
      const int cnt = min(a.T, pc.p1 - pos);
      mbar_wait(&full[stage], phase);
      const uint8_t* Ks = ring + stage * stage_bytes;
      const uint8_t* Vs = Ks + a.stage_region;
      const float* ksc = nullptr;
      const float* vsc = nullptr;
      if (QNT) {
        if (a.sc_region) {
          ksc = reinterpret_cast<const float*>(Ks + 2 * a.stage_region);
          vsc = reinterpret_cast<const float*>(Ks + 2 * a.stage_region + a.sc_region);
        } else {
          const int grp = pt[pos >> g.log2P];
          const uint8_t* lb = layer_base + static_cast<int64_t>(grp) * g.group_bytes;
          const int off = pos & (g.P - 1);
          ksc = reinterpret_cast<const float*>(lb + g.ks_off) + off * hkv;
          vsc = reinterpret_cast<const float*>(lb + g.vs_off) + off * hkv;
        }
      }
      // warp-uniform trip count: every lane runs every shuffle
      for (int t0 = 0; t0 < a.T; t0 += tstep) {
        float sc[MAXH][PB][G];
        // (A) all K dots of the batch, independent chains
#pragma unroll
        for (int hh = 0; hh < MAXH; ++hh) {
          const int hk = h0 + hh * hstride;
#pragma unroll
          for (int i = 0; i < PB; ++i) {
            const int t = t0 + cls + ncls * i;
            const bool act = t < cnt && hh < nh;
#pragma unroll
            for (int gg = 0; gg < G; ++gg) sc[hh][i][gg] = 0.0f;
            if (act) {
              const uint8_t* kr = Ks + static_cast<size_t>(t * hkv + hk) * row_bytes;
              float2 d2[G];
#pragma unroll
              for (int gg = 0; gg < G; ++gg) d2[gg] = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int c = 0; c < NC; ++c) {
                float2 kx[4];
                Fmt<FMT>::load8(kr + kv_row_bytes(FMT, (c * LPR + li) * 8), kx);
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    d2[gg] = __ffma2_rn(make_float2(q[hh * G + gg][c * 8 + 2 * e], q[hh * G + gg][c * 8 + 2 * e + 1]),
                                        kx[e], d2[gg]);
                }
              }
#pragma unroll
              for (int gg = 0; gg < G; ++gg) sc[hh][i][gg] = d2[gg].x + d2[gg].y;
            }
          }
        }
        // (B) reductions over the LPR lanes of each row, pipelined
#pragma unroll
        for (int sh = LPR / 2; sh > 0; sh >>= 1) {
#pragma unroll
          for (int hh = 0; hh < MAXH; ++hh)
#pragma unroll
            for (int i = 0; i < PB; ++i)
#pragma unroll
              for (int gg = 0; gg < G; ++gg) sc[hh][i][gg] += __shfl_xor_sync(0xffffffffu, sc[hh][i][gg], sh);
        }
        // (C) block online softmax per (head, query)
        float p[MAXH][PB][G];
        float vs[MAXH][PB];
#pragma unroll
        for (int hh = 0; hh < MAXH; ++hh) {
          const int hk = h0 + hh * hstride;
#pragma unroll
          for (int i = 0; i < PB; ++i) {
            const int t = t0 + cls + ncls * i;
            const bool act = t < cnt && hh < nh;
            float ks = 1.0f;
            vs[hh][i] = 1.0f;
            if (QNT && act) {
              ks = ksc[t * hkv + hk];
              vs[hh][i] = vsc[t * hkv + hk];
            }
#pragma unroll
            for (int gg = 0; gg < G; ++gg) sc[hh][i][gg] = act ? sc[hh][i][gg] * ks : -INFINITY;
          }
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            const int j = hh * G + gg;
            float mb = sc[hh][0][gg];
#pragma unroll
            for (int i = 1; i < PB; ++i) mb = fmaxf(mb, sc[hh][i][gg]);
            // branchless: an all-masked batch with no history gives c = p = 0
            const float mn = fmaxf(m[j], mb);
            const float ms = mn == -INFINITY ? 0.0f : mn;
            const float c = fast_exp2(m[j] - ms);
            float ps = 0.0f;
#pragma unroll
            for (int i = 0; i < PB; ++i) {
              p[hh][i][gg] = fast_exp2(sc[hh][i][gg] - ms);
              ps += p[hh][i][gg];
            }
            l[j] = fmaf(l[j], c, ps);
            m[j] = mn;
#pragma unroll
            for (int e = 0; e < EPL; ++e) acc[j][e] *= c;
          }
        }
        // (D) V accumulation
#pragma unroll
        for (int hh = 0; hh < MAXH; ++hh) {
          const int hk = h0 + hh * hstride;
#pragma unroll
          for (int i = 0; i < PB; ++i) {
            const int t = t0 + cls + ncls * i;
            const bool act = t < cnt && hh < nh;
            if (act) {
              const uint8_t* vr = Vs + static_cast<size_t>(t * hkv + hk) * row_bytes;
#pragma unroll
              for (int c = 0; c < NC; ++c) {
                float2 vx[4];
                Fmt<FMT>::load8(vr + kv_row_bytes(FMT, (c * LPR + li) * 8), vx);
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                  const float pv = QNT ? p[hh][i][gg] * vs[hh][i] : p[hh][i][gg];
                  const float2 pv2 = make_float2(pv, pv);
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    float* ac = &acc[hh * G + gg][c * 8 + 2 * e];
                    const float2 r = __ffma2_rn(pv2, vx[e], make_float2(ac[0], ac[1]));
                    ac[0] = r.x;
                    ac[1] = r.y;
                  }
                }
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == a.nstages) {
        stage = 0;
        phase ^= 1;
      }
    }

    // ---- finalize the piece: merge position classes through shared memory
    if (ncls > 1) {
      const int slot_stride = MAXQ * (HD + 2);
      if (nh > 0 && cls > 0) {
        float* dst = scratch + static_cast<size_t>(rg) * slot_stride;
#pragma unroll
        for (int j = 0; j < MAXQ; ++j) {
          if (j / G < nh) {
            float* d = dst + j * (HD + 2);
            if (li == 0) {
              d[0] = m[j];
              d[1] = l[j];
            }
#pragma unroll
            for (int i = 0; i < EPL; ++i) d[2 + ((i / 8) * LPR + li) * 8 + (i % 8)] = acc[j][i];
          }
        }
      }
      named_bar(1, kConsumerWarps * 32);
      if (nh > 0 && cls == 0) {
        for (int c = 1; c < ncls; ++c) {
          const float* src = scratch + static_cast<size_t>(c * hkv + h0) * slot_stride;
#pragma unroll
          for (int j = 0; j < MAXQ; ++j) {
            if (j / G < nh) {
              const float* sp = src + j * (HD + 2);
              const float m2 = sp[0], l2 = sp[1];
              const float M = fmaxf(m[j], m2);
              const float ca = m[j] == -INFINITY ? 0.0f : fast_exp2(m[j] - M);
              const float cb2 = m2 == -INFINITY ? 0.0f : fast_exp2(m2 - M);
              l[j] = l[j] * ca + l2 * cb2;
#pragma unroll
              for (int i = 0; i < EPL; ++i) {
                acc[j][i] = acc[j][i] * ca + sp[2 + ((i / 8) * LPR + li) * 8 + (i % 8)] * cb2;
              }
              m[j] = M;
            }
          }
        }
      }
      named_bar(1, kConsumerWarps * 32);
    }
    if (nh > 0 && cls == 0) {
      const bool direct = pc.flags & 1;
      float* orow = a.o + static_cast<int64_t>(pc.item) * a.o_stride;
#pragma unroll
      for (int j = 0; j < MAXQ; ++j) {
        if (j / G < nh) {
          const int qh = (h0 + (j / G) * hstride) * G + (j % G);
          if (direct) {
            const float inv = 1.0f / l[j];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              float4* dst = reinterpret_cast<float4*>(orow + qh * HD + (c * LPR + li) * 8);
              dst[0] = make_float4(acc[j][8 * c] * inv, acc[j][8 * c + 1] * inv,
                                   acc[j][8 * c + 2] * inv, acc[j][8 * c + 3] * inv);
              dst[1] = make_float4(acc[j][8 * c + 4] * inv, acc[j][8 * c + 5] * inv,
                                   acc[j][8 * c + 6] * inv, acc[j][8 * c + 7] * inv);
            }
          } else {
            float* pbase = a.part_acc + static_cast<int64_t>(w) * Hq * HD + qh * HD;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              float4* pa = reinterpret_cast<float4*>(pbase + (c * LPR + li) * 8);
              pa[0] = make_float4(acc[j][8 * c], acc[j][8 * c + 1], acc[j][8 * c + 2], acc[j][8 * c + 3]);
              pa[1] = make_float4(acc[j][8 * c + 4], acc[j][8 * c + 5], acc[j][8 * c + 6], acc[j][8 * c + 7]);
            }
            if (li == 0) {
              float* pm = a.part_ml + (static_cast<int64_t>(w) * Hq + qh) * 2;
              pm[0] = m[j];
              pm[1] = l[j];
            }
          }
        }
      }
    }
  }
}

// ----------------------------------------------------- K2 generic path ---
// Any head_dim / format / geometry (reference unit-test shapes such as
// hd = 4 or 12). One warp per (piece, query head); positions sequential,
// elements strided over lanes. Same online-softmax math as the fast path.
__device__ __forceinline__ float load_elem(const KvGeom& g, const uint8_t* lb, int off, int hk,
                                           int d, bool is_v) {
  const uint8_t* rows = lb + (is_v ? g.v_off : 0) + static_cast<int64_t>(off) * g.pos_bytes;
  const int idx = hk * g.hd + d;
  switch (g.fmt) {
    case SD_KV_SINGLE: return reinterpret_cast<const float*>(rows)[idx];
    case SD_KV_HALF: return __half2float(reinterpret_cast<const __half*>(rows)[idx]);
    case SD_KV_INT4: {
      const float sc = reinterpret_cast<const float*>(lb + (is_v ? g.vs_off : g.ks_off))[off * g.hc + hk];
      return static_cast<float>(static_cast<int>((rows[idx >> 1] >> ((idx & 1) * 4)) & 0xF) - 8) * sc;
    }
    default: {
      const float sc = reinterpret_cast<const float*>(lb + (is_v ? g.vs_off : g.ks_off))[off * g.hc + hk];
      return static_cast<float>(static_cast<int>(rows[idx]) - 128) * sc;
    }
  }
}

constexpr int kGenericMaxPerLane = 8;  // hd <= 256

__global__ void attn_generic_kernel(const AttnArgs a) {
  pdl_trigger();
  pdl_wait();
  const KvGeom& g = a.g;
  const int w = blockIdx.x;
  const int qh = blockIdx.y;
  const int lane = threadIdx.x;
  const Piece pc = a.pieces[w];
  const int hk = qh / a.G;
  const int Hq = g.hc * a.G;
  const int slot = a.item_slot[pc.item];
  const int32_t* pt = g.page_table + static_cast<int64_t>(slot) * g.max_pages;
  const uint8_t* layer_base = g.pool + static_cast<int64_t>(a.layer) * g.layer_bytes;
  const float* qrow = a.q + static_cast<int64_t>(pc.item) * a.q_stride + qh * g.hd;
  float qv[kGenericMaxPerLane], acc[kGenericMaxPerLane];
#pragma unroll
  for (int r = 0; r < kGenericMaxPerLane; ++r) {
    const int d = lane + 32 * r;
    qv[r] = d < g.hd ? qrow[d] * a.qscale : 0.0f;
    acc[r] = 0.0f;
  }
  float m = -INFINITY, l = 0.0f;
  for (int pos = pc.p0; pos < pc.p1; ++pos) {
    const uint8_t* lb = layer_base + static_cast<int64_t>(pt[pos >> g.log2P]) * g.group_bytes;
    const int off = pos & (g.P - 1);
    float s = 0.0f;
#pragma unroll
    for (int r = 0; r < kGenericMaxPerLane; ++r) {
      const int d = lane + 32 * r;
      if (d < g.hd) s = fmaf(qv[r], load_elem(g, lb, off, hk, d, false), s);
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) s += __shfl_xor_sync(0xffffffffu, s, sh);
    if (s > m) {
      const float c = fast_exp2(m - s);
      l *= c;
#pragma unroll
      for (int r = 0; r < kGenericMaxPerLane; ++r) acc[r] *= c;
      m = s;
    }
    const float p = fast_exp2(s - m);
    l += p;
#pragma unroll
    for (int r = 0; r < kGenericMaxPerLane; ++r) {
      const int d = lane + 32 * r;
      if (d < g.hd) acc[r] = fmaf(p, load_elem(g, lb, off, hk, d, true), acc[r]);
    }
  }
  if (pc.flags & 1) {
    float* orow = a.o + static_cast<int64_t>(pc.item) * a.o_stride + qh * g.hd;
    const float inv = 1.0f / l;
#pragma unroll
    for (int r = 0; r < kGenericMaxPerLane; ++r) {
      const int d = lane + 32 * r;
      if (d < g.hd) orow[d] = acc[r] * inv;
    }
  } else {
    float* pa = a.part_acc + static_cast<int64_t>(w) * Hq * g.hd + qh * g.hd;
#pragma unroll
    for (int r = 0; r < kGenericMaxPerLane; ++r) {
      const int d = lane + 32 * r;
      if (d < g.hd) pa[d] = acc[r];
    }
    if (lane == 0) {
      a.part_ml[(static_cast<int64_t>(w) * Hq + qh) * 2] = m;
      a.part_ml[(static_cast<int64_t>(w) * Hq + qh) * 2 + 1] = l;
    }
  }
}

// --------------------------------------------------------------- K3 ------
// Deterministic combine of an item's pieces in piece order.
__global__ void combine_kernel(const CombineArgs a) {
  pdl_trigger();
  pdl_wait();
  const int4 it = a.items[blockIdx.x];
  const int width = a.Hq * a.hd;
  float* orow = a.o + static_cast<int64_t>(it.x) * a.o_stride;
  for (int e = threadIdx.x; e < width; e += blockDim.x) {
    const int qh = e / a.hd;
    float M = -INFINITY;
    for (int p = 0; p < it.z; ++p) M = fmaxf(M, a.part_ml[(static_cast<int64_t>(it.y + p) * a.Hq + qh) * 2]);
    float L = 0.0f, acc = 0.0f;
    for (int p = 0; p < it.z; ++p) {
      const int64_t pi = it.y + p;
      const float wgt = fast_exp2(a.part_ml[(pi * a.Hq + qh) * 2] - M);
      L = fmaf(wgt, a.part_ml[(pi * a.Hq + qh) * 2 + 1], L);
      acc = fmaf(wgt, a.part_acc[pi * width + e], acc);
    }
    orow[e] = acc / L;
  }
}

// --------------------------------------------------------------- K1 ------
// One warp quantizes one head row (hd values from get(e)): int8 follows
// quantize_int8 (attention.cpp:28-46) bit for bit — scale = max|x| / 127.0f
// (IEEE fp32 division), q = clamp(rint((double)x * (1.0 / (double)scale)),
// +-127); int4 the same rules at +-7, two per byte, element 2i low. Stored
// offset-binary: q + 128 (int8), q + 8 (int4 nibbles), so the readers turn
// bytes into exact fp16 / fp32 integers without an xor; export_lane gives
// the reference's two's-complement bytes back.
template <class Get>
__device__ __forceinline__ void quantize_head(int fmt, int hd, const Get& get, uint8_t* dst, float* scale,
                                              int lane) {
  float mx = 0.0f;
  for (int e = lane; e < hd; e += 32) mx = fmaxf(mx, fabsf(get(e)));
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, sh));
  const double qmax = fmt == SD_KV_INT4 ? 7.0 : 127.0;
  const float sc = mx == 0.0f ? 0.0f : __fdiv_rn(mx, static_cast<float>(qmax));
  const double inv = sc == 0.0f ? 0.0 : 1.0 / static_cast<double>(sc);
  auto q = [&](int e) { return static_cast<int>(fmin(fmax(rint(static_cast<double>(get(e)) * inv), -qmax), qmax)); };
  if (fmt == SD_KV_INT4) {
    for (int e = lane; e < hd / 2; e += 32) dst[e] = static_cast<uint8_t>((q(2 * e) + 8) | ((q(2 * e + 1) + 8) << 4));
  } else {
    for (int e = lane; e < hd; e += 32) dst[e] = static_cast<uint8_t>(q(e) + 128);
  }
  if (lane == 0) *scale = sc;
}

// One block per (item, K|V) row: convert the fp32 row into the storage
// format at (slot, layer, position).
__global__ void append_kernel(const AppendArgs a) {
  pdl_trigger();
  pdl_wait();
  const KvGeom& g = a.g;
  // page-table updates for pages opened by this call
  if (blockIdx.x == 0 && blockIdx.y == 0) {
    for (int u = threadIdx.x; u < a.nupd; u += blockDim.x) g.page_table[a.upd[2 * u]] = a.upd[2 * u + 1];
  }
  const int i = blockIdx.x;
  if (i >= a.n) return;
  const bool is_v = blockIdx.y == 1;
  const float* src = (is_v ? a.v + i * a.v_stride : a.k + i * a.k_stride);
  const int pos = a.pos[i];
  const int off = pos & (g.P - 1);
  uint8_t* lb = g.pool + static_cast<int64_t>(a.group[i]) * g.group_bytes +
                static_cast<int64_t>(a.layer) * g.layer_bytes;
  uint8_t* row = lb + (is_v ? g.v_off : 0) + static_cast<int64_t>(off) * g.pos_bytes;
  if (g.fmt == SD_KV_SINGLE) {
    float* d = reinterpret_cast<float*>(row);
    for (int e = threadIdx.x; e < g.width; e += blockDim.x) d[e] = src[e];
  } else if (g.fmt == SD_KV_HALF) {
    __half* d = reinterpret_cast<__half*>(row);
    if ((g.width & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) | (reinterpret_cast<uintptr_t>(d) & 7)) == 0) {
      // 16-B loads, 8-B stores (same round-to-nearest-even as the scalar path)
      for (int e = 4 * threadIdx.x; e < g.width; e += 4 * blockDim.x) {
        const float4 x = *reinterpret_cast<const float4*>(src + e);
        const __half2 lo = __floats2half2_rn(x.x, x.y), hi = __floats2half2_rn(x.z, x.w);
        *reinterpret_cast<uint2*>(d + e) =
            make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
      }
    } else {
      for (int e = threadIdx.x; e < g.width; e += blockDim.x) d[e] = __float2half_rn(src[e]);
    }
  } else {
    // one warp per head
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    float* scales = reinterpret_cast<float*>(lb + (is_v ? g.vs_off : g.ks_off)) + off * g.hc;
    for (int h = warp; h < g.hc; h += nw) {
      const float* x = src + h * g.hd;
      quantize_head(g.fmt, g.hd, [&](int e) { return x[e]; }, row + kv_row_bytes(g.fmt, h * g.hd), scales + h, lane);
    }
  }
}

// Synthetic prefill, keyed by sequence id, not by store slot,
// so a sequence's context is the same in any shard and any allocation order:
// element (seq, layer, pos, kv, global kv head h, d) = synth_value(salt ^ idx),
// idx = ((((seq * 4096 + layer) * 2^20 + pos) * 2 + kv) * Hkv_total + h) * hd + d
// (kv_prefill_index in sd_common.h; the oracle restates it).
__global__ void prefill_kernel(const KvGeom g, int num_layers, const int32_t* slots, const uint64_t* seq_ids,
                               int n, int length, uint64_t salt, int h0, int kv_heads_total) {
  pdl_trigger();
  pdl_wait();
  const int64_t rows = static_cast<int64_t>(n) * num_layers * length * 2;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    int64_t t = r;
    const int kv = static_cast<int>(t & 1);
    t >>= 1;
    const int pos = static_cast<int>(t % length);
    t /= length;
    const int layer = static_cast<int>(t % num_layers);
    const int item = static_cast<int>(t / num_layers);
    const int slot = slots[item];
    const int grp = g.page_table[static_cast<int64_t>(slot) * g.max_pages + (pos >> g.log2P)];
    const int off = pos & (g.P - 1);
    uint8_t* lb = g.pool + static_cast<int64_t>(grp) * g.group_bytes +
                  static_cast<int64_t>(layer) * g.layer_bytes;
    uint8_t* row = lb + (kv ? g.v_off : 0) + static_cast<int64_t>(off) * g.pos_bytes;
    const uint64_t base = kv_prefill_index(seq_ids[item], layer, pos, kv, h0, 0, kv_heads_total, g.hd);
    if (g.fmt == SD_KV_SINGLE) {
      float* d = reinterpret_cast<float*>(row);
      for (int e = threadIdx.x; e < g.width; e += blockDim.x) d[e] = synth_value(salt ^ (base + e));
    } else if (g.fmt == SD_KV_HALF) {
      __half* d = reinterpret_cast<__half*>(row);
      for (int e = threadIdx.x; e < g.width; e += blockDim.x) d[e] = __float2half_rn(synth_value(salt ^ (base + e)));
    } else {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      float* scales = reinterpret_cast<float*>(lb + (kv ? g.vs_off : g.ks_off)) + off * g.hc;
      for (int h = warp; h < g.hc; h += nw) {
        const uint64_t hb = base + static_cast<uint64_t>(h) * g.hd;
        quantize_head(g.fmt, g.hd, [&](int e) { return synth_value(salt ^ (hb + e)); },
                      row + kv_row_bytes(g.fmt, h * g.hd), scales + h, lane);
      }
    }
  }
}

// ------------------------------------------------------------ dispatch ---
using AttnFn = void (*)(const AttnArgs);

template <int FMT, int LPR, int EPL>
AttnFn pick_mh(int maxh, int G) {
  if (G == 1) {
    switch (maxh) {
      case 1: return attn_kernel<FMT, LPR, EPL, 1, 1>;
      case 2: return attn_kernel<FMT, LPR, EPL, 2, 1>;
      case 3: return attn_kernel<FMT, LPR, EPL, 3, 1>;
      default: return nullptr;
    }
  }
  if (maxh != 1 || EPL != 8) return nullptr;
  switch (G) {
    case 2: return attn_kernel<FMT, LPR, 8, 1, 2>;
    case 4: return attn_kernel<FMT, LPR, 8, 1, 4>;
    default: return nullptr;
  }
}

template <int FMT>
AttnFn pick_fmt(const AttnConfig& c, int G) {
  if (c.cw == 10) return c.epl == 16 && c.lpr == 8 && c.maxh == 1 && G == 1 ? attn_kernel<FMT, 8, 16, 1, 1, 10> : nullptr;
  if (c.epl == 16) {
    switch (c.lpr) {
      case 8: return pick_mh<FMT, 8, 16>(c.maxh, G);
      case 16: return pick_mh<FMT, 16, 16>(c.maxh, G);
      default: return nullptr;
    }
  }
  switch (c.lpr) {
    case 2: return pick_mh<FMT, 2, 8>(c.maxh, G);
    case 4: return pick_mh<FMT, 4, 8>(c.maxh, G);
    case 8: return pick_mh<FMT, 8, 8>(c.maxh, G);
    case 16: return pick_mh<FMT, 16, 8>(c.maxh, G);
    case 32: return pick_mh<FMT, 32, 8>(c.maxh, G);
    default: return nullptr;
  }
}

AttnFn pick(const KvGeom& g, int G) {
  const AttnConfig c = choose_attn_config(g, G);
  if (!c.supported) return nullptr;
  switch (g.fmt) {
    case SD_KV_SINGLE: return pick_fmt<SD_KV_SINGLE>(c, G);
    case SD_KV_HALF: return pick_fmt<SD_KV_HALF>(c, G);
    case SD_KV_INT8: return pick_fmt<SD_KV_INT8>(c, G);
    case SD_KV_INT4: return pick_fmt<SD_KV_INT4>(c, G);
    default: return nullptr;
  }
}

}  // namespace

// Lanes per head row (LPR) and elements per lane (EPL): EPL = 16 when it
// balances the heads over the row groups at least as well as EPL = 8 (fewer
// shuffles per element), else 8. Heads per row group MAXH <= 3, G <= 4.
AttnConfig choose_attn_config(const KvGeom& g, int G) {
  AttnConfig best{false, 0, 0, 0, 0, kConsumerWarps};
  if (g.hd % 8 != 0 || g.pos_bytes % 16 != 0) return best;
  double best_eff = -1.0;
  for (int cw : {kConsumerWarps, 10}) {
    for (int epl : {16, 8}) {
      if (g.hd % epl != 0) continue;
      const int lpr = g.hd / epl;
      if (lpr < 2 || lpr > 32 || (lpr & (lpr - 1))) continue;
      // EPL 16 with grouped heads needs ~220 registers: over the 168 a thread
      // may hold when 9 warps share 4 SM sub-partitions
      if (epl == 16 && (G != 1 || (lpr != 8 && lpr != 16))) continue;
      if (cw != kConsumerWarps && (epl != 16 || lpr != 8 || G != 1)) continue;  // the one 10-warp instantiation
      const int rg = cw * (32 / lpr);
      const int maxh = g.hc >= rg ? (g.hc + rg - 1) / rg : 1;
      if (maxh > 3 || (G > 1 && maxh != 1) || (G != 1 && G != 2 && G != 4)) continue;
      if (cw != kConsumerWarps && maxh != 1) continue;
      const double eff = g.hc >= rg ? static_cast<double>(g.hc) / (rg * maxh) : 1.0;
      // the wider CTA only when it balances strictly better (e.g. 40 heads: 1.0 vs 0.83)
      if (eff > best_eff + 1e-9 && (cw == kConsumerWarps || eff > best_eff + 0.05)) {
        best_eff = eff;
        best = AttnConfig{true, lpr, epl, maxh, rg, cw};
      }
    }
  }
  return best;
}

int attention_consumer_warps() { return kConsumerWarps; }

size_t attention_smem_bytes(const KvGeom& g, int T, int nstages, int G, int* stage_region,
                            int* sc_region) {
  const int region = ((T * g.pos_bytes + 127) / 128) * 128;
  *stage_region = region;
  *sc_region = 0;
  if (kv_quantized(g.fmt) && g.hc % 4 == 0) *sc_region = ((T * g.hc * 4 + 127) / 128) * 128;
  size_t bytes = 128 * ((16 * nstages + 127) / 128) +
                 static_cast<size_t>(nstages) * (2 * region + 2 * *sc_region);
  const AttnConfig c = choose_attn_config(g, G);
  if (c.supported && g.hc < c.rg) {
    // class-merge scratch: RG x MAXQ x (hd + 2) floats
    bytes += static_cast<size_t>(c.rg) * G * (g.hd + 2) * sizeof(float);
  }
  return bytes;
}

bool launch_attention(const AttnArgs& a, int grid, size_t smem, cudaStream_t s) {
  AttnFn fn = pick(a.g, a.G);
  if (!fn) return false;
  if (smem > 48 * 1024) {
    SD_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  }
  const int threads = (choose_attn_config(a.g, a.G).cw + 1) * 32;
  SD_CUDA(launch_pdl(fn, dim3(grid), dim3(threads), smem, s, 1, a));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, fn);
    fail(SD_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e) + " (regs " +
                          std::to_string(fa.numRegs) + ", max threads " + std::to_string(fa.maxThreadsPerBlock) +
                          ", dyn smem " + std::to_string(smem) + ", static smem " +
                          std::to_string(fa.sharedSizeBytes) + ", grid " + std::to_string(grid) + ")");
  }
  ::sd::count_launch();
  return true;
}

void launch_attention_generic(const AttnArgs& a, int npieces, cudaStream_t s) {
  if (a.g.hd > 32 * kGenericMaxPerLane) fail(SD_ERR_CONFIG, "head_dim > 256 is not supported");
  dim3 grid(npieces, a.g.hc * a.G);
  SD_CUDA(launch_pdl(attn_generic_kernel, dim3(grid), dim3(32), 0, s, 1, a));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

void launch_combine(const CombineArgs& a, cudaStream_t s) {
  if (a.m == 0) return;
  SD_CUDA(launch_pdl(combine_kernel, dim3(a.m), dim3(256), 0, s, 1, a));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

void launch_append(const AppendArgs& a, cudaStream_t s) {
  if (a.n == 0 && a.nupd == 0) return;
  dim3 grid(a.n > 0 ? a.n : 1, 2);
  SD_CUDA(launch_pdl(append_kernel, grid, dim3(256), 0, s, 1, a));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

void launch_prefill_synthetic(const KvGeom& g, int num_layers, const int32_t* slots, const uint64_t* seq_ids,
                              int n, int length, uint64_t salt, int h0, int kv_heads_total, cudaStream_t s) {
  if (n == 0 || length == 0) return;
  SD_CUDA(launch_pdl(prefill_kernel, dim3(148 * 16), dim3(256), 0, s, 1, g, num_layers, slots, seq_ids, n, length,
                     salt, h0, kv_heads_total));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

}  // namespace sd
