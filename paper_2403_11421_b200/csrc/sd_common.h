// Internal shared definitions for libsd_b200 (host C++ and CUDA).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../../include/sd_abi.h"

namespace sd {

// Typed errors mirroring the reference's exception classes (core.hpp:25-38,
// attention.hpp:19-22); `code` is the C-ABI status they map to.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(SD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define SD_CUDA(x) ::sd::cuda_check((x), #x)

// Every kernel launch of this library bumps one process-wide counter
// (sd_launch_count in the C-ABI): the bench's "gpu_launches" evidence.
inline std::atomic<long long> g_launches{0};
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct Spec {
  int L, D, H, hd, F, V, Hkv;
  int kv_width() const { return Hkv * hd; }
  int qkv_width() const { return (H + 2 * Hkv) * hd; }
};

inline Spec make_spec(int L, int D, int H, int F, int V, int Hkv) {
  if (L < 1 || D < 1 || H < 1 || F < 1 || V < 1) {
    fail(SD_ERR_CONFIG, "model spec fields must all be >= 1");
  }
  if (D % H != 0) {
    fail(SD_ERR_CONFIG, "model_dim not divisible by heads (model_dim=" + std::to_string(D) +
                            ", num_heads=" + std::to_string(H) + ")");
  }
  if (Hkv == 0) Hkv = H;
  if (Hkv < 1 || H % Hkv != 0) fail(SD_ERR_CONFIG, "num_heads not divisible by num_kv_heads");
  return Spec{L, D, H, D / H, F, V, Hkv};
}

inline Spec from_abi(const sd_model_spec* s) {
  if (!s) fail(SD_ERR_CONFIG, "null model spec");
  Spec r = make_spec(s->num_layers, s->model_dim, s->num_heads, s->mlp_dim, s->vocab_size,
                     s->num_kv_heads);
  if (s->head_dim != 0 && s->head_dim != r.hd) {
    fail(SD_ERR_CONFIG, "head_dim inconsistent with model_dim / num_heads");
  }
  return r;
}

// SplitMix64 finalizer (core.cpp:161-166)
__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// Process-wide tuning switches (sd_tune in sd_abi.h). The defaults are the
// measured-best paths; A/B measurements and the variant-equivalence tests
// flip them. Read on the host when a launch is planned.
struct Tuning {
  int gemm_bn = 0;       // force the pair-tile width (16 | bn, 64..256); 0 = the wave cost model
  int gemm_pair = 1;     // 0: single-CTA tiles even when M spans two 128-row blocks
  int fused_append = 1;  // append_lane in the QKV GEMM epilogue (lockstep fp16 pages)
  int fused_argmax = 1;  // argmax_token in the head GEMM epilogue
  int dist_fuse = 1;     // multi-GPU exchange fused into its producers (else a scatter kernel)
  int attn_mma = 1;      // tensor-core attention where the geometry allows it
  int pdl = 1;           // programmatic dependent launch between the step's kernels
  int dist_phases = 0;   // per-phase CUDA events in DistEngine, printed to stderr at destroy
  int attn_i8_quad = 1;  // int8 tensor-core attention: four positions per bulk copy (else two; set when a store is built)
  int attn_l2_prefetch = 0;  // the attention prefetches the W_o weights into L2 at its end
  int attn_max_stages = 0;   // tensor-core attention ring depth (0: the per-format default)
  int attn_imma = 1;          // int8 / int4 KV: scores on integer tensor cores (q as byte limbs)
  int attn_rps8 = 1;          // shards of <= 2 kv heads copy 8 positions at a time (set when a store is built)
  int attn_ivalue = 1;        // int8 / int4 KV, G <= 4, with attn_imma: the value product on integer tensor cores
                              // too; > 1 also forces its int32 -> fp32 flush every that many stages (tests)
};
inline Tuning& tuning() {
  static Tuning t;
  return t;
}

// Bits of a 16-bit activation copy (bf16 or fp16 per the S-Part's dense mode).
using act16 = uint16_t;

// The 16-bit copy of an activation that a kind::f16 GEMM reads as its A
// operand: bf16, or fp16 when the S-Part runs fp16 operands; RNE either way.
__device__ __forceinline__ uint16_t to16(float x, int f16) {
  return f16 ? __half_as_ushort(__float2half_rn(x)) : __bfloat16_as_ushort(__float2bfloat16_rn(x));
}
__device__ __forceinline__ uint32_t pack16x2(float lo, float hi, int f16) {
  return static_cast<uint32_t>(to16(lo, f16)) | (static_cast<uint32_t>(to16(hi, f16)) << 16);
}

// KV storage formats: the quantized ones carry per-(position, head) fp32
// scales; bytes of n elements of a row (int4: two per byte)
__host__ __device__ constexpr bool kv_quantized(int fmt) { return fmt == SD_KV_INT8 || fmt == SD_KV_INT4; }
__host__ __device__ constexpr int kv_row_bytes(int fmt, int n) {
  return fmt == SD_KV_SINGLE ? 4 * n : fmt == SD_KV_HALF ? 2 * n : fmt == SD_KV_INT8 ? n : n / 2;
}

// Counter-based synthetic value in [-1, 1) (SURVEY §8d bench prefill)
__host__ __device__ inline float synth_value(uint64_t idx) {
  return 2.0f * (static_cast<float>(mix64(0x5EEDull ^ idx) >> 40) * 0x1p-24f) - 1.0f;
}

// Element index of the synthetic KV prefill: sequence id,
// layer (< 4096), position (< 2^20), K (0) / V (1), global kv head h of
// Hkv, element d of hd. Shard- and slot-independent.
__host__ __device__ inline uint64_t kv_prefill_index(uint64_t seq, int layer, int pos, int kv, int h, int d,
                                                     int kv_heads_total, int hd) {
  return ((((seq * 4096u + static_cast<uint64_t>(layer)) * 1048576u + static_cast<uint64_t>(pos)) * 2u +
           static_cast<uint64_t>(kv)) * static_cast<uint64_t>(kv_heads_total) + static_cast<uint64_t>(h)) *
             static_cast<uint64_t>(hd) + static_cast<uint64_t>(d);
}

// Device scratch buffer that only grows.
// Growth is geometric: a reallocation's cudaFree synchronizes the device, so
// a buffer that grows by a few bytes per decode step must not reallocate per
// step (callers on hot paths also pre-size to their upper bound).
inline size_t grow_bytes(size_t need, size_t have) {
  size_t n = have * 2 > need ? have * 2 : need;
  return (n + 4095) / 4096 * 4096;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      const size_t n = grow_bytes(need, bytes);
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      SD_CUDA(cudaMalloc(&p, n));
      bytes = n;
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct HostBuf {  // pinned
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      const size_t n = grow_bytes(need, bytes);
      if (p) cudaFreeHost(p);
      p = nullptr;
      bytes = 0;
      SD_CUDA(cudaMallocHost(&p, n));
      bytes = n;
    }
    return p;
  }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
};

// RAII device guard
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) SD_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace sd
