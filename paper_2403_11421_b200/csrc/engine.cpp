// Weights upload, the GPU StepComputation, the admission scheduler and
// drive_schedule — host C++ around the kernels.
#include "engine.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_set>

namespace sd {

// ======================================================== weight packing ===
namespace {

// Reference storage src = W^T row-major [in][out] (Eigen column-major
// out x in). Exact mode: copy into columns [col_off, col_off+out) of a
// [in][ld] fp32 matrix. Tensor modes: transpose into rows
// [row_off, row_off+out) of a [N][in] K-major matrix (bf16 or fp32).
__global__ void pack_kernel(const float* __restrict__ src, int in, int out, void* dst, int64_t ld,
                            int off, int mode) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r, j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (k < in && j < out) ? src[static_cast<int64_t>(k) * out + j] : 0.0f;
  }
  __syncthreads();
  if (mode == SD_DENSE_EXACT_F32) {
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const int k = k0 + r, j = j0 + threadIdx.x;
      if (k < in && j < out) static_cast<float*>(dst)[static_cast<int64_t>(k) * ld + off + j] = tile[r][threadIdx.x];
    }
  } else {
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const int j = j0 + r, k = k0 + threadIdx.x;
      if (k < in && j < out) {
        const float v = tile[threadIdx.x][r];
        const int64_t idx = static_cast<int64_t>(off + j) * ld + k;
        if (mode == SD_DENSE_BF16 || mode == SD_DENSE_F16) {
          static_cast<uint16_t*>(dst)[idx] = to16(v, mode == SD_DENSE_F16);
        } else {
          static_cast<float*>(dst)[idx] = v;
        }
      }
    }
  }
}

// Synthetic weights: w(j,k) = (2u-1)*scale, u from a counter hash; written
// straight into the target layout.
__global__ void synth_weight_kernel(int in, int out, void* dst, int64_t ld, int off, int mode,
                                    uint64_t salt, float scale) {
  const int64_t n = static_cast<int64_t>(in) * out;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e % out), k = static_cast<int>(e / out);
    const float v = synth_value(salt + static_cast<uint64_t>(e)) * scale;
    if (mode == SD_DENSE_EXACT_F32) {
      static_cast<float*>(dst)[static_cast<int64_t>(k) * ld + off + j] = v;
    } else if (mode == SD_DENSE_BF16 || mode == SD_DENSE_F16) {
      static_cast<uint16_t*>(dst)[static_cast<int64_t>(off + j) * ld + k] = to16(v, mode == SD_DENSE_F16);
    } else {
      static_cast<float*>(dst)[static_cast<int64_t>(off + j) * ld + k] = v;
    }
  }
}

__global__ void synth_embedding_kernel(int64_t n, float* dst, uint64_t salt) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    dst[e] = synth_value(salt + static_cast<uint64_t>(e));
  }
}

}  // namespace

int Weights::out_dim(int which) const {
  switch (which) {
    case 0: return spec_.qkv_width();
    case 1: return spec_.D;
    case 2:
    case 3: return spec_.kv_width();
    case 4: return spec_.D;
    case 5: return spec_.F;
    case 6: return spec_.D;
    case 7: return spec_.V;
    default: fail(SD_ERR_CONFIG, "bad weight index");
  }
}

int Weights::in_dim(int which) const { return which == 6 ? spec_.F : spec_.D; }

int64_t Weights::weight_bytes(int which) const {
  const int64_t es = mode_ == SD_DENSE_BF16 || mode_ == SD_DENSE_F16 ? 2 : 4;
  return es * out_dim(which) * in_dim(which);
}

void Weights::alloc() {
  DeviceGuard dg(device_);
  const size_t es = mode_ == SD_DENSE_BF16 || mode_ == SD_DENSE_F16 ? 2 : 4;
  size_t off = 0;
  auto take = [&](size_t elems) {
    const size_t o = off;
    off += (elems * es + 255) / 256 * 256;
    return o;
  };
  off_.assign(static_cast<size_t>(spec_.L) * 8, 0);
  for (int l = 0; l < spec_.L; ++l) {
    off_[l * 8 + 0] = take(static_cast<size_t>(spec_.D) * spec_.qkv_width());
    off_[l * 8 + 4] = take(static_cast<size_t>(spec_.D) * spec_.D);
    off_[l * 8 + 5] = take(static_cast<size_t>(spec_.D) * spec_.F);
    off_[l * 8 + 6] = take(static_cast<size_t>(spec_.F) * spec_.D);
  }
  head_off_ = take(static_cast<size_t>(spec_.D) * spec_.V);
  SD_CUDA(cudaMalloc(&blob_, off));
  SD_CUDA(cudaMalloc(&emb_, static_cast<size_t>(spec_.D) * spec_.V * sizeof(float)));
}

const void* Weights::tensor(int layer, int which) const {
  const uint8_t* b = static_cast<const uint8_t*>(blob_);
  if (which == 7) return b + head_off_;
  const size_t es = mode_ == SD_DENSE_BF16 || mode_ == SD_DENSE_F16 ? 2 : 4;
  const int D = spec_.D, kvw = spec_.kv_width();
  const size_t base = off_[static_cast<size_t>(layer) * 8 + (which <= 3 ? 0 : which)];
  if (which <= 3) {
    // slice of the fused qkv tensor: exact mode offsets columns, tensor modes rows
    const size_t slice = which == 0 ? 0 : which == 1 ? 0 : which == 2 ? D : static_cast<size_t>(D) + kvw;
    const size_t elem_off = mode_ == SD_DENSE_EXACT_F32 ? slice : slice * D;
    return b + base + elem_off * es;
  }
  return b + base;
}

Weights::Weights(const Spec& spec, const float* const* tensors, int mode, int device)
    : spec_(spec), mode_(mode), device_(device) {
  if (mode < SD_DENSE_EXACT_F32 || mode > SD_DENSE_F16) fail(SD_ERR_CONFIG, "unknown dense mode");
  alloc();
  DeviceGuard dg(device_);
  const int D = spec.D, F = spec.F, V = spec.V, kvw = spec.kv_width();
  SD_CUDA(cudaMemcpy(emb_, tensors[0], static_cast<size_t>(D) * V * 4, cudaMemcpyHostToDevice));
  DevBuf tmp;
  auto pack = [&](const float* host, int in, int out, void* dst, int64_t ld, int off) {
    const size_t bytes = static_cast<size_t>(in) * out * 4;
    tmp.get(bytes);
    SD_CUDA(cudaMemcpy(tmp.p, host, bytes, cudaMemcpyHostToDevice));
    dim3 grid((out + 31) / 32, (in + 31) / 32);
    pack_kernel<<<grid, dim3(32, 8)>>>(static_cast<const float*>(tmp.p), in, out, dst, ld, off, mode_);
    SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
  };
  uint8_t* b = static_cast<uint8_t*>(blob_);
  for (int l = 0; l < spec.L; ++l) {
    const float* const* t = tensors + 1 + 6 * l;
    void* qkv = b + off_[l * 8 + 0];
    const int64_t ld_qkv = mode == SD_DENSE_EXACT_F32 ? spec.qkv_width() : D;
    pack(t[0], D, D, qkv, ld_qkv, 0);
    pack(t[1], D, kvw, qkv, ld_qkv, D);
    pack(t[2], D, kvw, qkv, ld_qkv, D + kvw);
    pack(t[3], D, D, b + off_[l * 8 + 4], D, 0);
    pack(t[4], D, F, b + off_[l * 8 + 5], mode == SD_DENSE_EXACT_F32 ? F : D, 0);
    pack(t[5], F, D, b + off_[l * 8 + 6], mode == SD_DENSE_EXACT_F32 ? D : F, 0);
  }
  pack(tensors[1 + 6 * spec.L], D, V, b + head_off_, mode == SD_DENSE_EXACT_F32 ? V : D, 0);
  SD_CUDA(cudaDeviceSynchronize());
}

Weights::Weights(const Spec& spec, int mode, uint64_t seed, int device)
    : spec_(spec), mode_(mode), device_(device) {
  if (mode < SD_DENSE_EXACT_F32 || mode > SD_DENSE_F16) fail(SD_ERR_CONFIG, "unknown dense mode");
  alloc();
  DeviceGuard dg(device_);
  const int D = spec.D, F = spec.F, V = spec.V, kvw = spec.kv_width();
  const float ds = 1.0f / std::sqrt(static_cast<float>(D));
  const float ms = 1.0f / std::sqrt(static_cast<float>(F));
  uint64_t salt = mix64(seed);
  auto gen = [&](int in, int out, void* dst, int64_t ld, int off, float scale) {
    synth_weight_kernel<<<148 * 8, 256>>>(in, out, dst, ld, off, mode_, salt, scale);
    SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
    salt = mix64(salt);
  };
  synth_embedding_kernel<<<148 * 8, 256>>>(static_cast<int64_t>(D) * V, emb_, salt);
  salt = mix64(salt);
  uint8_t* b = static_cast<uint8_t*>(blob_);
  for (int l = 0; l < spec.L; ++l) {
    void* qkv = b + off_[l * 8 + 0];
    const int64_t ld_qkv = mode == SD_DENSE_EXACT_F32 ? spec.qkv_width() : D;
    gen(D, D, qkv, ld_qkv, 0, ds);
    gen(D, kvw, qkv, ld_qkv, D, ds);
    gen(D, kvw, qkv, ld_qkv, D + kvw, ds);
    gen(D, D, b + off_[l * 8 + 4], D, 0, ds);
    gen(D, F, b + off_[l * 8 + 5], mode == SD_DENSE_EXACT_F32 ? F : D, 0, ds);
    gen(F, D, b + off_[l * 8 + 6], mode == SD_DENSE_EXACT_F32 ? D : F, 0, ms);
  }
  gen(D, V, b + head_off_, mode == SD_DENSE_EXACT_F32 ? V : D, 0, ds);
  SD_CUDA(cudaDeviceSynchronize());
}

namespace {

// UniformSource (core.cpp:72-93): std::mt19937 seeded with
// uint32(seed ^ (seed >> 32)); u = (gen() >> 8) * 2^-24; value (2u - 1) *
// scale; tensors filled in memory (Eigen column-major) order. The 624-word
// twist is done in bulk and the tempering in a loop the compiler vectorizes
// (~1 ns per value; bit-identical to std::mt19937's stream).
class Mt19937Source {
 public:
  explicit Mt19937Source(uint64_t seed) {
    s_[0] = static_cast<uint32_t>(seed ^ (seed >> 32));
    for (int k = 1; k < 624; ++k) s_[k] = 1812433253u * (s_[k - 1] ^ (s_[k - 1] >> 30)) + static_cast<uint32_t>(k);
    i_ = 624;
  }
  void fill(float* out, size_t n, float scale) {
    size_t o = 0;
    while (o < n) {
      if (i_ == 624) twist();
      const size_t m = std::min<size_t>(static_cast<size_t>(624 - i_), n - o);
      const uint32_t* st = s_ + i_;
      for (size_t k = 0; k < m; ++k) {
        uint32_t y = st[k];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        out[o + k] = (2.0f * (static_cast<float>(y >> 8) * 0x1p-24f) - 1.0f) * scale;
      }
      i_ += static_cast<int>(m);
      o += m;
    }
  }

 private:
  void twist() {
    auto mix = [](uint32_t a, uint32_t b, uint32_t c) {
      const uint32_t y = (a & 0x80000000u) | (b & 0x7fffffffu);
      return c ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    };
    for (int k = 0; k < 227; ++k) s_[k] = mix(s_[k], s_[k + 1], s_[k + 397]);
    for (int k = 227; k < 623; ++k) s_[k] = mix(s_[k], s_[k + 1], s_[k - 227]);
    s_[623] = mix(s_[623], s_[0], s_[396]);
    i_ = 0;
  }
  uint32_t s_[624];
  int i_;
};

}  // namespace

// seed_random_weights (core.cpp:97-127): the reference's generator on the
// host, streamed tensor by tensor through two pinned chunks into a device
// staging copy of the reference storage, then packed into the mode's layout.
Weights::Weights(const Spec& spec, int mode, uint64_t seed, int device, SeedRandom)
    : spec_(spec), mode_(mode), device_(device) {
  if (mode < SD_DENSE_EXACT_F32 || mode > SD_DENSE_F16) fail(SD_ERR_CONFIG, "unknown dense mode");
  alloc();
  DeviceGuard dg(device_);
  const int D = spec.D, F = spec.F, V = spec.V, kvw = spec.kv_width();
  const float ds = 1.0f / std::sqrt(static_cast<float>(D));
  const float ms = 1.0f / std::sqrt(static_cast<float>(F));
  constexpr size_t kChunk = size_t{1} << 23;  // floats per pinned chunk (32 MB)
  float* pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  SD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    SD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pin[i]), kChunk * 4, cudaHostAllocDefault));
    SD_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  }
  Mt19937Source src(seed);
  int cur = 0;
  // the next n values of the stream into dst (device), in order
  auto stream_into = [&](float* dst, size_t n, float scale) {
    for (size_t o = 0; o < n; o += kChunk) {
      const size_t m = std::min(kChunk, n - o);
      SD_CUDA(cudaEventSynchronize(ev[cur]));  // the chunk's previous copy is done
      src.fill(pin[cur], m, scale);
      SD_CUDA(cudaMemcpyAsync(dst + o, pin[cur], m * 4, cudaMemcpyHostToDevice, st));
      SD_CUDA(cudaEventRecord(ev[cur], st));
      cur ^= 1;
    }
  };
  DevBuf tmp;
  auto gen = [&](int in, int out, void* dst, int64_t ld, int off, float scale) {
    const size_t n = static_cast<size_t>(in) * out;
    tmp.get(n * 4);
    stream_into(static_cast<float*>(tmp.p), n, scale);
    dim3 grid((out + 31) / 32, (in + 31) / 32);
    pack_kernel<<<grid, dim3(32, 8), 0, st>>>(static_cast<const float*>(tmp.p), in, out, dst, ld, off, mode_);
    SD_CUDA(cudaGetLastError());
    ::sd::count_launch();
    SD_CUDA(cudaStreamSynchronize(st));  // tmp is reused by the next tensor
  };
  try {
    stream_into(emb_, static_cast<size_t>(D) * V, 1.0f);  // embedding (D x V), scale 1
    uint8_t* b = static_cast<uint8_t*>(blob_);
    for (int l = 0; l < spec.L; ++l) {
      void* qkv = b + off_[l * 8 + 0];
      const int64_t ld_qkv = mode == SD_DENSE_EXACT_F32 ? spec.qkv_width() : D;
      gen(D, D, qkv, ld_qkv, 0, ds);           // w_q
      gen(D, kvw, qkv, ld_qkv, D, ds);         // w_k
      gen(D, kvw, qkv, ld_qkv, D + kvw, ds);   // w_v
      gen(D, D, b + off_[l * 8 + 4], D, 0, ds);                                 // w_o
      gen(D, F, b + off_[l * 8 + 5], mode == SD_DENSE_EXACT_F32 ? F : D, 0, ds);  // w_mlp_in
      gen(F, D, b + off_[l * 8 + 6], mode == SD_DENSE_EXACT_F32 ? D : F, 0, ms);  // w_mlp_out
    }
    gen(D, V, b + head_off_, mode == SD_DENSE_EXACT_F32 ? V : D, 0, ds);  // head (V x D)
    SD_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    cudaStreamSynchronize(st);
    for (int i = 0; i < 2; ++i) {
      cudaFreeHost(pin[i]);
      cudaEventDestroy(ev[i]);
    }
    cudaStreamDestroy(st);
    throw;
  }
  for (int i = 0; i < 2; ++i) {
    cudaFreeHost(pin[i]);
    cudaEventDestroy(ev[i]);
  }
  cudaStreamDestroy(st);
}

Weights::~Weights() {
  DeviceGuard dg(device_);
  cudaFree(blob_);
  cudaFree(emb_);
}

void Weights::linear(int layer, int which, int B, const float* x, int64_t ldx,
                     const act16* xb, int64_t ldxb, float* y, int64_t ldy,
                     act16* yb, int64_t ldyb, int epi, const float* res, int64_t ldr,
                     cudaStream_t s, int max_ctas) const {
  if (which != 7 && (layer < 0 || layer >= spec_.L)) fail(SD_ERR_CONFIG, "layer out of range");
  const int in = in_dim(which), out = out_dim(which);
  const void* W = tensor(layer, which);
  if (mode_ == SD_DENSE_EXACT_F32) {
    int64_t ldw = out;
    if (which <= 3) ldw = spec_.qkv_width();
    launch_linear_exact(B, in, out, x, ldx, static_cast<const float*>(W), ldw, y, ldy, epi, res, ldr, s);
    if (yb) launch_to_16(B, out, y, ldy, yb, ldyb, 0, s);
    return;
  }
  const GemmArgs g = gemm_args(layer, which, B, x, ldx, xb, ldxb, y, ldy, yb, ldyb, epi, res, ldr, max_ctas);
  launch_gemm_sm100(g, s);
}

GemmArgs Weights::gemm_args(int layer, int which, int B, const float* x, int64_t ldx, const act16* xb,
                            int64_t ldxb, float* y, int64_t ldy, act16* yb, int64_t ldyb, int epi,
                            const float* res, int64_t ldr, int max_ctas) const {
  if (mode_ == SD_DENSE_EXACT_F32) fail(SD_ERR_INTERNAL, "gemm_args: exact mode has no tensor-core GEMM");
  if (which != 7 && (layer < 0 || layer >= spec_.L)) fail(SD_ERR_CONFIG, "layer out of range");
  GemmArgs g{};
  g.M = B;
  g.N = out_dim(which);
  g.K = in_dim(which);
  g.kind = mode_;
  if (mode_ == SD_DENSE_BF16 || mode_ == SD_DENSE_F16) {
    if (!xb) fail(SD_ERR_INTERNAL, "kind::f16 GEMM needs a 16-bit A operand");
    g.A = xb;
    g.lda = ldxb;
  } else {
    g.A = x;
    g.lda = ldx;
  }
  g.B = tensor(layer, which);
  g.ldb = g.K;
  g.C = y;
  g.ldc = ldy;
  g.Cb = yb;
  g.ldcb = ldyb;
  g.epi = epi;
  g.res = res;
  g.ldr = ldr;
  g.max_ctas = max_ctas;
  if (!gemm_sm100_supported(g)) fail(SD_ERR_CONFIG, "shape not supported by the tcgen05 GEMM");
  return g;
}

// ============================================================= scheduler ===
int micro_batch_size(int b, int f, int s) {  // scheduler.cpp:10-21
  if (b < 1 || f < 1 || s < 1) fail(SD_ERR_ADMISSION, "micro_batch_size: arguments must be >= 1");
  const int64_t p = static_cast<int64_t>(b) * f;
  if (p < s) {
    fail(SD_ERR_ADMISSION, "interval too short for target batch: B*F = " + std::to_string(p) +
                               " < S = " + std::to_string(s));
  }
  return static_cast<int>(std::max<int64_t>(1, p / s));
}

LoadTracker::LoadTracker(int64_t limit) : limit_(limit) {
  if (limit < 1) fail(SD_ERR_ADMISSION, "load limit must be >= 1");
}

int64_t LoadTracker::earliest_start(int m, int s) const {  // scheduler.cpp:44-60
  if (static_cast<int64_t>(m) * s > limit_) fail(SD_ERR_ADMISSION, "micro-batch exceeds load limit");
  int64_t r = cur_;
  for (size_t i = 0; i < b_.size(); ++i) r = std::max(r, b_[i].end - (limit_ - w_[i]) / m);
  return r;
}

int LoadTracker::add(int64_t t, int m, int s) {  // scheduler.cpp:62-106
  if (m < 1 || s < 1) fail(SD_ERR_ADMISSION, "add_micro_batch: size and target length must be >= 1");
  if (t < cur_) fail(SD_ERR_ADMISSION, "cannot admit in the past");
  const int64_t own = static_cast<int64_t>(m) * s;
  if (own > limit_) fail(SD_ERR_ADMISSION, "admission rejected: batch workload exceeds limit");
  for (size_t i = 0; i < b_.size(); ++i) {
    if (b_[i].end > t && w_[i] + (b_[i].end - t) * m > limit_) {
      fail(SD_ERR_ADMISSION, "admission rejected: end-step workload of batch " +
                                 std::to_string(b_[i].id) + " exceeds the limit");
    }
  }
  for (size_t i = 0; i < b_.size(); ++i) {
    if (b_[i].end > t) w_[i] += (b_[i].end - t) * m;
  }
  b_.push_back(MB{next_id_, m, t, t + s});
  w_.push_back(own);
  return next_id_++;
}

LoadTracker::Plan LoadTracker::step() {  // scheduler.cpp:108-135
  cur_ += 1;
  Plan p;
  p.step = cur_;
  for (const MB& mb : b_) {
    if (mb.start < cur_ && cur_ <= mb.end) {
      p.active_ids.push_back(mb.id);
      p.total_load += static_cast<int64_t>(mb.size) * (cur_ - mb.start);
      if (mb.end == cur_) p.ending.push_back(mb.id);
    }
  }
  size_t keep = 0;
  for (size_t i = 0; i < b_.size(); ++i) {
    if (b_[i].end > cur_) {
      b_[keep] = b_[i];
      w_[keep] = w_[i];
      ++keep;
    }
  }
  b_.resize(keep);
  w_.resize(keep);
  return p;
}

namespace {
int admission_size(int64_t k, int64_t b, int64_t f, int64_t s) {
  return static_cast<int>(((k + 1) * b * f) / s - (k * b * f) / s);
}
int64_t ramp_limit(int64_t u, int64_t b, int64_t s, int64_t f) {
  const double steady = static_cast<double>(b) * (s + f) / 2.0;
  if (u >= s) return static_cast<int64_t>(steady);
  const double bd = static_cast<double>(b);
  const double v = bd * f + bd * static_cast<double>(u) * (2.0 * s - f - u) / (2.0 * s);
  return static_cast<int64_t>(std::floor(v + 1e-9));
}
}  // namespace

std::vector<Admission> cold_start_schedule(int b, int s, int f, int mode, int64_t horizon) {
  micro_batch_size(b, f, s);  // scheduler.cpp:179-214
  std::vector<Admission> out;
  if (mode == 0) {
    int64_t k = 0;
    for (int64_t t = 0; t <= horizon; t += f, ++k) {
      const int m = admission_size(k, b, f, s);
      if (m > 0) out.push_back({t, m, s});
    }
    return out;
  }
  if (mode != 1) fail(SD_ERR_CONFIG, "unknown cold start mode");
  const int64_t steady = static_cast<int64_t>(b) * (s + f) / 2;
  LoadTracker tr(std::max<int64_t>(1, ramp_limit(0, b, s, f)));
  int64_t k = 0;
  int64_t limit = 0;
  for (int64_t u = 0; u <= horizon; ++u) {
    limit = std::max<int64_t>(1, std::min(steady, ramp_limit(u, b, s, f)));
    tr.set_limit(limit);
    for (;;) {
      const int m = admission_size(k, b, f, s);
      if (static_cast<int64_t>(m) * s > limit) break;
      if (tr.earliest_start(m, s) != tr.current()) break;
      tr.add(tr.current(), m, s);
      out.push_back({tr.current(), m, s});
      ++k;
    }
    tr.step();
  }
  return out;
}

// ============================================================== ShardMap ===
namespace {
std::pair<int, int> range_of(int index, int groups, int total) {
  const int base = total / groups, rem = total % groups;
  return {index * base + std::min(index, rem), base + (index < rem ? 1 : 0)};
}
int group_of_head(int head, int groups, int total) {
  for (int g = 0; g < groups; ++g) {
    auto [st, c] = range_of(g, groups, total);
    if (head >= st && head < st + c) return g;
  }
  fail(SD_ERR_CONFIG, "head index out of range");
}
void check_map(int mode, int heads, int workers) {
  if (workers < 1) fail(SD_ERR_CONFIG, "shard map needs at least one worker");
  if (heads < 1) fail(SD_ERR_CONFIG, "shard map needs at least one head");
  if (mode < 0 || mode > 2) fail(SD_ERR_CONFIG, "invalid shard mode");
  if (mode == SD_SHARD_BY_HEAD && workers > heads) {
    fail(SD_ERR_CONFIG, "by-head sharding cannot use more workers than heads");
  }
}
}  // namespace

int shard_worker_for(int mode, int heads, int workers, uint64_t seq, int head) {
  check_map(mode, heads, workers);
  if (head < 0 || head >= heads) fail(SD_ERR_CONFIG, "head index out of range");
  switch (mode) {
    case SD_SHARD_BY_SEQUENCE: return static_cast<int>(mix64(seq) % static_cast<uint64_t>(workers));
    case SD_SHARD_BY_HEAD: return group_of_head(head, workers, heads);
    default: {
      const int hg_n = std::gcd(workers, heads);
      const int sg_n = workers / hg_n;
      return group_of_head(head, hg_n, heads) * sg_n +
             static_cast<int>(mix64(seq) % static_cast<uint64_t>(sg_n));
    }
  }
}

std::pair<int, int> shard_head_range(int mode, int heads, int workers, int w) {
  check_map(mode, heads, workers);
  if (w < 0 || w >= workers) fail(SD_ERR_CONFIG, "worker index out of range");
  switch (mode) {
    case SD_SHARD_BY_SEQUENCE: return {0, heads};
    case SD_SHARD_BY_HEAD: return range_of(w, workers, heads);
    default: {
      const int hg_n = std::gcd(workers, heads);
      return range_of(w / (workers / hg_n), hg_n, heads);
    }
  }
}

// ================================================================= drive ===
DriveResult drive(StepComputation& e, const sd_drive_config& c) {
  if (c.batch < 1 || c.target_len < 1 || c.interval < 1) {
    fail(SD_ERR_CONFIG, "generation config: batch, target_len, interval must be >= 1");
  }
  const auto t0 = std::chrono::steady_clock::now();
  struct {
    int D, V;
  } s{e.model_dim(), e.vocab()};
  const bool to_completion = c.steps <= 0;
  int64_t adm_h;
  if (to_completion) {
    const int m = micro_batch_size(c.batch, c.interval, c.target_len);
    const int64_t waves = std::max<int64_t>(1, (c.batch + m - 1) / m);
    adm_h = (waves - 1) * c.interval;
  } else {
    adm_h = c.steps;
  }
  std::vector<Admission> adm = cold_start_schedule(c.batch, c.target_len, c.interval, c.cold_start, adm_h);
  if (to_completion) {
    int64_t total = 0;
    std::vector<Admission> tr;
    for (Admission a : adm) {
      if (total >= c.batch) break;
      a.size = static_cast<int>(std::min<int64_t>(a.size, c.batch - total));
      total += a.size;
      tr.push_back(a);
    }
    adm = tr;
  }
  const int64_t horizon = to_completion ? (adm.empty() ? 0 : adm.back().step + c.target_len) : c.steps;
  int64_t limit = c.load_limit;
  if (limit <= 0) {  // workers.cpp:536-543
    const int64_t b = c.batch, S = c.target_len, f = c.interval;
    limit = (S % f == 0 && (b * f) % S == 0) ? b * (S + f) / 2 : b * S + b * f;
  }
  LoadTracker tr(limit);
  std::unordered_map<int, std::vector<uint64_t>> batch_seqs;
  std::unordered_map<uint64_t, std::pair<int, int>> states;  // (current, target)
  std::unordered_map<uint64_t, int> last;
  uint64_t next_id = 1;
  size_t next_adm = 0;
  auto admit_due = [&](int64_t step) {
    while (next_adm < adm.size() && adm[next_adm].step == step) {
      const Admission& a = adm[next_adm];
      const int id = tr.add(a.step, a.size, a.target);
      auto& v = batch_seqs[id];
      for (int i = 0; i < a.size; ++i) {
        const uint64_t q = next_id++;
        v.push_back(q);
        states[q] = {0, a.target};
        last[q] = static_cast<int>(mix64(c.seed ^ mix64(q)) % static_cast<uint64_t>(s.V));
      }
      ++next_adm;
    }
  };
  DriveResult res;
  admit_due(0);
  std::vector<uint64_t> ids;
  std::vector<int32_t> toks, next;
  std::vector<float> fx;
  for (int64_t u = 1; u <= horizon; ++u) {
    LoadTracker::Plan plan = tr.step();
    if (plan.active_ids.empty() && next_adm >= adm.size()) break;
    if (!plan.active_ids.empty()) {
      ids.clear();
      for (int id : plan.active_ids) for (uint64_t q : batch_seqs[id]) ids.push_back(q);
      const int B = static_cast<int>(ids.size());
      toks.resize(static_cast<size_t>(B));
      next.resize(static_cast<size_t>(B));
      for (int i = 0; i < B; ++i) toks[static_cast<size_t>(i)] = last.at(ids[static_cast<size_t>(i)]);
      if (c.record_activations) fx.resize(static_cast<size_t>(B) * s.D);
      e.compute(B, ids.data(), toks.data(), next.data(), c.record_activations ? fx.data() : nullptr);
      for (int i = 0; i < B; ++i) {
        const uint64_t q = ids[static_cast<size_t>(i)];
        last[q] = next[static_cast<size_t>(i)];
        auto& st = states.at(q);
        st.first += 1;
        if (st.first > st.second) fail(SD_ERR_LOGIC, "sequence ran past its target length");
        if (!e.owns(q)) continue;  // another rank produced this row's token
        res.steps.push_back(u);
        res.seqs.push_back(q);
        res.tokens.push_back(next[static_cast<size_t>(i)]);
        if (c.record_activations) {
          res.activations.insert(res.activations.end(), fx.begin() + static_cast<int64_t>(i) * s.D,
                                 fx.begin() + static_cast<int64_t>(i + 1) * s.D);
        }
      }
    }
    if (!plan.ending.empty()) {
      std::vector<uint64_t> retiring;
      for (int id : plan.ending) {
        auto it = batch_seqs.find(id);
        if (it == batch_seqs.end()) continue;
        for (uint64_t q : it->second) {
          if (states.at(q).first != states.at(q).second) {
            fail(SD_ERR_LOGIC, "retiring a sequence short of its target");
          }
          retiring.push_back(q);
          last.erase(q);
          states.erase(q);
        }
        batch_seqs.erase(it);
      }
      e.retire(static_cast<int>(retiring.size()), retiring.data());
    }
    admit_due(u);
  }
  res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

}  // namespace sd
