// S-Part CUDA-core kernels: the exact-order fp32 linear (K7), embedding
// gather, argmax, bf16 staging.
#include <cuda_bf16.h>

#include <cfloat>

#include "dense_kernels.cuh"
#include "pdl.cuh"
#include "sd_common.h"

namespace sd {

namespace {

constexpr int kRows = 8;     // batch rows per block
constexpr int kCols = 128;   // output columns per block (one per thread)
constexpr int kKTile = 64;   // x tile staged in shared memory

// One thread owns one output column j for kRows batch rows. For each k the
// weight element w(j,k) is one coalesced load across the block (the
// reference's column-major storage puts consecutive j at consecutive
// addresses) and the per-element sequence is acc = acc + w*x with explicit
// round-to-nearest multiply and add, i.e. no FMA contraction — bitwise
// identical to apply_linear built with -ffp-contract=off (dense.cpp:16-31).
__global__ void __launch_bounds__(kCols) linear_exact_kernel(int B, int in, int out,
                                                             const float* __restrict__ x, int64_t ldx,
                                                             const float* __restrict__ w, int64_t ldw,
                                                             float* __restrict__ y, int64_t ldy, int epi,
                                                             const float* __restrict__ res, int64_t ldr) {
  pdl_trigger();
  pdl_wait();
  __shared__ float xs[kRows][kKTile];
  const int j = blockIdx.x * kCols + threadIdx.x;
  const int b0 = blockIdx.y * kRows;
  float acc[kRows];
#pragma unroll
  for (int r = 0; r < kRows; ++r) acc[r] = 0.0f;
  for (int k0 = 0; k0 < in; k0 += kKTile) {
    const int kt = min(kKTile, in - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kRows * kKTile; e += kCols) {
      const int r = e / kKTile, kk = e % kKTile;
      xs[r][kk] = (b0 + r < B && kk < kt) ? x[static_cast<int64_t>(b0 + r) * ldx + k0 + kk] : 0.0f;
    }
    __syncthreads();
    if (j < out) {
      for (int kk = 0; kk < kt; ++kk) {
        const float wv = w[static_cast<int64_t>(k0 + kk) * ldw + j];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = __fadd_rn(acc[r], __fmul_rn(wv, xs[r][kk]));
      }
    }
  }
  if (j >= out) return;
#pragma unroll
  for (int r = 0; r < kRows; ++r) {
    const int b = b0 + r;
    if (b >= B) break;
    float v = acc[r];
    if (epi == kEpiResidual) {
      v = __fadd_rn(v, res[static_cast<int64_t>(b) * ldr + j]);
    } else if (epi == kEpiSilu) {
      v = __fdiv_rn(v, __fadd_rn(1.0f, expf(-v)));
    }
    y[static_cast<int64_t>(b) * ldy + j] = v;
  }
}

__global__ void embed_kernel(int B, int D, const int32_t* __restrict__ tokens,
                             const float* __restrict__ emb, float* __restrict__ x, int64_t ldx,
                             uint16_t* __restrict__ xb, int f16) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  const float* col = emb + static_cast<int64_t>(tokens[b]) * D;  // column-major D x V
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const float v = col[d];
    x[static_cast<int64_t>(b) * ldx + d] = v;
    if (xb) xb[static_cast<int64_t>(b) * D + d] = to16(v, f16);
  }
}

// First index wins ties: reduce (value, index) preferring the larger value,
// then the smaller index. NaN logits never win (the reference's `>` test).
__global__ void argmax_kernel(int V, const float* __restrict__ logits, int64_t ld,
                              int32_t* __restrict__ tokens) {
  pdl_trigger();
  pdl_wait();
  const float* row = logits + static_cast<int64_t>(blockIdx.x) * ld;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
    if (v > bv || (v == bv && i < bi)) {
      bv = v;
      bi = i;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, sh);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, sh);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, sh);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, sh);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) tokens[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
  }
}

__global__ void to16_kernel(int rows, int cols, const float* __restrict__ x, int64_t ldx,
                            uint16_t* __restrict__ y, int64_t ldy, int f16) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.y;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
    y[static_cast<int64_t>(r) * ldy + c] = to16(x[static_cast<int64_t>(r) * ldx + c], f16);
  }
}

}  // namespace

__global__ void fill_synthetic_kernel(float* p, int64_t n, uint64_t salt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    p[i] = synth_value(salt + static_cast<uint64_t>(i));
  }
}

void launch_fill_synthetic(float* p, int64_t n, uint64_t salt, cudaStream_t s) {
  if (n <= 0) return;
  fill_synthetic_kernel<<<148 * 4, 256, 0, s>>>(p, n, salt);
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

void launch_linear_exact(int B, int in, int out, const float* x, int64_t ldx, const float* w,
                         int64_t ldw, float* y, int64_t ldy, int epi, const float* res,
                         int64_t ldr, cudaStream_t s) {
  if (B == 0 || out == 0) return;
  dim3 grid((out + kCols - 1) / kCols, (B + kRows - 1) / kRows);
  SD_CUDA(launch_pdl(linear_exact_kernel, grid, dim3(kCols), 0, s, 1, B, in, out, x, ldx, w, ldw, y, ldy, epi, res, ldr));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

void launch_embed(int B, int D, const int32_t* tokens, const float* emb, float* x, int64_t ldx,
                  void* xb, int f16, cudaStream_t s) {
  if (B == 0) return;
  SD_CUDA(launch_pdl(embed_kernel, dim3(B), dim3(256), 0, s, 1, B, D, tokens, emb, x, ldx,
                     static_cast<uint16_t*>(xb), f16));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

__global__ void argmax_keys_kernel(int B, unsigned long long* keys, int32_t* tokens) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) {
    const unsigned long long k = keys[i];
    tokens[i] = k ? static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k)) : 0;  // all-NaN row: index 0
    keys[i] = 0;
  }
  pdl_trigger();
}

void launch_argmax_keys(int B, unsigned long long* keys, int32_t* tokens, cudaStream_t s) {
  if (B <= 0) return;
  SD_CUDA(launch_pdl(argmax_keys_kernel, dim3((B + 127) / 128), dim3(128), 0, s, 1, B, keys, tokens));
  SD_CUDA(cudaGetLastError());
  count_launch();
}

void launch_argmax(int B, int V, const float* logits, int64_t ld, int32_t* tokens,
                   cudaStream_t s) {
  if (B == 0) return;
  SD_CUDA(launch_pdl(argmax_kernel, dim3(B), dim3(512), 0, s, 1, V, logits, ld, tokens));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

void launch_to_16(int rows, int cols, const float* x, int64_t ldx, void* y, int64_t ldy, int f16,
                  cudaStream_t s) {
  if (rows == 0 || cols == 0) return;
  dim3 grid((cols + 255) / 256 < 64 ? (cols + 255) / 256 : 64, rows);
  SD_CUDA(launch_pdl(to16_kernel, grid, dim3(256), 0, s, 1, rows, cols, x, ldx, static_cast<uint16_t*>(y), ldy,
                     f16));
  SD_CUDA(cudaGetLastError());
  ::sd::count_launch();
}

}  // namespace sd
