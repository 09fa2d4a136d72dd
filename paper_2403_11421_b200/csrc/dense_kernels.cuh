// S-Part device interfaces (dense_kernels.cu, gemm_sm100.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sd {

enum Epilogue : int {
  kEpiNone = 0,      // y = acc
  kEpiResidual = 1,  // y = acc + res          (finish_block's `y += residual`, dense.cpp:60)
  kEpiSilu = 2,      // y = silu(acc)          (dense.cpp:47-49, 63-65)
};

// K7: out[b][j] = sum_k w(j,k) * x[b][k] with the reference's per-element
// operation order (k ascending, one accumulator, multiply then add, no FMA;
// dense.cpp:16-31). w is the reference storage: w(j,k) at w[k*ldw + j].
void launch_linear_exact(int B, int in, int out, const float* x, int64_t ldx, const float* w,
                         int64_t ldw, float* y, int64_t ldy, int epi, const float* res,
                         int64_t ldr, cudaStream_t s);
// x[b][:] = embedding(:, tokens[b]); embedding is D x V column-major;
// xb (optional): its 16-bit copy (fp16 when f16, else bf16)
void launch_embed(int B, int D, const int32_t* tokens, const float* emb, float* x, int64_t ldx,
                  void* xb, int f16, cudaStream_t s);
// argmax_token per row (first index wins ties, dense.cpp:78-88)
// tokens[i] from the fused-argmax keys (first maximum wins, as
// argmax_token dense.cpp:80-88); resets the keys to zero for the next launch
void launch_argmax_keys(int B, unsigned long long* keys, int32_t* tokens, cudaStream_t s);
void launch_argmax(int B, int V, const float* logits, int64_t ld, int32_t* tokens,
                   cudaStream_t s);
// counter-hash values in [-1, 1) (synth_value(salt + i)): benchmark operands
void launch_fill_synthetic(float* p, int64_t n, uint64_t salt, cudaStream_t s);
// fp32 -> 16-bit copy (the A operand of a kind::f16 GEMM; fp16 when f16, else bf16)
void launch_to_16(int rows, int cols, const float* x, int64_t ldx, void* y, int64_t ldy, int f16,
                  cudaStream_t s);

// tcgen05 GEMM: C[M][N] = A[M][K] . B[N][K]^T with fused epilogue; A, B
// K-major (bf16 / fp16 for kind::f16, fp32 bits for kind::tf32). Writes fp32 C
// and, if Cb != nullptr, a 16-bit copy (the operand format) for the next
// GEMM's A operand.
// Multi-GPU exchange fused into a producer's epilogue (dist.cpp): output row
// m is stored straight into base[rank[m]] + row[m] * ld (a peer's receive
// buffer through its CUDA IPC mapping, or this rank's own), and the last CTA
// to finish publishes flag[d][slot * 8 + self] = epoch (release, system
// scope) for every rank d in `notify`.
struct RowRoute {
  const int32_t* rank;
  const int32_t* row;
  float* base[8];
  int64_t ld;
  int32_t rows;  // rows of every base buffer (tensor-map extent)
  int64_t* flag[8];
  int32_t* done;  // grid arrival counter, zero between launches
  int64_t epoch;
  uint32_t notify;
  int slot, self;
};

// append_lane (attention.cpp:91-112) folded into the QKV GEMM's epilogue:
// the K and V columns of row r are rounded to fp16 (RNE, as the append
// kernel) and stored into the row's KV page for this layer instead of C.
struct KvAppendOut {
  uint8_t* layer_base;     // pool + layer * layer_bytes
  int64_t group_bytes, v_off;
  int32_t pos_bytes, pmask;  // bytes per position row; positions per page - 1
  const int32_t* group;    // [M] page group holding row r's position
  const int32_t* pos;      // [M] position of row r
  int32_t col_k, width;    // K columns [col_k, col_k + width), V the next width
};

struct GemmArgs {
  int M, N, K;
  const void* A;
  int64_t lda;  // elements
  const void* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
  void* Cb;      // 16-bit copy of C in the operand format (bf16 / fp16)
  int64_t ldcb;
  int epi;
  const float* res;
  int64_t ldr;
  int kind;      // SD_DENSE_BF16 (kind::f16, bf16), SD_DENSE_TF32 (kind::tf32), SD_DENSE_F16 (kind::f16, fp16)
  int max_ctas;  // SM budget of the persistent grid (0 = every SM)
  const RowRoute* route = nullptr;  // fp32 C rows routed to peers (C unused)
  // argmax_token fused into the epilogue: per row, atomicMax of (ordered
  // value << 32 | ~column) over every tile (zero before the launch); C and
  // Cb may be null. launch_argmax_keys turns the keys into tokens.
  unsigned long long* amax = nullptr;
  const KvAppendOut* kvapp = nullptr;  // QKV rows' K/V straight into the KV pages (C keeps q)
};
bool gemm_sm100_supported(const GemmArgs& g);
void launch_gemm_sm100(const GemmArgs& g, cudaStream_t s);


}  // namespace sd
