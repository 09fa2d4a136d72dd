// NVLink peer bandwidth probe (standalone, one process, all visible GPUs):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/p2p_bw tools/p2p_bw.cu && /tmp/p2p_bw
// Measures SM-store push, SM-load pull and copy-engine copies between GPU 0
// and GPU 1, then an all-to-all push among every GPU, each at a large size
// and at the burst size of one routed QKV GEMM epilogue.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__global__ void push(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    dst[i] = src[i];
  }
}

// all-to-all: this GPU writes n4 float4 to each of `np` destinations
struct Dsts {
  float4* d[8];
  int np;
};
__global__ void push_multi(const float4* __restrict__ src, Dsts d, size_t n4) {
  const int p = blockIdx.y;
  float4* dst = d.d[p];
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
    dst[i] = src[i];
  }
}

int main() {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) {
    std::printf("need >= 2 GPUs\n");
    return 0;
  }
  for (int a = 0; a < ng; ++a) {
    CK(cudaSetDevice(a));
    for (int b = 0; b < ng; ++b) {
      if (a != b) CK(cudaDeviceEnablePeerAccess(b, 0));
    }
  }
  const size_t big = 256ull << 20, burst = 12ull << 20;
  std::vector<float*> buf(ng), src(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&buf[g], big * 8));
    CK(cudaMalloc(&src[g], big));
    CK(cudaMemset(src[g], 1, big));
  }
  auto timed = [&](int dev, auto fn, int reps) -> double {
    cudaSetDevice(dev);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
  };
  for (size_t bytes : {big, burst}) {
    const size_t n4 = bytes / 16;
    for (int blocks : {148, 296, 592}) {
      double ms = timed(0, [&] { push<<<blocks, 512>>>((const float4*)src[0], (float4*)buf[1], n4); }, 10);
      std::printf("push  0->1 %6.1f MB grid %4d: %8.1f us %7.1f GB/s\n", bytes / 1e6, blocks, ms * 1e3,
                  bytes / ms / 1e6);
    }
    {
      double ms = timed(0, [&] { push<<<592, 512>>>((const float4*)buf[1], (float4*)src[0], n4); }, 10);
      std::printf("pull  1->0 %6.1f MB grid  592: %8.1f us %7.1f GB/s\n", bytes / 1e6, ms * 1e3, bytes / ms / 1e6);
    }
    {
      double ms = timed(0, [&] { cudaMemcpyPeerAsync(buf[1], 1, src[0], 0, bytes, 0); }, 10);
      std::printf("CE    0->1 %6.1f MB          : %8.1f us %7.1f GB/s\n", bytes / 1e6, ms * 1e3, bytes / ms / 1e6);
    }
    {
      double ms = timed(0, [&] { push<<<592, 512>>>((const float4*)src[0], (float4*)buf[0], n4); }, 10);
      std::printf("local 0->0 %6.1f MB grid  592: %8.1f us %7.1f GB/s\n", bytes / 1e6, ms * 1e3, bytes / ms / 1e6);
    }
    // all-to-all push: every GPU writes bytes/(ng-1) to each peer, concurrently
    const size_t per = bytes / (ng - 1) / 16;
    std::vector<cudaEvent_t> e0(ng), e1(ng);
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaDeviceSynchronize());
      cudaEventCreate(&e0[g]);
      cudaEventCreate(&e1[g]);
    }
    for (int rep = 0; rep < 2; ++rep) {
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        Dsts d{};
        d.np = ng - 1;
        int k = 0;
        for (int p = 0; p < ng; ++p) {
          if (p != g) d.d[k++] = (float4*)(buf[p] + (size_t)g * (bytes / 4));
        }
        cudaEventRecord(e0[g]);
        push_multi<<<dim3(148 * 2 / (ng - 1) + 1, ng - 1), 512>>>((const float4*)src[g], d, per);
        cudaEventRecord(e1[g]);
      }
      double worst = 0;
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0[g], e1[g]);
        worst = ms > worst ? ms : worst;
      }
      if (rep) {
        std::printf("a2a  x%d   %6.1f MB/GPU egress: %8.1f us %7.1f GB/s per GPU\n", ng, bytes / 1e6, worst * 1e3,
                    bytes / worst / 1e6);
      }
    }
  }
  return 0;
}
