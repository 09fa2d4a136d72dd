#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out) {
  __shared__ __align__(128) uint8_t sm[16 * 32];
  for (int i = threadIdx.x; i < 16 * 32; i += 32) sm[i] = (uint8_t)((i / 32) * 16 + (i % 32));  // row r (pitch 32), col c
  __syncwarp();
  const int lane = threadIdx.x;
  uint32_t addr = (uint32_t)__cvta_generic_to_shared(sm + (lane % 16) * 32);
  uint32_t r0, r1;
  asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
  out[lane * 2] = r0;
  out[lane * 2 + 1] = r1;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 64 * 4);
  k<<<1, 32>>>(d);
  uint32_t h[64]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int l = 0; l < 32; ++l) {
    printf("lane %2d:", l);
    for (int j = 0; j < 2; ++j) for (int b = 0; b < 4; ++b) { int v = (h[2*l+j] >> (8*b)) & 0xff; printf(" (%d,%d)", v / 16, v % 16); }
    printf("\n");
  }
}
