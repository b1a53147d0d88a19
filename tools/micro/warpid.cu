// Which warp slot (%warpid) each warp of two co-resident 256-thread CTAs gets.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  extern __shared__ char sm[];
  unsigned wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if ((threadIdx.x & 31) == 0) {
    int i = blockIdx.x * 8 + threadIdx.x / 32;
    out[3 * i] = smid; out[3 * i + 1] = wid; out[3 * i + 2] = blockIdx.x;
  }
  sm[threadIdx.x] = 0;
  long long t0 = clock64(); while (clock64() - t0 < 1000000) {}
}
int main() {
  int* d; cudaMalloc(&d, 3 * 296 * 8 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  k<<<296, 256, 110000>>>(d);
  int h[3 * 296 * 8]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int b = 0; b < 296; ++b) {
    if (h[3 * b * 8] != 0) continue;  // SM 0 only
    printf("cta %3d sm %d warpids:", b, h[3 * b * 8]);
    for (int w = 0; w < 8; ++w) printf(" %d", h[3 * (b * 8 + w) + 1]);
    printf("\n");
  }
}
