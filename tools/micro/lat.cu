// Latency / throughput probes for the FP64 and shared-memory ops the C1 kernel chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* o, double a, double b, int it, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) { x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); }
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dadd(double* o, double a, double b, int it, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) { x = x + b; x = x - a; x = x + b; x = x - a; }
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_rcp(double* o, double a, double b, int it, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) {
    double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r;
  }
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double* o, double a, double b, int it, long long* cyc) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) { j = idx[j]; j = idx[j]; j = idx[j]; j = idx[j]; }
  long long t1 = clock64();
  o[threadIdx.x] = j; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* o, double a, double b, int it, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) { x = __shfl_xor_sync(~0u, x, 1); x = __shfl_xor_sync(~0u, x, 2); x = __shfl_xor_sync(~0u, x, 4); x = __shfl_xor_sync(~0u, x, 8); }
  long long t1 = clock64();
  o[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: many independent chains per thread, warps per SM = blockDim/32
__global__ void k_dfma_tp(double* o, double a, double b, int it, long long* cyc) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  __syncthreads();
  long long t1 = clock64();
  o[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* o, double a, double b, int it, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
typedef void (*K)(double*, double, double, int, long long*);
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  struct { const char* n; K k; int threads; double per; } ks[] = {
    {"dfma dep latency", k_dfma, 32, 4}, {"dadd dep latency", k_dadd, 32, 4}, {"rcp64h dep latency", k_rcp, 32, 4},
    {"lds dep latency", k_lds, 32, 4}, {"shfl dep latency", k_shfl, 32, 4},
    {"dfma tp (cyc per warp-inst per SM), 1 warp", k_dfma_tp, 32, 8}, {"dfma tp 4 warps", k_dfma_tp, 128, 8},
    {"dfma tp 8 warps", k_dfma_tp, 256, 8}, {"dfma tp 16 warps", k_dfma_tp, 512, 8},
    {"bar.sync 256 thr", k_bar, 256, 4}, {"bar.sync 512 thr", k_bar, 512, 4}};
  const int it = 4096;
  for (auto& k : ks) {
    k.k<<<1, k.threads>>>(o, 1.0000001, 0.9999999, it, c);
    k.k<<<1, k.threads>>>(o, 1.0000001, 0.9999999, it, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double per = (double)h / (it * k.per);
    if (k.k == k_dfma_tp) per /= (k.threads / 32);
    printf("%-44s %.2f cycles\n", k.n, per);
  }
  return 0;
}
