// FP64 pipe peak probe (diagnostics for the roofline denominator; not on the hot path).
// MEASURED_PEAKS.json carries HBM and bf16 peaks only, so bench.py measures the
// FP64 FMA peak on the same box with this dependent-chain DFMA kernel.
#include <cuda_runtime.h>

#include "../../include/curvalign_cuda.h"

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_kernel(double* sink, int iters, double a, double b) {
  double v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fma(v[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 1.2345) sink[threadIdx.x] = s;  // keep the chains alive
}

}  // namespace

extern "C" int cva_probe_fp64_tflops(double* tflops) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return CVA_CUDA_ERROR;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(double)) != cudaSuccess) return CVA_CUDA_ERROR;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(sink, iters, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) dfma_kernel<<<blocks, threads>>>(sink, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess || ms <= 0.f) return CVA_CUDA_ERROR;
  const double flops = 2.0 * kChains * (double)iters * threads * blocks * reps;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return CVA_OK;
}
