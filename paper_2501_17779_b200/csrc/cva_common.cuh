// Shared device helpers for the curvalign sm_100a kernels.
//
// Layout convention (matches curvalign::Point2, proj/include/curvalign/geometry.hpp:9-33):
// a curve of n nodes is n interleaved (x, y) doubles, read and written as double2
// (16-byte vector accesses); the complex sequence z = x + i y is the same bytes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cva {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- complex math
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulconj(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }
// multiply by +i
__device__ __forceinline__ double2 cmul_pi(double2 a) { return make_double2(-a.y, a.x); }

// ------------------------------------------------------- fast fp64 rcp / sqrt
// Fast reciprocal: MUFU seed + one cubic step (<= 1 ulp; the reference's
// divisions are correctly rounded, the difference is far below the 1e-10 bar).
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  // one cubically convergent step: r (1 + e + e^2), e = 1 - x r (seed error
  // <= 2^-19 -> <= 2^-57 before the final rounding)
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Fast sqrt: MUFU rsqrt seed, one third-order step, one final correction (<= 1 ulp).
__device__ __forceinline__ double fsqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  // one third-order step on the rsqrt seed: r (1 + e/2 + 3e^2/8), e = 1 - x r^2
  const double e = fma(-x * r, r, 1.0);
  r = fma(r * e, fma(0.375, e, 0.5), r);
  double y = x * r;
  y = fma(fma(-y, y, x), 0.5 * r, y);
  return x > 0.0 ? y : (x == 0.0 ? 0.0 : __longlong_as_double(0x7ff8000000000000ULL));
}

// sqrt without the zero / negative select (no branch in the SASS): x == 0 or
// x = inf give NaN (MUFU seed inf / 0); callers test the argument or result.
// x times the refined rsqrt (~2^-56): within ~1 ulp, no Heron step (used for
// polygon lengths, sums of many edges).
__device__ __forceinline__ double fsqrt_nb(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x * r, r, 1.0);
  r = fma(r * e, fma(0.375, e, 0.5), r);
  return x * r;
}

// --------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_min_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_or(int v) {
  return __any_sync(0xffffffffu, v != 0) ? 1 : 0;
}

// Block-wide reductions. `red` is shared scratch of >= 32 double2. All threads of
// the block must call; every thread receives the result.
__device__ __forceinline__ double2 block_sum2(double2 v, double2* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum2(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double2 r = lane < nw ? red[lane] : make_double2(0.0, 0.0);
  r = warp_sum2(r);
  return r;
}
__device__ __forceinline__ double block_sum(double v, double2* red) {
  return block_sum2(make_double2(v, 0.0), red).x;
}
__device__ __forceinline__ double block_max(double v, double2* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid].x = v;
  __syncthreads();
  double r = lane < nw ? red[lane].x : -INFINITY;
  return warp_max(r);
}
__device__ __forceinline__ int block_min_int(int v, double2* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_min_int(v);
  __syncthreads();
  if (lane == 0) reinterpret_cast<int*>(red)[wid] = v;
  __syncthreads();
  int r = lane < nw ? reinterpret_cast<int*>(red)[lane] : 0x7fffffff;
  return warp_min_int(r);
}
__device__ __forceinline__ int block_or(int v, double2* red) {
  return block_min_int(v ? 0 : 1, red) == 0 ? 1 : 0;
}

// Status codes written per pair / per curve (mirror cva_status in include/curvalign_cuda.h).
enum : int32_t { kOk = 0, kInvalid = 1, kRuntime = 2 };

}  // namespace cva
