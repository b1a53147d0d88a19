// Complex FFT of any length on the GPU for the single-call drop-in API:
// real_dft / real_idft / circular_cross_correlation (proj/src/fft.cpp:81-125)
// and correlation_all_shifts_fft (proj/src/rigid_align.cpp:147-183), which the
// reference runs through FFTW for any n >= 2 (fft.cpp:24-40).
//
// Power-of-two n: bit-reversal copy, then log2 n radix-2 passes in place (one
// launch each, twiddles exp(s 2 pi i k / len) from sincospi(2k / len), exact
// arguments). Other n: Bluestein's chirp-z transform over a power-of-two
// convolution of length M >= 2n - 1 (chirp angles pi (j^2 mod 2n) / n, exact
// integer reduction). O(n log n) everywhere; the batched hot path uses the
// shared-memory transforms of pairfft.cuh / largen.cu instead.
//
// The correlation stack follows SURVEY.md §8(b): with z = x + i y and Z = DFT(z),
//   D_m = sum_l conj(z1_l) z2_{l+m} = IDFT(conj(Z1) Z2)_m,
//   E_m = sum_l z1_l z2_{l+m}       = IDFT(Z1[-k] Z2[k])_m,
// A11 = (Re D + Re E) / 2, A22 = (Re D - Re E) / 2, A12 = (Im D + Im E) / 2,
// A21 = (Im E - Im D) / 2: two forward and two inverse transforms per pair of
// curves instead of the reference's four r2c + four c2r.
#include <cuda_runtime.h>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "gfft.h"

namespace cva {
namespace gf {

constexpr int kT = 256;

__host__ __device__ inline bool pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

__global__ void bitrev_kernel(const double2* __restrict__ in, double2* __restrict__ out, int64_t n, int lg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = __brevll((unsigned long long)i) >> (64 - lg);
    out[r] = in[i];
  }
}

// one radix-2 pass of butterflies of span 2 * half (in place)
__global__ void pass_kernel(double2* a, int64_t n, int64_t half, int sign) {
  const int64_t nb = n / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nb; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t % half, i = (t / half) * 2 * half + k, j = i + half;
    double s, c;
    sincospi((double)k / (double)half, &s, &c);  // exp(sign 2 pi i k / (2 half))
    const double2 w = make_double2(c, sign * s);
    const double2 u = a[i], v = cmul(a[j], w);
    a[i] = cadd(u, v);
    a[j] = csub(u, v);
  }
}

// chirp c_j = exp(sign pi i (j^2 mod 2n) / n): with jk = (j^2 + k^2 - (k-j)^2) / 2,
// X_k = c_k sum_j (x_j c_j) conj(c_{k-j})
__device__ inline double2 chirp(int64_t j, int64_t n, int sign) {
  const int64_t jj = (int64_t)(((unsigned long long)(j % (2 * n)) * (unsigned long long)(j % (2 * n))) %
                               (unsigned long long)(2 * n));
  double s, c;
  sincospi((double)jj / (double)n, &s, &c);
  return make_double2(c, sign * s);
}

__global__ void blue_in_kernel(const double2* __restrict__ x, int64_t n, int64_t M, int sign, double2* __restrict__ u,
                               double2* __restrict__ v) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
    u[j] = j < n ? cmul(x[j], chirp(j, n, sign)) : make_double2(0, 0);
    // v_k = conj(c_k) on both wraps (k < n and M - k for 0 < k < n), 0 between
    const int64_t k = j < n ? j : (M - j < n ? M - j : -1);
    if (k >= 0) {
      const double2 c = chirp(k, n, sign);
      v[j] = make_double2(c.x, -c.y);
    } else {
      v[j] = make_double2(0, 0);
    }
  }
}

__global__ void mul_kernel(double2* __restrict__ u, const double2* __restrict__ v, int64_t M) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x)
    u[j] = cmul(u[j], v[j]);
}

__global__ void blue_out_kernel(const double2* __restrict__ w, int64_t n, int64_t M, int sign, double2* __restrict__ x) {
  const double inv = 1.0 / (double)M;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    x[k] = cscale(cmul(w[k], chirp(k, n, sign)), inv);
}

unsigned grid_for(int64_t items) {
  const int64_t b = (items + kT - 1) / kT;
  return (unsigned)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

// in-place power-of-two transform of a (n points) using tmp (n points)
cudaError_t fft_pow2(double2* a, double2* tmp, int64_t n, int sign, cudaStream_t s) {
  if (n <= 1) return cudaSuccess;
  int lg = 0;
  while ((int64_t(1) << lg) < n) ++lg;
  bitrev_kernel<<<grid_for(n), kT, 0, s>>>(a, tmp, n, lg);
  for (int64_t half = 1; half < n; half *= 2) pass_kernel<<<grid_for(n / 2), kT, 0, s>>>(tmp, n, half, sign);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(a, tmp, sizeof(double2) * (size_t)n, cudaMemcpyDeviceToDevice, s);
}

}  // namespace gf

int64_t gfft_workspace(int64_t n) {
  if (gf::pow2(n)) return n;
  int64_t M = 1;
  while (M < 2 * n - 1) M *= 2;
  return 3 * M;  // u, v, transform temporary
}

cudaError_t gfft(double2* x, int64_t n, int sign, double2* ws, cudaStream_t s) {
  if (n <= 1) return cudaSuccess;
  if (gf::pow2(n)) return gf::fft_pow2(x, ws, n, sign, s);
  int64_t M = 1;
  while (M < 2 * n - 1) M *= 2;
  double2 *u = ws, *v = ws + M, *t = ws + 2 * M;
  gf::blue_in_kernel<<<gf::grid_for(M), gf::kT, 0, s>>>(x, n, M, sign, u, v);
  cudaError_t e;
  if ((e = gf::fft_pow2(u, t, M, -1, s)) != cudaSuccess) return e;
  if ((e = gf::fft_pow2(v, t, M, -1, s)) != cudaSuccess) return e;
  gf::mul_kernel<<<gf::grid_for(M), gf::kT, 0, s>>>(u, v, M);
  if ((e = gf::fft_pow2(u, t, M, +1, s)) != cudaSuccess) return e;
  gf::blue_out_kernel<<<gf::grid_for(n), gf::kT, 0, s>>>(u, n, M, sign, x);
  return cudaGetLastError();
}

namespace gf {
// PD_k = conj(Z1_k) Z2_k, PE_k = Z1_{-k} Z2_k
__global__ void corr_products_kernel(const double2* __restrict__ z1, const double2* __restrict__ z2, int64_t n,
                                     double2* __restrict__ pd, double2* __restrict__ pe) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = z1[k], b = z2[k], am = z1[k == 0 ? 0 : n - k];
    pd[k] = cmulconj(b, a);
    pe[k] = cmul(am, b);
  }
}

__global__ void corr_pack_kernel(const double2* __restrict__ d, const double2* __restrict__ e, int64_t n,
                                 double* __restrict__ out4) {
  const double h = 0.5 / (double)n;  // 1/n of the inverse transform, 1/2 of the combination
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    const double2 D = d[m], E = e[m];
    out4[4 * m + 0] = (D.x + E.x) * h;  // A11
    out4[4 * m + 1] = (D.y + E.y) * h;  // A12
    out4[4 * m + 2] = (E.y - D.y) * h;  // A21
    out4[4 * m + 3] = (D.x - E.x) * h;  // A22
  }
}
}  // namespace gf

int64_t gfft_correlation_workspace(int64_t n) { return 4 * n + gfft_workspace(n); }

cudaError_t gfft_correlation(const double2* c1, const double2* c2, int64_t n, double* out4, double2* ws,
                             cudaStream_t s) {
  double2 *z1 = ws, *z2 = ws + n, *pd = ws + 2 * n, *pe = ws + 3 * n, *w = ws + 4 * n;
  cudaError_t e = cudaMemcpyAsync(z1, c1, sizeof(double2) * (size_t)n, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(z2, c2, sizeof(double2) * (size_t)n, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = gfft(z1, n, -1, w, s);
  if (e == cudaSuccess) e = gfft(z2, n, -1, w, s);
  if (e != cudaSuccess) return e;
  gf::corr_products_kernel<<<gf::grid_for(n), gf::kT, 0, s>>>(z1, z2, n, pd, pe);
  if ((e = gfft(pd, n, +1, w, s)) != cudaSuccess) return e;
  if ((e = gfft(pe, n, +1, w, s)) != cudaSuccess) return e;
  gf::corr_pack_kernel<<<gf::grid_for(n), gf::kT, 0, s>>>(pd, pe, n, out4);
  return cudaGetLastError();
}

}  // namespace cva
