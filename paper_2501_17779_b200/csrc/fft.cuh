// Block-cooperative fp64 complex FFT held in shared memory (sm_100a).
//
// Replaces the reference's FFTW r2c/c2r calls (proj/src/fft.cpp:81-114): instead
// of 4 real forward + 4 real inverse transforms per alignment
// (proj/src/rigid_align.cpp:147-183) the path runs 2 complex forward transforms
// (z = x + i y) and 1 more forward transform for the correlation (the inverse
// is taken as conj(FFT(conj(.))) so only the forward kernel exists).
//
// Algorithm: Stockham autosort, decimation in time, natural order in and out:
//   for Ns = 1; Ns < N; Ns *= R:
//     for each butterfly j in [0, N/R):
//       v[r] = in[j + r N/R] * w_N^{r (j mod Ns) N/(Ns R)},  r < R
//       v    = DFT_R(v)
//       out[(j / Ns) Ns R + (j mod Ns) + r Ns] = v[r]
// with w_N = exp(-2 pi i / N) read from a per-N device table (exact sincospi
// values, never a recurrence). Radices 8/4/2; one __syncthreads per pass.
#pragma once

#include "cva_common.cuh"

namespace cva {

// In-register forward DFTs, X_k = sum_n v_n exp(-2 pi i n k / R).
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  const double2 a = cadd(v0, v2), b = csub(v0, v2), c = cadd(v1, v3), d = csub(v1, v3);
  v0 = cadd(a, c);
  v2 = csub(a, c);
  v1 = cadd(b, cmul_mi(d));  // b - i d
  v3 = csub(b, cmul_mi(d));  // b + i d
}

__device__ __forceinline__ void dft8(double2* v) {
  // evens / odds
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4(e0, e1, e2, e3);
  dft4(o0, o1, o2, o3);
  constexpr double r2 = 0.70710678118654752440084436210484904;
  // o_k *= w8^k, w8 = (1 - i)/sqrt2
  const double2 t1 = make_double2(r2 * (o1.x + o1.y), r2 * (o1.y - o1.x));
  const double2 t2 = cmul_mi(o2);
  const double2 t3 = make_double2(r2 * (o3.y - o3.x), -r2 * (o3.x + o3.y));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, t1);
  v[5] = csub(e1, t1);
  v[2] = cadd(e2, t2);
  v[6] = csub(e2, t2);
  v[3] = cadd(e3, t3);
  v[7] = csub(e3, t3);
}

// 16-point DFT as 4 x 4: X[k1 + 4 k2] = sum_n2 W4^{n2 k2} W16^{n2 k1} sum_n1 x[n2 + 4 n1] W4^{n1 k1}.
// Leaves X[k1 + 4 k2] in v[4 k1 + k2] (no register transpose): read outputs
// through dft16_slot(k).
__device__ __forceinline__ void dft16(double2* v) {
#pragma unroll
  for (int c = 0; c < 4; ++c) dft4(v[c], v[c + 4], v[c + 8], v[c + 12]);
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  constexpr double r2 = 0.70710678118654752440;
  // v[c + 4 k1] *= W16^{c k1}
  v[5] = cmul(v[5], make_double2(c1, -s1));
  v[6] = cmul(v[6], make_double2(r2, -r2));
  v[7] = cmul(v[7], make_double2(s1, -c1));
  v[9] = cmul(v[9], make_double2(r2, -r2));
  v[10] = cmul_mi(v[10]);
  v[11] = cmul(v[11], make_double2(-r2, -r2));
  v[13] = cmul(v[13], make_double2(s1, -c1));
  v[14] = cmul(v[14], make_double2(-r2, -r2));
  v[15] = cmul(v[15], make_double2(-c1, s1));
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
}
__host__ __device__ constexpr int dft16_slot(int k) { return 4 * (k & 3) + (k >> 2); }

template <int R>
__device__ __forceinline__ void dft_r(double2* v);
template <>
__device__ __forceinline__ void dft_r<2>(double2* v) { dft2(v[0], v[1]); }
template <>
__device__ __forceinline__ void dft_r<4>(double2* v) { dft4(v[0], v[1], v[2], v[3]); }
template <>
__device__ __forceinline__ void dft_r<8>(double2* v) { dft8(v); }
template <>
__device__ __forceinline__ void dft_r<16>(double2* v) { dft16(v); }
// register holding output k of dft_r<R>
template <int R>
__host__ __device__ constexpr int dft_slot(int k) {
  return R == 16 ? dft16_slot(k) : k;
}

// One Stockham pass of radix R over a length-N sequence, threads t in [0, T).
template <int R>
__device__ __forceinline__ void stockham_pass(const double2* in, double2* out,
                                              int N, int Ns, const double2* __restrict__ tw, int t,
                                              int T) {
  const int nb = N / R;
  const int tw_stride = N / (Ns * R);
  for (int j = t; j < nb; j += T) {
    double2 v[R];
    const int jm = j & (Ns - 1);  // Ns is a power of two
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[j + r * nb];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[r * jm * tw_stride]));
    }
    dft_r<R>(v);
    const int base = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) out[base + r * Ns] = v[r];
  }
}

// Forward FFT of buf[0..N) (N = 2^p, N >= 2) by threads t in [0, T) of the
// block, ping-ponging with `scratch`. Returns the buffer holding the result.
// Contains __syncthreads(); every thread of the block must call it.
__device__ inline double2* fft_forward(double2* buf, double2* scratch, int N, const double2* tw,
                                       int t, int T) {
  double2* src = buf;
  double2* dst = scratch;
  int Ns = 1;
  while (Ns < N) {
    const int rem = N / Ns;
    if (rem >= 8 && (rem % 8) == 0) {
      stockham_pass<8>(src, dst, N, Ns, tw, t, T);
      Ns *= 8;
    } else if (rem >= 4) {
      stockham_pass<4>(src, dst, N, Ns, tw, t, T);
      Ns *= 4;
    } else {
      stockham_pass<2>(src, dst, N, Ns, tw, t, T);
      Ns *= 2;
    }
    __syncthreads();
    double2* tmp = src;
    src = dst;
    dst = tmp;
  }
  return src;
}

}  // namespace cva
