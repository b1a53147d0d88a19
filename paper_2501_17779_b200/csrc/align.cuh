// Block-level tail of the alignment: FFT cross-correlation -> tie-broken argmax
// -> rotation, trace, energy -> aligned curve. Replaces
// correlation_all_shifts_fft + pick_best + optimal_rotation_svd
// (proj/src/rigid_align.cpp:147-183, :31-61, :82-102) for one pair.
#pragma once

#include <climits>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "fft.cuh"

namespace cva {

constexpr double kTieRelTol = 1e-12;  // proj/src/rigid_align.cpp:16

// Sum of squared norms of buf[0..n) (proj/src/rigid_align.cpp:23-27), block-wide.
__device__ __forceinline__ double block_sum_norm2(const double2* buf, int n, double2* red) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 p = buf[i];
    acc = fma(p.x, p.x, fma(p.y, p.y, acc));
  }
  return block_sum(acc, red);
}

// z1: curve 1 (destroyed). c2: curve 2 (preserved). w1, w2: N-element scratch.
// s1, s2: sum_norm2 of the two curves. Writes *out (thread 0) and, if aligned is
// non-null, aligned[l] = R(theta) c2[(l + m) mod N] (all threads).
__device__ inline void block_align_tail(double2* z1, const double2* c2, double2* w1, double2* w2,
                                        int N, const double2* __restrict__ tw, double s1, double s2,
                                        cva_alignment* out, double2* __restrict__ aligned,
                                        double2* red) {
  const int t = threadIdx.x, T = blockDim.x;
  for (int i = t; i < N; i += T) w1[i] = c2[i];
  __syncthreads();
  double2* X1 = fft_forward(z1, w2, N, tw, t, T);
  double2* fr = (X1 == z1) ? w2 : z1;
  double2* X2 = fft_forward(w1, fr, N, tw, t, T);
  for (int k = t; k < N; k += T) X1[k] = cmulconj(X1[k], X2[k]);  // Z1 conj(Z2)
  __syncthreads();
  // D_m = sum_l conj(z1_l) z2_{l+m} = IDFT(conj Z1 . Z2)_m = conj(FFT(Z1 conj Z2)_m) / N
  double2* F = fft_forward(X1, X2, N, tw, t, T);

  const double invN = 1.0 / (double)N;
  double best = -INFINITY;
  for (int k = t; k < N; k += T) {
    const double2 f = F[k];
    best = fmax(best, sqrt(fma(f.x, f.x, f.y * f.y)) * invN);
  }
  best = block_max(best, red);
  const double thr = best - kTieRelTol * fmax(1.0, fabs(best));
  int cand = INT_MAX;
  for (int k = t; k < N; k += T) {
    const double2 f = F[k];
    if (sqrt(fma(f.x, f.x, f.y * f.y)) * invN >= thr) {
      cand = k;
      break;  // k ascending per thread: first hit is this thread's minimum
    }
  }
  const int m = block_min_int(cand, red);

  __shared__ double2 bc;  // (cos theta, sin theta)
  __shared__ int bm;
  if (t == 0) {
    cva_alignment r;
    if (!isfinite(best) || m == INT_MAX) {
      r.shift = 0;
      r.t0 = 0.0;
      r.theta = __longlong_as_double(0x7ff8000000000000ULL);
      r.trace = r.theta;
      r.energy = r.theta;
      r.degenerate = 0;
      r.status = CVA_INVALID_ARGUMENT;  // non-finite correlation (rigid_align.cpp:83)
      bm = -1;
    } else {
      const double2 f = F[m];
      const double trace = sqrt(fma(f.x, f.x, f.y * f.y)) * invN;
      double theta = 0.0;
      int degenerate = 0;
      if (trace == 0.0) {
        degenerate = 1;  // rigid_align.cpp:86-88
      } else {
        theta = atan2(-f.y, f.x);  // arg D_m, D_m = conj(F_m) / N
      }
      const double h = invN;
      double e = h * (s1 + s2) - 2.0 * h * trace;
      if (e < 0.0) e = 0.0;
      r.shift = m;
      r.t0 = (double)m / (double)N;
      r.theta = theta;
      r.trace = degenerate ? 0.0 : trace;
      r.energy = e;
      r.degenerate = degenerate;
      r.status = CVA_OK;
      bm = m;
      double sn, cs;
      sincos(theta, &sn, &cs);
      bc = make_double2(cs, sn);
    }
    *out = r;
  }
  __syncthreads();
  if (aligned != nullptr) {
    const int mm = bm;
    if (mm < 0) {
      const double nan = __longlong_as_double(0x7ff8000000000000ULL);
      for (int l = t; l < N; l += T) aligned[l] = make_double2(nan, nan);
    } else {
      const double2 r = bc;
      for (int l = t; l < N; l += T) {
        int j = l + mm;
        if (j >= N) j -= N;
        const double2 q = c2[j];
        aligned[l] = make_double2(fma(r.x, q.x, r.y * q.y), fma(-r.y, q.x, r.x * q.y));
      }
    }
  }
}

}  // namespace cva
