// Elastic (SRV) matching on the GPU — the rigid path's caller in the
// reference's elastic distance:
//
//   * dp_kernel        batched dp_reparam (proj/src/srv.cpp:180-257): the
//                      monotone lattice path of least discretised SRV mismatch;
//   * elastic_kernel   batched elastic_distance_approach2
//                      (proj/src/elastic.cpp:102-174): rigid pre-alignment,
//                      then alternating DP gamma-steps and FFT (t0, R)-steps
//                      with the raw-pair SVD refit, each accepted only if the
//                      realised energy does not increase.
//
// One 256-thread CTA per pair (a grid-stride loop over pairs). The DP walks
// its rows in order (row i depends on rows i-1 .. i-W) with the cells of a row
// spread over the threads; dp values live in a (W+1)-row ring in shared
// memory, parent steps in shared memory (N <= 256) or a per-CTA global slab.
//
// Exactness. dp_step_cost, apply_srv_action, compose/rebase and the DP
// recurrence are restated operation for operation with __dadd_rn/__dmul_rn
// (no FMA contraction) and the reference's summation order, so dp_reparam is
// bitwise the reference's for the same inputs. Inside approach 2 the rigid
// alignments run on the FFT pair stage (rotation within ulps of the
// reference's SVD) and cos/sin come from CUDA's libm (<= 2 ulp), so the
// alternating search agrees with the reference to rounding, not bitwise.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <stdint.h>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "elastic.h"
#include "pairfft.cuh"

namespace cva {
namespace el {

constexpr int kT = 256;
constexpr double kGridSnap = 1e-9;  // srv.cpp:14
constexpr int kMaxSteps = 64;   // shared step table (W <= 8: 43 steps)
constexpr int kMaxSlope = 20;   // 255 steps: parent indices stay below the 0xff sentinel (srv.cpp:222)
#ifndef CVA_EL_MINB
#define CVA_EL_MINB 2
#endif

// ------------------------------------------------------------ exact arithmetic
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double norm2(double2 p) { return add(mul(p.x, p.x), mul(p.y, p.y)); }

// geometry.hpp:90-94
__device__ __forceinline__ double wrap_unit(double t) {
  double r = sub(t, floor(t));
  if (r >= 1.0) r = sub(r, 1.0);
  return r;
}

// srv.cpp:19-37 (periodic linear interpolation with grid snapping)
__device__ __forceinline__ double2 interp_periodic(const double2* q, int n, double u) {
  const double x = mul(u, (double)n);
  double i0f = floor(x);
  double frac = sub(x, i0f);
  if (frac > 1.0 - kGridSnap) {
    i0f = add(i0f, 1.0);
    frac = 0.0;
  } else if (frac < kGridSnap) {
    frac = 0.0;
  }
  long long i0 = (long long)i0f % (long long)n;
  if (i0 < 0) i0 += n;
  if (frac == 0.0) return q[i0];
  const long long i1 = (i0 + 1) % n;
  const double2 a = q[i0], b = q[i1];
  return make_double2(add(a.x, mul(frac, sub(b.x, a.x))), add(a.y, mul(frac, sub(b.y, a.y))));
}

// Rotation2::apply (geometry.hpp:70-73) with (c, s) = (cos, sin)(theta)
__device__ __forceinline__ double2 rot_apply(double c, double s, double2 p) {
  return make_double2(add(mul(c, p.x), mul(s, p.y)), add(mul(-s, p.x), mul(c, p.y)));
}

// apply_srv_action element l (srv.cpp:100-118)
__device__ __forceinline__ double2 action_at(const double2* q, int n, double t0, double c, double s,
                                             const double* g, int l) {
  const double gdot = mul(sub(g[l + 1], g[l]), (double)n);
  const double u = wrap_unit(add(t0, g[l]));
  const double2 v = interp_periodic(q, n, u);
  const double k = sqrt(fmax(gdot, 0.0));
  const double2 r = rot_apply(c, s, v);
  return make_double2(mul(r.x, k), mul(r.y, k));
}

// Sequential sum of x[0..n) by thread 0 (the reference's loop order), returned
// to every thread. `cell`: one shared double.
__device__ __forceinline__ double seq_sum(const double* x, int n, double* cell) {
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0;
    for (int l = 0; l < n; ++l) e = add(e, x[l]);
    *cell = e;
  }
  __syncthreads();
  return *cell;
}

// elastic_energy (srv.cpp:120-128): terms computed in parallel into T, summed
// in order, / n.
__device__ double energy(const double2* q1, const double2* q2, int n, double t0, double theta,
                         const double* g, double* T, double* cell) {
  double s, c;
  sincos(theta, &s, &c);
  for (int l = threadIdx.x; l < n; l += kT) {
    const double2 w = action_at(q2, n, t0, c, s, g, l);
    T[l] = norm2(make_double2(sub(q1[l].x, w.x), sub(q1[l].y, w.y)));
  }
  return dvd(seq_sum(T, n, cell), (double)n);
}

// srv_transform (srv.cpp:71-88)
__device__ void srv_transform(const double2* c, int n, double2* q) {
  const double nn = (double)n;
  const double eps = mul(1e-8, nn);
  for (int l = threadIdx.x; l < n; l += kT) {
    const double2 nx = c[l + 1 == n ? 0 : l + 1], pv = c[l == 0 ? n - 1 : l - 1];
    const double h = dvd(nn, 2.0);
    const double2 d = make_double2(mul(sub(nx.x, pv.x), h), mul(sub(nx.y, pv.y), h));
    const double mag = sqrt(norm2(d));
    if (mag < eps) {
      q[l] = make_double2(0.0, 0.0);
    } else {
      const double r = dvd(1.0, sqrt(mag));
      q[l] = make_double2(mul(d.x, r), mul(d.y, r));
    }
  }
}

// srv_center (srv.cpp:90-98): mean by the reference's sequential sum.
__device__ void srv_center(const double2* q, int n, double2* out, double* cell2) {
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0, my = 0.0;
    for (int l = 0; l < n; ++l) {
      mx = add(mx, q[l].x);
      my = add(my, q[l].y);
    }
    const double r = dvd(1.0, (double)n);
    cell2[0] = mul(mx, r);
    cell2[1] = mul(my, r);
  }
  __syncthreads();
  const double mx = cell2[0], my = cell2[1];
  for (int l = threadIdx.x; l < n; l += kT) out[l] = make_double2(sub(q[l].x, mx), sub(q[l].y, my));
  __syncthreads();
}

// ------------------------------------------------------------------- DP

// Admissible steps (srv.cpp:130-139): (a, b) in 1..W, gcd 1, a-major order.
struct Steps {
  int count;
  int a[kMaxSteps], b[kMaxSteps];
};
__host__ __device__ constexpr int gcd_i(int x, int y) { return y == 0 ? x : gcd_i(y, x % y); }
__host__ __device__ constexpr Steps make_steps(int W) {
  Steps s{};
  s.count = 0;
  for (int a = 1; a <= W; ++a)
    for (int b = 1; b <= W; ++b)
      if (gcd_i(a, b) == 1 && s.count < kMaxSteps) {
        s.a[s.count] = a;
        s.b[s.count] = b;
        ++s.count;
      }
  return s;
}

// Per-step constants of dp_step_cost, formed once per CTA with the reference's
// operations: sq = sqrt((double)b / a) and the interpolation offsets
// (double)(k b) / a, so the per-cell work has no division or square root.
// StepTab: shared-memory table for W <= 8; StepView: the table the DP reads,
// either that one or a per-CTA global table (slab mode, W up to kMaxSlope).
struct StepTab {
  double sq[kMaxSteps];
  double fr[kMaxSteps][9];
  int a[kMaxSteps], b[kMaxSteps];
};
struct StepView {
  double* sq;
  double* fr;  // count x frs
  int frs;
  int* a;
  int* b;
};

// dp_step_cost (srv.cpp:145-176) with q1, q2 in shared memory. sq, fr: the
// step's StepTab row; inv_n: 1/n when n is a power of two (then cost * inv_n
// == cost / n exactly), else 0 (divide).
__device__ __forceinline__ double step_cost_t(const double2* q1, const double2* q2, int n, int i0, int j0, int a,
                                              int b, double sq, const double* fr, double inv_n) {
  double cost = 0.0;
  for (int k = 0; k <= a; ++k) {
    int i = i0 + k;
    if (i >= n) i %= n;
    const int num = k * b;
    double2 s;
    if (num % a == 0) {
      int jj = j0 + num / a;
      if (jj >= n) jj %= n;
      s = q2[jj];
    } else {
      const double pos = add((double)j0, fr[k]);
      const int base = (int)pos;
      const double frac = sub(pos, (double)base);
      int b0 = base, b1 = base + 1;
      if (b0 >= n) b0 %= n;
      if (b1 >= n) b1 %= n;
      const double2 u = q2[b0];
      const double2 v = q2[b1];
      s = make_double2(add(u.x, mul(frac, sub(v.x, u.x))), add(u.y, mul(frac, sub(v.y, u.y))));
    }
    const double2 d = make_double2(sub(q1[i].x, mul(s.x, sq)), sub(q1[i].y, mul(s.y, sq)));
    const double nd = norm2(d);
    cost = add(cost, (k == 0 || k == a) ? mul(0.5, nd) : nd);  // w = 1 multiplies exactly
  }
  return inv_n != 0.0 ? mul(cost, inv_n) : dvd(cost, (double)n);
}

// Reference-order constants for one step (used by the table and the single-call utility).
__device__ __forceinline__ void step_consts(int a, int b, double* sq, double* fr) {
  *sq = sqrt(dvd((double)b, (double)a));
  for (int k = 0; k <= a; ++k) fr[k] = dvd((double)(k * b), (double)a);
}

__device__ __forceinline__ double step_cost(const double2* q1, const double2* q2, int n, int i0, int j0, int a,
                                            int b) {
  double sq, fr[9];
  step_consts(a, b, &sq, fr);
  return step_cost_t(q1, q2, n, i0, j0, a, b, sq, fr, 0.0);
}

__device__ __forceinline__ int jmin_of(int i, int n, int W) {
  const int lo1 = (i + W - 1) / W;
  const int lo2 = n - W * (n - i);
  return max(max(lo1, lo2), 0);
}
__device__ __forceinline__ int jmax_of(int i, int n, int W) {
  const int hi1 = W * i;
  const int hi2 = n - (n - i + W - 1) / W;
  return min(min(hi1, hi2), n);
}

// Interpolation offsets (k b) / a of the compile-time step set: constant-
// evaluated IEEE divisions, the same correctly rounded values dvd() forms.
struct FrTab {
  double fr[kMaxSteps][9];
};
__host__ __device__ constexpr FrTab make_fr(int W) {
  FrTab t{};
  const Steps s = make_steps(W);
  for (int q = 0; q < s.count; ++q)
    for (int k = 0; k <= s.a[q]; ++k) t.fr[q][k] = (double)(k * s.b[q]) / (double)s.a[q];
  return t;
}

// (a-1, b-1) of every step, 4 bits per step (W <= 4: at most 11 steps).
__host__ __device__ constexpr unsigned long long pack_steps(int W) {
  const Steps s = make_steps(W);
  unsigned long long v = 0;
  for (int q = 0; q < s.count; ++q) v |= (unsigned long long)((s.a[q] - 1) | ((s.b[q] - 1) << 2)) << (4 * q);
  return v;
}

// Offsets of each step's interior samples (k = 1..a-1) in a column's cache.
struct OffTab {
  int v[kMaxSteps];
  int total;
};
__host__ __device__ constexpr OffTab make_off(int W) {
  OffTab t{};
  const Steps s = make_steps(W);
  int o = 0;
  for (int q = 0; q < s.count; ++q) {
    t.v[q] = o;
    o += s.a[q] - 1;
  }
  t.total = o;
  return t;
}

// q2 operand window of column j: q2[(j - c) mod n], q2[j-c+1] - q2[j-c] and
// (double)(j - c) for c = 0..kW (j - c < 0: unused slots).
template <int kW>
__device__ __forceinline__ void column_window(const double2* q2, int n, int j, double2* q2w, double2* dq,
                                              double* jd) {
#pragma unroll
  for (int c = 0; c <= kW; ++c) {
    const int x = j - c;
    q2w[c] = q2[x < 0 ? 0 : (x >= n ? x - n : x)];
    jd[c] = (double)x;
  }
#pragma unroll
  for (int c = 1; c <= kW; ++c) dq[c] = make_double2(sub(q2w[c - 1].x, q2w[c].x), sub(q2w[c - 1].y, q2w[c].y));
}

// Interior sample k of step (a, b) (0 < k < a) into column j, scaled by
// sqrt(b/a): dp_step_cost's interpolation (srv.cpp:156-166) at base column
// j - cu (cu = b - floor(k b / a)) with offset fr = k b / a, then the sq product.
__device__ __forceinline__ double2 scaled_interior(const double2* q2w, const double2* dq, const double* jd, int b,
                                                   int cu, double fr, double sq) {
  const double frac = sub(add(jd[b], fr), jd[cu]);
  const double2 sv = make_double2(add(q2w[cu].x, mul(frac, dq[cu].x)), add(q2w[cu].y, mul(frac, dq[cu].y)));
  return make_double2(mul(sv.x, sq), mul(sv.y, sq));
}

// The DP rows for a compile-time slope bound: dp_step_cost's operand fetches
// hoisted out of the step loop. Every step into cell (i, j) reads q1 at rows
// i-kW..i and q2 at columns j-kW..j only, so each thread holds those two
// windows, the column differences q2[c+1]-q2[c] and (double)(j-c) in
// registers, and the interpolation base of sample k of step (a, b) is the
// compile-time offset floor(k b / a) from j-b: (int)((double)(j-b) + kb/a) ==
// j-b+floor(kb/a) because the fraction is >= 1/a away from an integer and the
// addition's rounding error is < 2^-32 for any n < 2^20 (the parent matrix
// alone bounds n far below that). Same operations, same order, same values as
// step_cost_t; no modulo, no integer/float conversions, no shared loads in the
// sample loop.
// A thread's first column (threadIdx.x) is the same in every row and its
// scaled interior samples do not depend on the row, so they are formed once
// per DP and kept in registers (kCached cells); only q1's side changes per
// row. Further columns (n >= kT) take the window path.
template <int kW, bool kPow2, bool kCached>
__device__ __forceinline__ void dp_cell(const double2* q2, int n, int i, int j, const double2* q1w,
                                        const double* const* prv, const double2* Sc, const double* sqt,
                                        double inv_n, double* cur, uint8_t* par) {
  constexpr Steps kS = make_steps(kW);
  constexpr FrTab kF = make_fr(kW);
  constexpr OffTab kO = make_off(kW);
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double2 q2w[kW + 1], dq[kW + 1];
  double jd[kW + 1];
  if constexpr (kCached) {
#pragma unroll
    for (int c = 0; c <= kW; ++c) {
      const int x = j - c;
      q2w[c] = q2[x < 0 ? 0 : (x >= n ? x - n : x)];
    }
  } else {
    column_window<kW>(q2, n, j, q2w, dq, jd);
  }
  // Branch-free over the steps: an inadmissible predecessor reads as +inf and
  // inf + cost never compares below best (cost is finite), which is the
  // reference's `continue` (srv.cpp:214-216) without a divergent region per
  // step, so the steps' sample chains interleave.
  double best = inf;
  uint8_t best_s = 0xff;
#pragma unroll
  for (int s = 0; s < kS.count; ++s) {
    const int a = kS.a[s], b = kS.b[s];
    const double base = (i - a < 0 || j - b < 0) ? inf : prv[a][max(j - b, 0)];
    const double sq = sqt[s];
    double cost = 0.0;
#pragma unroll
    for (int k = 0; k <= a; ++k) {
      double2 d;
      if (k == 0 || k == a) {
        const double2 sv = q2w[k == 0 ? b : 0];
        d = make_double2(sub(q1w[a - k].x, mul(sv.x, sq)), sub(q1w[a - k].y, mul(sv.y, sq)));
      } else {
        double2 S;
        if constexpr (kCached)
          S = Sc[kO.v[s] + k - 1];
        else
          S = scaled_interior(q2w, dq, jd, b, b - (k * b) / a, kF.fr[s][k], sq);
        d = make_double2(sub(q1w[a - k].x, S.x), sub(q1w[a - k].y, S.y));
      }
      const double nd = norm2(d);
      cost = add(cost, (k == 0 || k == a) ? mul(0.5, nd) : nd);
    }
    const double cand = add(base, kPow2 ? mul(cost, inv_n) : dvd(cost, (double)n));
    if (cand < best) {
      best = cand;
      best_s = (uint8_t)s;
    }
  }
  *cur = best;
  *par = best_s;
}

template <int kW, bool kPow2>
__device__ __forceinline__ void dp_rows_hoisted(const double2* q1, const double2* q2, int n, double* ring,
                                                uint8_t* parent, const double* sqt, double inv_n) {
  constexpr Steps kS = make_steps(kW);
  constexpr FrTab kF = make_fr(kW);
  constexpr OffTab kO = make_off(kW);
  const int stride = n + 1;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const int jc = threadIdx.x;
  double2 Sc[kO.total];
  if (jc <= n) {
    double2 q2w[kW + 1], dq[kW + 1];
    double jd[kW + 1];
    column_window<kW>(q2, n, jc, q2w, dq, jd);
#pragma unroll
    for (int s = 0; s < kS.count; ++s)
#pragma unroll
      for (int k = 1; k < kS.a[s]; ++k)
        Sc[kO.v[s] + k - 1] =
            scaled_interior(q2w, dq, jd, kS.b[s], kS.b[s] - (k * kS.b[s]) / kS.a[s], kF.fr[s][k], sqt[s]);
  }
  int ri = 0;  // i % (kW + 1)
  for (int i = 1; i <= n; ++i) {
    ri = ri == kW ? 0 : ri + 1;
    const int lo = jmin_of(i, n, kW), hi = jmax_of(i, n, kW);
    double* cur = ring + (size_t)ri * stride;
    uint8_t* par = parent + (size_t)i * stride;
    const double* prv[kW + 1];
    double2 q1w[kW + 1];
#pragma unroll
    for (int c = 0; c <= kW; ++c) {
      const int r = ri - c < 0 ? ri - c + kW + 1 : ri - c;
      prv[c] = ring + (size_t)r * stride;
      const int x = i - c;
      q1w[c] = q1[x < 0 ? 0 : (x >= n ? x - n : x)];
    }
    for (int j = jc; j <= n; j += kT) {
      if (j < lo || j > hi) {
        cur[j] = inf;
        par[j] = 0xff;
      } else if (j == jc) {
        dp_cell<kW, kPow2, true>(q2, n, i, j, q1w, prv, Sc, sqt, inv_n, cur + j, par + j);
      } else {
        dp_cell<kW, kPow2, false>(q2, n, i, j, q1w, prv, Sc, sqt, inv_n, cur + j, par + j);
      }
    }
    __syncthreads();
  }
}

// dp_reparam (srv.cpp:180-257) on q1, q2 (n samples; shared memory, or the
// CTA's global slab in slab mode). ring: (W+1) x (n+1) doubles; parent:
// (n+1)^2 bytes (shared or global); gamma: n+1. gtab: null = the shared step
// table (W <= 8), else a global StepView with room for W's steps. Returns the
// path energy (thread-uniform); +inf if no admissible path.
template <int kW>
__device__ double dp_reparam(const double2* q1, const double2* q2, int n, int Wrt, double* ring,
                             uint8_t* parent, double* gamma, double* cell, const StepView* gtab = nullptr) {
  const int W = kW > 0 ? kW : Wrt;
  const int stride = n + 1;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const double inv_n = (n & (n - 1)) == 0 ? dvd(1.0, (double)n) : 0.0;
  __shared__ StepTab stab;
  const StepView tab = gtab ? *gtab : StepView{stab.sq, &stab.fr[0][0], 9, stab.a, stab.b};
  {
    int s = 0;
    for (int a = 1; a <= W; ++a)
      for (int b = 1; b <= W; ++b)
        if (gcd_i(a, b) == 1) {
          if (threadIdx.x == s) {
            step_consts(a, b, &tab.sq[s], tab.fr + (size_t)s * tab.frs);
            tab.a[s] = a;
            tab.b[s] = b;
          }
          ++s;
        }
  }
  auto row = [&](int i) { return ring + (size_t)(i % (W + 1)) * stride; };
  for (int j = threadIdx.x; j <= n; j += kT) row(0)[j] = j == 0 ? 0.0 : inf;
  __syncthreads();
  if constexpr (kW > 0) {
    if (inv_n != 0.0)
      dp_rows_hoisted<kW, true>(q1, q2, n, ring, parent, tab.sq, inv_n);
    else
      dp_rows_hoisted<kW, false>(q1, q2, n, ring, parent, tab.sq, inv_n);
  } else
  for (int i = 1; i <= n; ++i) {
    const int lo = jmin_of(i, n, W), hi = jmax_of(i, n, W);
    double* cur = row(i);
    for (int j = threadIdx.x; j <= n; j += kT) {
      double best = inf;
      uint8_t best_s = 0xff;
      if (j >= lo && j <= hi) {
        auto try_step = [&](int s, int a, int b) {
          const int pi = i - a, pj = j - b;
          if (pi < 0 || pj < 0) return;
          const double base = row(pi)[pj];
          if (base == inf) return;
          const double cand =
              add(base, step_cost_t(q1, q2, n, pi, pj, a, b, tab.sq[s], tab.fr + (size_t)s * tab.frs, inv_n));
          if (cand < best) {
            best = cand;
            best_s = (uint8_t)s;
          }
        };
        if constexpr (kW > 0) {
          constexpr Steps kS = make_steps(kW);
#pragma unroll
          for (int s = 0; s < kS.count; ++s) try_step(s, kS.a[s], kS.b[s]);
        } else {
          int s = 0;
          for (int a = 1; a <= W; ++a)
            for (int b = 1; b <= W; ++b)
              if (gcd_i(a, b) == 1) try_step(s++, a, b);
        }
      }
      cur[j] = best;
      parent[(size_t)i * stride + j] = best_s;
    }
    __syncthreads();
  }
  const double e = row(n)[n];
  // Backtrack (srv.cpp:235-255). Thread 0 walks the parent steps and leaves, in
  // gamma[l] for every row l of the path, the step that covers it (pj, s, k);
  // the threads then form gamma[pi + k] = (pj + k b / a) / n in parallel (the
  // walk is a dependent chain of shared loads; the divisions are not).
  if (threadIdx.x == 0) {
    int count = 0;
    for (int a = 1; a <= W; ++a)
      for (int b = 1; b <= W; ++b) count += gcd_i(a, b) == 1;
    int ok = e != inf;
    if (ok) {
      int i = n, j = n;
      const uint8_t* pp = parent + (size_t)n * stride + n;
      while (i > 0) {
        const uint8_t s = *pp;
        if (s == 0xff || s >= count) {
          ok = 0;
          break;
        }
        int a, b;
        if constexpr (kW > 0 && kW <= 4) {  // (a-1, b-1) of every step in one constant: no table load in the chain
          constexpr unsigned long long kPack = pack_steps(kW);
          const int f = (int)((kPack >> (4 * s)) & 15);
          a = (f & 3) + 1;
          b = (f >> 2) + 1;
        } else {
          a = tab.a[s];
          b = tab.b[s];
        }
        const int pi = i - a, pj = j - b;
        pp -= (size_t)a * stride + b;
        for (int k = 0; k < a; ++k) gamma[pi + k] = __longlong_as_double(((long long)pj << 16) | (s << 8) | k);
        i = pi;
        j = pj;
      }
    }
    *cell = ok ? e : inf;
  }
  __syncthreads();
  const double r = *cell;
  if (r != inf) {
    for (int l = threadIdx.x; l < n; l += kT) {
      const long long code = __double_as_longlong(gamma[l]);
      const int k = (int)(code & 255), s = (int)((code >> 8) & 255), pj = (int)(code >> 16);
      const int a = tab.a[s], b = tab.b[s];
      const double jj = add((double)pj, dvd((double)(k * b), (double)a));
      gamma[l] = l == 0 ? 0.0 : dvd(jj, (double)n);
    }
    if (threadIdx.x == 0) gamma[n] = 1.0;
  }
  __syncthreads();
  return r;
}

// Reparameterization::eval (srv.cpp:39-50)
__device__ __forceinline__ double reparam_eval(const double* g, int n, double t) {
  if (t <= 0.0) return g[0];
  if (t >= 1.0) return g[n];
  const double x = mul(t, (double)n);
  const int i = min((int)x, n - 1);
  const double frac = sub(x, (double)i);
  return add(g[i], mul(frac, sub(g[i + 1], g[i])));
}

// compose_reparam(outer, inner) (elastic.cpp:21-33) -> out (n+1)
__device__ void compose(const double* outer, const double* inner, int n, double* out) {
  for (int l = threadIdx.x; l <= n; l += kT) out[l] = reparam_eval(outer, n, inner[l]);
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = 0.0;
    out[n] = 1.0;
    for (int l = 1; l <= n; ++l) out[l] = fmax(out[l], out[l - 1]);
  }
  __syncthreads();
}

// rebase_reparam(gamma, m) (elastic.cpp:37-50) -> out (n+1)
__device__ void rebase(const double* g, int n, int m, double* out) {
  const double gm = g[m];
  for (int l = threadIdx.x; l <= n; l += kT) {
    const int lm = l + m;
    out[l] = lm <= n ? sub(g[lm], gm) : sub(add(g[lm - n], 1.0), gm);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = 0.0;
    out[n] = 1.0;
  }
  __syncthreads();
}

// ------------------------------------------------------------- kernels

struct Smem {
  double2 *c1, *c2, *q1, *q2, *q1c, *w, *wc, *fft;
  double *g, *gc, *gd, *T, *ring, *cell;
  uint8_t* parent;
  cva_alignment* rec;
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Layout shared by the host size query and the kernel. Slab mode (fft ==
// false): the same arrays in the CTA's global slab, without the transform
// buffers (the rigid steps run the direct correlation, align_direct).
__host__ __device__ inline size_t smem_layout(int n, int W, bool parent_in_smem, char* base, Smem* S,
                                              bool fft_bufs = true) {
  const int M = pf::fft_len(n);
  const size_t fft = fft_bufs ? 4 * sizeof(double2) * (size_t)pf::padded_len(M) : 0;
  const size_t dp = align_up(sizeof(double) * (size_t)(W + 1) * (n + 1)) +
                    (parent_in_smem ? align_up((size_t)(n + 1) * (n + 1)) : 0);
  const size_t scratch = fft > dp ? fft : dp;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes);
    return base ? base + o : nullptr;
  };
  char* X = take(scratch);
  char* q1 = take(sizeof(double2) * n);
  char* q2 = take(sizeof(double2) * n);
  char* q1c = take(sizeof(double2) * n);
  char* w = take(sizeof(double2) * n);
  char* wc = take(sizeof(double2) * n);
  char* g = take(sizeof(double) * (n + 1));
  char* gc = take(sizeof(double) * (n + 1));
  char* gd = take(sizeof(double) * (n + 1));
  char* T = take(sizeof(double) * n);
  char* cell = take(sizeof(double) * 4);
  char* rec = take(sizeof(cva_alignment));
  if (S) {
    S->c1 = (double2*)w;  // raw curves: only before the first iteration
    S->c2 = (double2*)wc;
    S->fft = (double2*)X;
    S->ring = (double*)X;
    S->parent = parent_in_smem ? (uint8_t*)(X + align_up(sizeof(double) * (size_t)(W + 1) * (n + 1))) : nullptr;
    S->q1 = (double2*)q1;
    S->q2 = (double2*)q2;
    S->q1c = (double2*)q1c;
    S->w = (double2*)w;
    S->wc = (double2*)wc;
    S->g = (double*)g;
    S->gc = (double*)gc;
    S->gd = (double*)gd;
    S->T = (double*)T;
    S->cell = (double*)cell;
    S->rec = (cva_alignment*)rec;
  }
  return off;
}

// Slab mode (n or W beyond the shared-memory kernels): every per-pair array,
// the dp ring, the parent matrix and the step table live in a per-CTA slab of
// global memory (L2-resident for moderate n); shared memory keeps only the
// reduction cells. Returns the slab bytes per CTA.
__host__ __device__ inline int step_count(int W) {
  int c = 0;
  for (int a = 1; a <= W; ++a)
    for (int b = 1; b <= W; ++b) c += gcd_i(a, b) == 1;
  return c;
}
__host__ __device__ inline size_t slab_layout(int n, int W, char* base, Smem* S, uint8_t** parent, StepView* tv,
                                              double2** D) {
  size_t off = smem_layout(n, W, false, base, S, false);
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes);
    return base ? base + o : nullptr;
  };
  const int cnt = step_count(W);
  char* par = take((size_t)(n + 1) * (n + 1));
  char* d = take(sizeof(double2) * (size_t)n);
  char* sq = take(sizeof(double) * cnt);
  char* fr = take(sizeof(double) * (size_t)cnt * (W + 1));
  char* a = take(sizeof(int) * cnt);
  char* b = take(sizeof(int) * cnt);
  if (base) {
    *parent = (uint8_t*)par;
    *D = (double2*)d;
    *tv = StepView{(double*)sq, (double*)fr, W + 1, (int*)a, (int*)b};
  }
  return off;
}

// align_fft(a, b) (rigid_align.cpp:204-208) by the direct correlation: D_m =
// sum_l conj(a_l) b_{(l+m) mod n} for every shift m, each thread summing its
// shifts in order of l, then the pair stage's selection on |D_m| (max, the
// reference's tie band, smallest shift in the band; theta = arg D_m). Used in
// slab mode, where n is past the shared-memory transforms and the DP costs
// O(n^2 W^2) per iteration anyway. D: n double2 of scratch.
__device__ cva_alignment align_direct(const double2* a, const double2* b, int n, double2* D, double2* red) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  double s1 = 0.0, s2 = 0.0;
  for (int l = t; l < n; l += kT) {
    s1 = fma(a[l].x, a[l].x, fma(a[l].y, a[l].y, s1));
    s2 = fma(b[l].x, b[l].x, fma(b[l].y, b[l].y, s2));
  }
  constexpr int kB = 4;  // shifts per pass of a thread: one read of a_l feeds kB products
  double best2 = -1.0;
  for (int m0 = t; m0 < n; m0 += kB * kT) {
    double2 acc[kB];
    int j[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      acc[q] = make_double2(0.0, 0.0);
      j[q] = (m0 + q * kT) % n;  // padding lanes (m >= n, discarded) stay in range
    }
    for (int l = 0; l < n; ++l) {
      const double2 x = a[l];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const double2 y = b[j[q]];
        acc[q].x = fma(x.x, y.x, fma(x.y, y.y, acc[q].x));
        acc[q].y = fma(x.x, y.y, fma(-x.y, y.x, acc[q].y));
        j[q] = j[q] + 1 == n ? 0 : j[q] + 1;
      }
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int m = m0 + q * kT;
      if (m < n) {
        D[m] = acc[q];
        best2 = fmax(best2, fma(acc[q].x, acc[q].x, acc[q].y * acc[q].y));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    best2 = fmax(best2, __shfl_xor_sync(0xffffffffu, best2, o));
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  __shared__ double r3[3][kT / 32];
  __shared__ int s_cand[kT / 32];
  if (lane == 0) {
    r3[0][wid] = best2;
    r3[1][wid] = s1;
    r3[2][wid] = s2;
  }
  __syncthreads();
  best2 = -1.0;
  s1 = s2 = 0.0;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) {
    best2 = fmax(best2, r3[0][w]);
    s1 += r3[1][w];
    s2 += r3[2][w];
  }
  const double best = sqrt(best2);  // NaN if the correlation is not finite
  const double thr = best - pf::kTieRelTol * fmax(1.0, fabs(best));
  const double thr2 = thr > 0.0 ? thr * thr : -1.0;
  int cand = INT_MAX;
  for (int m = t; m < n; m += kT) {  // own entries: written by this thread above
    const double2 d = D[m];
    if (fma(d.x, d.x, d.y * d.y) >= thr2) {
      cand = m;
      break;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
  if (lane == 0) s_cand[wid] = cand;
  __syncthreads();
  int m = INT_MAX;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) m = min(m, s_cand[w]);
  const bool ok = isfinite(best) && best2 >= 0.0 && m != INT_MAX;
  cva_alignment r;
  if (!ok) {
    r.shift = 0;
    r.t0 = 0.0;
    r.theta = r.trace = r.energy = pf::qnan();
    r.degenerate = 0;
    r.status = CVA_INVALID_ARGUMENT;  // non-finite correlation (rigid_align.cpp:83)
  } else {
    const double2 dm = D[m];  // written by thread m % kT before the barrier above
    const double trace = sqrt(fma(dm.x, dm.x, dm.y * dm.y));
    const int degenerate = trace == 0.0;
    const double invN = 1.0 / (double)n;
    double e = invN * (s1 + s2) - 2.0 * invN * trace;  // rigid_align.cpp:56-59
    if (e < 0.0) e = 0.0;
    r.shift = m;
    r.t0 = (double)m / (double)n;
    r.theta = degenerate ? 0.0 : atan2(dm.y, dm.x);
    r.trace = trace;
    r.energy = e;
    r.degenerate = degenerate;
    r.status = CVA_OK;
  }
  __syncthreads();  // D and the reduction cells are reused by the next call
  return r;
}

__device__ __forceinline__ void load_curve(const double2* src, double2* dst, int n) {
  for (int l = threadIdx.x; l < n; l += kT) dst[l] = src[l];
}

// Per-CTA working set: shared memory (with the parents there or in the slab),
// or, in slab mode, the CTA's slab with only the cells in shared memory.
struct Work {
  Smem S;
  uint8_t* parent;
  StepView tv;
  const StepView* tvp;  // null: the shared step table
  double2* D;           // slab mode: align_direct scratch
};
template <bool kSlab>
__device__ __forceinline__ void setup_work(Work& w, char* smem, int n, int W, int parent_in_smem,
                                           uint8_t* parent_slab) {
  if constexpr (kSlab) {
    const size_t per = slab_layout(n, W, nullptr, nullptr, nullptr, nullptr, nullptr);
    slab_layout(n, W, (char*)parent_slab + (size_t)blockIdx.x * per, &w.S, &w.parent, &w.tv, &w.D);
    w.S.cell = (double*)smem;
    w.S.rec = (cva_alignment*)(smem + 64);
    w.tvp = &w.tv;
  } else {
    smem_layout(n, W, parent_in_smem != 0, smem, &w.S);
    w.parent = parent_in_smem ? w.S.parent : parent_slab + (size_t)blockIdx.x * (n + 1) * (n + 1);
    w.tvp = nullptr;
    w.D = nullptr;
  }
}

// Batched dp_reparam on SRV pairs (q1, q2: pairs x n).
template <int kW, bool kSlab = false>
__global__ void __launch_bounds__(kT, CVA_EL_MINB)
    dp_kernel(const double2* __restrict__ q1, const double2* __restrict__ q2, int64_t pairs, int n, int W,
              int parent_in_smem, uint8_t* parent_slab, double* gamma, double* energy, int32_t* status) {
  extern __shared__ __align__(16) char smem[];
  Work wk;
  setup_work<kSlab>(wk, smem, n, W, parent_in_smem, parent_slab);
  Smem& S = wk.S;
  for (int64_t p = blockIdx.x; p < pairs; p += gridDim.x) {
    load_curve(q1 + p * n, S.q1, n);
    load_curve(q2 + p * n, S.q2, n);
    __syncthreads();
    const double e = dp_reparam<kW>(S.q1, S.q2, n, W, S.ring, wk.parent, S.gd, S.cell, wk.tvp);
    const bool ok = isfinite(e);
    for (int l = threadIdx.x; l <= n; l += kT)
      gamma[p * (n + 1) + l] = ok ? S.gd[l] : __longlong_as_double(0x7ff8000000000000LL);
    if (threadIdx.x == 0) {
      energy[p] = ok ? e : __longlong_as_double(0x7ff8000000000000LL);
      if (status) status[p] = ok ? CVA_OK : CVA_RUNTIME_ERROR;  // srv.cpp:233
    }
    __syncthreads();
  }
}

// align_fft(a, b) on shared curves via the pair stage; result in S.rec.
template <int kN>
__device__ __forceinline__ cva_alignment align(const double2* a, const double2* b, int n, const Smem& S,
                                              const double2* tw, double2* red) {
  pf::PairIn in{a, b, make_double2(0, 0), make_double2(0, 0), 1.0, 1.0};
  __syncthreads();
  pf::pair_stage<false, kN>(in, S.fft, n, tw, S.rec, nullptr, red);
  __syncthreads();
  const cva_alignment r = *S.rec;
  __syncthreads();
  return r;
}

// elastic_distance_approach2 per pair. Pair p matches c2 onto c1 where
// matrix_k == 0: c1 = A + p n, c2 = B + p n; else (distance matrix of
// matrix_k curves A): c1 = A + (p / k) n, c2 = A + (p % k) n.
template <int kN, int kW, bool kSlab = false>
__global__ void __launch_bounds__(kT, CVA_EL_MINB)
    elastic_kernel(const double2* __restrict__ A, const double2* __restrict__ B, int64_t pairs, int64_t matrix_k,
                   int n_rt, ElasticParams prm, int parent_in_smem, uint8_t* parent_slab, const double2* tw,
                   ElasticOut out) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[16];
  const int n = kN > 0 ? kN : n_rt;
  const int W = kW > 0 ? kW : prm.max_slope;
  Work wk;
  setup_work<kSlab>(wk, smem, n, W, parent_in_smem, parent_slab);
  Smem& S = wk.S;
  uint8_t* parent = wk.parent;
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  // rigid alignment of two curves held in S: align_fft, or with use_fft = 0
  // (and in slab mode) the direct per-shift sums (align_naive's semantics)
  auto rigid = [&](const double2* a, const double2* b) {
    if constexpr (kSlab) {
      return align_direct(a, b, n, wk.D, red);
    } else {
      if (!prm.use_fft) return align_direct(a, b, n, S.fft, red);  // the transform buffers as scratch
      return align<kN>(a, b, n, S, tw, red);
    }
  };
  for (int64_t p = blockIdx.x; p < pairs; p += gridDim.x) {
    const double2* c1 = matrix_k ? A + (p / matrix_k) * n : A + p * n;
    const double2* c2 = matrix_k ? A + (p % matrix_k) * n : B + p * n;
    if constexpr (kSlab) {  // read in place (global either way)
      S.c1 = const_cast<double2*>(c1);
      S.c2 = const_cast<double2*>(c2);
    } else {
      load_curve(c1, S.c1, n);
      load_curve(c2, S.c2, n);
    }
    __syncthreads();
    // finite input (validate_curve, curve.cpp:11-14)
    int bad = 0;
    for (int l = threadIdx.x; l < n; l += kT)
      bad |= !(isfinite(S.c1[l].x) && isfinite(S.c1[l].y) && isfinite(S.c2[l].x) && isfinite(S.c2[l].y));
    bad = __syncthreads_or(bad);
    int status = CVA_OK;
    double t0 = 0.0, theta = 0.0, en = qnan;
    int iters = 0, conv = 0;
    if (bad) {
      status = CVA_INVALID_ARGUMENT;
    } else {
      srv_transform(S.c1, n, S.q1);
      srv_transform(S.c2, n, S.q2);
      __syncthreads();
      srv_center(S.q1, n, S.q1c, S.cell);
      // rigid pre-alignment of the curves themselves (elastic.cpp:114-117)
      const cva_alignment pre = rigid(S.c1, S.c2);
      if (pre.status != CVA_OK) {
        status = CVA_INVALID_ARGUMENT;
      } else {
        t0 = pre.t0;
        theta = pre.theta;
        for (int l = threadIdx.x; l <= n; l += kT) S.g[l] = l == n ? 1.0 : dvd((double)l, (double)n);
        __syncthreads();
        en = energy(S.q1, S.q2, n, t0, theta, S.g, S.T, S.cell);
        if (out.trace && threadIdx.x == 0) out.trace[p * (prm.max_iters + 1)] = en;
        for (int iter = 1; iter <= prm.max_iters; ++iter) {
          const double prev = en;
          {  // gamma-step (elastic.cpp:124-133)
            double s, c;
            sincos(theta, &s, &c);
            for (int l = threadIdx.x; l < n; l += kT) S.w[l] = action_at(S.q2, n, t0, c, s, S.g, l);
            __syncthreads();
            const double de = dp_reparam<kW>(S.q1, S.w, n, W, S.ring, parent, S.gd, S.cell, wk.tvp);
            if (!isfinite(de)) {
              status = CVA_RUNTIME_ERROR;  // srv.cpp:233
              break;
            }
            compose(S.g, S.gd, n, S.gc);
            const double e = energy(S.q1, S.q2, n, t0, theta, S.gc, S.T, S.cell);
            if (e <= en) {
              for (int l = threadIdx.x; l <= n; l += kT) S.g[l] = S.gc[l];
              en = e;
            }
            __syncthreads();
          }
          {  // (t0, R)-step (elastic.cpp:135-158)
            for (int l = threadIdx.x; l < n; l += kT) S.w[l] = action_at(S.q2, n, t0, 1.0, 0.0, S.g, l);
            __syncthreads();
            srv_center(S.w, n, S.wc, S.cell);
            const cva_alignment ra = rigid(S.q1c, S.wc);
            if (ra.status != CVA_OK) {
              status = CVA_INVALID_ARGUMENT;
              break;
            }
            const int m = (int)ra.shift;
            const double t0c = wrap_unit(add(t0, S.g[m]));
            rebase(S.g, n, m, S.gc);
            // raw-pair refit: optimal_rotation_svd(cross_correlation_matrix(q1, w, m))
            if (threadIdx.x == 0) {
              double a11 = 0.0, a12 = 0.0, a21 = 0.0, a22 = 0.0;
              for (int l = 0; l < n; ++l) {
                const double2 pq = S.q1[l];
                int lm = l + m;
                if (lm >= n) lm -= n;
                const double2 qq = S.w[lm];
                a11 = add(a11, mul(pq.x, qq.x));
                a12 = add(a12, mul(pq.x, qq.y));
                a21 = add(a21, mul(pq.y, qq.x));
                a22 = add(a22, mul(pq.y, qq.y));
              }
              const bool finite = isfinite(a11) && isfinite(a12) && isfinite(a21) && isfinite(a22);
              const bool zero = a11 == 0.0 && a12 == 0.0 && a21 == 0.0 && a22 == 0.0;
              S.cell[2] = !finite ? qnan : (zero ? 0.0 : atan2(sub(a12, a21), add(a11, a22)));
            }
            __syncthreads();
            const double th_raw = S.cell[2];
            __syncthreads();
            if (!isfinite(th_raw)) {
              status = CVA_INVALID_ARGUMENT;  // rigid_align.cpp:83
              break;
            }
            const double e_c = energy(S.q1, S.q2, n, t0c, ra.theta, S.gc, S.T, S.cell);
            const double e_r = energy(S.q1, S.q2, n, t0c, th_raw, S.gc, S.T, S.cell);
            const double r_cand = e_r <= e_c ? th_raw : ra.theta;
            const double e = fmin(e_r, e_c);
            if (e <= en) {
              t0 = t0c;
              theta = r_cand;
              for (int l = threadIdx.x; l <= n; l += kT) S.g[l] = S.gc[l];
              en = e;
            }
            __syncthreads();
          }
          iters = iter;
          if (out.trace && threadIdx.x == 0) out.trace[p * (prm.max_iters + 1) + iter] = en;  // elastic.cpp:160
          if (prev - en < prm.energy_tol) {
            conv = 1;
            break;
          }
        }
      }
    }
    const bool ok = status == CVA_OK;
    if (out.gamma)
      for (int l = threadIdx.x; l <= n; l += kT) out.gamma[p * (n + 1) + l] = ok ? S.g[l] : qnan;
    if (out.trace)  // NaN past the last recorded iteration (and everywhere for a failed pair)
      for (int k = threadIdx.x; k <= prm.max_iters; k += kT)
        if (!ok || k > iters) out.trace[p * (prm.max_iters + 1) + k] = qnan;
    if (threadIdx.x == 0) {
      out.distance[p] = ok ? sqrt(fmax(en, 0.0)) : qnan;  // elastic.cpp:19
      out.energy[p] = ok ? en : qnan;
      out.t0[p] = ok ? t0 : qnan;
      out.theta[p] = ok ? theta : qnan;
      out.iterations[p] = iters;
      out.converged[p] = conv;
      out.status[p] = status;
    }
    __syncthreads();
  }
}

// elastic_distance_approach1 (elastic.cpp:62-100), one work item per (pair,
// shift m): Kabsch rotation of the SRV pair at shift m, the shifted rotated SRV,
// one DP, and the realised energy at t0 = m / n. Items write (energy, theta,
// gamma) to scratch; a1_pick_kernel keeps, per pair, the first m with the
// smallest energy (the reference's strict `e < best` scan over m).
template <int kN, int kW, bool kSlab = false>
__global__ void __launch_bounds__(kT, CVA_EL_MINB)
    a1_kernel(const double2* __restrict__ A, const double2* __restrict__ B, int64_t pairs, int64_t matrix_k,
              int n_rt, int Wrt, int parent_in_smem, uint8_t* parent_slab, double* item_e, double* item_theta,
              double* item_gamma, int32_t* item_status) {
  extern __shared__ __align__(16) char smem[];
  const int n = kN > 0 ? kN : n_rt;
  const int W = kW > 0 ? kW : Wrt;
  Work wk;
  setup_work<kSlab>(wk, smem, n, W, parent_in_smem, parent_slab);
  Smem& S = wk.S;
  uint8_t* parent = wk.parent;
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  const int64_t items = pairs * n;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t p = it / n;
    const int m = (int)(it % n);
    const double2* c1 = matrix_k ? A + (p / matrix_k) * n : A + p * n;
    const double2* c2 = matrix_k ? A + (p % matrix_k) * n : B + p * n;
    if constexpr (kSlab) {
      S.c1 = const_cast<double2*>(c1);
      S.c2 = const_cast<double2*>(c2);
    } else {
      load_curve(c1, S.c1, n);
      load_curve(c2, S.c2, n);
    }
    __syncthreads();
    int bad = 0;
    for (int l = threadIdx.x; l < n; l += kT)
      bad |= !(isfinite(S.c1[l].x) && isfinite(S.c1[l].y) && isfinite(S.c2[l].x) && isfinite(S.c2[l].y));
    bad = __syncthreads_or(bad);
    int status = CVA_OK;
    double e = qnan, th = qnan;
    if (bad) {
      status = CVA_INVALID_ARGUMENT;
    } else {
      srv_transform(S.c1, n, S.q1);
      srv_transform(S.c2, n, S.q2);
      __syncthreads();
      if (threadIdx.x == 0) {  // optimal_rotation_svd(cross_correlation_matrix(q1, q2, m))
        double a11 = 0.0, a12 = 0.0, a21 = 0.0, a22 = 0.0;
        for (int l = 0; l < n; ++l) {
          const double2 pq = S.q1[l];
          int lm = l + m;
          if (lm >= n) lm -= n;
          const double2 qq = S.q2[lm];
          a11 = add(a11, mul(pq.x, qq.x));
          a12 = add(a12, mul(pq.x, qq.y));
          a21 = add(a21, mul(pq.y, qq.x));
          a22 = add(a22, mul(pq.y, qq.y));
        }
        const bool fin = isfinite(a11) && isfinite(a12) && isfinite(a21) && isfinite(a22);
        const bool zero = a11 == 0.0 && a12 == 0.0 && a21 == 0.0 && a22 == 0.0;
        S.cell[2] = !fin ? qnan : (zero ? 0.0 : atan2(sub(a12, a21), add(a11, a22)));
      }
      __syncthreads();
      th = S.cell[2];
      __syncthreads();
      if (!isfinite(th)) {
        status = CVA_INVALID_ARGUMENT;  // rigid_align.cpp:83
      } else {
        double sn, cs;
        sincos(th, &sn, &cs);
        for (int l = threadIdx.x; l < n; l += kT) {
          int lm = l + m;
          if (lm >= n) lm -= n;
          S.w[l] = rot_apply(cs, sn, S.q2[lm]);
        }
        __syncthreads();
        const double de = dp_reparam<kW>(S.q1, S.w, n, W, S.ring, parent, S.gd, S.cell, wk.tvp);
        if (!isfinite(de)) {
          status = CVA_RUNTIME_ERROR;
        } else {
          const double t0 = dvd((double)m, (double)n);
          e = energy(S.q1, S.q2, n, t0, th, S.gd, S.T, S.cell);
        }
      }
    }
    if (item_gamma)  // only when the caller wants gamma (not for distance matrices)
      for (int l = threadIdx.x; l <= n; l += kT) item_gamma[it * (n + 1) + l] = status == CVA_OK ? S.gd[l] : qnan;
    if (threadIdx.x == 0) {
      item_e[it] = e;
      item_theta[it] = th;
      item_status[it] = status;
    }
    __syncthreads();
  }
}

// Per pair: the first shift with the smallest energy (elastic.cpp:92-98), or
// the first failing item's status (an exception in the reference).
__global__ void a1_pick_kernel(int64_t pairs, int n, const double* item_e, const double* item_theta,
                               const double* item_gamma, const int32_t* item_status, ElasticOut out) {
  const int64_t p = blockIdx.x;
  if (p >= pairs) return;
  __shared__ int s_m, s_st;
  if (threadIdx.x == 0) {
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bm = -1, st = CVA_OK;
    for (int m = 0; m < n; ++m) {
      const int64_t it = p * n + m;
      if (item_status[it] != CVA_OK) {
        st = item_status[it];
        break;
      }
      if (item_e[it] < best) {
        best = item_e[it];
        bm = m;
      }
    }
    if (st == CVA_OK && bm < 0) st = CVA_RUNTIME_ERROR;
    s_m = bm;
    s_st = st;
  }
  __syncthreads();
  const int m = s_m;
  const bool ok = s_st == CVA_OK;
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  if (out.gamma)
    for (int l = threadIdx.x; l <= n; l += blockDim.x)
      out.gamma[p * (n + 1) + l] = ok ? item_gamma[(p * n + m) * (n + 1) + l] : qnan;
  if (threadIdx.x == 0) {
    const double e = ok ? item_e[p * n + m] : qnan;
    out.energy[p] = e;
    out.distance[p] = ok ? sqrt(fmax(e, 0.0)) : qnan;
    out.t0[p] = ok ? dvd((double)m, (double)n) : qnan;
    out.theta[p] = ok ? item_theta[p * n + m] : qnan;
    out.iterations[p] = ok ? 1 : 0;  // elastic.cpp:96-98
    out.converged[p] = ok ? 1 : 0;
    out.status[p] = s_st;
  }
}

// ---- single-call utilities behind the C++ drop-in (apply_srv_action,
// elastic_energy, dp_step_cost), one CTA.
__global__ void action_kernel(const double2* q, int n, double t0, double theta, const double* g, double2* out) {
  double s, c;
  sincos(theta, &s, &c);
  for (int l = threadIdx.x; l < n; l += blockDim.x) out[l] = action_at(q, n, t0, c, s, g, l);
}
__global__ void __launch_bounds__(kT) energy_kernel(const double2* q1, const double2* q2, int n, double t0,
                                                    double theta, const double* g, double* T, double* out) {
  __shared__ double cell[4];
  const double e = energy(q1, q2, n, t0, theta, g, T, cell);
  if (threadIdx.x == 0) *out = e;
}
__global__ void step_cost_kernel(const double2* q1, const double2* q2, int n, int i0, int j0, int a, int b,
                                 double* out) {
  *out = step_cost(q1, q2, n, i0, j0, a, b);
}

}  // namespace el

// ------------------------------------------------------------- launchers

namespace {
constexpr size_t kMaxSmem = 227 * 1024;

bool parent_fits(int n, int W) {
  return el::smem_layout(n, W, true, nullptr, nullptr) <= 110 * 1024;  // keep 2 CTAs/SM
}

// Resident CTAs of fn on the device. The dynamic shared-memory attribute must
// be raised first: without it the occupancy query sees the 48 KB default and
// reports 0 (which silently halved the grid before).
int resident(const void* fn, size_t smem) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, el::kT, smem) != cudaSuccess || per < 1) per = 1;
  return sms * per;
}
}  // namespace

// Shared-memory kernels: W <= 8 (shared step table), the pair-stage transform
// (M <= 1024) and the per-pair arrays in shared memory. Anything else the
// reference accepts runs in slab mode.
bool elastic_slab_mode(int n, int W) {
  return !(W <= 8 && pf::fft_len(n) <= 1024 && el::smem_layout(n, W, false, nullptr, nullptr) <= kMaxSmem);
}
constexpr size_t kSlabBudget = size_t(4) << 30;  // slab-mode scratch: the grid shrinks to fit
constexpr size_t kSlabSmem = 256;                // cells + alignment record

size_t elastic_smem(int n, int W) {
  if (elastic_slab_mode(n, W)) return kSlabSmem;
  return el::smem_layout(n, W, parent_fits(n, W), nullptr, nullptr);
}
bool elastic_supported(int n, int W) { return n >= 8 && n <= (1 << 20) && W >= 1 && W <= el::kMaxSlope; }

size_t elastic_parent_slab(int64_t pairs, int n, int W) {
  if (elastic_slab_mode(n, W)) return el::slab_layout(n, W, nullptr, nullptr, nullptr, nullptr, nullptr);
  if (parent_fits(n, W)) return 0;
  return (size_t)(n + 1) * (n + 1);  // per CTA; the launcher multiplies by the grid
}

template <int kW, bool kSlab>
static cudaError_t launch_dp_w(const double2* q1, const double2* q2, int64_t pairs, int n, int W, uint8_t* slab,
                               int grid, double* gamma, double* energy, int32_t* status, cudaStream_t s) {
  const bool ps = !kSlab && parent_fits(n, W);
  const size_t sm = elastic_smem(n, W);
  const void* fn = (const void*)el::dp_kernel<kW, kSlab>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  el::dp_kernel<kW, kSlab><<<grid, el::kT, sm, s>>>(q1, q2, pairs, n, W, ps ? 1 : 0, slab, gamma, energy, status);
  return cudaGetLastError();
}

int elastic_grid(int64_t pairs, int n, int W) {
  const size_t sm = elastic_smem(n, W);
  int r;
  if (elastic_slab_mode(n, W)) {
    r = resident((const void*)el::elastic_kernel<0, 0, true>, sm);
    r = std::min(r, resident((const void*)el::dp_kernel<0, true>, sm));
    r = std::min(r, resident((const void*)el::a1_kernel<0, 0, true>, sm));
    const size_t per = elastic_parent_slab(pairs, n, W);
    r = (int)std::max<size_t>(1, std::min<size_t>((size_t)r, kSlabBudget / per));
  } else {
    // the largest-footprint instance (most static shared memory) bounds all three kernels
    r = resident((const void*)el::elastic_kernel<0, 0>, sm);
    r = std::min(r, resident((const void*)el::dp_kernel<0>, sm));
    r = std::min(r, resident((const void*)el::a1_kernel<0, 0>, sm));
  }
  return (int)(pairs < r ? pairs : r);
}

cudaError_t launch_dp_reparam(const double2* q1, const double2* q2, int64_t pairs, int n, int W, uint8_t* slab,
                              int grid, double* gamma, double* energy, int32_t* status, cudaStream_t s) {
  if (elastic_slab_mode(n, W)) {
    if (W == 4) return launch_dp_w<4, true>(q1, q2, pairs, n, W, slab, grid, gamma, energy, status, s);
    return launch_dp_w<0, true>(q1, q2, pairs, n, W, slab, grid, gamma, energy, status, s);
  }
  if (W == 4) return launch_dp_w<4, false>(q1, q2, pairs, n, W, slab, grid, gamma, energy, status, s);
  return launch_dp_w<0, false>(q1, q2, pairs, n, W, slab, grid, gamma, energy, status, s);
}

template <int kN, int kW, bool kSlab = false>
static cudaError_t launch_el(const double2* A, const double2* B, int64_t pairs, int64_t k, int n,
                             const ElasticParams& prm, uint8_t* slab, int grid, const double2* tw,
                             const ElasticOut& out, cudaStream_t s) {
  const bool ps = !kSlab && parent_fits(n, prm.max_slope);
  const size_t sm = elastic_smem(n, prm.max_slope);
  const void* fn = (const void*)el::elastic_kernel<kN, kW, kSlab>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  el::elastic_kernel<kN, kW, kSlab><<<grid, el::kT, sm, s>>>(A, B, pairs, k, n, prm, ps ? 1 : 0, slab, tw, out);
  return cudaGetLastError();
}

cudaError_t launch_elastic_approach2(const double2* A, const double2* B, int64_t pairs, int64_t matrix_k, int n,
                                     const ElasticParams& prm, uint8_t* slab, int grid, const double2* tw,
                                     const ElasticOut& out, cudaStream_t s) {
  if (elastic_slab_mode(n, prm.max_slope)) {
    if (prm.max_slope == 4) return launch_el<0, 4, true>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
    return launch_el<0, 0, true>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
  }
  if (prm.max_slope == 4) {
    switch (n) {
      case 64: return launch_el<64, 4>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
      case 128: return launch_el<128, 4>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
      case 256: return launch_el<256, 4>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
      case 512: return launch_el<512, 4>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
      default: return launch_el<0, 4>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
    }
  }
  return launch_el<0, 0>(A, B, pairs, matrix_k, n, prm, slab, grid, tw, out, s);
}

template <int kN, int kW, bool kSlab = false>
static cudaError_t launch_a1(const double2* A, const double2* B, int64_t pairs, int64_t k, int n, int W,
                             uint8_t* slab, int grid, double* ie, double* ith, double* ig, int32_t* ist,
                             cudaStream_t s) {
  const bool ps = !kSlab && parent_fits(n, W);
  const size_t sm = elastic_smem(n, W);
  const void* fn = (const void*)el::a1_kernel<kN, kW, kSlab>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  el::a1_kernel<kN, kW, kSlab><<<grid, el::kT, sm, s>>>(A, B, pairs, k, n, W, ps ? 1 : 0, slab, ie, ith, ig, ist);
  return cudaGetLastError();
}

// Per item (pair, shift): energy, theta, status, and the item's gamma only
// when the caller asked for gamma (n + 1 doubles per item).
size_t elastic_a1_scratch(int64_t pairs, int n, bool gamma) {
  const int64_t items = pairs * n;
  return (size_t)items * (2 * sizeof(double) + sizeof(int32_t) + (gamma ? sizeof(double) * (n + 1) : 0)) + 1024;
}

cudaError_t launch_elastic_approach1(const double2* A, const double2* B, int64_t pairs, int64_t matrix_k, int n,
                                     int W, uint8_t* slab, int grid, void* scratch, const ElasticOut& out,
                                     cudaStream_t s) {
  const int64_t items = pairs * n;
  double* ie = (double*)scratch;
  double* ith = ie + items;
  double* ig = out.gamma ? ith + items : nullptr;
  int32_t* ist = (int32_t*)(ith + items + (out.gamma ? items * (n + 1) : 0));
  cudaError_t e;
  if (elastic_slab_mode(n, W)) {
    e = W == 4 ? launch_a1<0, 4, true>(A, B, pairs, matrix_k, n, W, slab, grid, ie, ith, ig, ist, s)
               : launch_a1<0, 0, true>(A, B, pairs, matrix_k, n, W, slab, grid, ie, ith, ig, ist, s);
  } else if (W == 4) {
    switch (n) {
      case 64: e = launch_a1<64, 4>(A, B, pairs, matrix_k, n, W, slab, grid, ie, ith, ig, ist, s); break;
      case 128: e = launch_a1<128, 4>(A, B, pairs, matrix_k, n, W, slab, grid, ie, ith, ig, ist, s); break;
      case 256: e = launch_a1<256, 4>(A, B, pairs, matrix_k, n, W, slab, grid, ie, ith, ig, ist, s); break;
      default: e = launch_a1<0, 4>(A, B, pairs, matrix_k, n, W, slab, grid, ie, ith, ig, ist, s); break;
    }
  } else {
    e = launch_a1<0, 0>(A, B, pairs, matrix_k, n, W, slab, grid, ie, ith, ig, ist, s);
  }
  if (e != cudaSuccess) return e;
  el::a1_pick_kernel<<<(unsigned)pairs, 128, 0, s>>>(pairs, n, ie, ith, ig, ist, out);
  return cudaGetLastError();
}

int elastic_items_grid(int64_t items, int n, int W) { return elastic_grid(items, n, W); }

cudaError_t launch_srv_action(const double2* q, int n, double t0, double theta, const double* g, double2* out,
                              cudaStream_t s) {
  el::action_kernel<<<1, el::kT, 0, s>>>(q, n, t0, theta, g, out);
  return cudaGetLastError();
}
cudaError_t launch_elastic_energy(const double2* q1, const double2* q2, int n, double t0, double theta,
                                  const double* g, double* T, double* out, cudaStream_t s) {
  el::energy_kernel<<<1, el::kT, 0, s>>>(q1, q2, n, t0, theta, g, T, out);
  return cudaGetLastError();
}
cudaError_t launch_dp_step_cost(const double2* q1, const double2* q2, int n, int i0, int j0, int a, int b,
                                double* out, cudaStream_t s) {
  el::step_cost_kernel<<<1, 1, 0, s>>>(q1, q2, n, i0, j0, a, b, out);
  return cudaGetLastError();
}

}  // namespace cva
