// Block-cooperative arc-length resampling of one closed curve (sm_100a, fp64).
//
// Replaces, per curve and inside one CTA:
//   arc_length_params            proj/src/curve.cpp:50-65
//   PeriodicCubicSpline ctor     proj/src/spline.cpp:62-96 (+ solve_cyclic_tridiagonal :16-58)
//   PeriodicCubicSpline::eval    proj/src/spline.cpp:98-117
//   resample_uniform             proj/src/curve.cpp:67-91
//   center_curve/normalize_length proj/src/curve.cpp:27-48
//
// The reference solves the cyclic tridiagonal system for the second derivatives
// with a serial Thomas sweep plus a Sherman-Morrison correction, twice (x and y)
// on identical knots. Here the system (scaled by 6)
//     h_{i-1} m_{i-1} + 2 (h_{i-1} + h_i) m_i + h_i m_{i+1} = 6 (dy_i/h_i - dy_{i-1}/h_{i-1})
// is solved once for both coordinates (double2 right-hand sides) by an exact
// partition method:
//   phase 1  K chunks (K a power of two); each thread eliminates its chunk's
//            interior, expressing it through the two neighbouring interface
//            unknowns w_{k-1}, w_k (one forward sweep; the back-substitution
//            values needed at the chunk ends are accumulated as running sums);
//   phase 2  the K interface equations form a cyclic tridiagonal system, solved
//            by cyclic reduction (PCR, log2 K steps, closed 2x2 at the end);
//   phase 3  each chunk re-solves its interior with known boundary values.
// No truncation is involved, so the result equals the reference's up to
// rounding (~1e-15 relative; the matrix is diagonally dominant with ratio 1/2).
// Parity note: the system solved is the one the reference's code actually
// solves, whose last row differs from the textbook periodic spline when
// h_{n-2} != h_{n-1} (see phase 2 and DESIGN.md, parity trap P11).
#pragma once

#include "cva_common.cuh"

namespace cva {

constexpr int kMaxChunk = 32;  // knots per chunk held in the phase-3 local array

// s[0..n]: h(i) = s[i+1] - s[i] for i in [-1, n-1]; h(-1) = h(n-1).
__device__ __forceinline__ double knot_h(const double* s, int n, int i) {
  return i < 0 ? s[n] - s[n - 1] : s[i + 1] - s[i];
}

__device__ __forceinline__ int spline_chunks(int n, int T) {
  int K = 2;
  while (K * 2 <= T && K * 2 <= n / 2) K *= 2;
  return K;
}

// Exclusive block scan of one double per thread; returns this thread's prefix
// and the block total in *total. `red` holds >= 33 double2.
__device__ __forceinline__ double block_exclusive_scan(double v, double* total, double2* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  double inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __syncthreads();
  if (lane == 31) red[wid].x = inc;
  __syncthreads();
  if (wid == 0) {
    double w = lane < nw ? red[lane].x : 0.0;
    double winc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, winc, o);
      if (lane >= o) winc += u;
    }
    red[lane].y = winc - w;  // exclusive prefix of warp totals
    if (lane == 31) red[32].x = winc;
  }
  __syncthreads();
  *total = red[32].x;
  return red[wid].y + inc - v;
}

// Normalised chordal arc length s[0..n] (s[n] = 1) of the closed polygon xy[0..n).
// Returns the total length; sets *bad on a non-positive edge (the reference's
// "coincident adjacent nodes", proj/src/curve.cpp:58).
__device__ inline double block_arc_length(const double2* xy, int n, double* s, double2* red, int* bad) {
  const int T = blockDim.x, t = threadIdx.x;
  const int C = (n + T - 1) / T;
  const int lo = min(n, t * C), hi = min(n, lo + C);
  double local = 0.0;
  int badl = 0;
  for (int i = lo; i < hi; ++i) {
    const double2 p = xy[i], q = xy[i + 1 == n ? 0 : i + 1];
    const double dx = q.x - p.x, dy = q.y - p.y;
    const double d = sqrt(fma(dx, dx, dy * dy));
    badl |= !(d > 0.0);
    local += d;
    s[i + 1] = local;  // local inclusive prefix, offset added below
  }
  double total;
  const double off = block_exclusive_scan(local, &total, red);
  const double inv = 1.0 / total;
  if (t == 0) s[0] = 0.0;
  for (int i = lo; i < hi; ++i) s[i + 1] = (s[i + 1] + off) * inv;
  __syncthreads();
  if (t == 0) s[n] = 1.0;
  // knots must be strictly increasing (proj/src/spline.cpp:66-68)
  for (int i = t; i < n; i += T) badl |= !(s[i + 1] > s[i]);
  *bad |= block_or(badl, red);
  return total;
}

struct ChunkEnds {  // values at the first / last interior knot of a chunk
  double2 v0f, v0l;
  double vLf, vLl, vRf, vRl;
};

// Solve the periodic spline system for m[0..n) (both coordinates). On entry m is
// scratch; `ends` holds >= K ChunkEnds (K <= blockDim.x). n >= 4, n <= K * kMaxChunk
// unless cpv_g is given (then any n).
// cpv_g: optional n-double scratch (global) for the phase-3 pivot ratios; null
// = a per-thread local array (chunks of <= kMaxChunk knots).
__device__ inline void block_spline_solve(const double* s, const double2* xy, double2* m, int n,
                                          ChunkEnds* ends, double2* red, double* cpv_g = nullptr) {
  const int T = blockDim.x, t = threadIdx.x;
  const int K = spline_chunks(n, T);

  // phase 0: right-hand sides, 6 (dy_i / h_i - dy_{i-1} / h_{i-1})
  for (int i = t; i < n; i += T) {
    const double hm = knot_h(s, n, i - 1), hi = knot_h(s, n, i);
    const double2 yp = xy[i == 0 ? n - 1 : i - 1], y0 = xy[i], yn = xy[i + 1 == n ? 0 : i + 1];
    const double ihm = 1.0 / hm, ihi = 1.0 / hi;
    m[i] = make_double2(6.0 * ((yn.x - y0.x) * ihi - (y0.x - yp.x) * ihm),
                        6.0 * ((yn.y - y0.y) * ihi - (y0.y - yp.y) * ihm));
  }
  __syncthreads();

  // phase 1: chunk interiors [a, b-1), interface unknown at b-1
  if (t < K) {
    const int a = (int)(((long long)t * n) / K), b = (int)(((long long)(t + 1) * n) / K);
    const int L = b - 2;
    double hm = knot_h(s, n, a - 1), hi = knot_h(s, n, a);
    double ib = 1.0 / (2.0 * (hm + hi));
    double2 g = cscale(m[a], ib);
    double gL = -hm * ib;
    double Q = 1.0;
    double2 S = g;
    double SL = gL;
    for (int i = a + 1; i <= L; ++i) {
      hm = hi;
      hi = knot_h(s, n, i);
      const double cpr = hm * ib;
      ib = 1.0 / (2.0 * (hm + hi) - hm * cpr);
      const double2 r = m[i];
      g = make_double2((r.x - hm * g.x) * ib, (r.y - hm * g.y) * ib);
      gL = -hm * gL * ib;
      Q *= -cpr;
      S.x = fma(g.x, Q, S.x);
      S.y = fma(g.y, Q, S.y);
      SL = fma(gL, Q, SL);
    }
    ChunkEnds e;
    e.v0l = g;
    e.v0f = S;
    e.vLl = gL;
    e.vLf = SL;
    e.vRl = -hi * ib;
    e.vRf = e.vRl * Q;
    ends[t] = e;
  }
  __syncthreads();

  // phase 2: interface system row k (knot j = b_k - 1), then cyclic PCR
  double ra = 0, rd = 0, rc = 0;
  double2 rr = make_double2(0, 0);
  int j = 0;
  if (t < K) {
    j = (int)(((long long)(t + 1) * n) / K) - 1;
    const int kn = t + 1 == K ? 0 : t + 1;
    const double hL = knot_h(s, n, j - 1), hj = knot_h(s, n, j);
    const ChunkEnds e = ends[t], en = ends[kn];
    const double2 r = m[j];
    double dj = 2.0 * (hL + hj), sj = hj;
    if (t == K - 1) {
      // Row n-1 as the reference actually solves it. Its Sherman-Morrison split
      // (proj/src/spline.cpp:20-26, :43-46) takes u[n-1] = b[n-1] and
      // v[n-1] = a[n-1]/g where the cyclic corner is a[n-1] / b[0], so with
      // non-uniform knots the last row reads
      //   h_{n-2} m_{n-2} + (2(h_{n-2}+h_{n-1}) + h_{n-1}(h_{n-1}-h_{n-2}) / (2(h_{n-1}+h_0))) m_{n-1}
      //     + h_{n-2} m_0 = r_{n-1}
      // (scaled by 6). Identical to the textbook row when h_{n-2} = h_{n-1}.
      const double h0 = knot_h(s, n, 0);
      sj = hL;
      dj = 2.0 * (hL + hj) + hj * (hj - hL) / (2.0 * (hj + h0));
    }
    ra = hL * e.vLl;
    rd = dj + hL * e.vRl + sj * en.vLf;
    rc = sj * en.vRf;
    rr = make_double2(r.x - hL * e.v0l.x - sj * en.v0f.x, r.y - hL * e.v0l.y - sj * en.v0f.y);
  }
  // PCR storage reuses `ends` (>= K * 48 bytes needed, ChunkEnds is 64 bytes)
  double* pa = reinterpret_cast<double*>(ends);
  double* pd = pa + K;
  double* pc = pd + K;
  double2* pr = reinterpret_cast<double2*>(pc + K);
  __syncthreads();
  if (t < K) {
    pa[t] = ra;
    pd[t] = rd;
    pc[t] = rc;
    pr[t] = rr;
  }
  __syncthreads();
  for (int st = 1; st < K / 2; st *= 2) {
    if (t < K) {
      const int im = (t - st) & (K - 1), ip = (t + st) & (K - 1);
      const double al = -ra / pd[im], ga = -rc / pd[ip];
      const double na = al * pa[im], nc = ga * pc[ip];
      rd = rd + al * pc[im] + ga * pa[ip];
      const double2 rm = pr[im], rp = pr[ip];
      rr = make_double2(rr.x + al * rm.x + ga * rp.x, rr.y + al * rm.y + ga * rp.y);
      ra = na;
      rc = nc;
    }
    __syncthreads();
    if (t < K) {
      pa[t] = ra;
      pd[t] = rd;
      pc[t] = rc;
      pr[t] = rr;
    }
    __syncthreads();
  }
  double2 w = make_double2(0, 0);
  if (t < K) {
    const int jp = (t + K / 2) & (K - 1);
    const double ei = ra + rc, ej = pa[jp] + pc[jp], dj = pd[jp];
    const double2 rj = pr[jp];
    const double idet = 1.0 / (rd * dj - ei * ej);
    w = make_double2((rr.x * dj - ei * rj.x) * idet, (rr.y * dj - ei * rj.y) * idet);
  }
  __syncthreads();
  if (t < K) m[j] = w;
  __syncthreads();

  // phase 3: interior re-solve with known interface values
  if (t < K) {
    const int a = (int)(((long long)t * n) / K), b = (int)(((long long)(t + 1) * n) / K);
    const int L = b - 2;
    const double2 wl = m[a == 0 ? n - 1 : a - 1], wr = m[b - 1];
    double cpv_l[kMaxChunk];
    double* cpv = cpv_g ? cpv_g + a : cpv_l;
    double hm = knot_h(s, n, a - 1), hi = knot_h(s, n, a);
    double ib = 1.0 / (2.0 * (hm + hi));
    double2 r = m[a];
    r.x -= hm * wl.x;
    r.y -= hm * wl.y;
    if (a == L) {
      r.x -= hi * wr.x;
      r.y -= hi * wr.y;
    }
    double2 g = cscale(r, ib);
    m[a] = g;
    for (int i = a + 1; i <= L; ++i) {
      hm = hi;
      hi = knot_h(s, n, i);
      const double cpr = hm * ib;
      cpv[i - a - 1] = cpr;  // c'_i
      ib = 1.0 / (2.0 * (hm + hi) - hm * cpr);
      r = m[i];
      if (i == L) {
        r.x -= hi * wr.x;
        r.y -= hi * wr.y;
      }
      g = make_double2((r.x - hm * g.x) * ib, (r.y - hm * g.y) * ib);
      m[i] = g;
    }
    double2 v = g;
    for (int i = L - 1; i >= a; --i) {
      const double c = cpv[i - a];  // c'_{i+1}
      const double2 gi = m[i];
      v = make_double2(gi.x - c * v.x, gi.y - c * v.y);
      m[i] = v;
    }
  }
  __syncthreads();
}

// First output index l in [0, n_out] with l / n_out >= x.
__device__ __forceinline__ int first_sample_at_or_after(double x, int n_out) {
  const double nn = (double)n_out;
  int l = (int)ceil(x * nn);
  l = max(0, min(n_out, l));
  while (l > 0 && (double)(l - 1) / nn >= x) --l;
  while (l < n_out && (double)l / nn < x) ++l;
  return l;
}

// Evaluate the periodic spline at t_l = l / n_out, l in [0, n_out), into out[].
// Chunk-owner evaluation: the thread owning knots [a, b) emits the samples with
// s_a <= t < s_b (the reference's upper_bound interval rule, spline.cpp:98-105).
__device__ inline void block_spline_eval(const double* s, const double2* xy, const double2* m, int n,
                                         int n_out, double2* out) {
  const int T = blockDim.x, t = threadIdx.x;
  const int K = spline_chunks(n, T);
  if (t < K) {
    const int a = (int)(((long long)t * n) / K), b = (int)(((long long)(t + 1) * n) / K);
    const int l_lo = t == 0 ? 0 : first_sample_at_or_after(s[a], n_out);
    const int l_hi = t == K - 1 ? n_out : first_sample_at_or_after(s[b], n_out);
    const double nn = (double)n_out;
    int i = a;
    for (int l = l_lo; l < l_hi; ++l) {
      const double tt = (double)l / nn;
      while (i < b - 1 && s[i + 1] <= tt) ++i;
      const int i1 = i + 1 == n ? 0 : i + 1;
      const double s0 = s[i], s1 = s[i + 1];
      const double h = s1 - s0, ih = 1.0 / h;
      const double A = (s1 - tt) * ih, B = (tt - s0) * ih;
      const double ca = (A * A * A - A), cb = (B * B * B - B), h26 = h * h / 6.0;
      const double2 y0 = xy[i], y1 = xy[i1], m0 = m[i], m1 = m[i1];
      out[l] = make_double2(A * y0.x + B * y1.x + (ca * m0.x + cb * m1.x) * h26,
                            A * y0.y + B * y1.y + (ca * m0.y + cb * m1.y) * h26);
    }
  }
  __syncthreads();
}

// center_curve then normalize_length on buf[0..n) in place (proj/src/curve.cpp:27-48).
__device__ inline void block_center_normalize(double2* buf, int n, double2* red, int* bad) {
  const int T = blockDim.x, t = threadIdx.x;
  double2 acc = make_double2(0, 0);
  for (int i = t; i < n; i += T) acc = cadd(acc, buf[i]);
  acc = block_sum2(acc, red);
  const double invn = 1.0 / (double)n;
  const double2 g = make_double2(invn * acc.x, invn * acc.y);
  for (int i = t; i < n; i += T) buf[i] = csub(buf[i], g);
  __syncthreads();
  double len = 0.0;
  for (int i = t; i < n; i += T) {
    const double2 p = buf[i], q = buf[i + 1 == n ? 0 : i + 1];
    const double dx = q.x - p.x, dy = q.y - p.y;
    len += sqrt(fma(dx, dx, dy * dy));
  }
  len = block_sum(len, red);
  *bad |= !(len > 0.0);
  const double sc = 1.0 / len;
  __syncthreads();
  for (int i = t; i < n; i += T) buf[i] = cscale(buf[i], sc);
  __syncthreads();
}

}  // namespace cva
