// Arc-length spline resampling of one closed curve by one 256-thread CTA (v2).
//
// Replaces, per curve (reference file:line):
//   arc_length_params              proj/src/curve.cpp:50-65
//   PeriodicCubicSpline ctor/solve proj/src/spline.cpp:62-96, :16-58
//   PeriodicCubicSpline::eval      proj/src/spline.cpp:98-117
//   resample_uniform               proj/src/curve.cpp:67-91
//   centroid / curve_length        proj/src/curve.cpp:17-32 (returned, applied by the caller)
//
// Layout: the raw curve (n <= kNMax nodes, 16 B each) and its knots s[0..n]
// live in shared memory (24 B/node, 72 KB at the 3072-node maximum). Thread t
// owns chunk [a_t, a_{t+1}) of K <= 256 knots (<= kCMax = 12 per chunk), and
// keeps the chunk's right-hand sides and pivots in registers, so no per-knot
// solver state is stored.
//
// The spline system is solved in the scaled unknowns mu = m / 6:
//   h_{i-1} mu_{i-1} + 2 (h_{i-1} + h_i) mu_i + h_i mu_{i+1} = slope_i - slope_{i-1},
//   slope_i = (y_{i+1} - y_i) / h_i,
// and evaluated as  A y_i + B y_{i+1} + ((A^3 - A) mu_i + (B^3 - B) mu_{i+1}) h_i^2,
// which is the reference's system and cubic (spline.cpp:80-92, :107-117) with
// the factor 6 folded into mu.
//
// Solver (exact; no truncation):
//   phase 1  each chunk eliminates its interior [a, b-1) by a forward Thomas
//            sweep, expressing it through the interface unknowns w_{k-1}, w_k
//            (= mu at the chunk's last knot b-1); the end values of the three
//            back-substituted responses are accumulated as running sums.
//   phase 2  the K interface rows form a cyclic tridiagonal system, solved by
//            parallel cyclic reduction (log2 K steps, ping-pong buffers, one
//            barrier per step, closed 2x2 solve at stride K/2).
//   phase 3  each chunk re-sweeps its interior with the now-known boundary
//            values and evaluates the resampled nodes inside its knot
//            intervals during the back-substitution (no mu array is stored).
//
// Parity trap (P11): the reference's Sherman-Morrison split uses
// u[n-1] = b[n-1], v[n-1] = a[n-1]/g where the cyclic corner is a[n-1], b[0]
// (spline.cpp:20-26, :43-46), so the last row it solves is
//   h_{n-2} mu_{n-2} + (2(h_{n-2}+h_{n-1}) + h_{n-1}(h_{n-1}-h_{n-2})/(2(h_{n-1}+h_0))) mu_{n-1}
//     + h_{n-2} mu_0 = r_{n-1}.
// That row is always an interface row here (chunk K-1 ends at n-1) and is
// reproduced in phase 2.
#pragma once

#include "cva_common.cuh"
#include "prof.cuh"

namespace cva {
namespace rs {

constexpr int kT = 256;            // threads per CTA = max chunks
constexpr int kCMax = 12;          // knots per chunk
constexpr int kNMax = kT * kCMax;  // raw nodes per curve (3072)
constexpr int kScratchDoubles = 11 * kT + 2;  // PCR ping-pong (2 x 5 arrays; F / W / MB alias them) + chunk offsets

__device__ __forceinline__ void bar_sync() { __syncthreads(); }

// log2 of the chunk count K: the largest power of two <= min(kT, n / 2), >= 2.
__device__ __forceinline__ int log2_chunks(int n) {
  const int c = min(kT, n >> 1);
  return max(1, 31 - __clz(c));
}

// frcp / fsqrt: cva_common.cuh

// Block exclusive scan of one double per thread (kT threads); also returns the
// total. red: >= 16 double2 of shared scratch.
__device__ __forceinline__ double scan_excl(double v, double* total, double2* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bar_sync();  // previous readers of red are done
  double inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) red[wid].x = inc;
  bar_sync();
  double pre = 0.0, tot = 0.0;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) {
    const double x = red[w].x;
    if (w < wid) pre += x;
    tot += x;
  }
  *total = tot;
  return pre + inc - v;
}

// Sum of three doubles over the block (kT threads); every thread gets the sums.
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double2* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  bar_sync();
  if (lane == 0) {
    red[wid] = make_double2(a, b);
    red[8 + wid].x = c;
  }
  bar_sync();
  a = b = c = 0.0;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) {
    a += red[w].x;
    b += red[w].y;
    c += red[8 + w].x;
  }
}

struct CurveStats {
  double2 centroid;  // vertex mean of the resampled nodes (curve.cpp:27-32)
  double inv_len;    // 1 / polygon length incl. closing edge (curve.cpp:17-25, :41-48)
  int bad;           // invalid input (too few / non-finite / coincident nodes)
};

// First sample index l in [0, N] with t_l = l / N >= x, t_l computed as the
// reference does ((double)l / (double)N, curve.cpp:88). For N = 2^p, x * N is
// exact and the answer is ceil(x N). Clamped to [0, N] so that garbage knots
// of an invalid curve (NaN / inf, flagged separately) never index outside.
template <bool kPow2>
__device__ __forceinline__ int first_sample(double x, int N) {
  const double nn = (double)N;
  const double c = ceil(x * nn);
  int l = c >= 0.0 ? (c <= nn ? (int)c : N) : 0;  // NaN -> 0
  if (!kPow2) {
    while (l > 0 && (double)(l - 1) / nn >= x) --l;
    while (l < N && (double)l / nn < x) ++l;
  }
  return l;
}

template <bool kPow2>
__device__ __forceinline__ double sample_t(int l, int N, double invN) {
  return kPow2 ? (double)l * invN : (double)l / (double)N;
}

// Resample the raw curve already in xy[0..n) (shared) at t_l = l/N, l < N, into
// out[0..N) (shared or global), uncentered. Returns the centroid and 1/length of
// the resampled polygon so that preprocess(c) = (out - centroid) * inv_len.
//
// Knots follow the reference's rounding structure (curve.cpp:50-65,
// spline.cpp:85): s_i = S_i / T with S_i the chordal prefix sum and T the
// perimeter, and h_i = s_{i+1} - s_i (spacings taken from the normalised knots,
// as the reference does, not from the edge lengths: with uneven spacing the
// two differ by ~ulp(1)/h relative, which the spline system amplifies). S_i is a
// two-level sum: sequential within a chunk, exclusive scan across chunks.
//
// L: shared, >= n + 1 doubles (chunk-local prefix sums, normalised in place). scr: shared,
// kScratchDoubles. red: 16 double2. Requires 4 <= n <= kNMax, N >= 8 (kPow2:
// N = 2^p), blockDim.x == kT. NOTE: no __restrict__ on these pointers: they
// carry data between threads across __syncthreads(), and restrict lets the
// compiler forward stale loads across the barrier.
// kLen = false skips the polygon length (inv_len is then not set, bad covers
// the knots only): the fused pair kernel measures it while loading its FFT.
// kPadOut: out is shared memory indexed out[l + (l >> 3)] (one pad slot per
// 8 samples: the chunk-strided sample stores spread over all banks).
// kOutInScr: out may alias scr (>= N + N/8 double2): the PCR scratch is dead
// once phase 3 has read its boundary values, so the samples go there.
template <bool kPow2, bool kLen = true, bool kPadOut = false, bool kOutInScr = false>
__device__ inline CurveStats resample_block(const double2* xy, int n, double* L, double* scr,
                                            double2* red, double2* out, const int N,
                                            const int pb = 0 /* phase-stamp base */) {
  const int t = threadIdx.x;
  const int lane = t & 31, wid = t >> 5;
  const int lgK = log2_chunks(n);
  const int K = 1 << lgK;
  const bool own = t < K;
  const int a = own ? (t * n) >> lgK : 0;
  const int b = own ? ((t + 1) * n) >> lgK : 0;
  const int M = b - 1 - a;  // interior knots (>= 1); knot b-1 is the interface
  int bad = 0;

  // ---- phase 0: chordal edges, chunk-local prefix sums, cross-chunk scan
  double tot = 0.0;
  if (own) {
    double2 p = xy[a];
#pragma unroll 4
    for (int i = a; i < b; ++i) {
      const double2 q = xy[i + 1 == n ? 0 : i + 1];
      const double dx = q.x - p.x, dy = q.y - p.y;
      p = q;
      const double d = fsqrt(fma(dx, dx, dy * dy));  // curve.cpp:57
      bad |= !(d > 0.0);                             // coincident nodes (curve.cpp:58)
      tot += d;
      if (i + 1 < b) L[(i + 1 - a) * K + t] = tot;
    }
  }
  double inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  bar_sync();  // previous users of red are done
  if (lane == 31) red[wid].x = inc;
  bar_sync();
  double T = 0.0, pre = 0.0;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) {
    const double x = red[w].x;
    if (w < wid) pre += x;
    T += x;
  }
  bad |= !isfinite(T);
  const double invT = 1.0 / T;
  // normalise in place: s_i = (OFF_t + L_i) / T for this chunk's knots
  // a..b-1 (s_a = OFF_t / T); s_n = 1 (curve.cpp:63-64) is not stored.
  // Knot layout is chunk-major: s_{a_t + j} lives at sk[j K + t], so the
  // per-chunk sweeps (thread t at offset j) hit consecutive words.
  double* sk = L;
  if (own) {
    const double off = pre + inc - tot;
    sk[t] = off * invT;
#pragma unroll 4
    for (int j = 1; j < b - a; ++j) sk[j * K + t] = (off + sk[j * K + t]) * invT;
  }
  bar_sync();
  auto own_knot = [&](int j) -> double { return sk[j * K + t]; };  // s_{a+j}
  // s_b: the next chunk's first knot (s_n = 1 after the last chunk)
  auto next_knot = [&]() -> double { return t == K - 1 ? 1.0 : sk[t + 1]; };
  // s_{a-1}: the previous chunk's last knot (s_{n-1} before the first chunk)
  auto prev_knot = [&]() -> double {
    const int tp = t == 0 ? K - 1 : t - 1;
    const int ap = (tp * n) >> lgK;
    const int cp = (t == 0 ? n : a) - ap;
    return sk[(cp - 1) * K + tp];
  };
  CVA_MARK(pb + 0);

  // ---- phase 1: rhs, forward sweep, chunk-end responses
  double2 R[kCMax];  // right-hand sides, later forward values g
  double IB[kCMax];  // 1 / pivot of interior rows
  double2 v0f = make_double2(0, 0), v0l = make_double2(0, 0);
  double vLf = 0, vLl = 0, vRf = 0, vRl = 0;
  double hL = 0, hj = 0;            // h_{b-2}, h_{b-1}
  double2 rj = make_double2(0, 0);  // rhs of the interface row b-1
  if (own) {
    // h_{a-1} = s_a - s_{a-1} (h_{n-1} = s_n - s_{n-1} for the first chunk)
    const int ap = a == 0 ? n - 1 : a - 1;
    double si = own_knot(0);
    double hm = (a == 0 ? 1.0 : si) - prev_knot();
    const double2 yp = xy[ap];
    double2 y0 = xy[a];
    const double ihm = frcp(hm);
    double2 slp = make_double2((y0.x - yp.x) * ihm, (y0.y - yp.y) * ihm);
    double2 g = make_double2(0, 0);
    double gL = 0, Q = 1.0, ib = 0;
    double2 S = make_double2(0, 0);
    double SL = 0;
    // interior rows a .. b-2 (j < M); the interface row b-1 follows the loop,
    // so the unrolled rows carry no second data-dependent branch
#pragma unroll
    for (int j = 0; j < kCMax; ++j) {
      if (j < M) {
        const int i = a + j;
        const double sn = own_knot(j + 1);
        const double h = sn - si;
        bad |= !(h > 0.0);  // strictly increasing knots (spline.cpp:66-68)
        const double ih = frcp(h);
        const double2 y1 = xy[i + 1];  // i + 1 <= b - 1 < n
        const double2 sl = make_double2((y1.x - y0.x) * ih, (y1.y - y0.y) * ih);
        const double2 r = make_double2(sl.x - slp.x, sl.y - slp.y);
        R[j] = r;
        if (j == 0) {
          ib = frcp(2.0 * (hm + h));
          g = cscale(r, ib);
          gL = -hm * ib;
          S = g;
          SL = gL;
        } else {
          const double cpr = hm * ib;
          ib = frcp(fma(-hm, cpr, 2.0 * (hm + h)));
          g = make_double2(fma(-hm, g.x, r.x) * ib, fma(-hm, g.y, r.y) * ib);
          gL = -hm * gL * ib;
          Q *= -cpr;
          S.x = fma(g.x, Q, S.x);
          S.y = fma(g.y, Q, S.y);
          SL = fma(gL, Q, SL);
        }
        IB[j] = ib;
        hm = h;
        slp = sl;
        y0 = y1;
        si = sn;
      }
    }
    {  // interface row b-1: its spacing and right-hand side
      hL = hm;
      const double sn = next_knot();
      const double h = sn - si;
      bad |= !(h > 0.0);
      const double ih = frcp(h);
      const double2 y1 = xy[b == n ? 0 : b];
      rj = make_double2((y1.x - y0.x) * ih - slp.x, (y1.y - y0.y) * ih - slp.y);
      hj = h;
    }
    v0l = g;
    vLl = gL;
    vRl = -hL * ib;
    vRf = vRl * Q;
    v0f = S;
    vLf = SL;
  }

  // ---- exchange chunk-start responses
  double* F = scr + 5 * kT;  // PCR buffer 1 as [K][4]: v0f.x, v0f.y, vLf, vRf
  if (own) {
    F[4 * t + 0] = v0f.x;
    F[4 * t + 1] = v0f.y;
    F[4 * t + 2] = vLf;
    F[4 * t + 3] = vRf;
  }
  bar_sync();
  CVA_MARK(pb + 1);

  // ---- phase 2: interface rows -> cyclic PCR
  double ra = 0, rc = 0, rd = 1, rid = 1;
  double2 rr = make_double2(0, 0);
  if (own) {
    const int tn = t + 1 == K ? 0 : t + 1;
    const double2 nf = make_double2(F[4 * tn + 0], F[4 * tn + 1]);
    const double nL = F[4 * tn + 2], nR = F[4 * tn + 3];
    double dj = 2.0 * (hL + hj), sj = hj;
    if (t == K - 1) {  // the reference's last row (see header, P11); h_0 = s_1 - s_0
      const double h0 = sk[K] - sk[0];  // s_1 - s_0 (chunk 0, offsets 1 and 0)
      sj = hL;
      dj = 2.0 * (hL + hj) + hj * (hj - hL) / (2.0 * (hj + h0));
    }
    ra = hL * vLl;
    rd = dj + hL * vRl + sj * nL;
    rc = sj * nR;
    rr = make_double2(rj.x - hL * v0l.x - sj * nf.x, rj.y - hL * v0l.y - sj * nf.y);
    rid = frcp(rd);
  }
  {
    int buf = 0;
    auto P = [&](int bsel, int arr) { return scr + (bsel * 5 + arr) * kT; };
    if (own) {  // buffer 0 (F lives in buffer 1, read above)
      P(0, 0)[t] = ra;
      P(0, 1)[t] = rc;
      P(0, 2)[t] = rid;
      P(0, 3)[t] = rr.x;
      P(0, 4)[t] = rr.y;
    }
    bar_sync();
    // Early exit: the interface couplings shrink quadratically per PCR step
    // (|a|,|c| / d ~ rho^(C 2^k) for a chunk of C knots, rho <= 1/2); once every
    // row's off-diagonals are below 2^-64 of its diagonal the remaining
    // steps cannot change w in fp64, and the closing 2x2 below reduces to r/d.
    for (int st = 1; st < K / 2; st *= 2) {
      bool done = true;
      if (own) {
        const int im = (t - st) & (K - 1), ip = (t + st) & (K - 1);
        const double* A = P(buf, 0);
        const double* C = P(buf, 1);
        const double* ID = P(buf, 2);
        const double al = -ra * ID[im], ga = -rc * ID[ip];
        const double na = al * A[im], nc = ga * C[ip];
        rd = rd + al * C[im] + ga * A[ip];
        rr.x = rr.x + al * P(buf, 3)[im] + ga * P(buf, 3)[ip];
        rr.y = rr.y + al * P(buf, 4)[im] + ga * P(buf, 4)[ip];
        ra = na;
        rc = nc;
        rid = frcp(rd);
        const int nb = buf ^ 1;
        P(nb, 0)[t] = ra;
        P(nb, 1)[t] = rc;
        P(nb, 2)[t] = rid;
        P(nb, 3)[t] = rr.x;
        P(nb, 4)[t] = rr.y;
        done = fabs(ra) + fabs(rc) <= 0x1p-64 * fabs(rd);
      }
      buf ^= 1;
      if (__syncthreads_and(done)) break;  // the step's barrier doubles as the vote
    }
    double2 w = make_double2(0, 0);
    if (own) {
      const int jp = (t + K / 2) & (K - 1);
      const double ei = ra + rc, ej = P(buf, 0)[jp] + P(buf, 1)[jp];
      const double dj = 1.0 / P(buf, 2)[jp];
      const double2 rjp = make_double2(P(buf, 3)[jp], P(buf, 4)[jp]);
      const double idet = 1.0 / (rd * dj - ei * ej);
      w = make_double2((rr.x * dj - ei * rjp.x) * idet, (rr.y * dj - ei * rjp.y) * idet);
    }
    // W and MB go to the buffer not read in the final step
    double2* W = reinterpret_cast<double2*>(P(buf ^ 1, 0));
    double2* MB = W + kT;
    if (own) W[t] = w;
    bar_sync();
    double2 wl = make_double2(0, 0);
    if (own) {
      wl = W[t == 0 ? K - 1 : t - 1];
      // mu at this chunk's first knot a (its first interior row), published for chunk t-1
      MB[t] = make_double2(v0f.x + wl.x * vLf + w.x * vRf, v0f.y + wl.y * vLf + w.y * vRf);
    }
    bar_sync();
    CVA_MARK(pb + 2);

    // ---- phase 3: interior re-solve + fused evaluation
    double2 cacc = make_double2(0, 0);
    double2 mub = make_double2(0, 0);
    if (own) mub = MB[t + 1 == K ? 0 : t + 1];
    if constexpr (kOutInScr) bar_sync();  // out aliases scr (W, MB): every read above is done
    if (own) {
      // forward with known boundary values, in place (R[j] <- g_j): each row
      // reads its left spacing from the knots and g_{j-1} from R[j-1], so no
      // value rotates through the data-dependent guard
      {
        const double hm0 = (a == 0 ? 1.0 : own_knot(0)) - prev_knot();
        const double2 r0 = make_double2(fma(-hm0, wl.x, R[0].x), fma(-hm0, wl.y, R[0].y));
        R[0] = cscale(r0, IB[0]);
      }
#pragma unroll
      for (int j = 1; j < kCMax; ++j) {
        if (j < M) {
          const double hm = own_knot(j) - own_knot(j - 1);
          R[j] = make_double2(fma(-hm, R[j - 1].x, R[j].x) * IB[j], fma(-hm, R[j - 1].y, R[j].y) * IB[j]);
        }
      }
      CVA_MARK(pb + 5);
      // backward: intervals b-1, b-2, ..., a; samples walked downwards from the
      // last one below s_b (sample l lies in interval i iff s_i <= t_l < s_{i+1},
      // the reference's upper_bound rule, spline.cpp:98-105)
      const double invN = 1.0 / (double)N;
      double s1 = next_knot();
      int l = ((t == K - 1) ? N : first_sample<kPow2>(s1, N)) - 1;
      double tl = sample_t<kPow2>(l, N, invN);
      double2 y1 = xy[b == n ? 0 : b];
      double2 mu1 = mub;
      double2 mu0 = w;
      // one interval [s_i, s_{i+1}): samples l, l-1, ... with t_l >= s_i
      auto walk = [&](double s0, double2 y0) {
        if (l >= 0 && tl >= s0) {
          const double h = s1 - s0;
          const double ih = frcp(h), h2 = h * h;
          do {
            const double A = (s1 - tl) * ih, B = (tl - s0) * ih;
            const double ca = fma(A, A, -1.0) * A * h2, cb = fma(B, B, -1.0) * B * h2;
            const double2 v = make_double2(fma(A, y0.x, fma(B, y1.x, fma(ca, mu0.x, cb * mu1.x))),
                                           fma(A, y0.y, fma(B, y1.y, fma(ca, mu0.y, cb * mu1.y))));
            out[kPadOut ? l + (l >> 3) : l] = v;
            cacc.x += v.x;
            cacc.y += v.y;
            --l;
            tl = sample_t<kPow2>(l, N, invN);
          } while (l >= 0 && tl >= s0);
        }
      };
      {  // the interface interval [s_{b-1}, s_b): mu = (w, mu_b)
        const double s0 = own_knot(M);
        const double2 y0 = xy[b - 1];
        walk(s0, y0);
        s1 = s0;
        y1 = y0;
        mu1 = mu0;
      }
#pragma unroll
      for (int j = kCMax - 1; j >= 0; --j) {
        if (j < M) {
          const int i = a + j;  // interval [s_i, s_{i+1})
          const double s0 = own_knot(j);
          // mu_i = g_i - c'_i mu_{i+1}, c'_i = h_i / pivot_i (mu_{b-1} = w: the
          // interface coupling of the last interior row is back-substituted,
          // not moved to its right-hand side, so every row is the same update)
          const double cpr = (s1 - s0) * IB[j];
          mu0 = make_double2(fma(-cpr, mu1.x, R[j].x), fma(-cpr, mu1.y, R[j].y));
          const double2 y0 = xy[i];
          walk(s0, y0);
          s1 = s0;
          y1 = y0;
          mu1 = mu0;
        }
      }
    }
    CVA_MARK(pb + 6);
    bar_sync();  // all samples written
    CVA_MARK(pb + 3);

    // ---- polygon length of the resampled curve and centroid (one reduction)
    double len = 0.0;
    if constexpr (kLen) {
      for (int q = t; q < N; q += kT) {
        const int q1 = q + 1 == N ? 0 : q + 1;
        const double2 p = out[kPadOut ? q + (q >> 3) : q], o = out[kPadOut ? q1 + (q1 >> 3) : q1];
        const double dx = o.x - p.x, dy = o.y - p.y;
        len += fsqrt(fma(dx, dx, dy * dy));
      }
    }
    double sx = cacc.x, sy = cacc.y;
    double lb = len + (bad ? INFINITY : 0.0);
    block_sum3(sx, sy, lb, red);
    CVA_MARK(pb + 4);
    CurveStats cs;
    const double invn = 1.0 / (double)N;
    cs.centroid = make_double2(invn * sx, invn * sy);
    if constexpr (kLen) {
      cs.bad = !(lb > 0.0) || !isfinite(lb);
      cs.inv_len = 1.0 / lb;
    } else {
      cs.bad = lb != 0.0 || !isfinite(sx) || !isfinite(sy);
      cs.inv_len = 0.0;
    }
    return cs;
  }
}

}  // namespace rs
}  // namespace cva
