/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's elastic (SRV)
 * matching: the rigid path's callers.
 *
 *   or_apply_srv_action   proj/src/srv.cpp:100-118 (interp_periodic :19-37)
 *   or_elastic_energy     proj/src/srv.cpp:120-128
 *   or_dp_step_cost       proj/src/srv.cpp:145-176
 *   or_dp_reparam         proj/src/srv.cpp:180-257
 *   or_elastic_approach1  proj/src/elastic.cpp:62-100
 *   or_elastic_approach2  proj/src/elastic.cpp:102-174 (compose :21-33,
 *                         rebase :37-50, run_align :52-54)
 *
 * Expression order follows the reference's so that, compiled without FMA
 * contraction (ISO C, x86-64 baseline), the results are bitwise the
 * reference's; tests/test_oracle_elastic.py checks that against oracle/_ref
 * and tests/golden/elastic_kat.npz.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "curvalign_oracle.h"

static const double kGridSnap = 1e-9; /* srv.cpp:14 */
static const double kMonoTol = 1e-12; /* srv.cpp:15 */

/* geometry.hpp:90-94 */
double or_wrap_unit(double t) {
  double r = t - floor(t);
  if (r >= 1.0) r -= 1.0;
  return r;
}

/* srv.cpp:19-37 */
static void interp_periodic(const double* q, int64_t n, double u, double* px, double* py) {
  const double x = u * (double)n;
  double i0f = floor(x);
  double frac = x - i0f;
  if (frac > 1.0 - kGridSnap) {
    i0f += 1.0;
    frac = 0.0;
  } else if (frac < kGridSnap) {
    frac = 0.0;
  }
  long i0 = (long)i0f % (long)n;
  if (i0 < 0) i0 += (long)n;
  if (frac == 0.0) {
    *px = q[2 * i0];
    *py = q[2 * i0 + 1];
    return;
  }
  const long i1 = (i0 + 1) % (long)n;
  *px = q[2 * i0] + frac * (q[2 * i1] - q[2 * i0]);
  *py = q[2 * i0 + 1] + frac * (q[2 * i1 + 1] - q[2 * i0 + 1]);
}

/* srv.cpp:58-69 */
static int validate_reparam(const double* g, int64_t n) {
  if (n < 2) return OR_INVALID;
  if (fabs(g[0]) > kMonoTol || fabs(g[n] - 1.0) > kMonoTol) return OR_INVALID;
  for (int64_t i = 0; i < n; ++i)
    if (g[i + 1] < g[i] - kMonoTol) return OR_INVALID;
  return OR_OK;
}

/* srv.cpp:100-118; rotation R(theta) = [[c, s], [-s, c]] (geometry.hpp:48-73) */
int or_apply_srv_action(const double* q, int64_t n, double t0, double theta, const double* gamma,
                        double* out) {
  if (n == 0) return OR_INVALID;
  int rc = validate_reparam(gamma, n);
  if (rc) return rc;
  if (!isfinite(theta)) return OR_INVALID; /* geometry.hpp:59 */
  const double nn = (double)n;
  for (int64_t l = 0; l < n; ++l) {
    const double gdot = (gamma[l + 1] - gamma[l]) * nn;
    const double u = or_wrap_unit(t0 + gamma[l]);
    double sx, sy;
    interp_periodic(q, n, u, &sx, &sy);
    const double c = cos(theta), s = sin(theta);
    const double rx = c * sx + s * sy, ry = -s * sx + c * sy;
    const double k = sqrt(gdot > 0.0 ? gdot : 0.0);
    out[2 * l] = rx * k;
    out[2 * l + 1] = ry * k;
  }
  return OR_OK;
}

/* srv.cpp:120-128 */
int or_elastic_energy(const double* q1, const double* q2, int64_t n, double t0, double theta,
                      const double* gamma, double* out) {
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  if (!w) return OR_BAD_ALLOC;
  int rc = or_apply_srv_action(q2, n, t0, theta, gamma, w);
  if (!rc) {
    double e = 0.0;
    for (int64_t l = 0; l < n; ++l) {
      const double dx = q1[2 * l] - w[2 * l], dy = q1[2 * l + 1] - w[2 * l + 1];
      e += dx * dx + dy * dy;
    }
    *out = e / (double)n;
  }
  free(w);
  return rc;
}

/* srv.cpp:145-176 */
static double step_cost(const double* q1, const double* q2, int64_t n, int i0, int j0, int a, int b) {
  const double slope = (double)b / (double)a;
  const double sq = sqrt(slope);
  double cost = 0.0;
  for (int k = 0; k <= a; ++k) {
    const int64_t i = (int64_t)(i0 + k) % n;
    const int num = k * b;
    double sx, sy;
    if (num % a == 0) {
      const int64_t j = (int64_t)(j0 + num / a) % n;
      sx = q2[2 * j];
      sy = q2[2 * j + 1];
    } else {
      const double pos = (double)j0 + (double)num / (double)a;
      const int base = (int)pos;
      const double frac = pos - (double)base;
      const int64_t u = (int64_t)base % n, v = (int64_t)(base + 1) % n;
      sx = q2[2 * u] + frac * (q2[2 * v] - q2[2 * u]);
      sy = q2[2 * u + 1] + frac * (q2[2 * v + 1] - q2[2 * u + 1]);
    }
    const double dx = q1[2 * i] - sx * sq, dy = q1[2 * i + 1] - sy * sq;
    const double w = (k == 0 || k == a) ? 0.5 : 1.0;
    cost += w * (dx * dx + dy * dy);
  }
  return cost / (double)n;
}

int or_dp_step_cost(const double* q1, const double* q2, int64_t n, int i0, int j0, int di, int dj,
                    double* out) {
  if (di < 1 || dj < 1) return OR_INVALID;
  *out = step_cost(q1, q2, n, i0, j0, di, dj);
  return OR_OK;
}

/* srv.cpp:130-139 */
static int gcd_i(int a, int b) { return b == 0 ? a : gcd_i(b, a % b); }
static int admissible_steps(int W, int* A, int* B) {
  int c = 0;
  for (int a = 1; a <= W; ++a)
    for (int b = 1; b <= W; ++b)
      if (gcd_i(a, b) == 1) {
        A[c] = a;
        B[c] = b;
        ++c;
      }
  return c;
}

static int imax3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
static int imin3(int a, int b, int c) { return a < b ? (a < c ? a : c) : (b < c ? b : c); }

/* srv.cpp:180-257: gamma (n+1), energy */
int or_dp_reparam(const double* q1, const double* q2, int64_t n64, int max_slope, double* gamma,
                  double* energy) {
  const int n = (int)n64;
  if (n < 8) return OR_INVALID;
  if (max_slope < 1) return OR_INVALID;
  const int W = max_slope;
  int* A = (int*)malloc(sizeof(int) * (size_t)(W * W));
  int* B = (int*)malloc(sizeof(int) * (size_t)(W * W));
  const size_t stride = (size_t)n + 1;
  double* dp = (double*)malloc(sizeof(double) * stride * stride);
  uint8_t* parent = (uint8_t*)malloc(stride * stride);
  if (!A || !B || !dp || !parent) {
    free(A), free(B), free(dp), free(parent);
    return OR_BAD_ALLOC;
  }
  const int ns = admissible_steps(W, A, B);
  for (size_t k = 0; k < stride * stride; ++k) {
    dp[k] = INFINITY;
    parent[k] = 0xff;
  }
  dp[0] = 0.0;
  for (int i = 1; i <= n; ++i) {
    const int lo = imax3((i + W - 1) / W, n - W * (n - i), 0);
    const int hi = imin3(W * i, n - (n - i + W - 1) / W, n);
    for (int j = lo; j <= hi; ++j) {
      double best = INFINITY;
      uint8_t best_s = 0xff;
      for (int s = 0; s < ns; ++s) {
        const int pi = i - A[s], pj = j - B[s];
        if (pi < 0 || pj < 0) continue;
        const double base = dp[(size_t)pi * stride + (size_t)pj];
        if (base == INFINITY) continue;
        const double cand = base + step_cost(q1, q2, n, pi, pj, A[s], B[s]);
        if (cand < best) {
          best = cand;
          best_s = (uint8_t)s;
        }
      }
      dp[(size_t)i * stride + (size_t)j] = best;
      parent[(size_t)i * stride + (size_t)j] = best_s;
    }
  }
  int rc = OR_OK;
  if (dp[(size_t)n * stride + (size_t)n] == INFINITY) rc = OR_RUNTIME; /* srv.cpp:233 */
  if (!rc) {
    *energy = dp[(size_t)n * stride + (size_t)n];
    for (int k = 0; k <= n; ++k) gamma[k] = 0.0;
    int i = n, j = n;
    gamma[n] = 1.0;
    while (i > 0) {
      const uint8_t s = parent[(size_t)i * stride + (size_t)j];
      if (s == 0xff) {
        rc = OR_RUNTIME;
        break;
      }
      const int a = A[s], b = B[s], pi = i - a, pj = j - b;
      for (int k = 0; k < a; ++k) {
        const double jj = (double)pj + (double)(k * b) / (double)a;
        gamma[pi + k] = jj / (double)n;
      }
      i = pi;
      j = pj;
    }
    gamma[0] = 0.0;
  }
  free(A), free(B), free(dp), free(parent);
  return rc;
}

/* Reparameterization::eval (srv.cpp:39-50) */
static double reparam_eval(const double* g, int64_t n, double t) {
  if (t <= 0.0) return g[0];
  if (t >= 1.0) return g[n];
  const double x = t * (double)n;
  int64_t i = (int64_t)x;
  if (i > n - 1) i = n - 1;
  const double frac = x - (double)i;
  return g[i] + frac * (g[i + 1] - g[i]);
}

/* elastic.cpp:21-33 */
static void compose(const double* outer, const double* inner, int64_t n, double* out) {
  for (int64_t l = 0; l <= n; ++l) out[l] = reparam_eval(outer, n, inner[l]);
  out[0] = 0.0;
  out[n] = 1.0;
  for (int64_t l = 1; l <= n; ++l) out[l] = out[l] < out[l - 1] ? out[l - 1] : out[l];
}

/* elastic.cpp:37-50 */
static void rebase(const double* g, int64_t n, int64_t m, double* out) {
  const double gm = g[m];
  for (int64_t l = 0; l <= n; ++l) {
    const int64_t lm = l + m;
    out[l] = (lm <= n) ? g[lm] - gm : g[lm - n] + 1.0 - gm;
  }
  out[0] = 0.0;
  out[n] = 1.0;
}

/* elastic.cpp:102-174 on preprocessed curves c1, c2 (n nodes). use_fft
 * selects align_fft / align_naive for the rigid steps (run_align :52-54). */
int or_elastic_approach2(const double* c1, const double* c2, int64_t n, int max_iters, double energy_tol,
                         int use_fft, int max_slope, or_elastic_match* out) {
  if (n < 8) return OR_INVALID; /* elastic.cpp:55-58 */
  const size_t pb = sizeof(double) * 2 * (size_t)n, gb = sizeof(double) * ((size_t)n + 1);
  double *q1 = malloc(pb), *q2 = malloc(pb), *q1c = malloc(pb), *w = malloc(pb), *wc = malloc(pb);
  double *g = malloc(gb), *gd = malloc(gb), *gc = malloc(gb);
  int rc = OR_OK;
  if (!q1 || !q2 || !q1c || !w || !wc || !g || !gd || !gc) rc = OR_BAD_ALLOC;
  if (!rc) rc = or_srv_transform(c1, n, q1);
  if (!rc) rc = or_srv_transform(c2, n, q2);
  if (!rc) rc = or_srv_center(q1, n, q1c);
  or_alignment pre;
  if (!rc) rc = use_fft ? or_align_fft(c1, c2, n, &pre) : or_align_naive(c1, c2, n, &pre);
  double t0 = 0.0, theta = 0.0, en = 0.0;
  int iters = 0, conv = 0;
  if (!rc) {
    t0 = pre.t0;
    theta = pre.theta;
    for (int64_t i = 0; i <= n; ++i) g[i] = (double)i / (double)n; /* identity_reparam, srv.cpp:52-56 */
    g[n] = 1.0;
    rc = or_elastic_energy(q1, q2, n, t0, theta, g, &en);
  }
  for (int iter = 1; !rc && iter <= max_iters; ++iter) {
    const double prev = en;
    { /* gamma-step */
      double de, e;
      rc = or_apply_srv_action(q2, n, t0, theta, g, w);
      if (!rc) rc = or_dp_reparam(q1, w, n, max_slope, gd, &de);
      if (rc) break;
      compose(g, gd, n, gc);
      rc = or_elastic_energy(q1, q2, n, t0, theta, gc, &e);
      if (rc) break;
      if (e <= en) {
        memcpy(g, gc, gb);
        en = e;
      }
    }
    { /* (t0, R)-step */
      or_alignment ra;
      rc = or_apply_srv_action(q2, n, t0, 0.0, g, w);
      if (!rc) rc = or_srv_center(w, n, wc);
      if (!rc) rc = use_fft ? or_align_fft(q1c, wc, n, &ra) : or_align_naive(q1c, wc, n, &ra);
      if (rc) break;
      const int64_t m = ra.shift;
      const double t0c = or_wrap_unit(t0 + g[m]);
      rebase(g, n, m, gc);
      double a4[4], th_raw, tr;
      int32_t dg;
      rc = or_cross_correlation_matrix(q1, w, n, m, a4);
      if (!rc) rc = or_optimal_rotation_svd(a4, &th_raw, &tr, &dg);
      double e_c, e_r;
      if (!rc) rc = or_elastic_energy(q1, q2, n, t0c, ra.theta, gc, &e_c);
      if (!rc) rc = or_elastic_energy(q1, q2, n, t0c, th_raw, gc, &e_r);
      if (rc) break;
      const double r_cand = (e_r <= e_c) ? th_raw : ra.theta;
      const double e = (e_c < e_r) ? e_c : e_r; /* std::min(e_raw, e_centered) */
      if (e <= en) {
        t0 = t0c;
        theta = r_cand;
        memcpy(g, gc, gb);
        en = e;
      }
    }
    iters = iter;
    if (prev - en < energy_tol) {
      conv = 1;
      break;
    }
  }
  if (!rc) {
    out->t0 = t0;
    out->theta = theta;
    out->energy = en;
    out->distance = sqrt(en > 0.0 ? en : 0.0); /* elastic.cpp:19 */
    out->iterations = iters;
    out->converged = conv;
    if (out->gamma) memcpy(out->gamma, g, gb);
  }
  free(q1), free(q2), free(q1c), free(w), free(wc), free(g), free(gd), free(gc);
  return rc;
}

/* elastic.cpp:62-100: every start shift m: Kabsch rotation of the SRV pair, the
 * shifted rotated SRV, one DP, the realised energy; the first smallest wins. */
int or_elastic_approach1(const double* c1, const double* c2, int64_t n, int max_slope, int64_t n_max,
                         or_elastic_match* out) {
  if (n < 8) return OR_INVALID;
  if (n > n_max) return OR_INVALID; /* elastic.cpp:66-69 */
  const size_t pb = sizeof(double) * 2 * (size_t)n, gb = sizeof(double) * ((size_t)n + 1);
  double *q1 = malloc(pb), *q2 = malloc(pb), *w = malloc(pb), *gd = malloc(gb), *best_g = malloc(gb);
  int rc = (!q1 || !q2 || !w || !gd || !best_g) ? OR_BAD_ALLOC : OR_OK;
  if (!rc) rc = or_srv_transform(c1, n, q1);
  if (!rc) rc = or_srv_transform(c2, n, q2);
  double best = INFINITY, best_t0 = 0.0, best_th = 0.0;
  for (int64_t m = 0; !rc && m < n; ++m) {
    double a4[4], th, tr, de, e;
    int32_t dg;
    rc = or_cross_correlation_matrix(q1, q2, n, m, a4);
    if (!rc) rc = or_optimal_rotation_svd(a4, &th, &tr, &dg);
    if (rc) break;
    const double c = cos(th), s = sin(th);
    for (int64_t l = 0; l < n; ++l) {
      const int64_t k = (l + m) % n;
      w[2 * l] = c * q2[2 * k] + s * q2[2 * k + 1];
      w[2 * l + 1] = -s * q2[2 * k] + c * q2[2 * k + 1];
    }
    rc = or_dp_reparam(q1, w, n, max_slope, gd, &de);
    const double t0 = (double)m / (double)n;
    if (!rc) rc = or_elastic_energy(q1, q2, n, t0, th, gd, &e);
    if (rc) break;
    if (e < best) {
      best = e;
      best_t0 = t0;
      best_th = th;
      memcpy(best_g, gd, gb);
    }
  }
  if (!rc) {
    out->t0 = best_t0;
    out->theta = best_th;
    out->energy = best;
    out->distance = sqrt(best > 0.0 ? best : 0.0);
    out->iterations = 1;
    out->converged = 1;
    if (out->gamma) memcpy(out->gamma, best_g, gb);
  }
  free(q1), free(q2), free(w), free(gd), free(best_g);
  return rc;
}
