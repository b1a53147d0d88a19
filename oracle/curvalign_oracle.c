/* TEST INFRASTRUCTURE ONLY — CPU oracle; see curvalign_oracle.h for scope and rules.
 *
 * Every function restates the reference implementation at the cited
 * /root/reference/proj/... file:line, keeping its operation order where that
 * order fixes rounding (prefix sums, Thomas sweeps, tie scan).
 */
#define _POSIX_C_SOURCE 200809L
#include "curvalign_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_fft.h"

static const double kTieRelTol = 1e-12; /* proj/src/rigid_align.cpp:16 */

/* ------------------------------------------------------------------ curve */

/* proj/src/curve.cpp:10-15 */
int or_validate_curve(const double* xy, int64_t n, int64_t min_nodes) {
  if (n < min_nodes) return OR_INVALID;
  for (int64_t i = 0; i < 2 * n; ++i)
    if (!isfinite(xy[i])) return OR_INVALID;
  return OR_OK;
}

/* proj/src/curve.cpp:17-25 */
int or_curve_length(const double* xy, int64_t n, double* out) {
  int rc = or_validate_curve(xy, n, 3);
  if (rc) return rc;
  double len = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t j = (i + 1) % n;
    const double dx = xy[2 * j] - xy[2 * i], dy = xy[2 * j + 1] - xy[2 * i + 1];
    len += sqrt(dx * dx + dy * dy);
  }
  *out = len;
  return OR_OK;
}

/* proj/src/curve.cpp:27-32 */
int or_centroid(const double* xy, int64_t n, double* out2) {
  int rc = or_validate_curve(xy, n, 3);
  if (rc) return rc;
  double sx = 0.0, sy = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    sx += xy[2 * i];
    sy += xy[2 * i + 1];
  }
  const double inv = 1.0 / (double)n;
  out2[0] = inv * sx;
  out2[1] = inv * sy;
  return OR_OK;
}

/* proj/src/curve.cpp:34-39 */
int or_center_curve(const double* xy, int64_t n, double* out) {
  double g[2];
  int rc = or_centroid(xy, n, g);
  if (rc) return rc;
  for (int64_t i = 0; i < n; ++i) {
    out[2 * i] = xy[2 * i] - g[0];
    out[2 * i + 1] = xy[2 * i + 1] - g[1];
  }
  return OR_OK;
}

/* proj/src/curve.cpp:41-48 */
int or_normalize_length(const double* xy, int64_t n, double* out) {
  double len;
  int rc = or_curve_length(xy, n, &len);
  if (rc) return rc;
  if (len <= 0.0) return OR_INVALID;
  const double s = 1.0 / len;
  for (int64_t i = 0; i < 2 * n; ++i) out[i] = s * xy[i];
  return OR_OK;
}

/* proj/src/curve.cpp:50-65: sequential chordal prefix sum, s[n] forced to 1 */
int or_arc_length_params(const double* xy, int64_t n, double* s, double* total) {
  int rc = or_validate_curve(xy, n, 3);
  if (rc) return rc;
  s[0] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t j = (i + 1) % n;
    const double dx = xy[2 * j] - xy[2 * i], dy = xy[2 * j + 1] - xy[2 * i + 1];
    const double d = sqrt(dx * dx + dy * dy);
    if (d <= 0.0) return OR_INVALID; /* coincident adjacent nodes */
    s[i + 1] = s[i] + d;
  }
  *total = s[n];
  for (int64_t i = 0; i <= n; ++i) s[i] /= *total;
  s[n] = 1.0;
  return OR_OK;
}

/* ----------------------------------------------------------------- spline */

/* proj/src/spline.cpp:16-58: cyclic tridiagonal b[i] u[i-1] + d[i] u[i] + a[i] u[i+1] = r[i]
 * by Thomas on the corner-modified matrix plus a Sherman-Morrison correction.
 * Solves for two right-hand sides r (the spline's x or y data) in one pass each. */
static int solve_cyclic_tridiagonal(const double* b, const double* d, const double* a,
                                    const double* r, int64_t n, double* sol) {
  if (n < 3) return OR_INVALID;
  double* dd = (double*)malloc(sizeof(double) * n);
  double* c = (double*)malloc(sizeof(double) * n);
  double* y = (double*)malloc(sizeof(double) * n);
  double* z = (double*)malloc(sizeof(double) * n);
  double* u = (double*)calloc((size_t)n, sizeof(double));
  int rc = OR_OK;
  if (!dd || !c || !y || !z || !u) {
    rc = OR_BAD_ALLOC;
    goto done;
  }
  const double g = -d[0];
  memcpy(dd, d, sizeof(double) * n);
  dd[0] = d[0] - g;
  dd[n - 1] = d[n - 1] - a[n - 1] * b[0] / g;
  u[0] = g;
  u[n - 1] = b[n - 1];
  /* thomas(rhs) at spline.cpp:24-41, run for r then for u */
  for (int pass = 0; pass < 2; ++pass) {
    const double* rhs = pass == 0 ? r : u;
    double* out = pass == 0 ? y : z;
    double beta = dd[0];
    if (beta == 0.0) {
      rc = OR_RUNTIME;
      goto done;
    }
    c[0] = 0.0;
    out[0] = rhs[0] / beta;
    for (int64_t i = 1; i < n; ++i) {
      c[i] = a[i - 1] / beta;
      beta = dd[i] - b[i] * c[i];
      if (beta == 0.0) {
        rc = OR_RUNTIME;
        goto done;
      }
      out[i] = (rhs[i] - b[i] * out[i - 1]) / beta;
    }
    for (int64_t i = n - 1; i-- > 0;) out[i] -= c[i + 1] * out[i + 1];
  }
  {
    const double vy = y[0] + a[n - 1] / g * y[n - 1];
    const double vz = 1.0 + z[0] + a[n - 1] / g * z[n - 1];
    if (vz == 0.0) {
      rc = OR_RUNTIME;
      goto done;
    }
    const double factor = vy / vz;
    for (int64_t i = 0; i < n; ++i) sol[i] = y[i] - factor * z[i];
  }
done:
  free(dd);
  free(c);
  free(y);
  free(z);
  free(u);
  return rc;
}

/* proj/src/spline.cpp:62-96. m has n_knots entries; m[n] = m[0]. */
int or_spline_second_derivs(const double* x, const double* yin, int64_t n_knots, double* m) {
  if (n_knots < 4) return OR_INVALID;
  const int64_t n = n_knots - 1;
  for (int64_t i = 0; i < n; ++i)
    if (!(x[i] < x[i + 1])) return OR_INVALID;
  for (int64_t i = 0; i < n_knots; ++i)
    if (!isfinite(yin[i])) return OR_INVALID;
  double* h = (double*)malloc(sizeof(double) * n);
  double* sub = (double*)malloc(sizeof(double) * n);
  double* diag = (double*)malloc(sizeof(double) * n);
  double* sup = (double*)malloc(sizeof(double) * n);
  double* rhs = (double*)malloc(sizeof(double) * n);
  int rc = OR_OK;
  if (!h || !sub || !diag || !sup || !rhs) {
    rc = OR_BAD_ALLOC;
    goto done;
  }
  /* y[n] is replaced by y[0] (spline.cpp:74) */
#define YV(i) ((i) == n ? yin[0] : yin[i])
  for (int64_t i = 0; i < n; ++i) h[i] = x[i + 1] - x[i];
  for (int64_t i = 0; i < n; ++i) {
    const double hm = (i == 0) ? h[n - 1] : h[i - 1];
    const double hi = h[i];
    sub[i] = hm / 6.0;
    diag[i] = (hm + hi) / 3.0;
    sup[i] = hi / 6.0;
    const double yp = (i == 0) ? YV(n - 1) : YV(i - 1);
    rhs[i] = (YV(i + 1) - YV(i)) / hi - (YV(i) - yp) / hm;
  }
#undef YV
  rc = solve_cyclic_tridiagonal(sub, diag, sup, rhs, n, m);
  if (rc == OR_OK) m[n] = m[0];
done:
  free(h);
  free(sub);
  free(diag);
  free(sup);
  free(rhs);
  return rc;
}

/* proj/src/spline.cpp:98-117: wrap into [x0, xn), upper_bound interval, cubic. */
double or_spline_eval(const double* x, const double* y, const double* m, int64_t n_knots,
                      double t) {
  const int64_t n = n_knots - 1;
  const double p = x[n] - x[0];
  double xw = x[0] + fmod(t - x[0], p);
  if (xw < x[0]) xw += p;
  /* upper_bound over x[0..n]: first index with x[idx] > xw */
  int64_t lo = 0, hi = n_knots;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (xw < x[mid])
      hi = mid;
    else
      lo = mid + 1;
  }
  int64_t i;
  if (lo == 0)
    i = 0;
  else if (lo >= n_knots)
    i = n_knots - 2;
  else
    i = lo - 1;
  const double yi = (i == 0) ? y[0] : y[i];
  const double yi1 = (i + 1 == n) ? y[0] : y[i + 1];
  const double h = x[i + 1] - x[i];
  const double A = (x[i + 1] - xw) / h;
  const double B = (xw - x[i]) / h;
  return A * yi + B * yi1 + ((A * A * A - A) * m[i] + (B * B * B - B) * m[i + 1]) * h * h / 6.0;
}

/* proj/src/curve.cpp:67-91 */
int or_resample_uniform(const double* xy, int64_t n, int64_t n_out, double* out) {
  int rc = or_validate_curve(xy, n, 4);
  if (rc) return rc;
  if (n_out < 8) return OR_INVALID;
  double* s = (double*)malloc(sizeof(double) * (n + 1));
  double* xs = (double*)malloc(sizeof(double) * (n + 1));
  double* ys = (double*)malloc(sizeof(double) * (n + 1));
  double* mx = (double*)malloc(sizeof(double) * (n + 1));
  double* my = (double*)malloc(sizeof(double) * (n + 1));
  double total;
  if (!s || !xs || !ys || !mx || !my) {
    rc = OR_BAD_ALLOC;
    goto done;
  }
  rc = or_arc_length_params(xy, n, s, &total);
  if (rc) goto done;
  for (int64_t i = 0; i < n; ++i) {
    xs[i] = xy[2 * i];
    ys[i] = xy[2 * i + 1];
  }
  xs[n] = xy[0];
  ys[n] = xy[1];
  rc = or_spline_second_derivs(s, xs, n + 1, mx);
  if (rc) goto done;
  rc = or_spline_second_derivs(s, ys, n + 1, my);
  if (rc) goto done;
  for (int64_t l = 0; l < n_out; ++l) {
    const double t = (double)l / (double)n_out;
    out[2 * l] = or_spline_eval(s, xs, mx, n + 1, t);
    out[2 * l + 1] = or_spline_eval(s, ys, my, n + 1, t);
  }
done:
  free(s);
  free(xs);
  free(ys);
  free(mx);
  free(my);
  return rc;
}

/* proj/src/curve.cpp:93-97: resample (optional) -> center -> normalize */
int or_preprocess(const double* xy, int64_t n, int64_t n_out, int resample, double* out) {
  const int64_t m = resample ? n_out : n;
  double* tmp = (double*)malloc(sizeof(double) * 2 * (size_t)(m > 0 ? m : 1));
  if (!tmp) return OR_BAD_ALLOC;
  int rc;
  if (resample)
    rc = or_resample_uniform(xy, n, n_out, tmp);
  else {
    memcpy(tmp, xy, sizeof(double) * 2 * (size_t)n);
    rc = OR_OK;
  }
  if (!rc) rc = or_center_curve(tmp, m, tmp);
  if (!rc) rc = or_normalize_length(tmp, m, out);
  free(tmp);
  return rc;
}

/* ------------------------------------------------------------ rigid align */

/* proj/src/rigid_align.cpp:18-21 */
static int check_pair(int64_t n1, int64_t n2) {
  if (n1 != n2) return OR_INVALID;
  if (n1 < 4) return OR_INVALID;
  return OR_OK;
}

/* proj/src/rigid_align.cpp:65-80 */
int or_cross_correlation_matrix(const double* c1, const double* c2, int64_t n, int64_t shift,
                                double* a4) {
  int rc = check_pair(n, n);
  if (rc) return rc;
  if (shift < 0 || shift >= n) return OR_INVALID;
  double a11 = 0, a12 = 0, a21 = 0, a22 = 0;
  for (int64_t l = 0; l < n; ++l) {
    const double* p = c1 + 2 * l;
    const double* q = c2 + 2 * ((l + shift) % n);
    a11 += p[0] * q[0];
    a12 += p[0] * q[1];
    a21 += p[1] * q[0];
    a22 += p[1] * q[1];
  }
  a4[0] = a11;
  a4[1] = a12;
  a4[2] = a21;
  a4[3] = a22;
  return OR_OK;
}

/* proj/src/rigid_align.cpp:126-145 */
int or_correlation_all_shifts_naive(const double* c1, const double* c2, int64_t n, double* out) {
  int rc = check_pair(n, n);
  if (rc) return rc;
  for (int64_t m = 0; m < n; ++m) {
    double a11 = 0, a12 = 0, a21 = 0, a22 = 0;
    for (int64_t l = 0; l < n; ++l) {
      const int64_t lm = l + m < n ? l + m : l + m - n;
      const double* p = c1 + 2 * l;
      const double* q = c2 + 2 * lm;
      a11 += p[0] * q[0];
      a12 += p[0] * q[1];
      a21 += p[1] * q[0];
      a22 += p[1] * q[1];
    }
    out[4 * m] = a11;
    out[4 * m + 1] = a12;
    out[4 * m + 2] = a21;
    out[4 * m + 3] = a22;
  }
  return OR_OK;
}

/* proj/src/fft.cpp:81-95: n/2+1 unnormalised bins of exp(-2 pi i jk/n) */
int or_real_dft(const double* in, int64_t n, double* out) {
  if (n < 2) return OR_INVALID;
  return offt_r2c(in, (size_t)n, out) ? OR_BAD_ALLOC : OR_OK;
}

/* proj/src/fft.cpp:97-114: Hermitian half-spectrum back to n reals, scaled 1/n */
int or_real_idft(const double* spec, int64_t n_bins, int64_t n, double* out) {
  if (n < 1 || n_bins != n / 2 + 1) return OR_INVALID;
  if (offt_c2r(spec, (size_t)n, out)) return OR_BAD_ALLOC;
  const double scale = 1.0 / (double)n;
  for (int64_t j = 0; j < n; ++j) out[j] = out[j] * scale;
  return OR_OK;
}

/* proj/src/fft.cpp:116-125: r[m] = sum_l a[l] b[(l+m) mod n] = IDFT(conj(A) B) */
int or_circular_cross_correlation(const double* a, const double* b, int64_t n, double* out) {
  if (n < 2) return OR_INVALID;
  const int64_t nc = n / 2 + 1;
  double* fa = (double*)malloc(sizeof(double) * 2 * nc);
  double* fb = (double*)malloc(sizeof(double) * 2 * nc);
  int rc = (!fa || !fb) ? OR_BAD_ALLOC : OR_OK;
  if (!rc) rc = or_real_dft(a, n, fa);
  if (!rc) rc = or_real_dft(b, n, fb);
  if (!rc) {
    for (int64_t k = 0; k < nc; ++k) {
      const double ar = fa[2 * k], ai = -fa[2 * k + 1];
      const double br = fb[2 * k], bi = fb[2 * k + 1];
      fa[2 * k] = ar * br - ai * bi;
      fa[2 * k + 1] = ar * bi + ai * br;
    }
    rc = or_real_idft(fa, nc, n, out);
  }
  free(fa);
  free(fb);
  return rc;
}

/* proj/src/rigid_align.cpp:147-183: four real correlations A_kj(m) */
int or_correlation_all_shifts_fft(const double* c1, const double* c2, int64_t n, double* out) {
  int rc = check_pair(n, n);
  if (rc) return rc;
  double* buf = (double*)malloc(sizeof(double) * 7 * (size_t)n);
  if (!buf) return OR_BAD_ALLOC;
  double *x1 = buf, *y1 = buf + n, *x2 = buf + 2 * n, *y2 = buf + 3 * n, *r = buf + 4 * n;
  for (int64_t l = 0; l < n; ++l) {
    x1[l] = c1[2 * l];
    y1[l] = c1[2 * l + 1];
    x2[l] = c2[2 * l];
    y2[l] = c2[2 * l + 1];
  }
  const double* lhs[4] = {x1, x1, y1, y1};
  const double* rhs[4] = {x2, y2, x2, y2};
  for (int k = 0; k < 4 && !rc; ++k) {
    rc = or_circular_cross_correlation(lhs[k], rhs[k], n, r);
    if (!rc)
      for (int64_t m = 0; m < n; ++m) out[4 * m + k] = r[m];
  }
  free(buf);
  return rc;
}

/* proj/src/rigid_align.cpp:82-102 (JacobiSVD + determinant correction). The 2x2
 * SVD is restated in closed form (oracle/shim/Eigen/SVD documents why any
 * correct SVD gives the same R). */
int or_optimal_rotation_svd(const double* a4, double* theta, double* trace, int32_t* degenerate) {
  for (int i = 0; i < 4; ++i)
    if (!isfinite(a4[i])) return OR_INVALID;
  const double a = a4[0], b = a4[1], c = a4[2], d = a4[3];
  if (sqrt(a * a + b * b + c * c + d * d) == 0.0) {
    *theta = 0.0;
    *trace = 0.0;
    *degenerate = 1;
    return OR_OK;
  }
  const double E = 0.5 * (a + d), F = 0.5 * (a - d), G = 0.5 * (c + b), H = 0.5 * (c - b);
  const double Q = hypot(E, H), R = hypot(F, G);
  double s0 = Q + R, s1 = Q - R;
  const double a1 = atan2(G, F), a2 = atan2(H, E);
  const double th = 0.5 * (a2 - a1), ph = 0.5 * (a2 + a1);
  double U[4] = {cos(ph), -sin(ph), sin(ph), cos(ph)};
  const double V[4] = {cos(th), sin(th), -sin(th), cos(th)};
  if (s1 < 0.0) {
    s1 = -s1;
    U[1] = -U[1];
    U[3] = -U[3];
  }
  const double detU = U[0] * U[3] - U[1] * U[2], detV = V[0] * V[3] - V[1] * V[2];
  const double sign = (detU * detV > 0.0) ? 1.0 : -1.0;
  /* R = U diag(1, sign) V^T ; theta = atan2(R01, R00) */
  const double R00 = U[0] * V[0] + U[1] * sign * V[1];
  const double R01 = U[0] * V[2] + U[1] * sign * V[3];
  *theta = atan2(R01, R00);
  *trace = s0 + sign * s1;
  *degenerate = 0;
  return OR_OK;
}

/* proj/src/rigid_align.cpp:104-119 */
int or_optimal_rotation_closed_form(const double* a4, double* theta, double* trace,
                                    int32_t* degenerate) {
  for (int i = 0; i < 4; ++i)
    if (!isfinite(a4[i])) return OR_INVALID;
  const double c = a4[0] + a4[3], s = a4[1] - a4[2];
  if (c == 0.0 && s == 0.0) {
    *theta = 0.0;
    *trace = 0.0;
    *degenerate = 1;
    return OR_OK;
  }
  *theta = atan2(s, c);
  *trace = hypot(c, s);
  *degenerate = 0;
  return OR_OK;
}

/* proj/src/rigid_align.cpp:23-27 */
static double sum_norm2(const double* c, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += c[2 * i] * c[2 * i] + c[2 * i + 1] * c[2 * i + 1];
  return s;
}

/* proj/src/rigid_align.cpp:31-61: hypot scan, smallest shift in the 1e-12 band,
 * SVD on the winner, energy by the trace identity clamped at 0. */
static int pick_best(const double* corr, double s1, double s2, int64_t n, or_alignment* out) {
  double best = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    const double tr = hypot(corr[4 * i] + corr[4 * i + 3], corr[4 * i + 1] - corr[4 * i + 2]);
    if (tr > best) best = tr;
  }
  const double tol = kTieRelTol * fmax(1.0, fabs(best));
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double tr = hypot(corr[4 * i] + corr[4 * i + 3], corr[4 * i + 1] - corr[4 * i + 2]);
    if (tr >= best - tol) {
      m = i;
      break;
    }
  }
  double theta, trace;
  int32_t degen;
  int rc = or_optimal_rotation_svd(corr + 4 * m, &theta, &trace, &degen);
  if (rc) return rc;
  out->shift = m;
  out->t0 = (double)m / (double)n;
  out->theta = theta;
  out->trace = trace;
  out->degenerate = degen;
  out->status = 0;
  const double h = 1.0 / (double)n;
  double e = h * (s1 + s2) - 2.0 * h * trace;
  if (e < 0.0) e = 0.0;
  out->energy = e;
  return OR_OK;
}

/* proj/src/rigid_align.cpp:185-196; Rotation2::apply at geometry.hpp:70-73 */
int or_mismatch_energy(const double* c1, const double* c2, int64_t n, int64_t shift, double theta,
                       double* out) {
  int rc = check_pair(n, n);
  if (rc) return rc;
  if (shift < 0 || shift >= n || !isfinite(theta)) return OR_INVALID;
  const double c = cos(theta), s = sin(theta);
  double e = 0.0;
  for (int64_t l = 0; l < n; ++l) {
    const double* q = c2 + 2 * ((l + shift) % n);
    const double rx = c * q[0] + s * q[1], ry = -s * q[0] + c * q[1];
    const double dx = c1[2 * l] - rx, dy = c1[2 * l + 1] - ry;
    e += dx * dx + dy * dy;
  }
  *out = e / (double)n;
  return OR_OK;
}

void or_aligned_curve(const double* c2, int64_t n, int64_t shift, double theta, double* out) {
  const double c = cos(theta), s = sin(theta);
  for (int64_t l = 0; l < n; ++l) {
    const double* q = c2 + 2 * ((l + shift) % n);
    out[2 * l] = c * q[0] + s * q[1];
    out[2 * l + 1] = -s * q[0] + c * q[1];
  }
}

static int align_impl(const double* c1, const double* c2, int64_t n, int use_fft,
                      or_alignment* out) {
  int rc = check_pair(n, n);
  if (rc) return rc;
  double* corr = (double*)malloc(sizeof(double) * 4 * (size_t)n);
  if (!corr) return OR_BAD_ALLOC;
  rc = use_fft ? or_correlation_all_shifts_fft(c1, c2, n, corr)
               : or_correlation_all_shifts_naive(c1, c2, n, corr);
  if (!rc) rc = pick_best(corr, sum_norm2(c1, n), sum_norm2(c2, n), n, out);
  free(corr);
  return rc;
}

/* proj/src/rigid_align.cpp:198-202 */
int or_align_naive(const double* c1, const double* c2, int64_t n, or_alignment* out) {
  return align_impl(c1, c2, n, 0, out);
}

/* proj/src/rigid_align.cpp:204-208 */
int or_align_fft(const double* c1, const double* c2, int64_t n, or_alignment* out) {
  return align_impl(c1, c2, n, 1, out);
}

/* -------------------------------------------------------------------- srv */

/* proj/src/srv.cpp:71-88 */
int or_srv_transform(const double* xy, int64_t n, double* q) {
  int rc = or_validate_curve(xy, n, 8);
  if (rc) return rc;
  const double nn = (double)n;
  const double eps = 1e-8 * nn;
  for (int64_t l = 0; l < n; ++l) {
    const int64_t nx = (l + 1) % n, pv = (l + n - 1) % n;
    const double dx = (nn / 2.0) * (xy[2 * nx] - xy[2 * pv]);
    const double dy = (nn / 2.0) * (xy[2 * nx + 1] - xy[2 * pv + 1]);
    const double mag = sqrt(dx * dx + dy * dy);
    if (mag < eps) {
      q[2 * l] = 0.0;
      q[2 * l + 1] = 0.0;
    } else {
      const double s = 1.0 / sqrt(mag);
      q[2 * l] = s * dx;
      q[2 * l + 1] = s * dy;
    }
  }
  return OR_OK;
}

/* proj/src/srv.cpp:90-98 */
int or_srv_center(const double* q, int64_t n, double* out) {
  if (n < 1) return OR_INVALID;
  double mx = 0.0, my = 0.0;
  for (int64_t l = 0; l < n; ++l) {
    mx += q[2 * l];
    my += q[2 * l + 1];
  }
  const double inv = 1.0 / (double)n;
  mx *= inv;
  my *= inv;
  for (int64_t l = 0; l < n; ++l) {
    out[2 * l] = q[2 * l] - mx;
    out[2 * l + 1] = q[2 * l + 1] - my;
  }
  return OR_OK;
}

/* ----------------------------------------------------------------- batch */

typedef struct {
  const double* points;
  const int64_t* offsets;
  int64_t pairs, n_out;
  int resample, mode;
  or_alignment* out;
  double* aligned;
  int64_t next; /* guarded by mu */
  pthread_mutex_t mu;
  int first_err;
} batch_ctx;

static int run_pair(batch_ctx* ctx, int64_t p) {
  const int64_t a0 = ctx->offsets[2 * p], a1 = ctx->offsets[2 * p + 1], b1 = ctx->offsets[2 * p + 2];
  const int64_t na = a1 - a0, nb = b1 - a1;
  const double* ra = ctx->points + 2 * a0;
  const double* rb = ctx->points + 2 * a1;
  const int64_t mu = ctx->mode == 0 ? (ctx->resample ? ctx->n_out : na) : na;
  const int64_t mv = ctx->mode == 0 ? (ctx->resample ? ctx->n_out : nb) : nb;
  double* u = (double*)malloc(sizeof(double) * 2 * (size_t)(mu > 0 ? mu : 1));
  double* v = (double*)malloc(sizeof(double) * 2 * (size_t)(mv > 0 ? mv : 1));
  int rc = (!u || !v) ? OR_BAD_ALLOC : OR_OK;
  if (!rc) {
    if (ctx->mode == 0) {
      rc = or_preprocess(ra, na, ctx->n_out, ctx->resample, u);
      if (!rc) rc = or_preprocess(rb, nb, ctx->n_out, ctx->resample, v);
    } else if (ctx->mode == 1) {
      memcpy(u, ra, sizeof(double) * 2 * (size_t)na);
      memcpy(v, rb, sizeof(double) * 2 * (size_t)nb);
    } else {
      rc = or_srv_transform(ra, na, u);
      if (!rc) rc = or_srv_center(u, na, u);
      if (!rc) rc = or_srv_transform(rb, nb, v);
      if (!rc) rc = or_srv_center(v, nb, v);
    }
  }
  if (!rc) rc = check_pair(mu, mv);
  if (!rc) rc = or_align_fft(u, v, mu, &ctx->out[p]);
  if (!rc && ctx->aligned)
    or_aligned_curve(v, mv, ctx->out[p].shift, ctx->out[p].theta, ctx->aligned + 2 * p * mv);
  if (rc) {
    or_alignment bad = {0, 0.0, NAN, NAN, NAN, 0, rc};
    ctx->out[p] = bad;
  }
  free(u);
  free(v);
  return rc;
}

static void* batch_worker(void* arg) {
  batch_ctx* ctx = (batch_ctx*)arg;
  for (;;) {
    pthread_mutex_lock(&ctx->mu);
    const int64_t p = ctx->next++;
    pthread_mutex_unlock(&ctx->mu);
    if (p >= ctx->pairs) break;
    const int rc = run_pair(ctx, p);
    if (rc) {
      pthread_mutex_lock(&ctx->mu);
      if (!ctx->first_err) ctx->first_err = rc;
      pthread_mutex_unlock(&ctx->mu);
    }
  }
  return NULL;
}

int or_batch(const double* points, const int64_t* offsets, int64_t pairs, int64_t n_out,
             int resample, int mode, int threads, or_alignment* out, double* aligned) {
  batch_ctx ctx;
  ctx.points = points;
  ctx.offsets = offsets;
  ctx.pairs = pairs;
  ctx.n_out = n_out;
  ctx.resample = resample;
  ctx.mode = mode;
  ctx.out = out;
  ctx.aligned = aligned;
  ctx.next = 0;
  ctx.first_err = 0;
  pthread_mutex_init(&ctx.mu, NULL);
  if (threads <= 1) {
    batch_worker(&ctx);
  } else {
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    if (!tids) return OR_BAD_ALLOC;
    for (int t = 0; t < threads; ++t) pthread_create(&tids[t], NULL, batch_worker, &ctx);
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    free(tids);
  }
  pthread_mutex_destroy(&ctx.mu);
  return ctx.first_err;
}
