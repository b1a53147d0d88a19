/* TEST INFRASTRUCTURE ONLY — CPU oracle (see oracle/README.md).
 *
 * Complex DFT of any length; definition in oracle_fft.h. This restates the
 * textbook algorithms (Cooley-Tukey radix 2, Bluestein 1970) rather than any
 * particular library: the reference delegates to an unpinned FFTW3
 * (/root/reference/proj/CMakeLists.txt:13-22), and its FFT is pinned only
 * through the naive-scan equivalence tests (proj/tests/test_rigid_align.cpp:133-151).
 */
#include "oracle_fft.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846264338327950288;

static int is_pow2(size_t n) { return n && !(n & (n - 1)); }

/* Radix-2 decimation in time, in place; n power of two. */
static void fft_pow2(double* a, size_t n, int sign) {
  if (n <= 1) return;
  /* bit reversal permutation */
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double tr = a[2 * i], ti = a[2 * i + 1];
      a[2 * i] = a[2 * j];
      a[2 * i + 1] = a[2 * j + 1];
      a[2 * j] = tr;
      a[2 * j + 1] = ti;
    }
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len >> 1;
    for (size_t k = 0; k < half; ++k) {
      /* twiddle evaluated directly (no recurrence) for full accuracy */
      const double ang = (double)sign * 2.0 * kPi * (double)k / (double)len;
      const double wr = cos(ang), wi = sin(ang);
      for (size_t s = 0; s < n; s += len) {
        double* u = a + 2 * (s + k);
        double* v = a + 2 * (s + k + half);
        const double vr = v[0] * wr - v[1] * wi;
        const double vi = v[0] * wi + v[1] * wr;
        v[0] = u[0] - vr;
        v[1] = u[1] - vi;
        u[0] += vr;
        u[1] += vi;
      }
    }
  }
}

/* Bluestein: X_k = conj(w_k) sum_j (x_j conj(w_j)) w_{k-j}, w_k = exp(i pi k^2 / n)
 * (for sign = -1; conjugated chirp for sign = +1). */
static int fft_bluestein(double* a, size_t n, int sign) {
  size_t m = 1;
  while (m < 2 * n - 1) m <<= 1;
  double* w = (double*)malloc(sizeof(double) * 2 * n);
  double* u = (double*)calloc(2 * m, sizeof(double));
  double* v = (double*)calloc(2 * m, sizeof(double));
  if (!w || !u || !v) {
    free(w);
    free(u);
    free(v);
    return -1;
  }
  const unsigned long long two_n = 2ULL * (unsigned long long)n;
  for (size_t k = 0; k < n; ++k) {
    /* k^2 mod 2n keeps the chirp angle small and exact */
    const unsigned long long kk = ((unsigned long long)k * (unsigned long long)k) % two_n;
    const double ang = kPi * (double)kk / (double)n;
    w[2 * k] = cos(ang);
    w[2 * k + 1] = (double)(-sign) * sin(ang); /* exp(-sign * i pi k^2/n) */
  }
  /* u_j = x_j * conj(w_j) */
  for (size_t j = 0; j < n; ++j) {
    const double xr = a[2 * j], xi = a[2 * j + 1];
    const double wr = w[2 * j], wi = -w[2 * j + 1];
    u[2 * j] = xr * wr - xi * wi;
    u[2 * j + 1] = xr * wi + xi * wr;
  }
  /* v = w on both wraps */
  v[0] = w[0];
  v[1] = w[1];
  for (size_t k = 1; k < n; ++k) {
    v[2 * k] = w[2 * k];
    v[2 * k + 1] = w[2 * k + 1];
    v[2 * (m - k)] = w[2 * k];
    v[2 * (m - k) + 1] = w[2 * k + 1];
  }
  fft_pow2(u, m, -1);
  fft_pow2(v, m, -1);
  for (size_t k = 0; k < m; ++k) {
    const double ur = u[2 * k], ui = u[2 * k + 1];
    const double vr = v[2 * k], vi = v[2 * k + 1];
    u[2 * k] = ur * vr - ui * vi;
    u[2 * k + 1] = ur * vi + ui * vr;
  }
  fft_pow2(u, m, +1);
  const double inv_m = 1.0 / (double)m;
  for (size_t k = 0; k < n; ++k) {
    const double cr = u[2 * k] * inv_m, ci = u[2 * k + 1] * inv_m;
    const double wr = w[2 * k], wi = -w[2 * k + 1];
    a[2 * k] = cr * wr - ci * wi;
    a[2 * k + 1] = cr * wi + ci * wr;
  }
  free(w);
  free(u);
  free(v);
  return 0;
}

int offt_dft(double* data, size_t n, int sign) {
  if (n <= 1) return 0;
  if (is_pow2(n)) {
    fft_pow2(data, n, sign);
    return 0;
  }
  return fft_bluestein(data, n, sign);
}
