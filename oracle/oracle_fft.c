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
#include <pthread.h>
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

/* ------------------------------------------------------------------ real DFT
 * Real transforms of even power-of-two length n through one n/2-point complex
 * transform (the standard even/odd split: z_j = x_2j + i x_2j+1), with the
 * twiddles and the bit-reversal table computed once per n and cached (the
 * role FFTW's plan plays in the reference, proj/src/fft.cpp:22-57); other n
 * take the full complex transform above. Plans are created under a mutex and
 * read-only afterwards; the work buffer is per thread, so concurrent calls
 * (the reference's thread pool) do not share state. */
typedef struct {
  size_t n, m;       /* n = 2m */
  double* tw;        /* exp(-2 pi i k / m), k < m / 2 */
  double* post;      /* exp(-2 pi i k / n), k <= m */
  size_t* rev;       /* bit reversal of m */
} rplan;

#define RPLAN_MAX 64
static rplan g_plans[RPLAN_MAX];
static int g_nplans = 0;
static pthread_mutex_t g_plan_mu = PTHREAD_MUTEX_INITIALIZER;

static const rplan* get_rplan(size_t n) {
  for (int i = 0; i < __atomic_load_n(&g_nplans, __ATOMIC_ACQUIRE); ++i)
    if (g_plans[i].n == n) return &g_plans[i];
  pthread_mutex_lock(&g_plan_mu);
  for (int i = 0; i < g_nplans; ++i)
    if (g_plans[i].n == n) {
      pthread_mutex_unlock(&g_plan_mu);
      return &g_plans[i];
    }
  if (g_nplans == RPLAN_MAX) {
    pthread_mutex_unlock(&g_plan_mu);
    return NULL;
  }
  rplan* p = &g_plans[g_nplans];
  const size_t m = n / 2;
  p->n = n;
  p->m = m;
  p->tw = (double*)malloc(sizeof(double) * (m > 1 ? m : 2));
  p->post = (double*)malloc(sizeof(double) * 2 * (m + 1));
  p->rev = (size_t*)malloc(sizeof(size_t) * m);
  if (!p->tw || !p->post || !p->rev) {
    free(p->tw);
    free(p->post);
    free(p->rev);
    pthread_mutex_unlock(&g_plan_mu);
    return NULL;
  }
  for (size_t k = 0; k < m / 2; ++k) {
    const double ang = -2.0 * kPi * (double)k / (double)m;
    p->tw[2 * k] = cos(ang);
    p->tw[2 * k + 1] = sin(ang);
  }
  for (size_t k = 0; k <= m; ++k) {
    const double ang = -2.0 * kPi * (double)k / (double)n;
    p->post[2 * k] = cos(ang);
    p->post[2 * k + 1] = sin(ang);
  }
  for (size_t i = 0, j = 0; i < m; ++i) {
    p->rev[i] = j;
    size_t bit = m >> 1;
    for (; bit && (j & bit); bit >>= 1) j ^= bit;
    j ^= bit;
  }
  __atomic_store_n(&g_nplans, g_nplans + 1, __ATOMIC_RELEASE);
  pthread_mutex_unlock(&g_plan_mu);
  return p;
}

/* in-place radix-2 DIT transform of the bit-reversed sequence a (m points) */
static void rfft_core(const rplan* p, double* a, int sign) {
  const size_t m = p->m;
  for (size_t len = 2; len <= m; len <<= 1) {
    const size_t half = len >> 1, step = m / len;
    for (size_t s = 0; s < m; s += len) {
      for (size_t k = 0; k < half; ++k) {
        const double wr = p->tw[2 * k * step], wi = -sign * p->tw[2 * k * step + 1];
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

static _Thread_local double* t_buf = NULL;
static _Thread_local size_t t_cap = 0;

static double* work(size_t doubles) {
  if (doubles > t_cap) {
    free(t_buf);
    t_buf = (double*)malloc(sizeof(double) * doubles);
    t_cap = t_buf ? doubles : 0;
  }
  return t_buf;
}

int offt_r2c(const double* in, size_t n, double* out) {
  if (n < 1) return -1;
  if (n < 4 || !is_pow2(n)) {
    double* buf = work(2 * n);
    if (!buf) return -1;
    for (size_t j = 0; j < n; ++j) {
      buf[2 * j] = in[j];
      buf[2 * j + 1] = 0.0;
    }
    if (offt_dft(buf, n, -1)) return -1;
    memcpy(out, buf, sizeof(double) * 2 * (n / 2 + 1));
    return 0;
  }
  const rplan* p = get_rplan(n);
  if (!p) return -1;
  const size_t m = p->m;
  double* z = work(2 * m);
  if (!z) return -1;
  for (size_t j = 0; j < m; ++j) {  /* z_j = x_2j + i x_2j+1, bit reversed */
    z[2 * p->rev[j]] = in[2 * j];
    z[2 * p->rev[j] + 1] = in[2 * j + 1];
  }
  rfft_core(p, z, -1);
  /* X_k = E_k + W^k O_k, E_k = (Z_k + conj Z_{m-k}) / 2, O_k = (Z_k - conj Z_{m-k}) / 2i */
  for (size_t k = 0; k <= m; ++k) {
    const size_t a = k == m ? 0 : k, b = k == 0 ? 0 : m - k;
    const double zr = z[2 * a], zi = z[2 * a + 1], cr = z[2 * b], ci = -z[2 * b + 1];
    const double er = 0.5 * (zr + cr), ei = 0.5 * (zi + ci);
    const double orr = 0.5 * (zi - ci), oi = -0.5 * (zr - cr);
    const double wr = p->post[2 * k], wi = p->post[2 * k + 1];
    out[2 * k] = er + (wr * orr - wi * oi);
    out[2 * k + 1] = ei + (wr * oi + wi * orr);
  }
  return 0;
}

int offt_c2r(const double* spec, size_t n, double* out) {
  if (n < 1) return -1;
  if (n < 4 || !is_pow2(n)) {
    double* buf = work(2 * n);
    if (!buf) return -1;
    for (size_t k = 0; k <= n / 2; ++k) {
      buf[2 * k] = spec[2 * k];
      buf[2 * k + 1] = spec[2 * k + 1];
    }
    for (size_t k = n / 2 + 1; k < n; ++k) {
      buf[2 * k] = spec[2 * (n - k)];
      buf[2 * k + 1] = -spec[2 * (n - k) + 1];
    }
    if (offt_dft(buf, n, +1)) return -1;
    for (size_t j = 0; j < n; ++j) out[j] = buf[2 * j];
    return 0;
  }
  const rplan* p = get_rplan(n);
  if (!p) return -1;
  const size_t m = p->m;
  double* z = work(2 * m);
  if (!z) return -1;
  /* Z'_k = (X_k + conj X_{m-k}) + i W^{-k} (X_k - conj X_{m-k}); z = unnormalised inverse of Z' */
  for (size_t k = 0; k < m; ++k) {
    const double xr = spec[2 * k], xi = spec[2 * k + 1];
    const double cr = spec[2 * (m - k)], ci = -spec[2 * (m - k) + 1];
    const double sr = xr + cr, si = xi + ci;
    const double dr = xr - cr, di = xi - ci;
    const double wr = p->post[2 * k], wi = -p->post[2 * k + 1]; /* W^{-k} */
    const double tr = wr * dr - wi * di, ti = wr * di + wi * dr;
    z[2 * p->rev[k]] = sr - ti;
    z[2 * p->rev[k] + 1] = si + tr;
  }
  rfft_core(p, z, +1);
  for (size_t j = 0; j < m; ++j) {
    out[2 * j] = z[2 * j];
    out[2 * j + 1] = z[2 * j + 1];
  }
  return 0;
}
