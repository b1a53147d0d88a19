/* TEST INFRASTRUCTURE ONLY — FFTW3-API stand-in for compiling the reference's
 * own fft.cpp (/root/reference/proj/src/fft.cpp) into oracle/_ref. See fftw3.h
 * for the transform definitions restated here.
 */
#include "fftw3.h"

#include <stdlib.h>
#include <string.h>

#include "../oracle_fft.h"

struct fftw_plan_s {
  int n;
  int kind; /* 0 = r2c, 1 = c2r */
};

double* fftw_alloc_real(size_t n) { return (double*)malloc(sizeof(double) * (n ? n : 1)); }

fftw_complex* fftw_alloc_complex(size_t n) {
  return (fftw_complex*)malloc(sizeof(fftw_complex) * (n ? n : 1));
}

void fftw_free(void* p) { free(p); }

static fftw_plan make_plan(int n, int kind) {
  if (n < 1) return NULL;
  fftw_plan p = (fftw_plan)malloc(sizeof(struct fftw_plan_s));
  if (!p) return NULL;
  p->n = n;
  p->kind = kind;
  return p;
}

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags) {
  (void)in;
  (void)out;
  (void)flags;
  return make_plan(n, 0);
}

fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags) {
  (void)in;
  (void)out;
  (void)flags;
  return make_plan(n, 1);
}

void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
  const size_t n = (size_t)p->n;
  double* buf = (double*)malloc(sizeof(double) * 2 * n);
  if (!buf) abort();
  for (size_t j = 0; j < n; ++j) {
    buf[2 * j] = in[j];
    buf[2 * j + 1] = 0.0;
  }
  if (offt_dft(buf, n, -1) != 0) abort();
  for (size_t k = 0; k <= n / 2; ++k) {
    out[k][0] = buf[2 * k];
    out[k][1] = buf[2 * k + 1];
  }
  free(buf);
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
  const size_t n = (size_t)p->n;
  double* buf = (double*)malloc(sizeof(double) * 2 * n);
  if (!buf) abort();
  for (size_t k = 0; k <= n / 2; ++k) {
    buf[2 * k] = in[k][0];
    buf[2 * k + 1] = in[k][1];
  }
  for (size_t k = n / 2 + 1; k < n; ++k) { /* Hermitian extension */
    buf[2 * k] = in[n - k][0];
    buf[2 * k + 1] = -in[n - k][1];
  }
  if (offt_dft(buf, n, +1) != 0) abort();
  for (size_t j = 0; j < n; ++j) out[j] = buf[2 * j];
  free(buf);
}

void fftw_destroy_plan(fftw_plan p) { free(p); }
