/* TEST INFRASTRUCTURE ONLY — FFTW3-API stand-in for compiling the reference's
 * own fft.cpp (/root/reference/proj/src/fft.cpp) into oracle/_ref. See fftw3.h
 * for the transform definitions restated here. The transforms are
 * oracle_fft.c's offt_r2c / offt_c2r: per-n cached twiddles and one half-length
 * complex transform per real transform (about what an FFTW_ESTIMATE plan
 * does), so the CPU baseline is not handicapped by the stand-in.
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
  if (offt_r2c(in, (size_t)p->n, &out[0][0]) != 0) abort();
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
  if (offt_c2r(&in[0][0], (size_t)p->n, out) != 0) abort();
}

void fftw_destroy_plan(fftw_plan p) { free(p); }
