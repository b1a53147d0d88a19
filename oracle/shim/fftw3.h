/* TEST INFRASTRUCTURE ONLY — part of the CPU oracle (see oracle/README.md).
 *
 * Minimal stand-in for the FFTW3 API subset that the reference's FFT wrapper
 * calls (/root/reference/proj/src/fft.cpp:30-36, :90, :108). FFTW3 is not
 * installed in this image or on the GPU box, and the reference
 * pins no version (proj/CMakeLists.txt:13-22), so this shim restates FFTW's
 * published transform definitions:
 *
 *   r2c:  Y[k] = sum_j x[j] exp(-2 pi i j k / n),  k = 0..n/2   (unnormalised)
 *   c2r:  y[j] = sum_k X[k] exp(+2 pi i j k / n),  j = 0..n-1   (unnormalised,
 *         X extended by Hermitian symmetry; Im X[0], Im X[n/2] ignored)
 *
 * for every n >= 1 (mixed radix 2 + Bluestein, exactly like FFTW supports any n).
 * It is linked only into oracle/_ref/libcurvalign_ref.so.
 */
#ifndef CURVALIGN_ORACLE_FFTW3_SHIM_H
#define CURVALIGN_ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_MEASURE (0U)

double* fftw_alloc_real(size_t n);
fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
