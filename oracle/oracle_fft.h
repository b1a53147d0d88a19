/* TEST INFRASTRUCTURE ONLY — CPU oracle (see oracle/README.md). Never linked into
 * the product library.
 *
 * Plain-C complex DFT of any length n, used (a) by the FFTW-API shim that lets
 * the reference's own sources compile (oracle/shim/fftw3.h) and (b) by the C
 * restatement of the reference's FFT correlation (oracle/curvalign_oracle.c).
 *
 *   sign = -1:  X[k] = sum_j x[j] exp(-2 pi i j k / n)     (forward, unnormalised)
 *   sign = +1:  x[j] = sum_k X[k] exp(+2 pi i j k / n)     (backward, unnormalised)
 *
 * Power-of-two n: iterative radix-2 with directly evaluated twiddles.
 * Other n: Bluestein chirp-z over a power-of-two convolution.
 */
#ifndef CURVALIGN_ORACLE_FFT_H
#define CURVALIGN_ORACLE_FFT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* In-place transform of n interleaved complex values (re, im). Returns 0 on
 * success, -1 on allocation failure. */
int offt_dft(double* data, size_t n, int sign);

/* Real input x[0..n) -> n/2+1 unnormalised bins of exp(-2 pi i jk/n) (FFTW
 * r2c), and back (FFTW c2r: unnormalised, Hermitian input of n/2+1 bins).
 * Power-of-two n >= 4 go through one n/2-point complex transform with
 * per-n cached twiddles; thread-safe. 0 on success, -1 on failure. */
int offt_r2c(const double* in, size_t n, double* out_bins);
int offt_c2r(const double* bins, size_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif
