// Any-length complex FFT and the correlation stack on the GPU (gfft.cu), for the
// single-call drop-in entry points.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cva {

// double2 elements of scratch gfft / gfft_correlation need for length n
int64_t gfft_workspace(int64_t n);
int64_t gfft_correlation_workspace(int64_t n);
// in place: x_k <- sum_j x_j exp(sign 2 pi i j k / n), unnormalised, any n >= 1
cudaError_t gfft(double2* x, int64_t n, int sign, double2* ws, cudaStream_t s);
// out4[4 m + {0..3}] = A11, A12, A21, A22 of shift m (rigid_align.cpp:147-183)
cudaError_t gfft_correlation(const double2* c1, const double2* c2, int64_t n, double* out4, double2* ws,
                             cudaStream_t s);

}  // namespace cva
