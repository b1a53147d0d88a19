// Host-side declarations of the kernel launchers (kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/curvalign_cuda.h"

namespace cva {

size_t resample_smem_bytes(int nmax, int n_out);
int max_chunked_nodes();
// raw curves beyond shared memory: per-CTA global slabs (bytes per CTA, CTAs)
size_t resample_global_slab_bytes(int nmax);
int resample_global_grid(int64_t curves);
cudaError_t launch_preprocess_resample_global(const double2* pts, const int64_t* off, int64_t curves, int nmax,
                                              int n_out, int center_normalize, double2* out, int32_t* status,
                                              void* slab, cudaStream_t s);

// w_N^k for k < N, then (power-of-two N <= 2048) the pass twiddle tables of
// the compile-time transforms: twiddle_extra(N) more entries
cudaError_t launch_tw_init(double2* tw, int N, cudaStream_t s);
int twiddle_extra(int N);
cudaError_t launch_preprocess_resample(const double2* pts, const int64_t* off, int64_t curves,
                                       int nmax, int n_out, int center_normalize, double2* out,
                                       int32_t* status, cudaStream_t s);
cudaError_t launch_preprocess_center(const double2* pts, const int64_t* off, int64_t curves,
                                     double2* out, int32_t* status, cudaStream_t s);
}  // namespace cva
