// Host-side declarations of the v2 launchers (fused.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/curvalign_cuda.h"

namespace cva {

int v2_max_raw_nodes();
size_t v2_resample_align_smem(int N);
size_t v2_preprocess_smem(int n_out);
size_t v2_align_smem(int N);
int v2_fft_len(int N);  // power-of-two transform length used for N data points
bool v2_resample_align_supported(int N);

cudaError_t launch_v2_resample_align(const double2* pts, const int64_t* off, int64_t pairs, int N,
                                     const double2* tw, cva_alignment* out, double2* aligned,
                                     cudaStream_t s);
bool v3_resample_align_supported(int N);
int v3_max_raw_nodes();
cudaError_t launch_v3_resample_align(const double2* pts, const int64_t* off, int64_t pairs, int N,
                                     const double2* tw, cva_alignment* out, double2* aligned,
                                     cudaStream_t s);
cudaError_t launch_v2_preprocess(const double2* pts, const int64_t* off, int64_t curves, int n_out,
                                 int center_normalize, double2* out, int32_t* status,
                                 cudaStream_t s);
cudaError_t launch_v2_align(const double2* c1, const double2* c2, int64_t pairs, int N,
                            const double2* tw, cva_alignment* out, double2* aligned,
                            cudaStream_t s);
cudaError_t launch_v2_align_interleaved(const double2* rows, int64_t pairs, int N, const double2* tw,
                                        cva_alignment* out, double2* aligned, cudaStream_t s);
cudaError_t launch_v2_align_norm(const double2* c1, const double2* c2, int64_t pairs, int N, const double2* tw,
                                 const double4* norm1, const double4* norm2, const int32_t* bad1,
                                 const int32_t* bad2, cva_alignment* out, double2* aligned, cudaStream_t s);
cudaError_t launch_v2_align_row(const double2* row, const double2* curves, int64_t count, int N,
                                const double2* tw, cva_alignment* out, cudaStream_t s);
cudaError_t launch_unpack_row(const cva_alignment* in, int64_t count, double* energy, int32_t* shift,
                              double* theta, cudaStream_t s);

// all-pairs (allpairs.cu)
size_t allpairs_spectra_smem(int N);
cudaError_t launch_spectra(const double2* curves, int64_t count, int N, const double2* tw, double2* za,
                           double2* zb, double* ss, cudaStream_t s);
bool allpairs_fast_supported(int N);
size_t allpairs_scratch_cells(int64_t rows, int64_t count);  // bytes of the per-cell scratch `dm`
cudaError_t launch_allpairs(const double2* za, const double2* zb, const double* ss, int64_t count,
                            int64_t row_begin, int64_t row_end, const double2* tw, double* energy,
                            int32_t* shift, double* theta, double2* dm, cudaStream_t s);

// srv_center(srv_transform(c)) per curve, any N (global in/out)
cudaError_t launch_v2_srv_center(const double2* c, int64_t curves, int N, double2* q, cudaStream_t s);
cudaError_t launch_v2_srv_align(const double2* c1, const double2* c2, int64_t pairs, int N,
                                const double2* tw, cva_alignment* out, double2* aligned, cudaStream_t s);

}  // namespace cva
