// Host-side declarations of the large-N path (largen.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/curvalign_cuda.h"

namespace cva {

// Workspace for `chunk` pairs of N-node curves and the pair count per chunk
// that keeps the chunk's working set L2-resident.
size_t large_workspace_bytes(int64_t chunk, int N);
cudaError_t launch_broadcast_curve(const double2* c, int64_t n, int64_t copies, double2* out, cudaStream_t s);
int64_t large_chunk_pairs(int N);

// Twiddle tables of the four-step path (4096 <= M <= 65536, M = M1 x M2):
// s1 / s2 of lengths M1 / M2 for the sub-transforms, lo = the length-M table
// (entries < 256 used) and hi of length M / 256 for W_M^e = hi[e >> 8] lo[e & 255].
struct FourStepTw {
  const double2 *s1, *s2, *lo, *hi;
};
// M1 of the four-step split for transform length M (0: use the radix-16 passes)
int four_step_m1(int M);

// align_fft (normalize = 0) or preprocess(resample=false) + align_fft
// (normalize = 1) for pairs of N-node curves whose transform length exceeds the
// shared-memory kernels. tw: twiddles of length fft_len(N). aligned nullable.
cudaError_t launch_large_align(const double2* c1, const double2* c2, int64_t pairs, int N, int normalize,
                               const double2* tw, const FourStepTw* fst, cva_alignment* out, double2* aligned,
                               void* ws, int64_t chunk, cudaStream_t s);

// Per-curve centroid / 1/length (normalize = 1; else identity) and invalid
// flags, as (gx, gy, sc, 0) per curve; ws >= curve_stats_workspace(count).
size_t curve_stats_workspace(int64_t curves);
cudaError_t launch_curve_stats(const double2* curves, int64_t count, int N, int normalize, double4* norm,
                               int32_t* bad, void* ws, cudaStream_t s);

}  // namespace cva
