// Host-side declarations of the elastic (SRV) matching launchers (elastic.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace cva {

struct ElasticParams {
  int max_iters;      // ElasticOptions::max_iters (proj/include/curvalign/elastic.hpp:14)
  double energy_tol;  // ElasticOptions::energy_tol
  int max_slope;      // ElasticOptions::max_slope (DP step bound W)
  int use_fft = 1;    // ElasticOptions::use_fft: rigid steps by align_fft (1) or the direct sums (0)
};

struct ElasticOut {
  double* distance;
  double* energy;
  double* t0;
  double* theta;
  double* gamma;  // nullable: pairs x (n + 1)
  int32_t* iterations;
  int32_t* converged;
  int32_t* status;
  double* trace;  // nullable: pairs x (max_iters + 1) energies per accepted iteration, NaN-padded
};

// 8 <= n <= 2^20, 1 <= W <= 20 (255 steps: parent indices below the 0xff
// sentinel, srv.cpp:203-222). Slab mode: n or W past the shared-memory
// kernels; per-pair arrays, dp ring and parents in a per-CTA global slab.
bool elastic_supported(int n, int W);
bool elastic_slab_mode(int n, int W);
size_t elastic_smem(int n, int W);
// Bytes of per-CTA scratch in global memory (0: everything fits in shared
// memory; the parents alone, or in slab mode the whole working set).
size_t elastic_parent_slab(int64_t pairs, int n, int W);
int elastic_grid(int64_t pairs, int n, int W);

cudaError_t launch_dp_reparam(const double2* q1, const double2* q2, int64_t pairs, int n, int W,
                              uint8_t* slab, int grid, double* gamma, double* energy, int32_t* status,
                              cudaStream_t s);
cudaError_t launch_elastic_approach2(const double2* A, const double2* B, int64_t pairs, int64_t matrix_k, int n,
                                     const ElasticParams& prm, uint8_t* slab, int grid, const double2* tw,
                                     const ElasticOut& out, cudaStream_t s);

// approach 1: scratch bytes for pairs x n work items; grid for those items
size_t elastic_a1_scratch(int64_t pairs, int n, bool gamma);
int elastic_items_grid(int64_t items, int n, int W);
cudaError_t launch_elastic_approach1(const double2* A, const double2* B, int64_t pairs, int64_t matrix_k, int n,
                                     int W, uint8_t* slab, int grid, void* scratch, const ElasticOut& out,
                                     cudaStream_t s);

// single-call utilities (one CTA)
cudaError_t launch_srv_action(const double2* q, int n, double t0, double theta, const double* g, double2* out,
                              cudaStream_t s);
cudaError_t launch_elastic_energy(const double2* q1, const double2* q2, int n, double t0, double theta,
                                  const double* g, double* T, double* out, cudaStream_t s);
cudaError_t launch_dp_step_cost(const double2* q1, const double2* q2, int n, int i0, int j0, int a, int b,
                                double* out, cudaStream_t s);

}  // namespace cva
