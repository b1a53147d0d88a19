/* curvalign_cuda.h — C ABI of the B200-native (sm_100a) curve-alignment library
 * libcurvalign_cuda.so (paper_2501_17779_b200/).
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 2501.17779,
 * "FFT-based alignment of 2d closed curves"; reference C++ API in
 * /root/reference/proj/include/curvalign/). Plain pointers and sizes only: no
 * C++ or torch types cross it. The C++ API of the reference (namespace
 * curvalign: align_fft, preprocess, resample_uniform, srv_transform, ...) is
 * re-declared in the include/curvalign/ headers and implemented on top of these entry
 * points (paper_2501_17779_b200/csrc/dropin/, one .cpp per header); INTEGRATION.md shows the
 * ctypes / C++ bindings a maintainer adds.
 *
 * Data layout. A curve of n nodes is n interleaved (x, y) doubles — the layout
 * of curvalign::Point2 (proj/include/curvalign/geometry.hpp:9-33) and of
 * std::span<const Point2>::data(), so reference buffers pass through unchanged.
 * Batches are contiguous: pairs * n * 2 doubles. Ragged batches of raw curves
 * use an offsets array: curve c is points [offsets[c], offsets[c+1]).
 * Device curve buffers are accessed as 16-byte (x, y) pairs and must be
 * 16-byte aligned (cudaMalloc'd arrays at whole-point offsets are); an
 * 8-byte-aligned pointer is rejected with CVA_INVALID_ARGUMENT. The *_host
 * entry points copy into their own device buffers and accept any alignment.
 *
 * Conventions (identical to the reference):
 *  - shift m pairs c1[l] with c2[(l + m) mod N]            rigid_align.hpp:12-13
 *  - rotation R(theta) = [[cos, sin], [-sin, cos]] (clockwise); the aligned
 *    curve is aligned[l] = R(theta) c2[(l + shift) mod N]    geometry.hpp:48-73
 *  - best shift = smallest m with |D_m| >= max|D| - 1e-12 max(1, max|D|),
 *    D_m = sum_l conj(z1_l) z2_{(l+m) mod N}                 rigid_align.cpp:31-47
 *  - energy = max(0, h (|c1|^2 + |c2|^2) - 2 h trace), h = 1/N  rigid_align.cpp:56-59
 *
 * Errors. Every entry point returns a cva_status. Batched device entry points
 * validate what they can on the host (CVA_INVALID_ARGUMENT) and report
 * data-dependent failures per pair in cva_alignment.status (e.g. coincident
 * adjacent nodes -> CVA_INVALID_ARGUMENT, as proj/src/curve.cpp:58 throws),
 * with NaN theta/energy for that pair, like distance_matrix's NaN cells
 * (proj/src/elastic.cpp:210-217). cva_last_error() returns a thread-local
 * message for the last failing call on the calling thread.
 *
 * Streams. `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream). Device entry points are asynchronous on that stream; *_host entry
 * points are synchronous. All entry points are thread-safe (the twiddle-table
 * cache is guarded per device).
 */
#ifndef CURVALIGN_CUDA_H
#define CURVALIGN_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVA_ABI_VERSION 1

typedef enum cva_status {
  CVA_OK = 0,
  CVA_INVALID_ARGUMENT = 1, /* reference throws std::invalid_argument */
  CVA_RUNTIME_ERROR = 2,    /* reference throws std::runtime_error (singular spline) */
  CVA_BAD_ALLOC = 3,        /* reference throws std::bad_alloc */
  CVA_CUDA_ERROR = 4,       /* no device / launch failure / kernel fault */
  CVA_UNSUPPORTED = 5       /* size outside what this build's kernels cover */
} cva_status;

/* One alignment result; mirrors curvalign::RigidAlignment
 * (proj/include/curvalign/rigid_align.hpp:16-23). 48 bytes. */
typedef struct cva_alignment {
  int64_t shift;      /* m */
  double t0;          /* m / N */
  double theta;       /* Rotation2 angle, (-pi, pi] */
  double trace;       /* tr(R A^T) at the optimum = |D_m| */
  double energy;      /* mismatch energy */
  int32_t degenerate; /* rotation underdetermined (D_m == 0) */
  int32_t status;     /* cva_status of this pair */
} cva_alignment;

int cva_abi_version(void);
const char* cva_last_error(void);
/* Number of visible CUDA devices (0 when none); never fails. */
int cva_device_count(void);
/* Largest raw node count a single curve may have in the resampling entry points
 * (INT32_MAX: curves beyond shared memory are solved in global scratch). */
int64_t cva_max_resample_nodes(void);

/* ---------------------------------------------------------------------------
 * Hot-path batch entry points (device pointers, asynchronous on `stream`).
 * ------------------------------------------------------------------------- */

/* align_fft over a batch of pre-sampled pairs (proj/src/rigid_align.cpp:204-208).
 * c1, c2: pairs x n points. out: pairs results. aligned (nullable): pairs x n
 * points, aligned[l] = R c2[(l + shift) mod n]. Any n >= 4: n <= 2048 runs in
 * shared memory (non-powers of two zero-padded), larger n through the
 * L2-chunked multi-pass transform. */
int cva_align_batch(const double* c1, const double* c2, int64_t pairs, int64_t n,
                    cva_alignment* out, double* aligned, void* stream);

/* preprocess (proj/src/curve.cpp:93-97) of a ragged batch of raw curves.
 * resample != 0: periodic-cubic-spline arc-length resampling to n_out nodes,
 * then center, then normalize; out is curves x n_out points.
 * resample == 0: center + normalize only; out has the input's ragged layout.
 * max_n_in: largest curve size in the batch (host-known; sizes the kernels'
 *   scratch), or 0 to have it computed from the offsets; a curve longer than a
 *   positive max_n_in is reported CVA_INVALID_ARGUMENT in status (never read).
 * status (nullable): per-curve cva_status. */
int cva_preprocess_batch(const double* points, const int64_t* offsets, int64_t curves,
                         int64_t max_n_in, int64_t n_out, int resample, double* out,
                         int32_t* status, void* stream);

/* resample_uniform (proj/src/curve.cpp:67-91) of a ragged batch: periodic cubic
 * spline through the raw nodes on chordal arc length, sampled at t_l = l/n_out.
 * No centering / normalisation. out is curves x n_out points. */
int cva_resample_batch(const double* points, const int64_t* offsets, int64_t curves,
                       int64_t max_n_in, int64_t n_out, double* out, int32_t* status,
                       void* stream);

/* Fused C1 path (the BASELINE headline): pair p = (curve 2p, curve 2p+1) of
 * the ragged raw batch; preprocess both to n_out nodes (resample != 0;
 * proj/src/curve.cpp:93-97) then align_fft (proj/src/rigid_align.cpp:204-208),
 * the sequence of cmd_align / run_align (proj/src/cli.cpp:41-44, :99). aligned
 * (nullable): pairs x n_out points. Any raw node count and any n_out >= 8:
 * n_out = 512 / 1024 with raw curves <= 3072 nodes run one fused kernel, other
 * sizes preprocess into scratch and align (multi-pass beyond n_out = 2048). */
int cva_preprocess_align_batch(const double* points, const int64_t* offsets, int64_t pairs,
                               int64_t max_n_in, int64_t n_out, int resample,
                               cva_alignment* out, double* aligned, void* stream);

/* preprocess(resample = false) of both curves (center, then normalize to unit
 * length; proj/src/curve.cpp:93-97) fused with align_fft, for equal-size pairs
 * (BASELINE configs C0 and C3). Any N >= 4; large N runs the L2-chunked
 * multi-pass transform. aligned (nullable): pairs x n points. */
int cva_preprocess_align_uniform(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                 cva_alignment* out, double* aligned, void* stream);

/* SRV-space alignment: align_fft(srv_center(srv_transform(c1)).q,
 * srv_center(srv_transform(c2)).q) (proj/src/srv.cpp:71-98; the (t0,R) step
 * pattern of proj/src/elastic.cpp:138-139). aligned_q (nullable): the rotated,
 * shifted centered SRV of c2. Requires n >= 8; any n (n <= 2048 fused on chip,
 * larger n: SRV curves in scratch, then the multi-pass alignment). */
int cva_srv_align_batch(const double* c1, const double* c2, int64_t pairs, int64_t n,
                        cva_alignment* out, double* aligned_q, void* stream);

/* All ordered pairs of `count` pre-sampled curves of n nodes (BASELINE config
 * C2; the cells of distance_matrix, proj/src/elastic.cpp:176-236, each an
 * align_fft). Rows [row_begin, row_end) of the count x count matrices:
 * energy[r][j] (f64), shift[r][j] (i32), theta[r][j] (f64) for pair
 * (curve row_begin + r, curve j), row-major. Each curve's spectrum is computed
 * once and reused across its row and column. Multi-GPU callers shard rows. */
int cva_allpairs(const double* curves, int64_t count, int64_t n, int64_t row_begin, int64_t row_end,
                 double* energy, int32_t* shift, double* theta, void* stream);

/* ---------------------------------------------------------------------------
 * Host-buffer entry points (synchronous; host <-> device copies included).
 * These are what the C++ drop-in API (include/curvalign/ headers) calls; each
 * replaces the reference function its device twin above cites.
 * ------------------------------------------------------------------------- */

int cva_align_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                         cva_alignment* out, double* aligned);
int cva_preprocess_batch_host(const double* points, const int64_t* offsets, int64_t curves,
                              int64_t n_out, int resample, double* out, int32_t* status);
int cva_resample_batch_host(const double* points, const int64_t* offsets, int64_t curves,
                            int64_t n_out, double* out, int32_t* status);
int cva_preprocess_align_batch_host(const double* points, const int64_t* offsets, int64_t pairs,
                                    int64_t n_out, int resample, cva_alignment* out,
                                    double* aligned);
int cva_srv_align_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                             cva_alignment* out, double* aligned_q);
int cva_preprocess_align_uniform_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                      cva_alignment* out, double* aligned);
int cva_allpairs_host(const double* curves, int64_t count, int64_t n, int64_t row_begin,
                      int64_t row_end, double* energy, int32_t* shift, double* theta);

/* ---------------------------------------------------------------------------
 * Single-curve utilities behind the C++ drop-in API (synchronous, host
 * buffers, GPU compute). cva_dropin_last_error() describes their failures.
 * ------------------------------------------------------------------------- */

const char* cva_dropin_last_error(void);
/* A(m), m in [m_begin, m_begin + m_count): out4[4 i + {0,1,2,3}] = a11, a12, a21, a22
 * (cross_correlation_matrix / correlation_all_shifts_*, rigid_align.cpp:65-80, :126-183). */
int cva_correlation_matrices_host(const double* c1, const double* c2, int64_t n, int64_t m_begin,
                                  int64_t m_count, double* out4);
/* mismatch_energy (rigid_align.cpp:185-196) */
int cva_mismatch_energy_host(const double* c1, const double* c2, int64_t n, int64_t shift, double theta,
                             double* out);
/* centroid (curve.cpp:27-32) and curve_length (curve.cpp:17-25); either output nullable */
int cva_curve_stats_host(const double* xy, int64_t n, double* centroid2, double* length);
/* mode 1: center_curve (curve.cpp:34-39); mode 2: normalize_length (curve.cpp:41-48) */
int cva_center_or_normalize_host(const double* xy, int64_t n, int mode, double* out);
/* arc_length_params (curve.cpp:50-65): s[0..n], total */
int cva_arc_length_params_host(const double* xy, int64_t n, double* s, double* total);
/* PeriodicCubicSpline second derivatives m[0..n_knots) (spline.cpp:62-96) */
int cva_spline_solve_host(const double* x, const double* y, int64_t n_knots, double* m);
/* srv_transform (srv.cpp:71-88); center != 0 also applies srv_center (srv.cpp:90-98) */
int cva_srv_transform_host(const double* xy, int64_t n, int center, double* q);
/* X_k = scale * sum_j x_j exp(sign 2 pi i j k / n), k < kcount (any n, O(n log n):
 * radix 2 or Bluestein; real_dft / real_idft, proj/src/fft.cpp:81-114) */
int cva_dft_host(const double* x_complex, int64_t n, int64_t kcount, int sign, double scale,
                 double* out_complex);
/* A(m) for every shift m, out4[4 m + {0,1,2,3}] = a11, a12, a21, a22, by FFT
 * (correlation_all_shifts_fft, rigid_align.cpp:147-183; any n, O(n log n)) */
int cva_correlation_fft_host(const double* c1, const double* c2, int64_t n, double* out4);

/* ---------------------------------------------------------------------------
 * Elastic (SRV) matching: the rigid path's callers in the reference's elastic
 * distance (proj/src/srv.cpp:100-257, proj/src/elastic.cpp:102-236).
 * Device entry points are asynchronous on `stream`; *_host are synchronous.
 * Failures are per pair in `status` (NaN outputs), like distance_matrix's NaN
 * cells (elastic.cpp:210-217).
 * ------------------------------------------------------------------------- */

/* dp_reparam(q1[p], q2[p], max_slope) (srv.cpp:180-257) for pairs x n SRV samples:
 * gamma pairs x (n+1), energy pairs. Bitwise the reference's result.
 * status (nullable): CVA_RUNTIME_ERROR where no admissible path exists. */
int cva_dp_reparam_batch(const double* q1, const double* q2, int64_t pairs, int64_t n, int max_slope,
                         double* gamma, double* energy, int32_t* status, void* stream);
int cva_dp_reparam_batch_host(const double* q1, const double* q2, int64_t pairs, int64_t n,
                              int max_slope, double* gamma, double* energy, int32_t* status);

/* elastic_distance_approach2(c1[p], c2[p], opts) (elastic.cpp:102-174) on
 * preprocessed curves (pairs x n points each). Outputs per pair: distance,
 * energy, t0, theta (Rotation2 angle), gamma (nullable, pairs x (n+1)),
 * iterations, converged, status, energy_trace (nullable, pairs x (max_iters+1):
 * ElasticMatch::energy_trace, NaN after the last iteration). The rigid steps
 * use the FFT correlation (ElasticOptions::use_fft = true: align_fft); the
 * _ex entry points take use_fft, and 0 runs them on the direct per-shift sums
 * (align_naive, rigid_align.cpp:198-202). ElasticOptions defaults: max_iters
 * 30, energy_tol 1e-6, use_fft 1, max_slope 4. Supports 8 <= n <= 2^20 and 1 <= max_slope <= 20; n <= 1024
 * (non-powers of two <= 512) with max_slope <= 8 run the shared-memory
 * kernels, anything else slab mode (per-CTA global working set, direct
 * correlation for the rigid steps). */
int cva_elastic_approach2_batch(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                int max_iters, double energy_tol, int max_slope, double* distance,
                                double* energy, double* t0, double* theta, double* gamma,
                                int32_t* iterations, int32_t* converged, int32_t* status,
                                double* energy_trace, void* stream);
int cva_elastic_approach2_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                     int max_iters, double energy_tol, int max_slope, double* distance,
                                     double* energy, double* t0, double* theta, double* gamma,
                                     int32_t* iterations, int32_t* converged, int32_t* status,
                                     double* energy_trace);
int cva_elastic_approach2_batch_ex(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                   int max_iters, double energy_tol, int max_slope, int use_fft,
                                   double* distance, double* energy, double* t0, double* theta, double* gamma,
                                   int32_t* iterations, int32_t* converged, int32_t* status,
                                   double* energy_trace, void* stream);
int cva_elastic_approach2_batch_ex_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                        int max_iters, double energy_tol, int max_slope, int use_fft,
                                        double* distance, double* energy, double* t0, double* theta,
                                        double* gamma, int32_t* iterations, int32_t* converged, int32_t* status,
                                        double* energy_trace);

/* elastic_distance_approach1(c1[p], c2[p], opts) (elastic.cpp:62-100): for every
 * start shift m, the Kabsch rotation of the SRV pair, one DP, the realised
 * energy; the first m with the smallest energy wins. n <= n_max_approach1
 * (ElasticOptions::n_max_approach1, default 512) else CVA_INVALID_ARGUMENT.
 * Outputs as cva_elastic_approach2_batch (iterations = converged = 1). */
int cva_elastic_approach1_batch(const double* c1, const double* c2, int64_t pairs, int64_t n, int max_slope,
                                int64_t n_max_approach1, double* distance, double* energy, double* t0,
                                double* theta, double* gamma, int32_t* iterations, int32_t* converged,
                                int32_t* status, void* stream);
int cva_elastic_approach1_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                     int max_slope, int64_t n_max_approach1, double* distance, double* energy,
                                     double* t0, double* theta, double* gamma, int32_t* iterations,
                                     int32_t* converged, int32_t* status);

/* distance_matrix(curves, method, n) cells (elastic.cpp:176-236) for `count`
 * preprocessed curves of n nodes: d[i * count + j] = distance of matching curve j
 * onto curve i (method 1: approach 1, 2: approach 2); NaN for a failed pair. */
int cva_elastic_distance_matrix(const double* curves, int64_t count, int64_t n, int method, int max_iters,
                                double energy_tol, int max_slope, int64_t n_max_approach1, double* d,
                                void* stream);
int cva_elastic_distance_matrix_host(const double* curves, int64_t count, int64_t n, int method, int max_iters,
                                     double energy_tol, int max_slope, int64_t n_max_approach1, double* d);
int cva_elastic_distance_matrix_ex(const double* curves, int64_t count, int64_t n, int method, int max_iters,
                                   double energy_tol, int max_slope, int use_fft, int64_t n_max_approach1,
                                   double* d, void* stream);
int cva_elastic_distance_matrix_ex_host(const double* curves, int64_t count, int64_t n, int method,
                                        int max_iters, double energy_tol, int max_slope, int use_fft,
                                        int64_t n_max_approach1, double* d);

/* Single-call SRV utilities behind the C++ drop-in (synchronous, host buffers,
 * GPU compute; failures in cva_dropin_last_error()):
 * apply_srv_action (srv.cpp:100-118), elastic_energy (:120-128), dp_step_cost
 * (:145-176). gamma: n + 1 values; theta: Rotation2 angle. */
int cva_apply_srv_action_host(const double* q, int64_t n, double t0, double theta, const double* gamma,
                              double* out);
int cva_elastic_energy_host(const double* q1, const double* q2, int64_t n, double t0, double theta,
                            const double* gamma, double* out);
int cva_dp_step_cost_host(const double* q1, const double* q2, int64_t n, int i0, int j0, int di, int dj,
                          double* out);

/* ---------------------------------------------------------------------------
 * Diagnostics (not on the hot path).
 * ------------------------------------------------------------------------- */

/* Measured FP64 FMA throughput of the current device (dependent DFMA chains,
 * 8 per thread, CUDA-event timed), for the FP64 roofline denominator. */
int cva_probe_fp64_tflops(double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* CURVALIGN_CUDA_H */
