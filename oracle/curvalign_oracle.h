/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the curve-alignment hot path.
 *
 * A plain-C restatement of the reference's algorithm (arXiv 2501.17779,
 * /root/reference/proj/src/ sources), each function citing the reference
 * file:line it follows. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, and only as the checker.
 * The product (paper_2501_17779_b200/, libcurvalign_cuda.so) never links it.
 *
 * Parity pins (tests/test_oracle_*.py): the reference's own sources compiled in
 * place (oracle/_ref/libcurvalign_ref.so, see oracle/Makefile) and the
 * reference's known-answer tests restated in tests/golden/.
 *
 * Points are interleaved (x, y) doubles, i.e. the layout of
 * curvalign::Point2 (proj/include/curvalign/geometry.hpp:9-33).
 * Status codes: 0 ok, 1 invalid_argument, 2 runtime_error, 3 bad_alloc.
 */
#ifndef CURVALIGN_ORACLE_H
#define CURVALIGN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_INVALID = 1, OR_RUNTIME = 2, OR_BAD_ALLOC = 3 };

/* Same layout as cva_alignment (include/curvalign_cuda.h) and RigidAlignment
 * (proj/include/curvalign/rigid_align.hpp:16-23). */
typedef struct or_alignment {
  int64_t shift;
  double t0;
  double theta;
  double trace;
  double energy;
  int32_t degenerate;
  int32_t status;
} or_alignment;

/* curve core (proj/src/curve.cpp) */
int or_validate_curve(const double* xy, int64_t n, int64_t min_nodes);
int or_curve_length(const double* xy, int64_t n, double* out);
int or_centroid(const double* xy, int64_t n, double* out2);
int or_center_curve(const double* xy, int64_t n, double* out);
int or_normalize_length(const double* xy, int64_t n, double* out);
int or_arc_length_params(const double* xy, int64_t n, double* s /* n+1 */, double* total);
int or_resample_uniform(const double* xy, int64_t n, int64_t n_out, double* out);
int or_preprocess(const double* xy, int64_t n, int64_t n_out, int resample, double* out);

/* periodic cubic spline (proj/src/spline.cpp): solve for second derivatives
 * m[0..n] (m[n] = m[0]) of knots x[0..n], values y[0..n]; evaluate. */
int or_spline_second_derivs(const double* x, const double* y, int64_t n_knots, double* m);
double or_spline_eval(const double* x, const double* y, const double* m, int64_t n_knots, double t);

/* rigid alignment (proj/src/rigid_align.cpp) */
int or_cross_correlation_matrix(const double* c1, const double* c2, int64_t n, int64_t shift,
                                double* a4);
int or_correlation_all_shifts_naive(const double* c1, const double* c2, int64_t n, double* out4n);
int or_correlation_all_shifts_fft(const double* c1, const double* c2, int64_t n, double* out4n);
int or_optimal_rotation_svd(const double* a4, double* theta, double* trace, int32_t* degenerate);
int or_optimal_rotation_closed_form(const double* a4, double* theta, double* trace,
                                    int32_t* degenerate);
int or_mismatch_energy(const double* c1, const double* c2, int64_t n, int64_t shift, double theta,
                       double* out);
int or_align_naive(const double* c1, const double* c2, int64_t n, or_alignment* out);
int or_align_fft(const double* c1, const double* c2, int64_t n, or_alignment* out);
/* aligned[l] = R(theta) c2[(l + shift) mod n], R clockwise (geometry.hpp:64-73) */
void or_aligned_curve(const double* c2, int64_t n, int64_t shift, double theta, double* out);

/* real FFT wrappers (proj/src/fft.cpp) */
int or_real_dft(const double* in, int64_t n, double* out_complex /* n/2+1 */);
int or_real_idft(const double* spec, int64_t n_bins, int64_t n, double* out);
int or_circular_cross_correlation(const double* a, const double* b, int64_t n, double* out);

/* SRV (proj/src/srv.cpp:71-98) */
int or_srv_transform(const double* xy, int64_t n, double* q);
int or_srv_center(const double* q, int64_t n, double* out);

/* elastic (SRV) matching (oracle/elastic_oracle.c; proj/src/srv.cpp:100-257,
 * proj/src/elastic.cpp:21-174). gamma arrays hold n+1 values. */
typedef struct or_elastic_match {
  double t0, theta, energy, distance;
  int32_t iterations, converged;
  double* gamma; /* nullable: n+1 values */
} or_elastic_match;
double or_wrap_unit(double t);
int or_apply_srv_action(const double* q, int64_t n, double t0, double theta, const double* gamma,
                        double* out);
int or_elastic_energy(const double* q1, const double* q2, int64_t n, double t0, double theta,
                      const double* gamma, double* out);
int or_dp_step_cost(const double* q1, const double* q2, int64_t n, int i0, int j0, int di, int dj,
                    double* out);
int or_dp_reparam(const double* q1, const double* q2, int64_t n, int max_slope, double* gamma,
                  double* energy);
int or_elastic_approach2(const double* c1, const double* c2, int64_t n, int max_iters, double energy_tol,
                         int use_fft, int max_slope, or_elastic_match* out);
int or_elastic_approach1(const double* c1, const double* c2, int64_t n, int max_slope, int64_t n_max,
                         or_elastic_match* out);

/* Batched drivers over a ragged point array: pair p aligns curve 2p against
 * curve 2p+1, curve c = points [offsets[c], offsets[c+1]).
 *   mode 0: preprocess(raw, n_out, resample) both curves, then align_fft
 *   mode 1: inputs already uniform: align_fft
 *   mode 2: SRV: align_fft(srv_center(srv_transform(c1)), srv_center(srv_transform(c2)))
 * aligned (nullable): pairs * n_out points. threads <= 1 runs serially.
 * Returns the first nonzero per-pair status (per-pair status in out[p].status). */
int or_batch(const double* points, const int64_t* offsets, int64_t pairs, int64_t n_out,
             int resample, int mode, int threads, or_alignment* out, double* aligned);

#ifdef __cplusplus
}
#endif

#endif
