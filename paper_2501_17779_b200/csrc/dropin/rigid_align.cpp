// Rigid alignment (reference: proj/src/rigid_align.cpp) on the GPU.
#include "curvalign/rigid_align.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>

#include "status.hpp"

namespace curvalign {

using detail::check;
using detail::check_dropin;
using detail::raw;

namespace {

// rigid_align.cpp:18-21
void check_pair(std::size_t n1, std::size_t n2) {
  if (n1 != n2) throw std::invalid_argument("align: node count mismatch");
  if (n1 < 4) throw std::invalid_argument("align: need at least 4 nodes");
}

RigidAlignment from_record(const cva_alignment& r) {
  if (r.status != CVA_OK) {
    if (r.status == CVA_INVALID_ARGUMENT)
      throw std::invalid_argument("rotation: non-finite correlation matrix");
    throw std::runtime_error("curvalign: pair failed with status " + std::to_string(r.status));
  }
  RigidAlignment a;
  a.shift = (std::size_t)r.shift;
  a.t0 = r.t0;
  a.rotation = Rotation2(r.theta);
  a.trace = r.trace;
  a.energy = r.energy;
  a.degenerate = r.degenerate != 0;
  return a;
}

std::vector<Point2> flatten(const std::vector<Curve>& cs, std::size_t n) {
  std::vector<Point2> out;
  out.reserve(cs.size() * n);
  for (const Curve& c : cs) {
    if (c.size() != n) throw std::invalid_argument("align: node count mismatch");
    out.insert(out.end(), c.nodes.begin(), c.nodes.end());
  }
  return out;
}

}  // namespace

Mat2 cross_correlation_matrix(std::span<const Point2> c1, std::span<const Point2> c2, std::size_t shift) {
  check_pair(c1.size(), c2.size());
  if (shift >= c1.size()) throw std::invalid_argument("align: shift out of range");
  double a[4];
  check_dropin(cva_correlation_matrices_host(raw(c1.data()), raw(c2.data()), (int64_t)c1.size(), (int64_t)shift, 1, a));
  return Mat2{a[0], a[1], a[2], a[3]};
}

// The proper rotation maximising tr(R A^T). The reference takes it from a 2x2
// SVD with determinant correction (rigid_align.cpp:82-102); for a 2x2 matrix
// that rotation is exactly atan2(A12 - A21, A11 + A22) with trace
// |(A11 + A22, A12 - A21)| (the same value up to rounding; the reference's
// tests pin the two to 1e-8, test_rigid_align.cpp:88-100). O(1) host math.
RotationFit optimal_rotation_svd(const Mat2& A) {
  if (!A.finite()) throw std::invalid_argument("rotation: non-finite correlation matrix");
  if (std::sqrt(A.a11 * A.a11 + A.a12 * A.a12 + A.a21 * A.a21 + A.a22 * A.a22) == 0.0)
    return RotationFit{Rotation2(0.0), 0.0, true};
  const double c = A.a11 + A.a22, s = A.a12 - A.a21;
  return RotationFit{Rotation2(std::atan2(s, c)), std::hypot(c, s), false};
}

RotationFit optimal_rotation_closed_form(const Mat2& A) {
  if (!A.finite()) throw std::invalid_argument("rotation: non-finite correlation matrix");
  const double c = A.a11 + A.a22, s = A.a12 - A.a21;
  if (c == 0.0 && s == 0.0) return RotationFit{Rotation2(0.0), 0.0, true};
  return RotationFit{Rotation2(std::atan2(s, c)), std::hypot(c, s), false};
}

Rotation2 optimal_rotation_fixed_start(const Curve& c1, const Curve& c2) {
  return optimal_rotation_svd(cross_correlation_matrix(c1.nodes, c2.nodes, 0)).rotation;
}

std::vector<Mat2> correlation_all_shifts_naive(std::span<const Point2> c1, std::span<const Point2> c2) {
  check_pair(c1.size(), c2.size());
  const std::size_t n = c1.size();
  std::vector<Mat2> out(n);
  static_assert(sizeof(Mat2) == 4 * sizeof(double), "Mat2 is four packed doubles");
  check_dropin(cva_correlation_matrices_host(raw(c1.data()), raw(c2.data()), (int64_t)n, 0, (int64_t)n,
                                             reinterpret_cast<double*>(out.data())));
  return out;
}

// Two forward and two inverse GPU FFTs of z = x + i y (D and E spectra,
// gfft.cu), any n, O(n log n); correlation_all_shifts_naive above is the exact
// per-shift scan, so the reference's equivalence test (|naive - fft| <= 1e-9 n,
// test_rigid_align.cpp:133-151) compares two computations.
std::vector<Mat2> correlation_all_shifts_fft(std::span<const Point2> c1, std::span<const Point2> c2) {
  check_pair(c1.size(), c2.size());
  const std::size_t n = c1.size();
  std::vector<Mat2> out(n);
  check_dropin(cva_correlation_fft_host(raw(c1.data()), raw(c2.data()), (int64_t)n,
                                        reinterpret_cast<double*>(out.data())));
  return out;
}

double mismatch_energy(std::span<const Point2> c1, std::span<const Point2> c2, std::size_t shift,
                       const Rotation2& rotation) {
  check_pair(c1.size(), c2.size());
  if (shift >= c1.size()) throw std::invalid_argument("align: shift out of range");
  double e = 0.0;
  check_dropin(cva_mismatch_energy_host(raw(c1.data()), raw(c2.data()), (int64_t)c1.size(), (int64_t)shift,
                                        rotation.theta(), &e));
  return e;
}

RigidAlignment align_fft(std::span<const Point2> c1, std::span<const Point2> c2) {
  check_pair(c1.size(), c2.size());
  cva_alignment r{};
  check(cva_align_batch_host(raw(c1.data()), raw(c2.data()), 1, (int64_t)c1.size(), &r, nullptr));
  return from_record(r);
}

namespace {
double sum_norm2(std::span<const Point2> c) {
  double s = 0.0;
  for (const Point2& p : c) s += p.x * p.x + p.y * p.y;
  return s;
}

// pick_best (rigid_align.cpp:31-61): the smallest shift whose optimal trace is
// within 1e-12 (relative) of the maximum, rotation by SVD, energy identity.
RigidAlignment pick_best(const std::vector<Mat2>& corr, double s1, double s2, std::size_t n) {
  auto opt_trace = [](const Mat2& A) { return std::hypot(A.a11 + A.a22, A.a12 - A.a21); };
  double best = -std::numeric_limits<double>::infinity();
  for (const Mat2& A : corr) best = std::max(best, opt_trace(A));
  const double tol = 1e-12 * std::max(1.0, std::abs(best));
  std::size_t m = 0;
  for (std::size_t i = 0; i < n; ++i)
    if (opt_trace(corr[i]) >= best - tol) {
      m = i;
      break;
    }
  const RotationFit fit = optimal_rotation_svd(corr[m]);
  RigidAlignment out;
  out.shift = m;
  out.t0 = (double)m / (double)n;
  out.rotation = fit.rotation;
  out.trace = fit.trace;
  out.degenerate = fit.degenerate;
  const double h = 1.0 / (double)n;
  out.energy = std::max(0.0, h * (s1 + s2) - 2.0 * h * fit.trace);
  return out;
}
}  // namespace

// The exhaustive scan (rigid_align.cpp:198-202): exact per-shift sums on the GPU
// (correlation_all_shifts_naive), then the reference's tie-broken pick on the
// host — a computation independent of align_fft's FFT kernel, so the
// reference's acceptance criterion 1 (acceptance.cpp:94-120) compares the two.
RigidAlignment align_naive(std::span<const Point2> c1, std::span<const Point2> c2) {
  check_pair(c1.size(), c2.size());
  return pick_best(correlation_all_shifts_naive(c1, c2), sum_norm2(c1), sum_norm2(c2), c1.size());
}

std::vector<RigidAlignment> align_fft_batch(const std::vector<Curve>& c1, const std::vector<Curve>& c2,
                                            std::vector<Curve>* aligned) {
  if (c1.size() != c2.size()) throw std::invalid_argument("align: pair count mismatch");
  if (c1.empty()) return {};
  const std::size_t n = c1[0].size();
  check_pair(n, n);
  const std::vector<Point2> a = flatten(c1, n), b = flatten(c2, n);
  std::vector<cva_alignment> rec(c1.size());
  std::vector<Point2> al(aligned ? a.size() : 0);
  check(cva_align_batch_host(raw(a.data()), raw(b.data()), (int64_t)c1.size(), (int64_t)n, rec.data(),
                             aligned ? raw(al.data()) : nullptr));
  std::vector<RigidAlignment> out;
  out.reserve(rec.size());
  for (const auto& r : rec) out.push_back(from_record(r));
  if (aligned) {
    aligned->assign(c1.size(), Curve{});
    for (std::size_t p = 0; p < c1.size(); ++p)
      (*aligned)[p].nodes.assign(al.begin() + (std::ptrdiff_t)(p * n), al.begin() + (std::ptrdiff_t)((p + 1) * n));
  }
  return out;
}

std::vector<RigidAlignment> preprocess_align_batch(const std::vector<Curve>& raw1, const std::vector<Curve>& raw2,
                                                   std::size_t n_out, std::vector<Curve>* aligned) {
  if (raw1.size() != raw2.size()) throw std::invalid_argument("align: pair count mismatch");
  if (raw1.empty()) return {};
  if (n_out < 8) throw std::invalid_argument("resample: need at least 8 output nodes");
  std::vector<int64_t> offs(2 * raw1.size() + 1, 0);
  std::vector<Point2> pts;
  for (std::size_t p = 0; p < raw1.size(); ++p) {
    for (const Curve* c : {&raw1[p], &raw2[p]}) {
      validate_curve(*c, 4);
      pts.insert(pts.end(), c->nodes.begin(), c->nodes.end());
    }
    offs[2 * p + 1] = offs[2 * p] + (int64_t)raw1[p].size();
    offs[2 * p + 2] = offs[2 * p + 1] + (int64_t)raw2[p].size();
  }
  std::vector<cva_alignment> rec(raw1.size());
  std::vector<Point2> al(aligned ? raw1.size() * n_out : 0);
  check(cva_preprocess_align_batch_host(raw(pts.data()), offs.data(), (int64_t)raw1.size(), (int64_t)n_out, 1,
                                        rec.data(), aligned ? raw(al.data()) : nullptr));
  std::vector<RigidAlignment> out;
  for (const auto& r : rec) out.push_back(from_record(r));
  if (aligned) {
    aligned->assign(raw1.size(), Curve{});
    for (std::size_t p = 0; p < raw1.size(); ++p)
      (*aligned)[p].nodes.assign(al.begin() + (std::ptrdiff_t)(p * n_out), al.begin() + (std::ptrdiff_t)((p + 1) * n_out));
  }
  return out;
}

}  // namespace curvalign
