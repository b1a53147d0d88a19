// PeriodicCubicSpline (reference: proj/src/spline.cpp). The cyclic system for
// the second derivatives is solved on the GPU (cva_spline_solve_host, the
// partition solver of csrc/spline.cuh); eval / derivative apply the cubic.
#include "curvalign/spline.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "status.hpp"

namespace curvalign {

PeriodicCubicSpline::PeriodicCubicSpline(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size()) throw std::invalid_argument("spline: knot/value size mismatch");
  if (x.size() < 4) throw std::invalid_argument("spline: need at least 4 knots");
  for (std::size_t i = 0; i + 1 < x.size(); ++i)
    if (!(x[i] < x[i + 1])) throw std::invalid_argument("spline: knots must be strictly increasing");
  for (double v : y)
    if (!std::isfinite(v)) throw std::invalid_argument("spline: non-finite value");
  knots_.assign(x.begin(), x.end());
  vals_.assign(y.begin(), y.end());
  vals_.back() = vals_.front();
  m_.resize(knots_.size());
  detail::check_dropin(cva_spline_solve_host(knots_.data(), vals_.data(), (int64_t)knots_.size(), m_.data()));
}

double PeriodicCubicSpline::wrap(double x) const {
  const double p = period();
  double xw = knots_.front() + std::fmod(x - knots_.front(), p);
  if (xw < knots_.front()) xw += p;
  return xw;
}

std::size_t PeriodicCubicSpline::interval(double xw) const {
  const std::size_t i = (std::size_t)(std::upper_bound(knots_.begin(), knots_.end(), xw) - knots_.begin());
  if (i == 0) return 0;
  return std::min(i - 1, knots_.size() - 2);
}

double PeriodicCubicSpline::eval(double x) const {
  const double xw = wrap(x);
  const std::size_t i = interval(xw);
  const double h = knots_[i + 1] - knots_[i];
  const double a = (knots_[i + 1] - xw) / h, b = (xw - knots_[i]) / h;
  return a * vals_[i] + b * vals_[i + 1] + ((a * a * a - a) * m_[i] + (b * b * b - b) * m_[i + 1]) * h * h / 6.0;
}

double PeriodicCubicSpline::derivative(double x) const {
  const double xw = wrap(x);
  const std::size_t i = interval(xw);
  const double h = knots_[i + 1] - knots_[i];
  const double a = (knots_[i + 1] - xw) / h, b = (xw - knots_[i]) / h;
  return (vals_[i + 1] - vals_[i]) / h + ((1.0 - 3.0 * a * a) * m_[i] + (3.0 * b * b - 1.0) * m_[i + 1]) * h / 6.0;
}

}  // namespace curvalign
