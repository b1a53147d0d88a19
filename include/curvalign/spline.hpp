// Drop-in for /root/reference/proj/include/curvalign/spline.hpp:17-35.
// The second-derivative system is solved on the GPU at construction.
#pragma once

#include <span>
#include <vector>

namespace curvalign {

class PeriodicCubicSpline {
 public:
  // x strictly increasing, x.size() == y.size() >= 4; y.back() is replaced by y.front().
  PeriodicCubicSpline(std::span<const double> x, std::span<const double> y);

  double eval(double x) const;
  double derivative(double x) const;
  double period() const { return knots_.back() - knots_.front(); }

 private:
  std::vector<double> knots_;  // n + 1
  std::vector<double> vals_;   // n + 1, vals_[n] == vals_[0]
  std::vector<double> m_;      // second derivatives, n + 1
  std::size_t interval(double xw) const;
  double wrap(double x) const;
};

}  // namespace curvalign
