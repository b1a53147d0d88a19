// Real DFT helpers (reference: proj/src/fft.cpp:81-125) on the GPU.
#include "curvalign/fft.hpp"

#include <stdexcept>

#include "status.hpp"

namespace curvalign {

std::vector<std::complex<double>> real_dft(std::span<const double> in) {
  const std::size_t n = in.size();
  if (n < 2) throw std::invalid_argument("fft: length must be at least 2");
  std::vector<std::complex<double>> x(n), out(n / 2 + 1);
  for (std::size_t j = 0; j < n; ++j) x[j] = {in[j], 0.0};
  detail::check_dropin(cva_dft_host(reinterpret_cast<const double*>(x.data()), (int64_t)n, (int64_t)out.size(), -1,
                                    1.0, reinterpret_cast<double*>(out.data())));
  return out;
}

std::vector<double> real_idft(std::span<const std::complex<double>> spec, std::size_t n) {
  if (spec.size() != n / 2 + 1) throw std::invalid_argument("fft: spectrum size mismatch");
  std::vector<std::complex<double>> full(n), out(n);
  for (std::size_t k = 0; k < n; ++k) full[k] = k <= n / 2 ? spec[k] : std::conj(spec[n - k]);
  detail::check_dropin(cva_dft_host(reinterpret_cast<const double*>(full.data()), (int64_t)n, (int64_t)n, +1,
                                    1.0 / (double)n, reinterpret_cast<double*>(out.data())));
  std::vector<double> r(n);
  for (std::size_t j = 0; j < n; ++j) r[j] = out[j].real();
  return r;
}

std::vector<double> circular_cross_correlation(std::span<const double> a, std::span<const double> b) {
  if (a.size() != b.size()) throw std::invalid_argument("fft: correlation size mismatch");
  const std::size_t n = a.size();
  if (n < 2) throw std::invalid_argument("fft: length must be at least 2");
  // r[m] = A11(m) of the curves (a, 0), (b, 0), by FFT (O(n log n), fft.cpp:116-125)
  std::vector<Point2> pa(n), pb(n);
  for (std::size_t i = 0; i < n; ++i) {
    pa[i] = Point2(a[i], 0.0);
    pb[i] = Point2(b[i], 0.0);
  }
  std::vector<double> m4(4 * n), r(n);
  detail::check_dropin(cva_correlation_fft_host(detail::raw(pa.data()), detail::raw(pb.data()), (int64_t)n, m4.data()));
  for (std::size_t m = 0; m < n; ++m) r[m] = m4[4 * m];
  return r;
}

}  // namespace curvalign
