// Elastic distance (reference: proj/src/elastic.cpp) on the GPU: every pair of
// a call runs in one batched launch of the approach-1 / approach-2 kernels.
#include "curvalign/elastic.hpp"

#include <chrono>
#include <cmath>
#include <limits>
#include <stdexcept>

#include "status.hpp"

namespace curvalign {

using detail::check;
using detail::raw;

namespace {

void check_elastic_inputs(const Curve& c1, const Curve& c2) {  // elastic.cpp:55-58
  if (c1.size() != c2.size()) throw std::invalid_argument("elastic: node count mismatch");
  if (c1.size() < 8) throw std::invalid_argument("elastic: need at least 8 nodes");
}

struct Batch {
  std::vector<double> distance, energy, t0, theta, gamma, trace;
  int trace_len = 0;
  std::vector<int32_t> iterations, converged, status;
};

// c: pairs * n points each side; matrix_k > 0: curves is count x n and pairs = k^2 (matrix mode)
Batch run(const std::vector<Point2>& a, const std::vector<Point2>& b, int64_t pairs, int64_t n, int method,
          const ElasticOptions& o, bool want_gamma) {
  Batch r;
  r.distance.resize(pairs), r.energy.resize(pairs), r.t0.resize(pairs), r.theta.resize(pairs);
  r.iterations.resize(pairs), r.converged.resize(pairs), r.status.resize(pairs);
  if (want_gamma) r.gamma.resize((size_t)pairs * (n + 1));
  double* g = want_gamma ? r.gamma.data() : nullptr;
  if (method == 1)
    check(cva_elastic_approach1_batch_host(raw(a.data()), raw(b.data()), pairs, n, o.max_slope,
                                           (int64_t)o.n_max_approach1, r.distance.data(), r.energy.data(), r.t0.data(),
                                           r.theta.data(), g, r.iterations.data(), r.converged.data(),
                                           r.status.data()));
  else {
    r.trace_len = o.max_iters + 1;
    r.trace.resize((size_t)pairs * r.trace_len);
    check(cva_elastic_approach2_batch_ex_host(raw(a.data()), raw(b.data()), pairs, n, o.max_iters, o.energy_tol,
                                              o.max_slope, o.use_fft ? 1 : 0, r.distance.data(), r.energy.data(),
                                              r.t0.data(), r.theta.data(), g, r.iterations.data(),
                                              r.converged.data(), r.status.data(), r.trace.data()));
  }
  return r;
}

ElasticMatch to_match(const Batch& r, std::size_t p, std::size_t n) {
  if (r.status[p] == CVA_INVALID_ARGUMENT) throw std::invalid_argument("elastic: invalid input");
  if (r.status[p] == CVA_RUNTIME_ERROR) throw std::runtime_error("dp: no admissible path");
  if (r.status[p] != CVA_OK) throw std::runtime_error("elastic: GPU failure");
  ElasticMatch m;
  m.t0 = r.t0[p];
  m.rotation = Rotation2(r.theta[p]);
  if (!r.gamma.empty()) m.gamma.gamma.assign(r.gamma.begin() + p * (n + 1), r.gamma.begin() + (p + 1) * (n + 1));
  m.energy = r.energy[p];
  m.distance = r.distance[p];
  m.iterations = r.iterations[p];
  m.converged = r.converged[p] != 0;
  if (r.trace_len) {  // approach 2: initial energy + one entry per iteration (elastic.cpp:119, :160)
    for (int k = 0; k < r.trace_len; ++k) {
      const double v = r.trace[p * r.trace_len + k];
      if (std::isnan(v)) break;
      m.energy_trace.push_back(v);
    }
  } else {
    m.energy_trace = {m.energy};  // approach 1 (elastic.cpp:97)
  }
  return m;
}

}  // namespace

std::vector<ElasticMatch> elastic_distance_batch(const std::vector<Curve>& c1, const std::vector<Curve>& c2,
                                                 DistanceMethod method, const ElasticOptions& opts) {
  if (c1.size() != c2.size()) throw std::invalid_argument("elastic: pair count mismatch");
  if (c1.empty()) return {};
  const std::size_t n = c1[0].size();
  std::vector<Point2> a, b;
  for (std::size_t p = 0; p < c1.size(); ++p) {
    check_elastic_inputs(c1[p], c2[p]);
    if (c1[p].size() != n) throw std::invalid_argument("elastic: batch pairs must share one size");
    a.insert(a.end(), c1[p].nodes.begin(), c1[p].nodes.end());
    b.insert(b.end(), c2[p].nodes.begin(), c2[p].nodes.end());
  }
  if (method == DistanceMethod::approach1 && n > opts.n_max_approach1)
    throw std::invalid_argument("approach 1 is O(N^3); node count exceeds the configured limit, use approach 2");
  const Batch r = run(a, b, (int64_t)c1.size(), (int64_t)n, method == DistanceMethod::approach1 ? 1 : 2, opts, true);
  std::vector<ElasticMatch> out;
  for (std::size_t p = 0; p < c1.size(); ++p) out.push_back(to_match(r, p, n));
  return out;
}

ElasticMatch elastic_distance_approach1(const Curve& c1, const Curve& c2, const ElasticOptions& opts) {
  return elastic_distance_batch({c1}, {c2}, DistanceMethod::approach1, opts)[0];
}

ElasticMatch elastic_distance_approach2(const Curve& c1, const Curve& c2, const ElasticOptions& opts) {
  return elastic_distance_batch({c1}, {c2}, DistanceMethod::approach2, opts)[0];
}

std::vector<std::vector<double>> distance_matrix(const std::vector<Curve>& curves, DistanceMethod method,
                                                 std::size_t n, const ElasticOptions& opts, unsigned max_threads,
                                                 const CellCallback& on_cell) {
  (void)max_threads;
  if (curves.size() < 2) throw std::invalid_argument("distance_matrix: need at least 2 curves");
  const auto start = std::chrono::steady_clock::now();
  std::vector<Point2> prep;
  for (const Curve& p : preprocess_batch(curves, n, true))  // preprocess(curves[i], n, true) (elastic.cpp:184)
    prep.insert(prep.end(), p.nodes.begin(), p.nodes.end());
  const std::size_t k = curves.size();
  std::vector<double> d(k * k);
  check(cva_elastic_distance_matrix_ex_host(raw(prep.data()), (int64_t)k, (int64_t)n,
                                            method == DistanceMethod::approach1 ? 1 : 2, opts.max_iters,
                                            opts.energy_tol, opts.max_slope, opts.use_fft ? 1 : 0,
                                            (int64_t)opts.n_max_approach1, d.data()));
  std::vector<std::vector<double>> out(k, std::vector<double>(k));
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count() / (double)(k * k);
  for (std::size_t i = 0; i < k; ++i)
    for (std::size_t j = 0; j < k; ++j) {
      out[i][j] = d[i * k + j];
      if (on_cell) on_cell(i, j, out[i][j], secs);
    }
  return out;
}

}  // namespace curvalign
