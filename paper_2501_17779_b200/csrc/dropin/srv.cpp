// SRV helpers (reference: proj/src/srv.cpp) on the GPU: transform / center,
// the SRV action, the elastic energy and the reparameterisation DP. The small
// header-level helpers (identity_reparam, validate_reparam, Reparameterization::eval,
// dp_admissible_steps) are data-structure code and stay on the host, as in the
// reference's header.
#include "curvalign/srv.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "status.hpp"

namespace curvalign {

using detail::check;
using detail::check_dropin;
using detail::raw;

SrvCurve srv_transform(const Curve& c) {
  validate_curve(c, 8);
  SrvCurve out;
  out.h = 1.0 / (double)c.size();
  out.q.resize(c.size());
  check_dropin(cva_srv_transform_host(raw(c.nodes.data()), (int64_t)c.size(), 0, raw(out.q.data())));
  return out;
}

SrvCurve srv_center(const SrvCurve& q) {
  if (q.q.empty()) throw std::invalid_argument("srv: empty");
  SrvCurve out;
  out.h = q.h;
  out.q.resize(q.size());
  check_dropin(cva_center_or_normalize_host(raw(q.q.data()), (int64_t)q.size(), 1, raw(out.q.data())));
  return out;
}

std::vector<RigidAlignment> srv_align_batch(const std::vector<Curve>& c1, const std::vector<Curve>& c2) {
  if (c1.size() != c2.size()) throw std::invalid_argument("srv: pair count mismatch");
  if (c1.empty()) return {};
  const std::size_t n = c1[0].size();
  std::vector<Point2> a, b;
  for (std::size_t p = 0; p < c1.size(); ++p) {
    validate_curve(c1[p], 8);
    validate_curve(c2[p], 8);
    if (c1[p].size() != n || c2[p].size() != n) throw std::invalid_argument("srv: size mismatch");
    a.insert(a.end(), c1[p].nodes.begin(), c1[p].nodes.end());
    b.insert(b.end(), c2[p].nodes.begin(), c2[p].nodes.end());
  }
  std::vector<cva_alignment> rec(c1.size());
  check(cva_srv_align_batch_host(raw(a.data()), raw(b.data()), (int64_t)c1.size(), (int64_t)n, rec.data(), nullptr));
  std::vector<RigidAlignment> out;
  for (const auto& r : rec) {
    if (r.status != CVA_OK) throw std::invalid_argument("srv: invalid pair");
    RigidAlignment x;
    x.shift = (std::size_t)r.shift;
    x.t0 = r.t0;
    x.rotation = Rotation2(r.theta);
    x.trace = r.trace;
    x.energy = r.energy;
    x.degenerate = r.degenerate != 0;
    out.push_back(x);
  }
  return out;
}

// ---- reparameterisations (srv.cpp:39-69)

double Reparameterization::eval(double t) const {
  const std::size_t n = grid_size();
  if (n == 0) throw std::invalid_argument("reparam: empty");
  if (t <= 0.0) return gamma.front();
  if (t >= 1.0) return gamma.back();
  const double x = t * static_cast<double>(n);
  const std::size_t i = std::min(static_cast<std::size_t>(x), n - 1);
  const double frac = x - static_cast<double>(i);
  return gamma[i] + frac * (gamma[i + 1] - gamma[i]);
}

Reparameterization identity_reparam(std::size_t n) {
  Reparameterization g;
  g.gamma.resize(n + 1);
  for (std::size_t i = 0; i <= n; ++i) g.gamma[i] = static_cast<double>(i) / static_cast<double>(n);
  g.gamma[n] = 1.0;
  return g;
}

void validate_reparam(const Reparameterization& g) {
  const std::size_t n = g.grid_size();
  if (n < 2) throw std::invalid_argument("reparam: too few samples");
  if (std::abs(g.gamma.front()) > 1e-12 || std::abs(g.gamma.back() - 1.0) > 1e-12)
    throw std::invalid_argument("reparam: endpoints must be 0 and 1");
  for (std::size_t i = 0; i < n; ++i)
    if (g.gamma[i + 1] < g.gamma[i] - 1e-12) throw std::invalid_argument("reparam: not monotone");
}

// ---- action, energy, DP (GPU)

SrvCurve apply_srv_action(const SrvCurve& q, double t0, const Rotation2& rotation, const Reparameterization& gamma) {
  const std::size_t n = q.size();
  if (n == 0) throw std::invalid_argument("srv: empty");
  if (gamma.grid_size() != n) throw std::invalid_argument("srv: grid size mismatch");
  validate_reparam(gamma);
  SrvCurve out;
  out.h = q.h;
  out.q.resize(n);
  check_dropin(cva_apply_srv_action_host(raw(q.q.data()), (int64_t)n, t0, rotation.theta(), gamma.gamma.data(),
                                         raw(out.q.data())));
  return out;
}

double elastic_energy(const SrvCurve& q1, const SrvCurve& q2, double t0, const Rotation2& rotation,
                      const Reparameterization& gamma) {
  if (q1.size() != q2.size()) throw std::invalid_argument("srv: size mismatch");
  if (q2.size() == 0) throw std::invalid_argument("srv: empty");
  if (gamma.grid_size() != q2.size()) throw std::invalid_argument("srv: grid size mismatch");
  validate_reparam(gamma);
  double e = 0.0;
  check_dropin(cva_elastic_energy_host(raw(q1.q.data()), raw(q2.q.data()), (int64_t)q1.size(), t0, rotation.theta(),
                                       gamma.gamma.data(), &e));
  return e;
}

std::vector<std::pair<int, int>> dp_admissible_steps(int max_slope) {
  if (max_slope < 1) throw std::invalid_argument("dp: max_slope must be >= 1");
  std::vector<std::pair<int, int>> steps;
  for (int a = 1; a <= max_slope; ++a)
    for (int b = 1; b <= max_slope; ++b)
      if (std::gcd(a, b) == 1) steps.emplace_back(a, b);
  return steps;
}

double dp_step_cost(const SrvCurve& q1, const SrvCurve& q2, int i0, int j0, int di, int dj) {
  if (q1.size() != q2.size()) throw std::invalid_argument("dp: size mismatch");
  if (di < 1 || dj < 1) throw std::invalid_argument("dp: step increments must be positive");
  double c = 0.0;
  check_dropin(cva_dp_step_cost_host(raw(q1.q.data()), raw(q2.q.data()), (int64_t)q1.size(), i0, j0, di, dj, &c));
  return c;
}

std::vector<DpResult> dp_reparam_batch(const std::vector<SrvCurve>& q1, const std::vector<SrvCurve>& q2,
                                       int max_slope) {
  if (q1.size() != q2.size()) throw std::invalid_argument("dp: pair count mismatch");
  if (q1.empty()) return {};
  const std::size_t n = q1[0].size();
  std::vector<Point2> a, b;
  for (std::size_t p = 0; p < q1.size(); ++p) {
    if (q1[p].size() != q2[p].size()) throw std::invalid_argument("dp: size mismatch");
    if (q1[p].size() != n) throw std::invalid_argument("dp: batch pairs must share one size");
    a.insert(a.end(), q1[p].q.begin(), q1[p].q.end());
    b.insert(b.end(), q2[p].q.begin(), q2[p].q.end());
  }
  if (n < 8) throw std::invalid_argument("dp: need at least 8 samples");  // srv.cpp:183
  dp_admissible_steps(max_slope);                                          // validates max_slope
  std::vector<double> g(q1.size() * (n + 1)), e(q1.size());
  std::vector<int32_t> st(q1.size());
  check(cva_dp_reparam_batch_host(raw(a.data()), raw(b.data()), (int64_t)q1.size(), (int64_t)n, max_slope, g.data(),
                                  e.data(), st.data()));
  std::vector<DpResult> out(q1.size());
  for (std::size_t p = 0; p < q1.size(); ++p) {
    if (st[p] != CVA_OK) throw std::runtime_error("dp: no admissible path");  // srv.cpp:233
    out[p].gamma.gamma.assign(g.begin() + p * (n + 1), g.begin() + (p + 1) * (n + 1));
    out[p].energy = e[p];
  }
  return out;
}

DpResult dp_reparam(const SrvCurve& q1, const SrvCurve& q2, int max_slope) {
  if (q1.size() != q2.size()) throw std::invalid_argument("dp: size mismatch");
  return dp_reparam_batch({q1}, {q2}, max_slope)[0];
}

}  // namespace curvalign
