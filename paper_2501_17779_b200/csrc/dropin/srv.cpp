// SRV helpers of the alignment path (reference: proj/src/srv.cpp:71-98) on the GPU.
#include "curvalign/srv.hpp"

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

}  // namespace curvalign
