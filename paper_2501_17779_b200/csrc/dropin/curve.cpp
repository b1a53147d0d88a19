// curvalign curve core on the GPU (reference: proj/src/curve.cpp).
#include "curvalign/curve.hpp"

#include <stdexcept>

#include "status.hpp"

namespace curvalign {

using detail::check;
using detail::check_dropin;
using detail::raw;

// curve.cpp:10-15 (argument validation stays on the host so the same
// exceptions are thrown before any device work)
void validate_curve(const Curve& c, std::size_t min_nodes) {
  if (c.size() < min_nodes) throw std::invalid_argument("curve: too few nodes");
  for (const Point2& p : c.nodes)
    if (!p.finite()) throw std::invalid_argument("curve: non-finite node");
}

double curve_length(const Curve& c) {
  validate_curve(c);
  double len = 0.0;
  check_dropin(cva_curve_stats_host(raw(c.nodes.data()), (int64_t)c.size(), nullptr, &len));
  return len;
}

Point2 centroid(const Curve& c) {
  validate_curve(c);
  Point2 g;
  check_dropin(cva_curve_stats_host(raw(c.nodes.data()), (int64_t)c.size(), raw(&g), nullptr));
  return g;
}

Curve center_curve(const Curve& c) {
  validate_curve(c);
  Curve out;
  out.nodes.resize(c.size());
  check_dropin(cva_center_or_normalize_host(raw(c.nodes.data()), (int64_t)c.size(), 1, raw(out.nodes.data())));
  return out;
}

Curve normalize_length(const Curve& c) {
  validate_curve(c);
  Curve out;
  out.nodes.resize(c.size());
  check_dropin(cva_center_or_normalize_host(raw(c.nodes.data()), (int64_t)c.size(), 2, raw(out.nodes.data())));
  return out;
}

ArcLengthParams arc_length_params(const Curve& c) {
  validate_curve(c);
  ArcLengthParams ap;
  ap.s.resize(c.size() + 1);
  check_dropin(cva_arc_length_params_host(raw(c.nodes.data()), (int64_t)c.size(), ap.s.data(), &ap.total_length));
  return ap;
}

Curve resample_uniform(const Curve& c, std::size_t n_out) {
  validate_curve(c, 4);
  if (n_out < 8) throw std::invalid_argument("resample: need at least 8 output nodes");
  const int64_t offs[2] = {0, (int64_t)c.size()};
  Curve out;
  out.nodes.resize(n_out);
  int32_t st = 0;
  check(cva_resample_batch_host(raw(c.nodes.data()), offs, 1, (int64_t)n_out, raw(out.nodes.data()), &st));
  if (st != CVA_OK) throw std::invalid_argument("curve: coincident adjacent nodes");
  return out;
}

std::vector<Curve> preprocess_batch(const std::vector<Curve>& curves, std::size_t n_out, bool resample) {
  std::vector<int64_t> offs(curves.size() + 1, 0);
  for (std::size_t i = 0; i < curves.size(); ++i) {
    validate_curve(curves[i], resample ? 4 : 3);
    offs[i + 1] = offs[i] + (int64_t)curves[i].size();
  }
  if (resample && n_out < 8) throw std::invalid_argument("resample: need at least 8 output nodes");
  std::vector<Point2> pts;
  pts.reserve((std::size_t)offs.back());
  for (const Curve& c : curves) pts.insert(pts.end(), c.nodes.begin(), c.nodes.end());
  std::vector<Point2> out(resample ? curves.size() * n_out : pts.size());
  std::vector<int32_t> st(curves.size(), 0);
  if (!curves.empty())
    check(cva_preprocess_batch_host(raw(pts.data()), offs.data(), (int64_t)curves.size(), (int64_t)n_out,
                                    resample ? 1 : 0, raw(out.data()), st.data()));
  std::vector<Curve> res(curves.size());
  for (std::size_t i = 0; i < curves.size(); ++i) {
    if (st[i] != CVA_OK) throw std::invalid_argument("curve: invalid input (coincident / non-finite nodes)");
    const std::size_t b = resample ? i * n_out : (std::size_t)offs[i];
    const std::size_t e = resample ? b + n_out : (std::size_t)offs[i + 1];
    res[i].nodes.assign(out.begin() + (std::ptrdiff_t)b, out.begin() + (std::ptrdiff_t)e);
  }
  return res;
}

// curve.cpp:93-97: resample (optional) -> center -> normalize, composed from the
// same GPU primitives as the individual functions so that preprocess equals
// the manual composition bit for bit (test_curve_core.cpp:215-232). Batches go
// through preprocess_batch (one fused launch).
Curve preprocess(const Curve& c, std::size_t n_out, bool resample) {
  Curve out = resample ? resample_uniform(c, n_out) : c;
  out = center_curve(out);
  return normalize_length(out);
}

}  // namespace curvalign
