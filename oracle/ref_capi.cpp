// TEST INFRASTRUCTURE ONLY — C-ABI over the reference's OWN implementation.
//
// oracle/Makefile compiles the reference sources in place
// (/root/reference/proj/src/{fft,rigid_align,curve,spline,srv,synthetic,elastic}.cpp,
// unmodified, never copied) together with this file and the FFTW/Eigen shims
// into oracle/_ref/libcurvalign_ref.so. Tests use it to pin the C restatement
// (oracle/curvalign_oracle.c) and to generate golden vectors; bench.py uses it
// as the CPU baseline ("kind": "reference"). Nothing in the product links it.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <new>
#include <numbers>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "curvalign/curve.hpp"
#include "curvalign/elastic.hpp"
#include "curvalign/fft.hpp"
#include "curvalign/io.hpp"
#include "curvalign/rigid_align.hpp"
#include "curvalign/spline.hpp"
#include "curvalign/srv.hpp"
#include "curvalign/synthetic.hpp"

using namespace curvalign;

extern "C" {

// Layout shared with include/curvalign_cuda.h (cva_alignment).
struct ref_alignment {
  int64_t shift;
  double t0;
  double theta;
  double trace;
  double energy;
  int32_t degenerate;
  int32_t status;
};

}  // extern "C"

namespace {

enum { kOk = 0, kInvalid = 1, kRuntime = 2, kBadAlloc = 3, kOther = 4 };

template <typename F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const std::invalid_argument&) {
    return kInvalid;
  } catch (const std::bad_alloc&) {
    return kBadAlloc;
  } catch (const std::runtime_error&) {
    return kRuntime;
  } catch (...) {
    return kOther;
  }
}

Curve to_curve(const double* xy, int64_t n) {
  Curve c;
  c.nodes.resize(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) c.nodes[i] = Point2(xy[2 * i], xy[2 * i + 1]);
  return c;
}

std::vector<Point2> to_points(const double* xy, int64_t n) { return to_curve(xy, n).nodes; }

void from_points(const std::vector<Point2>& p, double* out) {
  for (std::size_t i = 0; i < p.size(); ++i) {
    out[2 * i] = p[i].x;
    out[2 * i + 1] = p[i].y;
  }
}

void fill(const RigidAlignment& a, ref_alignment* out) {
  out->shift = static_cast<int64_t>(a.shift);
  out->t0 = a.t0;
  out->theta = a.rotation.theta();
  out->trace = a.trace;
  out->energy = a.energy;
  out->degenerate = a.degenerate ? 1 : 0;
  out->status = 0;
}

// aligned[l] = R(theta).apply(c2[(l + shift) mod N])  (proj/src/elastic.cpp:80 pattern)
void aligned_curve(std::span<const Point2> c2, const RigidAlignment& a, double* out) {
  const std::size_t n = c2.size();
  for (std::size_t l = 0; l < n; ++l) {
    const Point2 p = a.rotation.apply(c2[(l + a.shift) % n]);
    out[2 * l] = p.x;
    out[2 * l + 1] = p.y;
  }
}

// Atomic-counter pool over work items: the pattern of proj/src/elastic.cpp:196-234.
void parallel_for(int64_t count, int threads, const std::function<void(int64_t)>& body) {
  if (threads <= 1 || count <= 1) {
    for (int64_t i = 0; i < count; ++i) body(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  const int t = static_cast<int>(std::min<int64_t>(threads, count));
  pool.reserve(static_cast<std::size_t>(t));
  for (int k = 0; k < t; ++k) {
    pool.emplace_back([&]() {
      for (int64_t i = next.fetch_add(1); i < count; i = next.fetch_add(1)) body(i);
    });
  }
  for (auto& th : pool) th.join();
}

std::function<double(double)> warp_fn(int kind, double u) {
  switch (kind) {
    case 1: return gamma1_warp;
    case 2: return gamma2_warp;
    case 3:  // C4 warp: t + 0.05 u sin(2 pi t)
      return [u](double t) { return t + 0.05 * u * std::sin(2.0 * std::numbers::pi * t); };
    default: return nullptr;
  }
}

}  // namespace

extern "C" {

int ref_align_fft(const double* c1, const double* c2, int64_t n, ref_alignment* out) {
  return guard([&] { fill(align_fft(to_points(c1, n), to_points(c2, n)), out); });
}

int ref_align_naive(const double* c1, const double* c2, int64_t n, ref_alignment* out) {
  return guard([&] { fill(align_naive(to_points(c1, n), to_points(c2, n)), out); });
}

int ref_align_fft_n(const double* c1, int64_t n1, const double* c2, int64_t n2,
                    ref_alignment* out) {
  return guard([&] { fill(align_fft(to_points(c1, n1), to_points(c2, n2)), out); });
}

// Mat2 stack, row-major per shift: out[4m + {0,1,2,3}] = a11, a12, a21, a22.
int ref_correlation_all_shifts(const double* c1, const double* c2, int64_t n, int use_fft,
                               double* out) {
  return guard([&] {
    const auto p1 = to_points(c1, n), p2 = to_points(c2, n);
    const auto st = use_fft ? correlation_all_shifts_fft(p1, p2) : correlation_all_shifts_naive(p1, p2);
    for (std::size_t m = 0; m < st.size(); ++m) {
      out[4 * m] = st[m].a11;
      out[4 * m + 1] = st[m].a12;
      out[4 * m + 2] = st[m].a21;
      out[4 * m + 3] = st[m].a22;
    }
  });
}

int ref_cross_correlation_matrix(const double* c1, const double* c2, int64_t n, int64_t shift,
                                 double* out4) {
  return guard([&] {
    const Mat2 a = cross_correlation_matrix(to_points(c1, n), to_points(c2, n),
                                            static_cast<std::size_t>(shift));
    out4[0] = a.a11;
    out4[1] = a.a12;
    out4[2] = a.a21;
    out4[3] = a.a22;
  });
}

int ref_optimal_rotation(const double* a4, int use_svd, double* theta, double* trace,
                         int32_t* degenerate) {
  return guard([&] {
    const Mat2 a{a4[0], a4[1], a4[2], a4[3]};
    const RotationFit f = use_svd ? optimal_rotation_svd(a) : optimal_rotation_closed_form(a);
    *theta = f.rotation.theta();
    *trace = f.trace;
    *degenerate = f.degenerate ? 1 : 0;
  });
}

int ref_mismatch_energy(const double* c1, const double* c2, int64_t n, int64_t shift,
                        double theta, double* out) {
  return guard([&] {
    *out = mismatch_energy(to_points(c1, n), to_points(c2, n), static_cast<std::size_t>(shift),
                           Rotation2(theta));
  });
}

int ref_arc_length_params(const double* xy, int64_t n, double* s_out, double* total) {
  return guard([&] {
    const ArcLengthParams ap = arc_length_params(to_curve(xy, n));
    std::memcpy(s_out, ap.s.data(), sizeof(double) * ap.s.size());
    *total = ap.total_length;
  });
}

int ref_curve_length(const double* xy, int64_t n, double* out) {
  return guard([&] { *out = curve_length(to_curve(xy, n)); });
}

int ref_centroid(const double* xy, int64_t n, double* out2) {
  return guard([&] {
    const Point2 g = centroid(to_curve(xy, n));
    out2[0] = g.x;
    out2[1] = g.y;
  });
}

int ref_center_curve(const double* xy, int64_t n, double* out) {
  return guard([&] { from_points(center_curve(to_curve(xy, n)).nodes, out); });
}

int ref_normalize_length(const double* xy, int64_t n, double* out) {
  return guard([&] { from_points(normalize_length(to_curve(xy, n)).nodes, out); });
}

int ref_resample_uniform(const double* xy, int64_t n, int64_t n_out, double* out) {
  return guard([&] {
    from_points(resample_uniform(to_curve(xy, n), static_cast<std::size_t>(n_out)).nodes, out);
  });
}

int ref_preprocess(const double* xy, int64_t n, int64_t n_out, int resample, double* out) {
  return guard([&] {
    from_points(preprocess(to_curve(xy, n), static_cast<std::size_t>(n_out), resample != 0).nodes,
                out);
  });
}

int ref_spline_eval(const double* x, const double* y, int64_t n_knots, const double* xq,
                    int64_t nq, int derivative, double* out) {
  return guard([&] {
    const PeriodicCubicSpline s(std::span<const double>(x, static_cast<std::size_t>(n_knots)),
                                std::span<const double>(y, static_cast<std::size_t>(n_knots)));
    for (int64_t i = 0; i < nq; ++i) out[i] = derivative ? s.derivative(xq[i]) : s.eval(xq[i]);
  });
}

int ref_srv_transform(const double* xy, int64_t n, double* q_out, double* h) {
  return guard([&] {
    const SrvCurve q = srv_transform(to_curve(xy, n));
    from_points(q.q, q_out);
    *h = q.h;
  });
}

int ref_srv_center(const double* q, int64_t n, double* out) {
  return guard([&] {
    SrvCurve s;
    s.q = to_points(q, n);
    s.h = n ? 1.0 / static_cast<double>(n) : 0.0;
    from_points(srv_center(s).q, out);
  });
}

int ref_real_dft(const double* in, int64_t n, double* out_complex) {
  return guard([&] {
    const auto spec = real_dft(std::span<const double>(in, static_cast<std::size_t>(n)));
    for (std::size_t k = 0; k < spec.size(); ++k) {
      out_complex[2 * k] = spec[k].real();
      out_complex[2 * k + 1] = spec[k].imag();
    }
  });
}

int ref_real_idft(const double* spec_complex, int64_t n_bins, int64_t n, double* out) {
  return guard([&] {
    std::vector<std::complex<double>> spec(static_cast<std::size_t>(n_bins));
    for (int64_t k = 0; k < n_bins; ++k) spec[k] = {spec_complex[2 * k], spec_complex[2 * k + 1]};
    const auto r = real_idft(spec, static_cast<std::size_t>(n));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

int ref_circular_cross_correlation(const double* a, int64_t na, const double* b, int64_t nb,
                                   double* out) {
  return guard([&] {
    const auto r = circular_cross_correlation(std::span<const double>(a, static_cast<std::size_t>(na)),
                                              std::span<const double>(b, static_cast<std::size_t>(nb)));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

int ref_gen_curve(int family, int64_t n, uint64_t seed, int harmonics, double* out) {
  return guard([&] {
    from_points(gen_curve(static_cast<CurveFamily>(family), static_cast<std::size_t>(n), seed,
                          harmonics)
                    .nodes,
                out);
  });
}

// warp_kind: 0 none, 1 gamma1, 2 gamma2, 3 t + 0.05 u sin(2 pi t)
int ref_transform_curve(const double* xy, int64_t n, double start_shift, double theta,
                        int warp_kind, double u, double* out) {
  return guard([&] {
    from_points(transform_curve(to_curve(xy, n), start_shift, theta, warp_fn(warp_kind, u)).nodes,
                out);
  });
}

// ---- batched drivers (CPU baseline / golden generation) -------------------

// Pair p aligns curve 2p against curve 2p+1 of a ragged point array:
// curve c occupies points [offsets[c], offsets[c+1]). mode 0: preprocess(raw, n_out,
// resample) both, then align_fft. mode 1: inputs already uniform (align_fft only).
// mode 2: SRV: align_fft(srv_center(srv_transform(c1)).q, srv_center(srv_transform(c2)).q).
// aligned (nullable): pairs * n_out points, R.apply(c2'[(l+k) mod N]).
int ref_batch(const double* points, const int64_t* offsets, int64_t pairs, int64_t n_out,
              int resample, int mode, int threads, ref_alignment* out, double* aligned) {
  std::atomic<int> first_err{0};
  parallel_for(pairs, threads, [&](int64_t p) {
    const int64_t a0 = offsets[2 * p], a1 = offsets[2 * p + 1], b1 = offsets[2 * p + 2];
    const int rc = guard([&] {
      const Curve ra = to_curve(points + 2 * a0, a1 - a0);
      const Curve rb = to_curve(points + 2 * a1, b1 - a1);
      std::vector<Point2> u, v;
      if (mode == 0) {
        u = preprocess(ra, static_cast<std::size_t>(n_out), resample != 0).nodes;
        v = preprocess(rb, static_cast<std::size_t>(n_out), resample != 0).nodes;
      } else if (mode == 1) {
        u = ra.nodes;
        v = rb.nodes;
      } else {
        u = srv_center(srv_transform(ra)).q;
        v = srv_center(srv_transform(rb)).q;
      }
      const RigidAlignment a = align_fft(u, v);
      fill(a, &out[p]);
      if (aligned) aligned_curve(v, a, aligned + 2 * p * static_cast<int64_t>(v.size()));
    });
    if (rc != kOk) {
      out[p] = ref_alignment{0, 0.0, std::nan(""), std::nan(""), std::nan(""), 0, rc};
      int expected = 0;
      first_err.compare_exchange_strong(expected, rc);
    }
  });
  return first_err.load();
}

// All ordered pairs of M uniform (preprocessed) curves of N nodes, rows
// [row_begin, row_end): energy/shift/theta matrices of (row_end-row_begin) x M.
int ref_allpairs(const double* curves, int64_t m, int64_t n, int64_t row_begin, int64_t row_end,
                 int threads, double* energy, int64_t* shift, double* theta) {
  std::atomic<int> first_err{0};
  const int64_t rows = row_end - row_begin;
  parallel_for(rows * m, threads, [&](int64_t cell) {
    const int64_t i = row_begin + cell / m, j = cell % m;
    const int rc = guard([&] {
      const RigidAlignment a =
          align_fft(std::span<const Point2>(reinterpret_cast<const Point2*>(curves) + i * n, n),
                    std::span<const Point2>(reinterpret_cast<const Point2*>(curves) + j * n, n));
      energy[cell] = a.energy;
      shift[cell] = static_cast<int64_t>(a.shift);
      theta[cell] = a.rotation.theta();
    });
    if (rc != kOk) {
      energy[cell] = std::nan("");
      int expected = 0;
      first_err.compare_exchange_strong(expected, rc);
    }
  });
  return first_err.load();
}

// ---- elastic (SRV) matching: the path's callers --

SrvCurve to_srv(const double* q, int64_t n) {
  SrvCurve s;
  s.q = to_points(q, n);
  s.h = n ? 1.0 / static_cast<double>(n) : 0.0;
  return s;
}

Reparameterization to_reparam(const double* g, int64_t n) {
  Reparameterization r;
  r.gamma.assign(g, g + n + 1);
  return r;
}

int ref_apply_srv_action(const double* q, int64_t n, double t0, double theta, const double* gamma,
                         double* out) {
  return guard([&] { from_points(apply_srv_action(to_srv(q, n), t0, Rotation2(theta), to_reparam(gamma, n)).q, out); });
}

int ref_elastic_energy(const double* q1, const double* q2, int64_t n, double t0, double theta,
                       const double* gamma, double* out) {
  return guard([&] { *out = elastic_energy(to_srv(q1, n), to_srv(q2, n), t0, Rotation2(theta), to_reparam(gamma, n)); });
}

int ref_dp_step_cost(const double* q1, const double* q2, int64_t n, int i0, int j0, int di, int dj,
                     double* out) {
  return guard([&] { *out = dp_step_cost(to_srv(q1, n), to_srv(q2, n), i0, j0, di, dj); });
}

// pairs x n SRV samples each; gamma_out pairs x (n+1).
int ref_dp_reparam_batch(const double* q1, const double* q2, int64_t pairs, int64_t n, int max_slope,
                         int threads, double* gamma_out, double* energy_out, int32_t* status) {
  std::atomic<int> first_err{0};
  parallel_for(pairs, threads, [&](int64_t p) {
    const int rc = guard([&] {
      const DpResult r = dp_reparam(to_srv(q1 + 2 * p * n, n), to_srv(q2 + 2 * p * n, n), max_slope);
      std::memcpy(gamma_out + p * (n + 1), r.gamma.gamma.data(), sizeof(double) * (n + 1));
      energy_out[p] = r.energy;
    });
    status[p] = rc;
    if (rc != kOk) {
      energy_out[p] = std::nan("");
      int expected = 0;
      first_err.compare_exchange_strong(expected, rc);
    }
  });
  return first_err.load();
}

// elastic_distance_approach2 (proj/src/elastic.cpp:102-174) on pairs of
// preprocessed curves (pairs x n points each). gamma_out (nullable) pairs x (n+1).
int ref_elastic_approach2_batch(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                int max_iters, double energy_tol, int use_fft, int max_slope,
                                int threads, double* distance, double* energy, double* t0,
                                double* theta, double* gamma_out, int32_t* iterations,
                                int32_t* converged, int32_t* status, double* trace) {
  ElasticOptions o;
  o.max_iters = max_iters;
  o.energy_tol = energy_tol;
  o.use_fft = use_fft != 0;
  o.max_slope = max_slope;
  std::atomic<int> first_err{0};
  parallel_for(pairs, threads, [&](int64_t p) {
    const int rc = guard([&] {
      const ElasticMatch m = elastic_distance_approach2(to_curve(c1 + 2 * p * n, n), to_curve(c2 + 2 * p * n, n), o);
      distance[p] = m.distance;
      energy[p] = m.energy;
      t0[p] = m.t0;
      theta[p] = m.rotation.theta();
      if (gamma_out) std::memcpy(gamma_out + p * (n + 1), m.gamma.gamma.data(), sizeof(double) * (n + 1));
      iterations[p] = m.iterations;
      converged[p] = m.converged ? 1 : 0;
      if (trace)
        for (int k = 0; k <= max_iters; ++k)
          trace[p * (max_iters + 1) + k] =
              k < (int)m.energy_trace.size() ? m.energy_trace[(std::size_t)k] : std::nan("");
    });
    status[p] = rc;
    if (rc != kOk) {
      distance[p] = energy[p] = std::nan("");
      int expected = 0;
      first_err.compare_exchange_strong(expected, rc);
    }
  });
  return first_err.load();
}

// elastic_distance_approach1 (proj/src/elastic.cpp:62-100), same outputs.
int ref_elastic_approach1_batch(const double* c1, const double* c2, int64_t pairs, int64_t n, int max_slope,
                                int64_t n_max, int threads, double* distance, double* energy, double* t0,
                                double* theta, double* gamma_out, int32_t* iterations, int32_t* converged,
                                int32_t* status) {
  ElasticOptions o;
  o.max_slope = max_slope;
  o.n_max_approach1 = static_cast<std::size_t>(n_max);
  std::atomic<int> first_err{0};
  parallel_for(pairs, threads, [&](int64_t p) {
    const int rc = guard([&] {
      const ElasticMatch m = elastic_distance_approach1(to_curve(c1 + 2 * p * n, n), to_curve(c2 + 2 * p * n, n), o);
      distance[p] = m.distance;
      energy[p] = m.energy;
      t0[p] = m.t0;
      theta[p] = m.rotation.theta();
      if (gamma_out) std::memcpy(gamma_out + p * (n + 1), m.gamma.gamma.data(), sizeof(double) * (n + 1));
      iterations[p] = m.iterations;
      converged[p] = m.converged ? 1 : 0;
    });
    status[p] = rc;
    if (rc != kOk) {
      distance[p] = energy[p] = std::nan("");
      int expected = 0;
      first_err.compare_exchange_strong(expected, rc);
    }
  });
  return first_err.load();
}

// distance_matrix(curves, approach2, n) (proj/src/elastic.cpp:176-236): count
// raw curves of n_in nodes each (uniform size), preprocessed to n inside.
int ref_distance_matrix(const double* curves, int64_t count, int64_t n_in, int64_t n, int method,
                        int max_iters, double energy_tol, int max_slope, int threads, double* out) {
  return guard([&] {
    std::vector<Curve> cs;
    for (int64_t i = 0; i < count; ++i) cs.push_back(to_curve(curves + 2 * i * n_in, n_in));
    ElasticOptions o;
    o.max_iters = max_iters;
    o.energy_tol = energy_tol;
    o.max_slope = max_slope;
    const auto d = distance_matrix(cs, method == 1 ? DistanceMethod::approach1 : DistanceMethod::approach2,
                                   static_cast<std::size_t>(n), o, static_cast<unsigned>(threads));
    for (int64_t i = 0; i < count; ++i)
      for (int64_t j = 0; j < count; ++j) out[i * count + j] = d[i][j];
  });
}

// ---- file formats (proj/src/io.cpp): strings returned through (buf, cap) ----

static int put(const std::string& v, char* buf, int64_t cap, int64_t* len) {
  *len = (int64_t)v.size();
  if ((int64_t)v.size() + 1 > cap) return kOther;
  std::memcpy(buf, v.c_str(), v.size() + 1);
  return kOk;
}

int ref_load_curve(const char* path, double* out, int64_t cap_nodes, int64_t* n) {
  return guard([&] {
    const Curve c = load_curve(path);
    *n = (int64_t)c.size();
    if ((int64_t)c.size() > cap_nodes) throw std::runtime_error("capacity");
    from_points(c.nodes, out);
  });
}

int ref_curve_to_csv(const double* xy, int64_t n, char* buf, int64_t cap, int64_t* len) {
  int rc = kOk;
  const int g = guard([&] { rc = put(curve_to_csv(to_curve(xy, n)), buf, cap, len); });
  return g ? g : rc;
}

int ref_curve_to_json(const double* xy, int64_t n, char* buf, int64_t cap, int64_t* len) {
  int rc = kOk;
  const int g = guard([&] { rc = put(curve_to_json(to_curve(xy, n)), buf, cap, len); });
  return g ? g : rc;
}

int ref_write_curve(const char* path, const double* xy, int64_t n, int json) {
  return guard([&] { json ? write_curve_json(path, to_curve(xy, n)) : write_curve_csv(path, to_curve(xy, n)); });
}

int ref_alignment_to_json(const ref_alignment* a, char* buf, int64_t cap, int64_t* len) {
  int rc = kOk;
  const int g = guard([&] {
    RigidAlignment r;
    r.shift = (std::size_t)a->shift;
    r.t0 = a->t0;
    r.rotation = Rotation2(a->theta);
    r.trace = a->trace;
    r.energy = a->energy;
    r.degenerate = a->degenerate != 0;
    rc = put(alignment_to_json(r), buf, cap, len);
  });
  return g ? g : rc;
}

int ref_elastic_to_json(double t0, double theta, const double* gamma, int64_t n_gamma, double distance,
                        int iterations, int converged, char* buf, int64_t cap, int64_t* len) {
  int rc = kOk;
  const int g = guard([&] {
    ElasticMatch m;
    m.t0 = t0;
    m.rotation = Rotation2(theta);
    m.gamma.gamma.assign(gamma, gamma + n_gamma);
    m.distance = distance;
    m.iterations = iterations;
    m.converged = converged != 0;
    rc = put(elastic_to_json(m), buf, cap, len);
  });
  return g ? g : rc;
}

// names: k labels separated by '\n'; d: k x k row-major
int ref_matrix_to_csv(const char* names, int64_t k, const double* d, char* buf, int64_t cap, int64_t* len) {
  int rc = kOk;
  const int g = guard([&] {
    std::vector<std::string> nm;
    std::string cur;
    for (const char* p = names; *p; ++p) {
      if (*p == '\n') {
        nm.push_back(cur);
        cur.clear();
      } else {
        cur += *p;
      }
    }
    nm.push_back(cur);
    std::vector<std::vector<double>> m((std::size_t)k, std::vector<double>((std::size_t)k));
    for (int64_t i = 0; i < k; ++i)
      for (int64_t j = 0; j < k; ++j) m[(std::size_t)i][(std::size_t)j] = d[i * k + j];
    rc = put(matrix_to_csv(nm, m), buf, cap, len);
  });
  return g ? g : rc;
}

}  // extern "C"
