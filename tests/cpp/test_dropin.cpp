#include <chrono>
// C++ tests of the drop-in API (include/curvalign/*.hpp over libcurvalign_cuda.so).
// Each case restates a hot-path test of the reference's own suite
// (/root/reference/proj/tests/test_rigid_align.cpp, test_curve_core.cpp,
// test_srv.cpp, test_elastic.cpp; file:line cited per case), written against the same API so a
// reference user's code compiles unchanged. Fixture curves are generated here
// (the reference's synthetic.cpp generators are outside this library).
// Exit status = number of failed checks.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <dirent.h>
#include <sys/stat.h>
#include <unistd.h>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "curvalign/curve.hpp"
#include "curvalign/elastic.hpp"
#include "curvalign/fft.hpp"
#include "curvalign/io.hpp"
#include "curvalign/rigid_align.hpp"
#include "curvalign/spline.hpp"
#include "curvalign/srv.hpp"

using namespace curvalign;

static int g_fail = 0, g_checks = 0;
static std::string g_case;
#define CHECK(cond)                                                                  \
  do {                                                                               \
    ++g_checks;                                                                      \
    if (!(cond)) {                                                                   \
      ++g_fail;                                                                      \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                \
  } while (0)
template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}
static void run(const char* name, const std::function<void()>& f) {
  g_case = name;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL [%s] unexpected exception: %s\n", name, e.what());
  }
}

static const double kPi = 3.14159265358979323846;

static Curve polar(std::size_t n, const std::function<double(double)>& r) {
  Curve c;
  c.nodes.resize(n);
  for (std::size_t l = 0; l < n; ++l) {
    const double phi = 2.0 * kPi * (double)l / (double)n;
    c.nodes[l] = Point2(r(phi) * std::cos(phi), r(phi) * std::sin(phi));
  }
  return c;
}
static Curve limacon(std::size_t n) { return polar(n, [](double p) { return 0.75 + 0.5 * std::cos(p); }); }
static Curve circle(std::size_t n) { return polar(n, [](double) { return 1.0; }); }
static Curve bumps(std::size_t n) { return polar(n, [](double p) { return 1.0 + 0.2 * std::sin(6.0 * p); }); }
static Curve hippopede(std::size_t n) {
  return polar(n, [](double p) { return std::sqrt(4.0 * 0.9 * (1.0 - 0.9 * std::sin(p) * std::sin(p))); });
}
static Curve random_curve(std::mt19937_64& rng, std::size_t n) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  Curve c;
  c.nodes.resize(n);
  for (auto& p : c.nodes) p = Point2(u(rng), u(rng));
  return c;
}
static double wrap_angle(double t) {
  while (t > kPi) t -= 2.0 * kPi;
  while (t < -kPi) t += 2.0 * kPi;
  return t;
}
// c2[l] = rotate_ccw(c1[(l - k) mod n], th): the reference recovers shift k, angle th
static Curve shift_rotate(const Curve& c1, std::size_t k, double th) {
  const std::size_t n = c1.size();
  Curve c2;
  c2.nodes.resize(n);
  for (std::size_t l = 0; l < n; ++l) c2.nodes[l] = rotate_ccw(c1[(l + n - k) % n], th);
  return c2;
}

int main() {
  // ---------------------------------------------------------- rigid_align
  run("diamond", [] {  // test_rigid_align.cpp:47-56
    Curve c;
    c.nodes = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    const Mat2 a = cross_correlation_matrix(c.nodes, c.nodes, 1);
    CHECK(std::fabs(a.a11) < 1e-15 && std::fabs(a.a12 - 2.0) < 1e-15 && std::fabs(a.a21 + 2.0) < 1e-15 &&
          std::fabs(a.a22) < 1e-15);
  });
  run("direct double loop", [] {  // :58-70
    std::mt19937_64 rng(7);
    Curve c1 = random_curve(rng, 37), c2 = random_curve(rng, 37);
    for (std::size_t m : {0u, 1u, 13u, 36u}) {
      Mat2 want;
      for (std::size_t l = 0; l < 37; ++l) {
        const Point2 p = c1[l], q = c2[(l + m) % 37];
        want.a11 += p.x * q.x, want.a12 += p.x * q.y, want.a21 += p.y * q.x, want.a22 += p.y * q.y;
      }
      const Mat2 got = cross_correlation_matrix(c1.nodes, c2.nodes, m);
      CHECK(std::fabs(got.a11 - want.a11) < 1e-12 && std::fabs(got.a12 - want.a12) < 1e-12 &&
            std::fabs(got.a21 - want.a21) < 1e-12 && std::fabs(got.a22 - want.a22) < 1e-12);
    }
  });
  run("closed form known matrix", [] {  // :79-86
    const RotationFit f = optimal_rotation_closed_form(Mat2{0.0, 1.0, -1.0, 0.0});
    CHECK(std::fabs(f.rotation.theta() - kPi / 2) < 1e-14 && std::fabs(f.trace - 2.0) < 1e-13 && !f.degenerate);
  });
  run("svd vs closed form", [] {  // :88-100
    std::mt19937_64 rng(23);
    std::uniform_real_distribution<double> u(-2.0, 2.0);
    for (int k = 0; k < 1000; ++k) {
      const Mat2 a{u(rng), u(rng), u(rng), u(rng)};
      const RotationFit s = optimal_rotation_svd(a), c = optimal_rotation_closed_form(a);
      CHECK(std::fabs(s.trace - c.trace) < 1e-10);
      if (!s.degenerate && !c.degenerate && std::fabs(s.trace) > 1e-6)
        CHECK(std::fabs(wrap_angle(s.rotation.theta() - c.rotation.theta())) < 1e-8);
    }
  });
  run("degenerate", [] {  // :102-108
    CHECK(optimal_rotation_svd(Mat2{}).degenerate);
    CHECK(optimal_rotation_closed_form(Mat2{}).degenerate);
  });
  run("fixed start rotation", [] {  // :125-131
    Curve c1 = bumps(128), c2 = c1;
    for (auto& p : c2.nodes) p = rotate_ccw(p, kPi / 3.0);
    CHECK(std::fabs(optimal_rotation_fixed_start(c1, c2).theta() - kPi / 3.0) < 1e-10);
  });
  run("naive == fft stacks", [] {  // :133-151
    std::mt19937_64 rng(43);
    // naive: exact per-shift sums; fft: two forward + two inverse GPU FFTs
    // (radix 2 for powers of two, Bluestein otherwise): two computations
    for (std::size_t n : {4u, 5u, 8u, 20u, 37u, 64u, 101u, 1000u, 4097u}) {
      Curve c1 = random_curve(rng, n), c2 = random_curve(rng, n);
      const auto a = correlation_all_shifts_naive(c1.nodes, c2.nodes);
      const auto b = correlation_all_shifts_fft(c1.nodes, c2.nodes);
      CHECK(a.size() == n && b.size() == n);
      for (std::size_t m = 0; m < n; ++m)
        CHECK(std::fabs(a[m].a11 - b[m].a11) < 1e-9 * n && std::fabs(a[m].a22 - b[m].a22) < 1e-9 * n &&
              std::fabs(a[m].a12 - b[m].a12) < 1e-9 * n && std::fabs(a[m].a21 - b[m].a21) < 1e-9 * n);
      const RigidAlignment f = align_fft(c1, c2), g = align_naive(c1, c2);
      CHECK(f.shift == g.shift && std::fabs(f.energy - g.energy) < 1e-9);
    }
  });
  run("fft stack at n = 65536 is O(n log n)", [] {
    std::mt19937_64 rng(44);
    const std::size_t n = 65536;
    Curve c1 = random_curve(rng, n), c2 = random_curve(rng, n);
    (void)correlation_all_shifts_fft(c1.nodes, c2.nodes);  // first call: context, workspace
    const auto t0 = std::chrono::steady_clock::now();
    const auto b = correlation_all_shifts_fft(c1.nodes, c2.nodes);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::printf("    correlation_all_shifts_fft(65536): %.2f ms\n", ms);
    CHECK(ms < 100.0);
    for (std::size_t m : {0u, 1u, 777u, 32768u, 65535u}) {
      const Mat2 a = cross_correlation_matrix(c1.nodes, c2.nodes, m);
      CHECK(std::fabs(a.a11 - b[m].a11) < 1e-9 * n && std::fabs(a.a12 - b[m].a12) < 1e-9 * n &&
            std::fabs(a.a21 - b[m].a21) < 1e-9 * n && std::fabs(a.a22 - b[m].a22) < 1e-9 * n);
    }
  });
  run("exact cyclic shift", [] {  // :153-168
    Curve c1 = limacon(96), c2;
    c2.nodes.resize(96);
    for (std::size_t l = 0; l < 96; ++l) c2.nodes[(l + 29) % 96] = c1[l];
    const RigidAlignment a = align_fft(c1, c2);
    CHECK(a.shift == 29 && std::fabs(a.rotation.theta()) < 1e-9 && a.energy < 1e-15);
    const RigidAlignment b = align_naive(c1, c2);
    CHECK(b.shift == a.shift);
  });
  run("circle tie -> shift 0", [] {  // :170-176
    Curve c = circle(64);
    const RigidAlignment a = align_fft(c, c);
    CHECK(a.shift == 0 && std::fabs(a.rotation.theta()) < 1e-9 && a.energy < 1e-12);
  });
  run("shift and rotation recovered", [] {  // :178-185 (fixture built by cyclic shift + rotation)
    Curve c1 = polar(256, [](double p) { return 1.0 + 0.2 * std::cos(3 * p + 0.4) + 0.1 * std::sin(5 * p); });
    Curve c2 = shift_rotate(c1, 64, kPi / 3.0);
    const RigidAlignment a = align_fft(c1, c2);
    CHECK(std::fabs(a.t0 - 0.25) < 1e-12 && std::fabs(a.rotation.theta() - kPi / 3.0) < 1e-9 && a.energy < 1e-12);
  });
  run("energy identity", [] {  // :187-197
    std::mt19937_64 rng(57);
    Curve c1 = random_curve(rng, 48), c2 = random_curve(rng, 48);
    const RigidAlignment a = align_naive(c1, c2);
    const double direct = mismatch_energy(c1.nodes, c2.nodes, a.shift, a.rotation);
    CHECK(std::fabs(a.energy - direct) <= 1e-9 * std::fabs(direct));
  });
  run("optimum beats random candidates", [] {  // :199-210
    std::mt19937_64 rng(61);
    Curve c1 = random_curve(rng, 40), c2 = random_curve(rng, 40);
    const RigidAlignment a = align_naive(c1, c2);
    std::uniform_real_distribution<double> ang(-kPi, kPi);
    std::uniform_int_distribution<std::size_t> sh(0, 39);
    for (int k = 0; k < 100; ++k) CHECK(a.energy <= mismatch_energy(c1.nodes, c2.nodes, sh(rng), Rotation2(ang(rng))) + 1e-12);
  });
  run("rotation covariance", [] {  // :212-220
    Curve c1 = hippopede(128), c2 = c1;
    for (auto& p : c2.nodes) p = rotate_ccw(p, 0.4);
    const RigidAlignment base = align_fft(c1, c1), rot = align_fft(c1, c2);
    CHECK(rot.shift == base.shift && std::fabs(wrap_angle(rot.rotation.theta() - base.rotation.theta()) - 0.4) < 1e-8);
  });
  run("shift covariance", [] {  // :222-235
    std::mt19937_64 rng(71);
    Curve c1 = random_curve(rng, 60), c2 = random_curve(rng, 60), c2s;
    const RigidAlignment base = align_naive(c1, c2);
    c2s.nodes.resize(60);
    for (std::size_t l = 0; l < 60; ++l) c2s.nodes[l] = c2[(l + 17) % 60];
    const RigidAlignment s = align_naive(c1, c2s);
    CHECK(s.shift == (base.shift + 60 - 17) % 60 && std::fabs(s.rotation.theta() - base.rotation.theta()) < 1e-10 &&
          std::fabs(s.energy - base.energy) <= 1e-10 * base.energy);
  });
  run("reflection", [] {  // :237-246
    Curve c1 = limacon(128), c2 = c1;
    for (auto& p : c2.nodes) p.y = -p.y;
    const RigidAlignment a = align_fft(c1, c2);
    const Mat2 r = a.rotation.matrix();
    CHECK(std::fabs(r.a11 * r.a22 - r.a12 * r.a21 - 1.0) < 1e-12 && a.energy > 1e-6);
  });
  run("validation", [] {  // :248-257
    Curve c1 = circle(32), c2 = circle(64), tiny;
    tiny.nodes = {{0, 0}, {1, 0}, {0, 1}};
    CHECK(throws<std::invalid_argument>([&] { align_fft(c1, c2); }));
    CHECK(throws<std::invalid_argument>([&] { cross_correlation_matrix(c1.nodes, c2.nodes, 0); }));
    CHECK(throws<std::invalid_argument>([&] { cross_correlation_matrix(c1.nodes, c1.nodes, 32); }));
    CHECK(throws<std::invalid_argument>([&] { align_fft(tiny, tiny); }));
  });

  // ----------------------------------------------------------- curve core
  run("curve_length", [] {  // test_curve_core.cpp:73-84
    Curve sq;
    sq.nodes = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    CHECK(std::fabs(curve_length(sq) - 4.0) < 1e-15);
    CHECK(std::fabs(curve_length(circle(256)) - 512.0 * std::sin(kPi / 256.0)) < 1e-12);
  });
  run("centroid / center", [] {  // :86-104
    Curve c;
    c.nodes = {{0, 0}, {2, 0}, {2, 2}, {0, 2}};
    const Point2 g = centroid(c);
    CHECK(std::fabs(g.x - 1.0) < 1e-15 && std::fabs(g.y - 1.0) < 1e-15);
    const Curve ce = center_curve(c);
    CHECK(std::fabs(ce[0].x + 1.0) < 1e-15 && std::fabs(ce[2].y - 1.0) < 1e-15);
    const Point2 m = centroid(ce);
    CHECK(std::hypot(m.x, m.y) < 1e-12);
  });
  run("normalize_length", [] {  // :106-113
    Curve sq;
    sq.nodes = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    const Curve c = normalize_length(sq);
    CHECK(std::fabs(curve_length(c) - 1.0) < 1e-14 && std::fabs(c[1].x - 0.25) < 1e-14);
  });
  run("arc_length_params", [] {  // :126-138
    Curve sq, rect;
    sq.nodes = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    rect.nodes = {{0, 0}, {2, 0}, {2, 1}, {0, 1}};
    const ArcLengthParams a = arc_length_params(sq), b = arc_length_params(rect);
    const double es[5] = {0, 0.25, 0.5, 0.75, 1.0}, er[5] = {0, 1.0 / 3.0, 0.5, 5.0 / 6.0, 1.0};
    CHECK(a.s.size() == 5 && std::fabs(a.total_length - 4.0) < 1e-14);
    for (int i = 0; i < 5; ++i) CHECK(std::fabs(a.s[i] - es[i]) < 1e-15 && std::fabs(b.s[i] - er[i]) < 1e-15);
    Curve dup;
    dup.nodes = {{0, 0}, {1, 0}, {1, 0}, {0, 1}};
    CHECK(throws<std::invalid_argument>([&] { arc_length_params(dup); }));
  });
  run("spline knots / smooth / bad knots", [] {  // :36-71
    std::vector<double> x = {0.0, 0.2, 0.45, 0.7, 1.0}, y = {1.0, -0.5, 2.0, 0.25, 1.0};
    PeriodicCubicSpline s(x, y);
    for (std::size_t i = 0; i + 1 < x.size(); ++i) CHECK(std::fabs(s.eval(x[i]) - y[i]) < 1e-14);
    CHECK(std::fabs(s.eval(0.0) - s.eval(1.0)) < 1e-14);
    std::vector<double> xs(65), ys(65);
    for (int i = 0; i <= 64; ++i) {
      xs[i] = i / 64.0;
      ys[i] = std::sin(2 * kPi * xs[i]);
    }
    PeriodicCubicSpline t(xs, ys);
    double worst = 0.0;
    for (int k = 0; k < 1000; ++k) worst = std::fmax(worst, std::fabs(t.eval(k / 1000.0) - std::sin(2 * kPi * k / 1000.0)));
    CHECK(worst < 1e-5);
    std::vector<double> bx = {0.0, 0.5, 0.25, 0.75}, by = {0, 1, 2, 3};
    CHECK(throws<std::invalid_argument>([&] { PeriodicCubicSpline(bx, by); }));
  });
  run("resample equalizes chords / reproduces uniform", [] {  // :154-189
    Curve c;
    c.nodes.resize(64);
    for (int i = 0; i < 64; ++i) {
      const double t = i / 64.0, u = t + 0.15 * t * (1.0 - t);
      c.nodes[i] = Point2(std::cos(2 * kPi * u), std::sin(2 * kPi * u));
    }
    const Curve r = resample_uniform(c, 256);
    double lo = 1e300, hi = 0.0;
    for (std::size_t i = 0; i < 256; ++i) {
      const double ch = (r[(i + 1) % 256] - r[i]).norm();
      lo = std::fmin(lo, ch), hi = std::fmax(hi, ch);
    }
    CHECK((hi - lo) / hi < 0.02);
    const Curve g = circle(128), rg = resample_uniform(g, 128);
    double worst = 0.0;
    for (std::size_t i = 0; i < 128; ++i) worst = std::fmax(worst, (rg[i] - g[i]).norm());
    CHECK(worst < 1e-4);
    Curve sq;
    sq.nodes = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    CHECK(throws<std::invalid_argument>([&] { resample_uniform(sq, 4); }));
  });
  run("preprocess composes", [] {  // :215-232
    const Curve c = hippopede(100), p = preprocess(c, 128);
    const Curve manual = normalize_length(center_curve(resample_uniform(c, 128)));
    CHECK(p.size() == 128);
    bool same = true;
    for (std::size_t i = 0; i < 128; ++i) same = same && p[i].x == manual[i].x && p[i].y == manual[i].y;
    CHECK(same);
    const Point2 m = centroid(p);
    CHECK(std::hypot(m.x, m.y) < 1e-12 && std::fabs(curve_length(p) - 1.0) < 1e-12);
    CHECK(preprocess(c, 64, false).size() == 100);
    // the batched (fused) path agrees to rounding
    const Curve b = preprocess_batch({c}, 128)[0];
    for (std::size_t i = 0; i < 128; ++i) CHECK((b[i] - p[i]).norm() < 1e-14);
  });

  // ------------------------------------------------------------------ srv
  run("srv of unit circle / equivariance / center", [] {  // test_srv.cpp:80-128
    const SrvCurve q = srv_transform(preprocess(circle(512), 256));
    CHECK(q.size() == 256 && std::fabs(q.h - 1.0 / 256.0) < 1e-15);
    for (const auto& p : q.q) CHECK(std::fabs(p.norm() - 1.0) < 1e-3);
    Curve c = preprocess(bumps(256), 128), cr = c;
    for (auto& p : cr.nodes) p = rotate_ccw(p, 0.7);
    const SrvCurve a = srv_transform(c), b = srv_transform(cr);
    for (std::size_t l = 0; l < a.size(); ++l) {
      const Point2 w = rotate_ccw(a.q[l], 0.7);
      CHECK(std::fabs(b.q[l].x - w.x) < 1e-14 && std::fabs(b.q[l].y - w.y) < 1e-14);
    }
    const SrvCurve z = srv_center(a);
    Point2 mean;
    for (const auto& p : z.q) mean += p;
    CHECK(std::hypot(mean.x, mean.y) / z.size() < 1e-12);
  });

  // ------------------------------------------------------------------ fft
  run("real dft / idft / correlation", [] {
    std::mt19937_64 rng(5);
    std::normal_distribution<double> g;
    for (std::size_t n : {2u, 3u, 8u, 33u, 101u, 256u, 1000u}) {
      std::vector<double> x(n), y(n);
      for (auto& v : x) v = g(rng);
      for (auto& v : y) v = g(rng);
      const auto X = real_dft(x);
      CHECK(X.size() == n / 2 + 1);
      double err = 0.0;
      for (std::size_t k = 0; k < X.size(); ++k) {
        std::complex<double> w;
        for (std::size_t j = 0; j < n; ++j) w += x[j] * std::polar(1.0, -2 * kPi * double((j * k) % n) / double(n));
        err = std::fmax(err, std::abs(w - X[k]));
      }
      CHECK(err < 1e-12 * n);
      const auto back = real_idft(X, n);
      for (std::size_t j = 0; j < n; ++j) CHECK(std::fabs(back[j] - x[j]) < 1e-12);
      const auto r = circular_cross_correlation(x, y);
      for (std::size_t m = 0; m < n; ++m) {
        double w = 0.0;
        for (std::size_t l = 0; l < n; ++l) w += x[l] * y[(l + m) % n];
        CHECK(std::fabs(w - r[m]) < 1e-12 * n);
      }
    }
  });

  // ---------------------------------------------------------------- batch
  run("batch == single", [] {
    std::mt19937_64 rng(9);
    std::vector<Curve> a, b;
    for (int p = 0; p < 5; ++p) {
      a.push_back(random_curve(rng, 128));
      b.push_back(shift_rotate(a.back(), 7 * p + 1, 0.3 * p));
    }
    std::vector<Curve> al;
    const auto res = align_fft_batch(a, b, &al);
    for (int p = 0; p < 5; ++p) {
      const RigidAlignment s = align_fft(a[p], b[p]);
      CHECK(res[p].shift == s.shift && res[p].shift == (std::size_t)(7 * p + 1));
      CHECK(std::fabs(res[p].energy - mismatch_energy(a[p].nodes, b[p].nodes, s.shift, s.rotation)) < 1e-12);
      for (std::size_t l = 0; l < 128; ++l) CHECK((al[p][l] - a[p][l]).norm() < 1e-12);
    }
    const auto pr = preprocess_align_batch(a, b, 256);
    CHECK(pr.size() == 5);
  });

  // --------------------------------------------------------- srv / DP / elastic
  // a monotone warp of [0, 1] (fixed endpoints) for the action cases
  auto warp = [](std::size_t n) {
    Reparameterization g;
    g.gamma.resize(n + 1);
    for (std::size_t l = 0; l <= n; ++l) {
      const double t = (double)l / (double)n;
      g.gamma[l] = t + 0.05 * std::sin(2.0 * kPi * t);
    }
    g.gamma[0] = 0.0;
    g.gamma[n] = 1.0;
    return g;
  };
  auto srv_norm2 = [](const SrvCurve& q) {
    double s = 0.0;
    for (const auto& p : q.q) s += p.norm2();
    return s * q.h;
  };
  run("identity action", [] {  // test_srv.cpp:130-137
    const SrvCurve q = srv_transform(preprocess(bumps(256), 128));
    const SrvCurve out = apply_srv_action(q, 0.0, Rotation2(0.0), identity_reparam(q.size()));
    for (std::size_t l = 0; l < q.size(); ++l) CHECK((out.q[l] - q.q[l]).norm() < 1e-12);
  });
  run("shift action relabels", [] {  // test_srv.cpp:139-147
    const std::size_t n = 128, m = 48;
    const SrvCurve q = srv_transform(preprocess(bumps(256), n));
    const SrvCurve out = apply_srv_action(q, double(m) / double(n), Rotation2(0.0), identity_reparam(n));
    for (std::size_t l = 0; l < n; ++l) CHECK(out.q[l].x == q.q[(l + m) % n].x && out.q[l].y == q.q[(l + m) % n].y);
  });
  run("action norm", [&] {  // test_srv.cpp:149-155
    const SrvCurve q = srv_transform(preprocess(bumps(512), 256));
    const SrvCurve out = apply_srv_action(q, 0.37, Rotation2(1.1), warp(256));
    CHECK(std::fabs(srv_norm2(out) - srv_norm2(q)) <= 0.02 * srv_norm2(q));
  });
  run("energy resummation", [&] {  // test_srv.cpp:157-170
    const std::size_t n = 128;
    const SrvCurve q1 = srv_transform(preprocess(bumps(256), n));
    const SrvCurve q2 = srv_transform(preprocess(limacon(256), n));
    const Reparameterization g = warp(n);
    const double e = elastic_energy(q1, q2, 0.21, Rotation2(0.8), g);
    const SrvCurve act = apply_srv_action(q2, 0.21, Rotation2(0.8), g);
    double direct = 0.0;
    for (std::size_t l = 0; l < n; ++l) direct += (q1.q[l] - act.q[l]).norm2();
    direct *= q1.h;
    CHECK(std::fabs(e - direct) <= 1e-12 * direct);
    CHECK(elastic_energy(q1, q1, 0.0, Rotation2(0.0), identity_reparam(n)) < 1e-15);
  });
  run("admissible steps", [] {  // test_srv.cpp:179-187
    const auto st = dp_admissible_steps(4);
    CHECK(st.size() == 11);
    CHECK(dp_admissible_steps(1).size() == 1);
    CHECK(throws<std::invalid_argument>([] { dp_admissible_steps(0); }));
  });
  run("dp identity / bound / valid", [] {  // test_srv.cpp:189-229
    const std::size_t n = 64;
    const SrvCurve q = srv_transform(preprocess(bumps(256), n));
    const DpResult r = dp_reparam(q, q);
    CHECK(r.gamma.gamma.size() == n + 1 && r.energy < 1e-12);
    for (std::size_t l = 0; l <= n; ++l) CHECK(std::fabs(r.gamma.gamma[l] - double(l) / double(n)) < 1e-10);
    const SrvCurve q2 = srv_transform(preprocess(hippopede(256), n));
    const DpResult s = dp_reparam(q, q2);
    CHECK(s.energy <= elastic_energy(q, q2, 0.0, Rotation2(0.0), identity_reparam(n)) + 1e-12);
    validate_reparam(s.gamma);
    std::mt19937_64 rng(5);
    for (int k = 0; k < 2; ++k) {
      const SrvCurve a = srv_transform(preprocess(random_curve(rng, 48), 48, false));
      const SrvCurve b = srv_transform(preprocess(random_curve(rng, 48), 48, false));
      const DpResult t = dp_reparam(a, b);
      CHECK(t.gamma.gamma.front() == 0.0 && t.gamma.gamma.back() == 1.0 && std::isfinite(t.energy) && t.energy >= 0);
      for (std::size_t l = 0; l < 48; ++l) CHECK(t.gamma.gamma[l + 1] >= t.gamma.gamma[l]);
    }
    CHECK(throws<std::invalid_argument>([&] { dp_step_cost(q, q2, 0, 0, 0, 1); }));
  });
  run("elastic self distance", [] {  // test_elastic.cpp:35-44
    const Curve c = preprocess(bumps(256), 64);
    const ElasticMatch m1 = elastic_distance_approach1(c, c);
    CHECK(m1.distance <= 1e-6 && m1.converged);
    const ElasticMatch m2 = elastic_distance_approach2(c, c);
    CHECK(m2.distance <= 1e-6 && m2.converged && m2.iterations >= 1);
  });
  run("energy traces", [] {  // test_elastic.cpp:46-61
    const Curve c1 = preprocess(limacon(256), 64), c2 = preprocess(bumps(256), 64);
    const ElasticMatch m2 = elastic_distance_approach2(c1, c2);
    CHECK(!m2.energy_trace.empty() && m2.energy_trace.size() == (std::size_t)m2.iterations + 1);
    for (std::size_t i = 1; i < m2.energy_trace.size(); ++i) CHECK(m2.energy_trace[i] <= m2.energy_trace[i - 1] + 1e-12);
    CHECK(std::fabs(m2.energy - m2.energy_trace.back()) <= 1e-12 * m2.energy);
    CHECK(std::fabs(m2.distance - std::sqrt(m2.energy)) <= 1e-12 * m2.distance);
    const ElasticMatch m1 = elastic_distance_approach1(c1, c2);
    CHECK(m1.energy >= 0.0 && m1.energy <= 4.0 + 1e-9);
    CHECK(std::fabs(m1.distance - std::sqrt(m1.energy)) <= 1e-12 * m1.distance);
  });
  run("elastic invariance", [] {  // test_elastic.cpp:63-73
    const std::size_t n = 128;
    const Curve c1 = preprocess(hippopede(256), n);
    Curve c2;
    c2.nodes.resize(n);
    for (std::size_t l = 0; l < n; ++l) c2.nodes[l] = rotate_ccw(c1[(l + n / 3) % n], 0.9);
    CHECK(elastic_distance_approach2(c1, c2).distance <= 0.005);
    CHECK(elastic_distance_approach1(c1, c2).distance <= 0.005);
  });
  run("approach 1 limit", [] {  // test_elastic.cpp:91-101
    const Curve c = preprocess(circle(1024), 600);
    bool threw = false;
    try {
      elastic_distance_approach1(c, c);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()).find("approach 2") != std::string::npos;
    }
    CHECK(threw);
  });
  run("elastic validation", [] {  // test_elastic.cpp:103-111
    const Curve a = preprocess(circle(64), 32), b = preprocess(circle(64), 16);
    CHECK(throws<std::invalid_argument>([&] { elastic_distance_approach2(a, b); }));
    Curve tiny;
    tiny.nodes = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    CHECK(throws<std::invalid_argument>([&] { elastic_distance_approach2(tiny, tiny); }));
  });
  run("distance matrix", [] {  // test_elastic.cpp:113-160
    const std::vector<Curve> dup = {bumps(200), bumps(200)};
    const auto d = distance_matrix(dup, DistanceMethod::approach2, 64);
    CHECK(d.size() == 2 && d[0].size() == 2);
    for (const auto& row : d)
      for (double v : row) CHECK(v <= 1e-6);
    const std::vector<Curve> three = {bumps(128), limacon(128), hippopede(128)};
    const auto d1 = distance_matrix(three, DistanceMethod::approach2, 64, {}, 1);
    const auto d4 = distance_matrix(three, DistanceMethod::approach2, 64, {}, 4);
    for (std::size_t i = 0; i < 3; ++i)
      for (std::size_t j = 0; j < 3; ++j) CHECK(d1[i][j] == d4[i][j]);
    CHECK(d1[0][1] > 0.01 && d1[0][2] > 0.01);
    ElasticOptions o;
    o.n_max_approach1 = 16;
    for (const auto& row : distance_matrix(three, DistanceMethod::approach1, 64, o, 1))
      for (double v : row) CHECK(std::isnan(v));
    int calls = 0;
    distance_matrix(dup, DistanceMethod::approach2, 64, {}, 1, [&](std::size_t, std::size_t, double, double) { ++calls; });
    CHECK(calls == 4);
  });
  run("elastic use_fft = false and slab-mode sizes", [] {  // ElasticOptions (elastic.hpp:13-19)
    const Curve c1 = preprocess(limacon(256), 64), c2 = preprocess(bumps(256), 64);
    ElasticOptions naive;
    naive.use_fft = false;
    const ElasticMatch f = elastic_distance_approach2(c1, c2), g = elastic_distance_approach2(c1, c2, naive);
    // the two correlations agree to rounding, so the searches end at the same distance
    CHECK(std::fabs(f.distance - g.distance) <= 1e-9 * f.distance && f.iterations == g.iterations);
    ElasticOptions steep;  // 9 <= max_slope <= 20 and n > 1024 run with the working set in global memory
    steep.max_slope = 9;
    steep.max_iters = 2;
    const ElasticMatch s9 = elastic_distance_approach2(c1, c2, steep);
    CHECK(std::isfinite(s9.distance) && s9.distance >= 0.0 && s9.iterations >= 1);
    const Curve big1 = preprocess(limacon(1500), 1100), big2 = preprocess(bumps(1500), 1100);
    ElasticOptions two;
    two.max_iters = 2;
    const ElasticMatch b = elastic_distance_approach2(big1, big2, two);
    CHECK(std::isfinite(b.distance) && b.gamma.gamma.size() == 1101 && b.gamma.gamma.back() == 1.0);
  });
  run("elastic batch == single", [] {
    const std::vector<Curve> a = {preprocess(bumps(200), 64), preprocess(limacon(200), 64)};
    const std::vector<Curve> b = {preprocess(hippopede(200), 64), preprocess(bumps(200), 64)};
    const auto r = elastic_distance_batch(a, b, DistanceMethod::approach2);
    for (int p = 0; p < 2; ++p) CHECK(r[p].distance == elastic_distance_approach2(a[p], b[p]).distance);
  });

  // ------------------------------------------------- concurrent callers
  // The reference's functions are pure and re-entrant and distance_matrix calls
  // align_fft from a thread pool (elastic.cpp:196-234): every thread must get
  // the answer a lone caller gets.
  run("concurrent align_fft / preprocess / srv from 8 threads", [&] {
    std::mt19937_64 rng(77);
    const int T = 8, per = 6;
    std::vector<std::pair<Curve, Curve>> in;
    for (int i = 0; i < T * per; ++i) {
      const Curve c = preprocess(random_curve(rng, 200 + 37 * i), 256);
      in.emplace_back(c, shift_rotate(c, (std::size_t)(rng() % 256), 0.1 * i));
    }
    std::vector<RigidAlignment> seq, par(in.size());
    std::vector<Curve> pseq, ppar(in.size());
    std::vector<RigidAlignment> sseq, spar(in.size());
    for (const auto& p : in) {
      seq.push_back(align_fft(p.first, p.second));
      pseq.push_back(preprocess(p.second, 128));
      sseq.push_back(align_fft(srv_center(srv_transform(p.first)).q, srv_center(srv_transform(p.second)).q));
    }
    std::vector<std::thread> th;
    std::vector<int> errors(T, 0);
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        try {
          for (int r = 0; r < 3; ++r)
            for (int i = t; i < (int)in.size(); i += T) {
              par[i] = align_fft(in[i].first, in[i].second);
              ppar[i] = preprocess(in[i].second, 128);
              spar[i] = align_fft(srv_center(srv_transform(in[i].first)).q,
                                  srv_center(srv_transform(in[i].second)).q);
            }
        } catch (...) {
          errors[t] = 1;
        }
      });
    for (auto& x : th) x.join();
    for (int t = 0; t < T; ++t) CHECK(errors[t] == 0);
    auto same = [](const RigidAlignment& a, const RigidAlignment& b) {
      return a.shift == b.shift && a.t0 == b.t0 && a.rotation.theta() == b.rotation.theta() && a.trace == b.trace &&
             a.energy == b.energy && a.degenerate == b.degenerate;
    };
    for (std::size_t i = 0; i < in.size(); ++i) {
      CHECK(same(seq[i], par[i]));
      CHECK(same(sseq[i], spar[i]));
      bool eq = pseq[i].size() == ppar[i].size();
      for (std::size_t l = 0; eq && l < pseq[i].size(); ++l)
        eq = pseq[i].nodes[l].x == ppar[i].nodes[l].x && pseq[i].nodes[l].y == ppar[i].nodes[l].y;
      CHECK(eq);
    }
  });

  // --------------------------------------------------------------- file formats
  const std::string tmpdir = "/tmp/cva_dropin_io_" + std::to_string((long)getpid());
  CHECK(mkdir(tmpdir.c_str(), 0700) == 0);
  auto tpath = [&](const char* n) { return tmpdir + "/" + n; };
  auto write_text = [](const std::string& p, const std::string& t) { std::ofstream(p, std::ios::binary) << t; };
  run("io round trips", [&] {  // test_io_cli.cpp:50-72, :110-118
    const Curve c = limacon(32);
    write_curve_csv(tpath("r.csv"), c);
    write_curve_json(tpath("r.json"), c);
    for (const char* f : {"r.csv", "r.json"}) {
      const Curve b = load_curve(tpath(f));
      CHECK(b.size() == c.size());
      for (std::size_t i = 0; i < c.size(); ++i) CHECK(b[i].x == c[i].x && b[i].y == c[i].y);
    }
  });
  run("io csv header / duplicate / malformed", [&] {  // test_io_cli.cpp:74-98
    write_text(tpath("h.csv"), "x,y\n1,0\n0,1\n-1,0\n0,-1\n1,0\n");
    const Curve c = read_curve_csv(tpath("h.csv"));
    CHECK(c.size() == 4 && c[0].x == 1.0 && c[3].y == -1.0);
    write_text(tpath("b1.csv"), "1,2\nthree\n4,5\n6,7\n");
    write_text(tpath("b2.csv"), "x,y\n1,2\nalpha,beta\n3,4\n5,6\n");
    write_text(tpath("few.csv"), "1,2\n3,4\n");
    CHECK(throws<std::runtime_error>([&] { read_curve_csv(tpath("b1.csv")); }));
    CHECK(throws<std::runtime_error>([&] { read_curve_csv(tpath("b2.csv")); }));
    CHECK(throws<std::invalid_argument>([&] { read_curve_csv(tpath("few.csv")); }));
    CHECK(throws<std::runtime_error>([&] { read_curve_csv(tpath("none.csv")); }));
  });
  run("io json schema", [&] {  // test_io_cli.cpp:100-108
    write_text(tpath("bad.json"), "{\"points\": [[0, 0]]}");
    write_text(tpath("rag.json"), "{\"nodes\": [[0, 0, 0], [1, 1]]}");
    CHECK(throws<std::runtime_error>([&] { read_curve_json(tpath("bad.json")); }));
    CHECK(throws<std::runtime_error>([&] { read_curve_json(tpath("rag.json")); }));
    write_text(tpath("ok.json"), " { \"closed\" : true , \"nodes\": [ [1,0], [0, 1.5e0], [-1,0],[0,-1],[1,0] ] } ");
    const Curve c = read_curve_json(tpath("ok.json"));
    CHECK(c.size() == 4 && c[1].y == 1.5);
  });
  run("io results", [] {  // test_io_cli.cpp:120-135
    const std::string csv = matrix_to_csv({"a", "b"}, {{0.0, 0.5}, {std::nan(""), 0.0}});
    CHECK(csv == "id,a,b\na,0,0.5\nb,nan,0\n");
    CHECK(throws<std::invalid_argument>([] { matrix_to_csv({"a"}, {{0.0, 0.5}, {0.0, 0.0}}); }));
    RigidAlignment r;
    r.shift = 29;
    r.t0 = 0.25;
    r.rotation = Rotation2(0.5);
    r.trace = 21.5;
    r.energy = 1e-07;
    CHECK(alignment_to_json(r) == "{\"energy\":1e-07,\"shift\":29,\"t0\":0.25,\"theta\":0.5,\"trace\":21.5}");
    CHECK(curve_to_json(Curve{{{1.0, 0.0}, {0.25, 2.0}}}) == "{\"closed\":true,\"nodes\":[[1.0,0.0],[0.25,2.0]]}");
  });
  if (DIR* d = opendir(tmpdir.c_str())) {
    while (dirent* e = readdir(d))
      if (std::string(e->d_name) != "." && std::string(e->d_name) != "..") std::remove(tpath(e->d_name).c_str());
    closedir(d);
  }
  rmdir(tmpdir.c_str());

  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail;
}
