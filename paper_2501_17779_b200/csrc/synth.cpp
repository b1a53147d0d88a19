// Seeded synthetic workloads for the BASELINE.json configs (bench harness; host only).
//
// The reference measures on no public dataset; these
// generators produce the configs' shapes, sizes and value distributions. RNG
// conventions follow proj/src/synthetic.cpp:19-22 (std::mt19937_64, top-53-bit
// uniforms); every pair has its own engine seeded from (seed, pair, stream) by
// splitmix64, so outputs are independent of the thread count.
//
// Shapes are star-shaped polar curves r(phi) = 1 + sum_{m=2}^{M+1} a_m cos(m phi + p_m),
// a_m ~ U(0, amp * m^-amp_exp), p_m ~ U(0, 2 pi).
//   C0  cva_synth_uniform_pairs(N=256, M=7,  amp=0.3, exp=1,   sigma=1e-3)
//   C1  cva_synth_sizes + cva_synth_ragged_pairs(N=1024, M=16, sigma=1e-3, n_in in [300, 3000])
//   C2  cva_synth_sizes + cva_synth_ragged_curves(M=16)
//   C3  cva_synth_uniform_pairs(N=65536, M=64, amp=0.3, exp=1.5, sigma=1e-4)
//   C4  cva_synth_srv_pairs(N=2048, M=16)
// Shift convention: curve 2 is curve 1 with its start moved by k (c2[l] ~ rot(c1[l-k], theta)),
// so the reference recovers shift k and theta (proj/tests/acceptance.cpp:67-74).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <functional>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr double kTwoPi = 2.0 * std::numbers::pi;

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

std::mt19937_64 engine(uint64_t seed, uint64_t item, uint64_t stream) {
  return std::mt19937_64(splitmix64(splitmix64(seed ^ (stream * 0xD1B54A32D192ED03ULL)) + item));
}

double u01(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }
double uab(std::mt19937_64& r, double a, double b) { return a + (b - a) * u01(r); }
int64_t uint_range(std::mt19937_64& r, int64_t lo, int64_t hi) {  // inclusive
  return lo + static_cast<int64_t>(r() % static_cast<uint64_t>(hi - lo + 1));
}
double gauss(std::mt19937_64& r) {  // Box-Muller
  double u = u01(r);
  while (u <= 0.0) u = u01(r);
  const double v = u01(r);
  return std::sqrt(-2.0 * std::log(u)) * std::cos(kTwoPi * v);
}

struct Shape {
  std::vector<int> m;
  std::vector<double> a, p;
  void draw(std::mt19937_64& r, int modes, double amp, double amp_exp) {
    m.resize(modes);
    a.resize(modes);
    p.resize(modes);
    for (int j = 0; j < modes; ++j) {
      m[j] = j + 2;
      a[j] = uab(r, 0.0, amp * std::pow(static_cast<double>(m[j]), -amp_exp));
      p[j] = uab(r, 0.0, kTwoPi);
    }
  }
  double radius(double phi) const {
    double rr = 1.0;
    for (size_t j = 0; j < m.size(); ++j) rr += a[j] * std::cos(m[j] * phi + p[j]);
    return rr;
  }
  void point(double phi, double* xy) const {
    const double rr = radius(phi);
    xy[0] = rr * std::cos(phi);
    xy[1] = rr * std::sin(phi);
  }
};

// Arc-length parameterisation of a shape through a fine polygon: phi(f) for an
// arc-length fraction f in [0, 1).
struct ArcMap {
  std::vector<double> L;  // cumulative chord length at phi_j = 2 pi j / F, j = 0..F
  int F = 0;
  double total = 0.0;
  void build(const Shape& s, int fine) {
    F = fine;
    L.assign(F + 1, 0.0);
    double prev[2], cur[2];
    s.point(0.0, prev);
    for (int j = 1; j <= F; ++j) {
      s.point(kTwoPi * j / F, cur);
      L[j] = L[j - 1] + std::hypot(cur[0] - prev[0], cur[1] - prev[1]);
      prev[0] = cur[0];
      prev[1] = cur[1];
    }
    total = L[F];
  }
  double phi(double f) const {
    const double target = f * total;
    const auto it = std::upper_bound(L.begin(), L.end(), target);
    int j = static_cast<int>(it - L.begin()) - 1;
    j = std::clamp(j, 0, F - 1);
    const double w = (target - L[j]) / (L[j + 1] - L[j]);
    return kTwoPi * (j + w) / F;
  }
};

double wrap_unit(double t) {
  double r = t - std::floor(t);
  if (r >= 1.0) r -= 1.0;
  return r;
}

void rotate_ccw(double* xy, double th) {
  const double c = std::cos(th), s = std::sin(th);
  const double x = xy[0], y = xy[1];
  xy[0] = c * x - s * y;
  xy[1] = s * x + c * y;
}

void parallel_for(int64_t n, int threads, const std::function<void(int64_t)>& f) {
  if (threads <= 1 || n < 2) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (int64_t i = next++; i < n; i = next++) f(i);
    });
  for (auto& th : pool) th.join();
}

// Nodes of a raw curve at jittered arc-length fractions (i + U(-0.4, 0.4)) / n,
// shifted by `shift` (fraction), rotated ccw by theta, plus N(0, sigma^2) noise.
void ragged_curve(const Shape& s, const ArcMap& am, int64_t n, double shift, double theta,
                  double sigma, std::mt19937_64& r, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double f = wrap_unit((static_cast<double>(i) + uab(r, -0.4, 0.4)) / n - shift);
    double* p = out + 2 * i;
    s.point(am.phi(f), p);
    if (theta != 0.0) rotate_ccw(p, theta);
    if (sigma > 0.0) {
      p[0] += sigma * gauss(r);
      p[1] += sigma * gauss(r);
    }
  }
}

}  // namespace

extern "C" {

// offsets[0..count] of `count` ragged curves with sizes U{n_min..n_max}.
int cva_synth_sizes(uint64_t seed, int64_t count, int64_t n_min, int64_t n_max, int64_t* offsets) {
  if (count < 0 || n_min < 1 || n_max < n_min) return 1;
  offsets[0] = 0;
  for (int64_t c = 0; c < count; ++c) {
    auto r = engine(seed, static_cast<uint64_t>(c), 0);
    offsets[c + 1] = offsets[c] + uint_range(r, n_min, n_max);
  }
  return 0;
}

// C1: pairs of raw curves (curve 2p, 2p+1) in the ragged layout given by offsets
// (2 * pairs + 1 entries). Curve 2 = curve 1's shape, start moved by k/N, rotated
// by theta, own jitter, plus noise. truth_* (nullable) receive k and theta.
int cva_synth_ragged_pairs(uint64_t seed, int64_t pairs, int64_t N, int modes, double amp,
                           double amp_exp, double sigma, const int64_t* offsets, double* points,
                           int64_t* truth_shift, double* truth_theta, int threads) {
  if (pairs < 0 || N < 1 || modes < 1) return 1;
  parallel_for(pairs, threads, [&](int64_t p) {
    auto r = engine(seed, static_cast<uint64_t>(p), 1);
    Shape s;
    s.draw(r, modes, amp, amp_exp);
    const int64_t k = uint_range(r, 0, N - 1);
    const double th = uab(r, 0.0, kTwoPi);
    ArcMap am;
    am.build(s, 8192);
    const int64_t a0 = offsets[2 * p], a1 = offsets[2 * p + 1], b1 = offsets[2 * p + 2];
    ragged_curve(s, am, a1 - a0, 0.0, 0.0, 0.0, r, points + 2 * a0);
    ragged_curve(s, am, b1 - a1, static_cast<double>(k) / N, th, sigma, r, points + 2 * a1);
    if (truth_shift) truth_shift[p] = k;
    if (truth_theta) truth_theta[p] = th;
  });
  return 0;
}

// C2: independent raw curves (no noise) in the ragged layout of offsets.
int cva_synth_ragged_curves(uint64_t seed, int64_t curves, int modes, double amp, double amp_exp,
                            const int64_t* offsets, double* points, int threads) {
  if (curves < 0 || modes < 1) return 1;
  parallel_for(curves, threads, [&](int64_t c) {
    auto r = engine(seed, static_cast<uint64_t>(c), 2);
    Shape s;
    s.draw(r, modes, amp, amp_exp);
    ArcMap am;
    am.build(s, 8192);
    ragged_curve(s, am, offsets[c + 1] - offsets[c], 0.0, 0.0, 0.0, r, points + 2 * offsets[c]);
  });
  return 0;
}

// C0 / C3: c1[l] = shape(2 pi l / N); c2[l] = rot_ccw(c1[(l - k) mod N], theta) + noise.
int cva_synth_uniform_pairs(uint64_t seed, int64_t pairs, int64_t N, int modes, double amp,
                            double amp_exp, double sigma, double* c1, double* c2,
                            int64_t* truth_shift, double* truth_theta, int threads) {
  if (pairs < 0 || N < 4 || modes < 1) return 1;
  parallel_for(pairs, threads, [&](int64_t p) {
    auto r = engine(seed, static_cast<uint64_t>(p), 3);
    Shape s;
    s.draw(r, modes, amp, amp_exp);
    const int64_t k = uint_range(r, 0, N - 1);
    const double th = uab(r, 0.0, kTwoPi);
    double* a = c1 + 2 * p * N;
    double* b = c2 + 2 * p * N;
    for (int64_t l = 0; l < N; ++l) s.point(kTwoPi * static_cast<double>(l) / N, a + 2 * l);
    for (int64_t l = 0; l < N; ++l) {
      const int64_t src = ((l - k) % N + N) % N;
      b[2 * l] = a[2 * src];
      b[2 * l + 1] = a[2 * src + 1];
      rotate_ccw(b + 2 * l, th);
      if (sigma > 0.0) {
        b[2 * l] += sigma * gauss(r);
        b[2 * l + 1] += sigma * gauss(r);
      }
    }
    if (truth_shift) truth_shift[p] = k;
    if (truth_theta) truth_theta[p] = th;
  });
  return 0;
}

// C4: c1 = unit-length shape at uniform arc length t_l = l/N; c2[l] = rot_ccw(c1(gamma(t_l) - k/N), theta)
// with gamma(t) = t + 0.05 u sin(2 pi t), u ~ U(-1, 1): the shift -> rotation -> warp
// order of transform_curve (proj/src/synthetic.cpp:120-157), evaluated on the exact shape.
int cva_synth_srv_pairs(uint64_t seed, int64_t pairs, int64_t N, int modes, double amp,
                        double amp_exp, double* c1, double* c2, int64_t* truth_shift,
                        double* truth_theta, double* truth_u, int threads) {
  if (pairs < 0 || N < 8 || modes < 1) return 1;
  parallel_for(pairs, threads, [&](int64_t p) {
    auto r = engine(seed, static_cast<uint64_t>(p), 4);
    Shape s;
    s.draw(r, modes, amp, amp_exp);
    const int64_t k = uint_range(r, 0, N - 1);
    const double th = uab(r, 0.0, kTwoPi);
    const double u = uab(r, -1.0, 1.0);
    ArcMap am;
    am.build(s, 16384);
    const double inv_len = 1.0 / am.total;
    double* a = c1 + 2 * p * N;
    double* b = c2 + 2 * p * N;
    for (int64_t l = 0; l < N; ++l) {
      const double t = static_cast<double>(l) / N;
      s.point(am.phi(t), a + 2 * l);
      a[2 * l] *= inv_len;
      a[2 * l + 1] *= inv_len;
      const double g = t + 0.05 * u * std::sin(kTwoPi * t);
      s.point(am.phi(wrap_unit(g - static_cast<double>(k) / N)), b + 2 * l);
      b[2 * l] *= inv_len;
      b[2 * l + 1] *= inv_len;
      rotate_ccw(b + 2 * l, th);
    }
    if (truth_shift) truth_shift[p] = k;
    if (truth_theta) truth_theta[p] = th;
    if (truth_u) truth_u[p] = u;
  });
  return 0;
}

}  // extern "C"
