// GPU kernels behind the scalar entry points of the C++ drop-in API
// (include/curvalign/*.hpp -> csrc/dropin/*.cpp). These serve the reference's
// single-curve utility functions; throughput work goes through the batched
// kernels (fused.cu, allpairs.cu, largen.cu). All fp64, one call = one curve.
#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "gfft.h"
#include "elastic.h"
#include "spline.cuh"

namespace cva {
namespace di {

constexpr int kT = 256;

// A(m) for m in [m0, m0 + count): A_kj = sum_l c1[l]_k c2[(l+m) mod n]_j
// (rigid_align.cpp:65-80, :126-145); one CTA per shift, fixed summation order.
__global__ void __launch_bounds__(kT) corr_kernel(const double2* __restrict__ c1, const double2* __restrict__ c2,
                                                  int64_t n, int64_t m0, double* out4) {
  __shared__ double2 red[64];
  const int64_t m = m0 + blockIdx.x;
  double2 a = make_double2(0, 0), b = make_double2(0, 0);  // (a11, a12), (a21, a22)
  for (int64_t l = threadIdx.x; l < n; l += kT) {
    int64_t j = l + m;
    if (j >= n) j -= n;
    const double2 p = c1[l], q = c2[j];
    a.x = fma(p.x, q.x, a.x);
    a.y = fma(p.x, q.y, a.y);
    b.x = fma(p.y, q.x, b.x);
    b.y = fma(p.y, q.y, b.y);
  }
  a = block_sum2(a, red);
  __syncthreads();
  b = block_sum2(b, red);
  if (threadIdx.x == 0) {
    double* o = out4 + 4 * blockIdx.x;
    o[0] = a.x;
    o[1] = a.y;
    o[2] = b.x;
    o[3] = b.y;
  }
}

// h sum_l |c1[l] - R(theta) c2[(l+shift) mod n]|^2 (rigid_align.cpp:185-196)
__global__ void __launch_bounds__(kT) mismatch_kernel(const double2* __restrict__ c1, const double2* __restrict__ c2,
                                                      int64_t n, int64_t shift, double theta, double* out) {
  __shared__ double2 red[64];
  double sn, cs;
  sincos(theta, &sn, &cs);
  double e = 0.0;
  for (int64_t l = threadIdx.x; l < n; l += kT) {
    int64_t j = l + shift;
    if (j >= n) j -= n;
    const double2 q = c2[j], p = c1[l];
    const double dx = p.x - (cs * q.x + sn * q.y), dy = p.y - (-sn * q.x + cs * q.y);
    e = fma(dx, dx, fma(dy, dy, e));
  }
  e = block_sum(e, red);
  if (threadIdx.x == 0) *out = e / (double)n;
}

// centroid (curve.cpp:27-32) and polygon length incl. closing edge (:17-25)
__global__ void __launch_bounds__(kT) stats_kernel(const double2* __restrict__ c, int64_t n, double* out3) {
  __shared__ double2 red[64];
  double2 s = make_double2(0, 0);
  double len = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kT) {
    const double2 p = c[i], q = c[i + 1 == n ? 0 : i + 1];
    s = cadd(s, p);
    const double dx = q.x - p.x, dy = q.y - p.y;
    len += sqrt(fma(dx, dx, dy * dy));
  }
  s = block_sum2(s, red);
  __syncthreads();
  len = block_sum(len, red);
  if (threadIdx.x == 0) {
    const double inv = 1.0 / (double)n;
    out3[0] = inv * s.x;
    out3[1] = inv * s.y;
    out3[2] = len;
  }
}

// out = c - g (center_curve, curve.cpp:34-39) or out = c / len (normalize_length, :41-48)
__global__ void affine_kernel(const double2* __restrict__ c, int64_t n, double gx, double gy, double sc,
                              double2* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double2 p = c[i];
    out[i] = make_double2((p.x - gx) * sc, (p.y - gy) * sc);
  }
}

// arc_length_params (curve.cpp:50-65) of one curve; status 1 on coincident nodes
__global__ void __launch_bounds__(kT) arclen_kernel(const double2* __restrict__ c, int n, double* s, double* total,
                                                    int* status) {
  __shared__ double2 red[64];
  int bad = 0;
  const double t = block_arc_length(c, n, s, red, &bad);
  if (threadIdx.x == 0) {
    *total = t;
    *status = bad;
  }
}

// Periodic spline second derivatives m[0..n] for knots x[0..n], values y[0..n]
// (spline.cpp:62-96), via the block partition solver of spline.cuh (the
// reference's system, P11 included). Values are carried as (y, 0) pairs.
__global__ void __launch_bounds__(kT) spline_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                    int n, double* m_out) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[64];
  double* s = reinterpret_cast<double*>(smem);
  double2* yy = reinterpret_cast<double2*>(s + ((n + 2) & ~1));
  double2* m = yy + n;
  ChunkEnds* ends = reinterpret_cast<ChunkEnds*>(m + n);
  for (int i = threadIdx.x; i <= n; i += kT) s[i] = x[i];
  for (int i = threadIdx.x; i < n; i += kT) yy[i] = make_double2(y[i], 0.0);
  __syncthreads();
  block_spline_solve(s, yy, m, n, ends, red);
  for (int i = threadIdx.x; i < n; i += kT) m_out[i] = m[i].x;
  if (threadIdx.x == 0) m_out[n] = m[0].x;
}

// srv_transform (srv.cpp:71-88) [+ srv_center, :90-98] of one curve
__global__ void __launch_bounds__(kT) srv_kernel(const double2* __restrict__ c, int64_t n, int center, double2* q) {
  __shared__ double2 red[64];
  const double nn = (double)n;
  double2 acc = make_double2(0, 0);
  for (int64_t l = threadIdx.x; l < n; l += kT) {
    const double2 nx = c[l + 1 == n ? 0 : l + 1], pv = c[l == 0 ? n - 1 : l - 1];
    const double2 d = make_double2((nn / 2.0) * (nx.x - pv.x), (nn / 2.0) * (nx.y - pv.y));
    const double mag = sqrt(fma(d.x, d.x, d.y * d.y));
    const double2 v = mag < 1e-8 * nn ? make_double2(0.0, 0.0) : cscale(d, 1.0 / sqrt(mag));
    q[l] = v;
    acc = cadd(acc, v);
  }
  if (!center) return;
  acc = block_sum2(acc, red);
  const double inv = 1.0 / nn;
  const double2 mean = make_double2(inv * acc.x, inv * acc.y);
  for (int64_t l = threadIdx.x; l < n; l += kT) q[l] = csub(q[l], mean);
}

// x *= scale (in place; the 1/n of real_idft, fft.cpp:111-112)
__global__ void scale_kernel(double2* x, int64_t n, double scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = cscale(x[i], scale);
}

}  // namespace di

// ----------------------------------------------------------------- host

namespace {
thread_local std::string t_err;

int err(int st, const char* what, cudaError_t e = cudaSuccess) {
  t_err = std::string(what) + (e != cudaSuccess ? std::string(": ") + cudaGetErrorString(e) : std::string());
  cudaStreamSynchronize(cudaStreamPerThread);  // no copy of this call still touches the caller's buffers
  return st;
}

// Single-call utilities run on the calling host thread's default stream
// (stream-ordered scratch), so concurrent callers do not serialise.
const cudaStream_t kS = cudaStreamPerThread;
struct Buf {
  void* p = nullptr;
  bool alloc(size_t b) { return cudaMallocAsync(&p, b ? b : 16, kS) == cudaSuccess; }
  ~Buf() {
    if (p) cudaFreeAsync(p, kS);
  }
};

int have_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return err(CVA_CUDA_ERROR, "no CUDA device available");
  return CVA_OK;
}

int up(Buf& b, const void* h, size_t bytes) {
  if (!b.alloc(bytes)) return err(CVA_BAD_ALLOC, "device allocation failed");
  cudaError_t e = cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, kS);
  return e == cudaSuccess ? CVA_OK : err(CVA_CUDA_ERROR, "H2D", e);
}

int down(void* h, const Buf& b, size_t bytes) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, b.p, bytes, cudaMemcpyDeviceToHost, kS);
  if (e == cudaSuccess) e = cudaStreamSynchronize(kS);
  return e == cudaSuccess ? CVA_OK : err(CVA_CUDA_ERROR, "kernel/D2H", e);
}
}  // namespace

}  // namespace cva

using cva::Buf;

extern "C" {

const char* cva_dropin_last_error(void) { return cva::t_err.c_str(); }

int cva_correlation_matrices_host(const double* c1, const double* c2, int64_t n, int64_t m_begin, int64_t m_count,
                                  double* out4) {
  if (n < 1 || m_begin < 0 || m_count < 0 || m_begin + m_count > n)
    return cva::err(CVA_INVALID_ARGUMENT, "correlation: bad shift range");
  if (m_count == 0) return CVA_OK;
  if (int rc = cva::have_device()) return rc;
  Buf a, b, o;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, c1, cb)) return rc;
  if (int rc = cva::up(b, c2, cb)) return rc;
  if (!o.alloc(sizeof(double) * 4 * (size_t)m_count)) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cva::di::corr_kernel<<<(unsigned)m_count, cva::di::kT, 0, cva::kS>>>((const double2*)a.p, (const double2*)b.p, n, m_begin,
                                                           (double*)o.p);
  return cva::down(out4, o, sizeof(double) * 4 * (size_t)m_count);
}

int cva_mismatch_energy_host(const double* c1, const double* c2, int64_t n, int64_t shift, double theta,
                             double* out) {
  if (n < 1 || shift < 0 || shift >= n) return cva::err(CVA_INVALID_ARGUMENT, "align: shift out of range");
  if (int rc = cva::have_device()) return rc;
  Buf a, b, o;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, c1, cb)) return rc;
  if (int rc = cva::up(b, c2, cb)) return rc;
  if (!o.alloc(sizeof(double))) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cva::di::mismatch_kernel<<<1, cva::di::kT, 0, cva::kS>>>((const double2*)a.p, (const double2*)b.p, n, shift, theta,
                                               (double*)o.p);
  return cva::down(out, o, sizeof(double));
}

int cva_curve_stats_host(const double* xy, int64_t n, double* centroid2, double* length) {
  if (n < 1) return cva::err(CVA_INVALID_ARGUMENT, "curve: too few nodes");
  if (int rc = cva::have_device()) return rc;
  Buf a, o;
  if (int rc = cva::up(a, xy, sizeof(double2) * (size_t)n)) return rc;
  if (!o.alloc(3 * sizeof(double))) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cva::di::stats_kernel<<<1, cva::di::kT, 0, cva::kS>>>((const double2*)a.p, n, (double*)o.p);
  double h[3];
  if (int rc = cva::down(h, o, sizeof(h))) return rc;
  if (centroid2) {
    centroid2[0] = h[0];
    centroid2[1] = h[1];
  }
  if (length) *length = h[2];
  return CVA_OK;
}

// mode 1: out = c - centroid(c); mode 2: out = c / curve_length(c)
int cva_center_or_normalize_host(const double* xy, int64_t n, int mode, double* out) {
  if (n < 1) return cva::err(CVA_INVALID_ARGUMENT, "curve: too few nodes");
  if (int rc = cva::have_device()) return rc;
  Buf a, o, st;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, xy, cb)) return rc;
  if (!o.alloc(cb) || !st.alloc(3 * sizeof(double))) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cva::di::stats_kernel<<<1, cva::di::kT, 0, cva::kS>>>((const double2*)a.p, n, (double*)st.p);
  double h[3];
  if (int rc = cva::down(h, st, sizeof(h))) return rc;
  if (mode == 2 && !(h[2] > 0.0)) return cva::err(CVA_INVALID_ARGUMENT, "curve: zero length");
  const double gx = mode == 1 ? h[0] : 0.0, gy = mode == 1 ? h[1] : 0.0, sc = mode == 2 ? 1.0 / h[2] : 1.0;
  cva::di::affine_kernel<<<(unsigned)((n + 255) / 256), 256, 0, cva::kS>>>((const double2*)a.p, n, gx, gy, sc, (double2*)o.p);
  return cva::down(out, o, cb);
}

int cva_arc_length_params_host(const double* xy, int64_t n, double* s, double* total) {
  if (n < 3) return cva::err(CVA_INVALID_ARGUMENT, "curve: too few nodes");
  if (int rc = cva::have_device()) return rc;
  Buf a, so, to, stt;
  if (int rc = cva::up(a, xy, sizeof(double2) * (size_t)n)) return rc;
  if (!so.alloc(sizeof(double) * (size_t)(n + 1)) || !to.alloc(sizeof(double)) || !stt.alloc(sizeof(int)))
    return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cva::di::arclen_kernel<<<1, cva::di::kT, 0, cva::kS>>>((const double2*)a.p, (int)n, (double*)so.p, (double*)to.p, (int*)stt.p);
  int bad = 0;
  if (int rc = cva::down(&bad, stt, sizeof(int))) return rc;
  if (bad) return cva::err(CVA_INVALID_ARGUMENT, "curve: coincident adjacent nodes");
  if (int rc = cva::down(s, so, sizeof(double) * (size_t)(n + 1))) return rc;
  return cva::down(total, to, sizeof(double));
}

int cva_spline_solve_host(const double* x, const double* y, int64_t n_knots, double* m) {
  if (n_knots < 4) return cva::err(CVA_INVALID_ARGUMENT, "spline: need at least 4 knots");
  const int n = (int)(n_knots - 1);
  if (n > cva::di::kT * cva::kMaxChunk) return cva::err(CVA_UNSUPPORTED, "spline: too many knots");
  if (int rc = cva::have_device()) return rc;
  Buf dx, dy, dm;
  if (int rc = cva::up(dx, x, sizeof(double) * (size_t)n_knots)) return rc;
  if (int rc = cva::up(dy, y, sizeof(double) * (size_t)n_knots)) return rc;
  if (!dm.alloc(sizeof(double) * (size_t)n_knots)) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  const size_t sm = sizeof(double) * (size_t)((n + 2) & ~1) + 2 * sizeof(double2) * (size_t)n +
                    sizeof(cva::ChunkEnds) * cva::di::kT;
  cudaFuncSetAttribute((const void*)cva::di::spline_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cva::di::spline_kernel<<<1, cva::di::kT, sm, cva::kS>>>((const double*)dx.p, (const double*)dy.p, n, (double*)dm.p);
  return cva::down(m, dm, sizeof(double) * (size_t)n_knots);
}

int cva_srv_transform_host(const double* xy, int64_t n, int center, double* q) {
  if (n < 1) return cva::err(CVA_INVALID_ARGUMENT, "srv: empty");
  if (int rc = cva::have_device()) return rc;
  Buf a, o;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, xy, cb)) return rc;
  if (!o.alloc(cb)) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cva::di::srv_kernel<<<1, cva::di::kT, 0, cva::kS>>>((const double2*)a.p, n, center, (double2*)o.p);
  return cva::down(q, o, cb);
}

// X_k, k < kcount, of the complex sequence x (n points); sign -1 forward, +1
// inverse; any n, O(n log n) (gfft.cu: radix 2 or Bluestein).
int cva_dft_host(const double* x_complex, int64_t n, int64_t kcount, int sign, double scale, double* out_complex) {
  if (n < 1 || kcount < 0 || kcount > n || (sign != 1 && sign != -1))
    return cva::err(CVA_INVALID_ARGUMENT, "fft: bad length");
  if (kcount == 0) return CVA_OK;
  if (int rc = cva::have_device()) return rc;
  Buf a, w;
  if (int rc = cva::up(a, x_complex, sizeof(double2) * (size_t)n)) return rc;
  if (!w.alloc(sizeof(double2) * (size_t)cva::gfft_workspace(n))) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cudaError_t e = cva::gfft((double2*)a.p, n, sign, (double2*)w.p, cva::kS);
  if (e != cudaSuccess) return cva::err(CVA_CUDA_ERROR, "fft launch", e);
  if (scale != 1.0) cva::di::scale_kernel<<<(unsigned)((kcount + 255) / 256), 256, 0, cva::kS>>>((double2*)a.p, kcount, scale);
  return cva::down(out_complex, a, sizeof(double2) * (size_t)kcount);
}

// A(m) for every shift m by FFT (correlation_all_shifts_fft, rigid_align.cpp:147-183).
int cva_correlation_fft_host(const double* c1, const double* c2, int64_t n, double* out4) {
  if (n < 1) return cva::err(CVA_INVALID_ARGUMENT, "correlation: empty");
  if (int rc = cva::have_device()) return rc;
  Buf a, b, o, w;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, c1, cb)) return rc;
  if (int rc = cva::up(b, c2, cb)) return rc;
  if (!o.alloc(sizeof(double) * 4 * (size_t)n) ||
      !w.alloc(sizeof(double2) * (size_t)cva::gfft_correlation_workspace(n)))
    return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cudaError_t e = cva::gfft_correlation((const double2*)a.p, (const double2*)b.p, n, (double*)o.p, (double2*)w.p,
                                        cva::kS);
  if (e != cudaSuccess) return cva::err(CVA_CUDA_ERROR, "correlation fft launch", e);
  return cva::down(out4, o, sizeof(double) * 4 * (size_t)n);
}

// ---- SRV / elastic utilities (srv.cpp:58-69 validation, :100-176)

namespace {
int check_reparam(const double* g, int64_t n) {  // validate_reparam (srv.cpp:58-69)
  if (n < 2) return cva::err(CVA_INVALID_ARGUMENT, "reparam: too few samples");
  if (std::abs(g[0]) > 1e-12 || std::abs(g[n] - 1.0) > 1e-12)
    return cva::err(CVA_INVALID_ARGUMENT, "reparam: endpoints must be 0 and 1");
  for (int64_t i = 0; i < n; ++i)
    if (g[i + 1] < g[i] - 1e-12) return cva::err(CVA_INVALID_ARGUMENT, "reparam: not monotone");
  return CVA_OK;
}
}  // namespace

int cva_apply_srv_action_host(const double* q, int64_t n, double t0, double theta, const double* gamma,
                              double* out) {
  if (n == 0) return cva::err(CVA_INVALID_ARGUMENT, "srv: empty");
  if (!std::isfinite(theta)) return cva::err(CVA_INVALID_ARGUMENT, "Rotation2: non-finite angle");
  if (int rc = check_reparam(gamma, n)) return rc;
  if (int rc = cva::have_device()) return rc;
  Buf a, g, o;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, q, cb)) return rc;
  if (int rc = cva::up(g, gamma, sizeof(double) * (size_t)(n + 1))) return rc;
  if (!o.alloc(cb)) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cudaError_t e = cva::launch_srv_action((const double2*)a.p, (int)n, t0, theta, (const double*)g.p, (double2*)o.p,
                                         cva::kS);
  if (e != cudaSuccess) return cva::err(CVA_CUDA_ERROR, "srv action launch", e);
  return cva::down(out, o, cb);
}

int cva_elastic_energy_host(const double* q1, const double* q2, int64_t n, double t0, double theta,
                            const double* gamma, double* out) {
  if (n == 0) return cva::err(CVA_INVALID_ARGUMENT, "srv: empty");
  if (!std::isfinite(theta)) return cva::err(CVA_INVALID_ARGUMENT, "Rotation2: non-finite angle");
  if (int rc = check_reparam(gamma, n)) return rc;
  if (int rc = cva::have_device()) return rc;
  Buf a, b, g, t, o;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, q1, cb)) return rc;
  if (int rc = cva::up(b, q2, cb)) return rc;
  if (int rc = cva::up(g, gamma, sizeof(double) * (size_t)(n + 1))) return rc;
  if (!t.alloc(sizeof(double) * (size_t)n) || !o.alloc(sizeof(double)))
    return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cudaError_t e = cva::launch_elastic_energy((const double2*)a.p, (const double2*)b.p, (int)n, t0, theta,
                                             (const double*)g.p, (double*)t.p, (double*)o.p, cva::kS);
  if (e != cudaSuccess) return cva::err(CVA_CUDA_ERROR, "elastic energy launch", e);
  return cva::down(out, o, sizeof(double));
}

int cva_dp_step_cost_host(const double* q1, const double* q2, int64_t n, int i0, int j0, int di, int dj,
                          double* out) {
  if (di < 1 || dj < 1) return cva::err(CVA_INVALID_ARGUMENT, "dp: step increments must be positive");
  if (n < 1 || i0 < 0 || j0 < 0) return cva::err(CVA_INVALID_ARGUMENT, "dp: bad step");
  if (int rc = cva::have_device()) return rc;
  Buf a, b, o;
  const size_t cb = sizeof(double2) * (size_t)n;
  if (int rc = cva::up(a, q1, cb)) return rc;
  if (int rc = cva::up(b, q2, cb)) return rc;
  if (!o.alloc(sizeof(double))) return cva::err(CVA_BAD_ALLOC, "device allocation failed");
  cudaError_t e = cva::launch_dp_step_cost((const double2*)a.p, (const double2*)b.p, (int)n, i0, j0, di, dj,
                                           (double*)o.p, cva::kS);
  if (e != cudaSuccess) return cva::err(CVA_CUDA_ERROR, "dp step launch", e);
  return cva::down(out, o, sizeof(double));
}

}  // extern "C"
