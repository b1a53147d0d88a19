// Large-N alignment (BASELINE config C3: N = 65536; any N whose transform
// length exceeds the shared-memory pair kernels, e.g. the reference tests'
// N = 4097). A curve is 1 MB at N = 65536, beyond one CTA's shared memory, so
// the three transforms run as batched multi-pass radix-16 Stockham kernels over
// global buffers; the host processes pairs in chunks whose working set stays
// resident in the 126 MB L2, so HBM sees the inputs, the aligned output and
// little else.
//
// Per chunk of P pairs (M = fft_len(N), data in the length-M padded form of
// pairfft.cuh: a = [z1', 0...], b = [z2', z2', 0...]):
//   stats_partial/final centroid / 1/length of each curve (curve.cpp:27-48) when
//                     the preprocess (resample=false) is fused, else identity
//   lpass<kLoadA/B>   first radix-16 pass reading the curves, normalising on load
//   lpass<kPlain>     remaining passes of the two forward transforms
//   lpass<kProduct>   first pass of the correlation transform on Z1 conj(Z2)
//   lmax_kernel       per-block max of |F|^2
//   lcand_kernel      global max, reference tie band, per-block smallest index
//   lpick_kernel      smallest index over blocks -> shift, rotation, energy
//   aligned_kernel    aligned[l] = R(theta) z2'[(l + m) mod N]
#include <cuda_runtime.h>

#include <climits>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "fft.cuh"
#include "largen.h"
#include "pairfft.cuh"

namespace cva {
namespace ln {

constexpr int kT = 256;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

template <int R>
__device__ __forceinline__ void dft_any(double2* v) {
  dft_r<R>(v);
}

enum Load { kPlain = 0, kLoadA = 1, kLoadB = 2, kProduct = 3 };

struct CurveNorm {
  double2 g;
  double sc;
};

// One Stockham pass of radix R over `nseq` sequences of length M (stride M).
// kLoadA / kLoadB: the pass reads curve c (N nodes) through its normalisation
// into the padded length-M form (first pass only, Ns = 1). kProduct: reads
// x1[k] conj(x2[k]) of two spectra (first pass only).
// Sum |z'|^2 of each curve (rigid_align.cpp:23-27) comes from the first pass
// of its transform: every load pass block writes one partial to sqp[block]
// (blocks never straddle sequences: M / R is a multiple of kT), and the pick
// kernel adds the partials of a sequence in a fixed order.
template <int R, int kMode>
__global__ void __launch_bounds__(kT)
    lpass(const double2* __restrict__ in, const double2* __restrict__ in2, double2* out, int M, int N,
          int Ns, const double2* __restrict__ tw, const CurveNorm* __restrict__ norm, int64_t nseq,
          double* sqp) {
  const int nb = M / R;
  const int64_t gid = (int64_t)blockIdx.x * kT + threadIdx.x;
  const int64_t seq = gid / nb;
  if (seq >= nseq) return;
  const int j = (int)(gid - seq * nb);
  const int jm = j & (Ns - 1);
  double2 v[R];
  if (kMode == kLoadA || kMode == kLoadB) {
    const double2* z = in + seq * N;
    const CurveNorm cn = norm[seq];
    const int lim = (kMode == kLoadA || M == N) ? N : 2 * N;
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = j + r * nb;
      if (i < lim) {
        const double2 q = __ldg(&z[i < N ? i : i - N]);
        v[r] = make_double2((q.x - cn.g.x) * cn.sc, (q.y - cn.g.y) * cn.sc);
        if (i < N) sq = fma(v[r].x, v[r].x, fma(v[r].y, v[r].y, sq));
      } else {
        v[r] = make_double2(0.0, 0.0);
      }
    }
    __shared__ double2 red[64];
    sq = block_sum(sq, red);
    if (threadIdx.x == 0) sqp[blockIdx.x] = sq;
  } else if (kMode == kProduct) {
    const double2* a = in + seq * M;
    const double2* b = in2 + seq * M;
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = cmulconj(__ldg(&a[j + r * nb]), __ldg(&b[j + r * nb]));
  } else {
    const double2* x = in + seq * M;
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = __ldg(&x[j + r * nb]);
  }
  if (Ns > 1) {
    const int tws = M / (Ns * R);
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[(int64_t)r * jm * tws]));
  }
  dft_any<R>(v);
  double2* o = out + seq * M;
  const int base = (j - jm) * R + jm;
#pragma unroll
  for (int r = 0; r < R; ++r) o[base + r * Ns] = v[dft_slot<R>(r)];
}

// Per-curve statistics, two deterministic stages (no atomics):
// stats_partial: grid (kStatBlocks, curves); each block sums its strided slice
//   of the curve: sum z, polygon edge lengths, and a non-finite flag.
// stats_final: one warp per curve adds the block partials in a fixed order and
//   forms the centroid and 1/length (center then normalize, curve.cpp:27-48).
//   The length is taken on the uncentred nodes (differences are translation
//   invariant; the reference centres first, a rounding-level difference).
constexpr int kStatBlocks = 32;

__global__ void __launch_bounds__(kT)
    stats_partial(const double2* __restrict__ curves, int N, double4* part) {
  __shared__ double2 red[64];
  const double2* z = curves + (int64_t)blockIdx.y * N;
  double2 acc = make_double2(0, 0);
  double len = 0.0;
  int nf = 0;
  for (int i = blockIdx.x * kT + threadIdx.x; i < N; i += kStatBlocks * kT) {
    const double2 p0 = __ldg(&z[i]), p1 = __ldg(&z[i + 1 == N ? 0 : i + 1]);
    nf |= !(isfinite(p0.x) && isfinite(p0.y));
    acc = cadd(acc, p0);
    const double dx = p1.x - p0.x, dy = p1.y - p0.y;
    len += sqrt(fma(dx, dx, dy * dy));
  }
  nf = block_or(nf, red);
  acc = block_sum2(acc, red);
  __syncthreads();
  len = block_sum(len, red);
  if (threadIdx.x == 0)
    part[(int64_t)blockIdx.y * kStatBlocks + blockIdx.x] = make_double4(acc.x, acc.y, len, nf ? 1.0 : 0.0);
}

__global__ void stats_final(const double4* __restrict__ part, int64_t curves, int N, int normalize,
                            CurveNorm* norm, int32_t* bad) {
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (c >= curves) return;
  double4 v = lane < kStatBlocks ? part[c * kStatBlocks + lane] : make_double4(0, 0, 0, 0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    v.z += __shfl_xor_sync(0xffffffffu, v.z, o);
    v.w += __shfl_xor_sync(0xffffffffu, v.w, o);
  }
  if (lane == 0) {
    CurveNorm cn{make_double2(0.0, 0.0), 1.0};
    int b = v.w != 0.0;
    if (normalize) {
      const double invn = 1.0 / (double)N;
      cn.g = make_double2(invn * v.x, invn * v.y);
      b |= !(v.z > 0.0);
      cn.sc = 1.0 / v.z;
    }
    norm[c] = cn;
    bad[c] = b;
  }
}

// per-block max of |F|^2 over the first N lags; grid (blocks_per_seq, nseq)
__global__ void __launch_bounds__(kT)
    lmax_kernel(const double2* __restrict__ F, int M, int N, double* bmax) {
  __shared__ double2 red[64];
  const double2* f = F + (int64_t)blockIdx.y * M;
  double m = -1.0;
  for (int k = blockIdx.x * kT + threadIdx.x; k < N; k += gridDim.x * kT) {
    const double2 v = __ldg(&f[k]);
    m = fmax(m, fma(v.x, v.x, v.y * v.y));
  }
  m = block_max(m, red);
  if (threadIdx.x == 0) bmax[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = m;
}

// Two-phase argmax with the reference's tie band (rigid_align.cpp:31-61) on
// |D| = |F| / M, spread over the same blocks as lmax_kernel:
// lcand_kernel: each block reduces the per-block maxima of its pair to the
//   global max (fixed order), forms the band threshold and reports its smallest
//   index in the band (INT_MAX if none).
__global__ void __launch_bounds__(kT)
    lcand_kernel(const double2* __restrict__ F, int M, int N, const double* __restrict__ bmax, int* bcand) {
  __shared__ double2 red[64];
  const int64_t p = blockIdx.y;
  const int nblk = gridDim.x;
  double best2 = -1.0;
  for (int b = threadIdx.x; b < nblk; b += kT) best2 = fmax(best2, bmax[p * nblk + b]);
  best2 = block_max(best2, red);
  const double best = sqrt(best2) / (double)M;
  const double thr = best - pf::kTieRelTol * fmax(1.0, fabs(best));
  const double thrM = thr * (double)M;
  const double thr2 = thr > 0.0 ? thrM * thrM : -1.0;
  const double2* f = F + p * M;
  int cand = INT_MAX;
  for (int k = blockIdx.x * kT + threadIdx.x; k < N; k += nblk * kT) {
    const double2 v = __ldg(&f[k]);
    if (fma(v.x, v.x, v.y * v.y) >= thr2) {
      cand = k;
      break;
    }
  }
  cand = block_min_int(cand, red);
  if (threadIdx.x == 0) bcand[p * nblk + blockIdx.x] = isfinite(best) && best2 >= 0.0 ? cand : INT_MAX;
}

// lpick_kernel: one warp per pair: smallest candidate -> shift, rotation,
// trace, energy (energy identity, rigid_align.cpp:56-59).
__global__ void lpick_kernel(const double2* __restrict__ F, int M, int N, const int* __restrict__ bcand,
                             int nblk, const double* __restrict__ sq1, const double* __restrict__ sq2, int sqn,
                             const int32_t* bad1, const int32_t* bad2, int64_t pairs, cva_alignment* out,
                             double2* rot) {
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (p >= pairs) return;
  int m = INT_MAX;
  for (int b = lane; b < nblk; b += 32) m = min(m, bcand[p * nblk + b]);
  double s1 = 0.0, s2 = 0.0;
  for (int b = lane; b < sqn; b += 32) {
    s1 += sq1[p * sqn + b];
    s2 += sq2[p * sqn + b];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane != 0) return;
  const double invM = 1.0 / (double)M, invN = 1.0 / (double)N;
  cva_alignment r;
  if (bad1[p] || bad2[p] || m == INT_MAX) {
    r.shift = 0;
    r.t0 = 0.0;
    r.theta = r.trace = r.energy = qnan();
    r.degenerate = 0;
    r.status = CVA_INVALID_ARGUMENT;
    rot[p] = make_double2(qnan(), qnan());
  } else {
    const double2 v = F[p * M + m];
    const double a2 = fma(v.x, v.x, v.y * v.y);
    const double trace = sqrt(a2) * invM;
    const int degenerate = trace == 0.0;
    double e = invN * (s1 + s2) - 2.0 * invN * trace;
    if (e < 0.0) e = 0.0;
    r.shift = m;
    r.t0 = (double)m / (double)N;
    r.theta = degenerate ? 0.0 : atan2(-v.y, v.x);
    r.trace = trace;
    r.energy = e;
    r.degenerate = degenerate;
    r.status = CVA_OK;
    const double ia = degenerate ? 0.0 : 1.0 / sqrt(a2);
    rot[p] = degenerate ? make_double2(1.0, 0.0) : make_double2(v.x * ia, -v.y * ia);
  }
  out[p] = r;
}

// aligned[l] = R(theta) z2'[(l + m) mod N]; grid (blocks, pairs)
__global__ void __launch_bounds__(kT)
    aligned_kernel(const double2* __restrict__ c2, int N, const CurveNorm* __restrict__ norm2,
                   const cva_alignment* __restrict__ res, const double2* __restrict__ rot, double2* aligned) {
  const int64_t p = blockIdx.y;
  const int64_t m = res[p].shift;
  const double2 r = rot[p];
  const CurveNorm cn = norm2[p];
  const double2* z = c2 + p * N;
  double2* a = aligned + p * N;
  for (int l = blockIdx.x * kT + threadIdx.x; l < N; l += gridDim.x * kT) {
    int64_t j = l + m;
    if (j >= N) j -= N;
    const double2 q = __ldg(&z[j]);
    const double2 v = make_double2((q.x - cn.g.x) * cn.sc, (q.y - cn.g.y) * cn.sc);
    a[l] = make_double2(fma(r.x, v.x, r.y * v.y), fma(-r.y, v.x, r.x * v.y));
  }
}

}  // namespace ln

// ------------------------------------------------------------------ host

namespace {

template <int R, int kMode>
cudaError_t pass(const double2* in, const double2* in2, double2* out, int M, int N, int Ns,
                 const double2* tw, const ln::CurveNorm* norm, int64_t nseq, double* sqp, cudaStream_t s) {
  const int64_t threads = nseq * (M / R);
  ln::lpass<R, kMode><<<(unsigned)((threads + ln::kT - 1) / ln::kT), ln::kT, 0, s>>>(in, in2, out, M, N, Ns, tw,
                                                                                     norm, nseq, sqp);
  return cudaGetLastError();
}

template <int kMode>
cudaError_t pass_r(int R, const double2* in, const double2* in2, double2* out, int M, int N, int Ns,
                   const double2* tw, const ln::CurveNorm* norm, int64_t nseq, double* sqp, cudaStream_t s) {
  switch (R) {
    case 16: return pass<16, kMode>(in, in2, out, M, N, Ns, tw, norm, nseq, sqp, s);
    case 8: return pass<8, kMode>(in, in2, out, M, N, Ns, tw, norm, nseq, sqp, s);
    case 4: return pass<4, kMode>(in, in2, out, M, N, Ns, tw, norm, nseq, sqp, s);
    default: return pass<2, kMode>(in, in2, out, M, N, Ns, tw, norm, nseq, sqp, s);
  }
}

// Forward FFT of nseq sequences: first pass in mode `first` (from `src`), the
// rest ping-ponging a -> b. Returns the buffer holding the spectra.
template <int kFirst>
cudaError_t fft_many(const double2* src, const double2* src2, double2* a, double2* b, int M, int N,
                     const double2* tw, const ln::CurveNorm* norm, int64_t nseq, double* sqp, cudaStream_t s,
                     double2** result) {
  int Ns = 1;
  double2* dst = a;
  double2* other = b;
  bool first = true;
  cudaError_t e = cudaSuccess;
  while (Ns < M && e == cudaSuccess) {
    const int rem = M / Ns;
    const int R = rem >= 16 ? 16 : rem;
    if (first)
      e = pass_r<kFirst>(R, src, src2, dst, M, N, Ns, tw, norm, nseq, sqp, s);
    else
      e = pass_r<ln::kPlain>(R, other, nullptr, dst, M, N, Ns, tw, norm, nseq, nullptr, s);
    first = false;
    Ns *= R;
    double2* t = dst;
    dst = other;
    other = t;
  }
  *result = other;
  return e;
}

struct Layout {
  int M, nblk, sqn;
};

Layout layout(int N) {
  Layout L;
  L.M = pf::fft_len(N);
  L.nblk = (N + ln::kT * 4 - 1) / (ln::kT * 4);
  L.sqn = L.M / 16 / ln::kT;  // first-pass blocks per sequence (M >= 4096)
  return L;
}

}  // namespace

size_t large_workspace_bytes(int64_t chunk, int N) {
  const Layout L = layout(N);
  const size_t seq = sizeof(double2) * (size_t)L.M;
  return 4 * seq * (size_t)chunk + 4096                                        // spectra ping-pong
         + 2 * sizeof(ln::CurveNorm) * (size_t)chunk                           // norms
         + 2 * sizeof(double4) * (size_t)(chunk * ln::kStatBlocks)             // stat partials
         + 2 * sizeof(double) * (size_t)(chunk * L.sqn)                        // |z'|^2 partials
         + 2 * sizeof(int32_t) * (size_t)chunk                                 // bad flags
         + sizeof(double2) * (size_t)chunk                                     // rotations
         + (sizeof(double) + sizeof(int)) * (size_t)(chunk * L.nblk) + 4096;   // argmax partials
}

int64_t large_chunk_pairs(int N) {
  // ~96 MB working set: 4 spectra of 16 M bytes per pair at N = 65536
  const int M = pf::fft_len(N);
  const int64_t per = 4 * (int64_t)sizeof(double2) * M;
  int64_t c = (96ll << 20) / per;
  return c < 1 ? 1 : c;
}

cudaError_t launch_large_align(const double2* c1, const double2* c2, int64_t pairs, int N, int normalize,
                               const double2* tw, cva_alignment* out, double2* aligned, void* ws,
                               int64_t chunk, cudaStream_t s) {
  const Layout Ly = layout(N);
  const int M = Ly.M, nblk = Ly.nblk, sqn = Ly.sqn;
  char* w = (char*)ws;
  auto take = [&](size_t bytes) {
    char* p = w;
    w += (bytes + 255) & ~size_t(255);
    return (void*)p;
  };
  double2* A = (double2*)take(sizeof(double2) * (size_t)M * chunk);
  double2* B = (double2*)take(sizeof(double2) * (size_t)M * chunk);
  double2* C = (double2*)take(sizeof(double2) * (size_t)M * chunk);
  double2* D = (double2*)take(sizeof(double2) * (size_t)M * chunk);
  ln::CurveNorm* n1 = (ln::CurveNorm*)take(sizeof(ln::CurveNorm) * chunk);
  ln::CurveNorm* n2 = (ln::CurveNorm*)take(sizeof(ln::CurveNorm) * chunk);
  double4* sp1 = (double4*)take(sizeof(double4) * chunk * ln::kStatBlocks);
  double4* sp2 = (double4*)take(sizeof(double4) * chunk * ln::kStatBlocks);
  double* q1 = (double*)take(sizeof(double) * chunk * sqn);
  double* q2 = (double*)take(sizeof(double) * chunk * sqn);
  int32_t* b1 = (int32_t*)take(sizeof(int32_t) * chunk);
  int32_t* b2 = (int32_t*)take(sizeof(int32_t) * chunk);
  double2* rot = (double2*)take(sizeof(double2) * chunk);
  double* bmax = (double*)take(sizeof(double) * chunk * nblk);
  int* bcand = (int*)take(sizeof(int) * chunk * nblk);
  cudaError_t e = cudaSuccess;
  for (int64_t p0 = 0; p0 < pairs && e == cudaSuccess; p0 += chunk) {
    const int64_t P = pairs - p0 < chunk ? pairs - p0 : chunk;
    const double2* z1 = c1 + p0 * N;
    const double2* z2 = c2 + p0 * N;
    ln::stats_partial<<<dim3(ln::kStatBlocks, (unsigned)P), ln::kT, 0, s>>>(z1, N, sp1);
    ln::stats_partial<<<dim3(ln::kStatBlocks, (unsigned)P), ln::kT, 0, s>>>(z2, N, sp2);
    ln::stats_final<<<(unsigned)((P + 7) / 8), 256, 0, s>>>(sp1, P, N, normalize, n1, b1);
    ln::stats_final<<<(unsigned)((P + 7) / 8), 256, 0, s>>>(sp2, P, N, normalize, n2, b2);
    double2 *Z1 = nullptr, *Z2 = nullptr, *F = nullptr;
    e = fft_many<ln::kLoadA>(z1, nullptr, A, B, M, N, tw, n1, P, q1, s, &Z1);
    if (e == cudaSuccess) e = fft_many<ln::kLoadB>(z2, nullptr, C, D, M, N, tw, n2, P, q2, s, &Z2);
    if (e != cudaSuccess) break;
    double2* fa = (Z1 == A) ? B : A;  // free buffers for the correlation transform
    double2* fb = (Z2 == C) ? D : C;
    e = fft_many<ln::kProduct>(Z1, Z2, fa, fb, M, N, tw, nullptr, P, nullptr, s, &F);
    if (e != cudaSuccess) break;
    ln::lmax_kernel<<<dim3((unsigned)nblk, (unsigned)P), ln::kT, 0, s>>>(F, M, N, bmax);
    ln::lcand_kernel<<<dim3((unsigned)nblk, (unsigned)P), ln::kT, 0, s>>>(F, M, N, bmax, bcand);
    ln::lpick_kernel<<<(unsigned)((P + 7) / 8), 256, 0, s>>>(F, M, N, bcand, nblk, q1, q2, sqn, b1, b2, P, out + p0,
                                                             rot);
    if (aligned)
      ln::aligned_kernel<<<dim3((unsigned)((N + 4 * ln::kT - 1) / (4 * ln::kT)), (unsigned)P), ln::kT, 0, s>>>(
          z2, N, n2, out + p0, rot, aligned + p0 * N);
    e = cudaGetLastError();
  }
  return e;
}

size_t curve_stats_workspace(int64_t curves) {
  return sizeof(double4) * (size_t)(curves * ln::kStatBlocks) + 256;
}

cudaError_t launch_curve_stats(const double2* curves, int64_t count, int N, int normalize, double4* norm,
                               int32_t* bad, void* ws, cudaStream_t s) {
  static_assert(sizeof(ln::CurveNorm) == sizeof(double4), "CurveNorm is (gx, gy, sc, pad)");
  double4* part = (double4*)ws;
  ln::stats_partial<<<dim3(ln::kStatBlocks, (unsigned)count), ln::kT, 0, s>>>(curves, N, part);
  ln::stats_final<<<(unsigned)((count + 7) / 8), 256, 0, s>>>(part, count, N, normalize, (ln::CurveNorm*)norm, bad);
  return cudaGetLastError();
}

}  // namespace cva
