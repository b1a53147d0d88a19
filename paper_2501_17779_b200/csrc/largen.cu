#include <algorithm>
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

// curves y < P2 come from `curves`, the rest from `curves2` (one launch for
// both curves of a chunk of pairs); P2 = gridDim.y when curves2 is null.
__global__ void __launch_bounds__(kT)
    stats_partial(const double2* __restrict__ curves, int N, double4* part,
                  const double2* __restrict__ curves2 = nullptr, int64_t P2 = 0) {
  __shared__ double2 red[64];
  const int64_t y = blockIdx.y;
  const double2* z = (curves2 && y >= P2) ? curves2 + (y - P2) * N : curves + y * N;
  double2 acc = make_double2(0, 0);
  double len = 0.0;
  int nf = 0;
  // kU strided elements per thread per round, all loads issued before use (the
  // pass streams the chunk's curves from HBM: memory-level parallelism)
  constexpr int kU = 4;
  constexpr int kS = kStatBlocks * kT;
  for (int i0 = blockIdx.x * kT + threadIdx.x; i0 < N; i0 += kU * kS) {
    double2 p0[kU], p1[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * kS;
      if (i < N) {
        p0[u] = __ldg(&z[i]);
        p1[u] = __ldg(&z[i + 1 == N ? 0 : i + 1]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (i0 + u * kS < N) {
        nf |= !(isfinite(p0[u].x) && isfinite(p0[u].y));
        acc = cadd(acc, p0[u]);
        const double dx = p1[u].x - p0[u].x, dy = p1[u].y - p0[u].y;
        len += sqrt(fma(dx, dx, dy * dy));
      }
    }
  }
  nf = block_or(nf, red);
  acc = block_sum2(acc, red);
  __syncthreads();
  len = block_sum(len, red);
  if (threadIdx.x == 0)
    part[(int64_t)blockIdx.y * kStatBlocks + blockIdx.x] = make_double4(acc.x, acc.y, len, nf ? 1.0 : 0.0);
}

// One warp: curve c's partials -> its CurveNorm and bad flag (every lane
// returns them; fixed reduction order, so every caller forms the same values).
__device__ __forceinline__ CurveNorm norm_of(const double4* __restrict__ part, int64_t c, int N, int normalize,
                                             int* bad) {
  const int lane = threadIdx.x & 31;
  double4 v = lane < kStatBlocks ? part[c * kStatBlocks + lane] : make_double4(0, 0, 0, 0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    v.z += __shfl_xor_sync(0xffffffffu, v.z, o);
    v.w += __shfl_xor_sync(0xffffffffu, v.w, o);
  }
  CurveNorm cn{make_double2(0.0, 0.0), 1.0};
  int b = v.w != 0.0;
  if (normalize) {
    const double invn = 1.0 / (double)N;
    cn.g = make_double2(invn * v.x, invn * v.y);
    b |= !(v.z > 0.0);
    cn.sc = 1.0 / v.z;
  }
  *bad = b;
  return cn;
}

__global__ void stats_final(const double4* __restrict__ part, int64_t curves, int N, int normalize,
                            CurveNorm* norm, int32_t* bad) {
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (c >= curves) return;
  int b;
  const CurveNorm cn = norm_of(part, c, N, normalize, &b);
  if (lane == 0) {
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
    lcand_kernel(const double2* __restrict__ F, int M, int N, const double* __restrict__ bmax, int nbmax,
                 int* bcand) {
  __shared__ double2 red[64];
  const int64_t p = blockIdx.y;
  const int nblk = gridDim.x;
  double best2 = -1.0;
  for (int b = threadIdx.x; b < nbmax; b += kT) best2 = fmax(best2, bmax[p * nbmax + b]);
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
  constexpr int kU = 4;  // loads of kU rounds in flight before their stores
  const int step = gridDim.x * kT;
  for (int l0 = blockIdx.x * kT + threadIdx.x; l0 < N; l0 += kU * step) {
    double2 q[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int l = l0 + u * step;
      int64_t j = l + m;
      if (j >= N) j -= N;
      q[u] = l < N ? __ldg(&z[j]) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int l = l0 + u * step;
      if (l < N) {
        const double2 v = make_double2((q[u].x - cn.g.x) * cn.sc, (q[u].y - cn.g.y) * cn.sc);
        a[l] = make_double2(fma(r.x, v.x, r.y * v.y), fma(-r.y, v.x, r.x * v.y));
      }
    }
  }
}

// ----------------------------------------------------------- four-step path
//
// For 4096 <= M <= 65536 the three transforms run as M = M1 x M2 four-step
// FFTs (M1, M2 in {64, 128, 256}) with every length-M1 / M2 sub-transform done
// by one warp on a shared-memory vector, so a correlation costs three passes
// over the data instead of twelve radix-16 passes:
//   f1_kernel  per curve, column FFTs (length M1, stride M2) of the normalised
//              curve + twiddle W_M^{n2 k1}  -> U[k1][n2]
//   fp_kernel  per pair and row k1: row FFTs of U1 and U2 (the spectra
//              Z[k1 + M1 k2]), the product Z1 conj(Z2), its row FFT and twiddle
//              W_M^{k1 m2}                   -> G[k1][m2]
//   p2_kernel  column FFTs of G: F[m2 + M2 m1] in natural order, + block max
//   pick_kernel tie-broken argmax + shift / rotation / energy (one CTA per pair)
// f1_kernel also reduces the stats partials into each curve's norm (no
// stats_final launch): per chunk, stats_partial, f1, fp, p2, pick, aligned.
// The product's transform is a forward FFT over the spectral index
// k = k1 + M1 k2 (D = conj(FFT(Z1 conj Z2)) / M, as in pairfft.cuh), which is
// why the second step of the forward transforms and the first of the third
// share one pass and the spectra are never stored.
namespace fs {
constexpr int kT = 256;  // 8 warps, one sub-FFT each
constexpr int kCT = 8;   // columns per column tile (128-byte row segments)
constexpr int kRT = 8;   // rows per row tile

__device__ __forceinline__ int padL(int i) { return i + (i >> 3); }
// shared vector stride: padded length + 1 so the 8 vectors of a tile start in
// different banks
template <int L>
__host__ __device__ constexpr int vstride() {
  return L + L / 8 + 1;
}

template <int L, int Ns>
__host__ __device__ constexpr int radix_at() {
  return pf::plan_radix_warp(L, Ns);  // the plan the pass twiddle tables are laid out for
}

// One in-place Stockham pass of radix R on a length-L shared vector by one warp.
// tw: the length-L table of get_twiddles (twstride 1); the pass reads its
// twiddles W_L^(r jm L/(Ns R)) from the table's one-warp pass tables
// ([r - 1][jm], pairfft.cuh ptw_off_warp: consecutive entries per warp load).
template <int L, int R, int Ns>
__device__ __forceinline__ void wpass(double2* x, const double2* __restrict__ tw, int twstride, int lane) {
  constexpr int nb = L / R;
  constexpr int B = (nb + 31) / 32;
  (void)twstride;  // always 1: sub-transform tables of their own length
  const double2* __restrict__ pt = tw + pf::ptw_off_warp(L, Ns);
  double2 v[B][R];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = lane + 32 * b;
    if (nb % 32 == 0 || j < nb) {
      const int jm = j & (Ns - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][r] = x[padL(j + r * nb)];
      if (Ns > 1) pf::twiddle<R>(v[b], pt, Ns, jm);  // (W^3, W^5..7 from W^1, W^2, W^4)
    }
  }
  __syncwarp();
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = lane + 32 * b;
    if (nb % 32 == 0 || j < nb) {
      const int jm = j & (Ns - 1);
      dft_r<R>(v[b]);
      const int base = (j - jm) * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) x[padL(base + r * Ns)] = v[b][dft_slot<R>(r)];
    }
  }
  __syncwarp();
}

// W_M^e for e < M from two short tables (L1-resident): W_M^(256 h + l) =
// hi[h] * lo[l], hi = W_{M/256}, lo = W_M^l (l < 256). One extra rounding
// against the direct table entry.
__device__ __forceinline__ double2 tw_m(const double2* __restrict__ lo, const double2* __restrict__ hi, int e) {
  return cmul(__ldg(&hi[e >> 8]), __ldg(&lo[e & 255]));
}

template <int L, int Ns = 1>
__device__ __forceinline__ void wfft(double2* x, const double2* __restrict__ tw, int twstride, int lane) {
  constexpr int R = radix_at<L, Ns>();
  wpass<L, R, Ns>(x, tw, twstride, lane);
  if constexpr (Ns * R < L) wfft<L, Ns * R>(x, tw, twstride, lane);
}

// Column pass of the forward transforms. grid (M2 / kCT, 2 P): sequence s < P is
// curve 1 of pair s (the a = [z1', 0...] form), s >= P curve 2 of pair s - P
// (b = [z2', z2', 0...]). Writes U[s][k1 M2 + n2] and sum |z'|^2 partials.
// The curve's CurveNorm comes from the stats partials (stats_final's reduction,
// done by warp 0 of every CTA of the curve; the first CTA also stores it and the
// bad flag for the pick and aligned-output kernels).
template <int M1>
__global__ void __launch_bounds__(kT)
    f1_kernel(const double2* __restrict__ z1, const double2* __restrict__ z2, int64_t P, int N, int M2,
              const double2* __restrict__ twS, const double2* __restrict__ lo, const double2* __restrict__ hi,
              const double4* __restrict__ part, int normalize, CurveNorm* norm, int32_t* bad, double2* U,
              double* sq1, double* sq2) {
  constexpr int VS = vstride<M1>();
  __shared__ __align__(16) double2 sm[kCT * VS];
  __shared__ double2 red[64];
  __shared__ CurveNorm s_cn;
  const int M = M1 * M2;
  const int64_t sidx = blockIdx.y;
  const bool second = sidx >= P;
  const int64_t p = second ? sidx - P : sidx;
  const double2* z = (second ? z2 : z1) + p * N;
  const int lim = (!second || M == N) ? N : 2 * N;
  const int c0 = blockIdx.x * kCT;
  constexpr int kLd = M1 * kCT / kT;
  double2 q[kLd];  // the tile's nodes, all loads in flight before the norm is formed
#pragma unroll
  for (int it = 0; it < kLd; ++it) {
    const int idx = threadIdx.x + it * kT;
    const int n = M2 * (idx / kCT) + c0 + idx % kCT;
    q[it] = n < lim ? __ldg(&z[n < N ? n : n - N]) : make_double2(0.0, 0.0);
  }
  if (threadIdx.x < 32) {  // curve sidx: curve 1s then curve 2s, as stats_partial numbers them
    int b;
    const CurveNorm c = norm_of(part, sidx, N, normalize, &b);
    if (threadIdx.x == 0) {
      s_cn = c;
      if (blockIdx.x == 0) {
        norm[sidx] = c;
        bad[sidx] = b;
      }
    }
  }
  __syncthreads();
  const CurveNorm cn = s_cn;
  double sq = 0.0;
#pragma unroll
  for (int it = 0; it < kLd; ++it) {
    const int idx = threadIdx.x + it * kT;
    const int n1i = idx / kCT, c = idx % kCT;
    const int n = M2 * n1i + c0 + c;
    double2 v = make_double2(0.0, 0.0);
    if (n < lim) {
      v = make_double2((q[it].x - cn.g.x) * cn.sc, (q[it].y - cn.g.y) * cn.sc);
      if (n < N) sq = fma(v.x, v.x, fma(v.y, v.y, sq));
    }
    sm[c * VS + padL(n1i)] = v;
  }
  sq = block_sum(sq, red);  // syncs the tile too
  if (threadIdx.x == 0) (second ? sq2 : sq1)[p * gridDim.x + blockIdx.x] = sq;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  wfft<M1>(sm + w * VS, twS, 1, lane);
  __syncthreads();
  double2* u = U + sidx * (int64_t)M;
  // a thread's column n2 is fixed and its k1 advance by kT / kCT per round, so
  // W_M^(n2 k1) is a geometric sequence: two table reads per thread instead of
  // two scattered reads per element (rounding drift <= a few ulps over the
  // M1 kCT / kT rounds)
  const int cn2 = c0 + (int)threadIdx.x % kCT;
  const int k10 = (int)threadIdx.x / kCT;
  double2 wt = tw_m(lo, hi, cn2 * k10);
  const double2 wstep = tw_m(lo, hi, (cn2 * (kT / kCT)) & (M - 1));
#pragma unroll
  for (int it = 0; it < M1 * kCT / kT; ++it) {
    const int k1 = k10 + it * (kT / kCT);
    u[(int64_t)k1 * M2 + cn2] = cmul(sm[(cn2 - c0) * VS + padL(k1)], wt);
    wt = cmul(wt, wstep);
  }
}

// Row pass: per pair p and rows k1 in [r0, r0 + kRT): spectra rows of both
// curves, product, its row FFT and twiddle. grid (M1 / kRT, P).
template <int M2>
__global__ void __launch_bounds__(kT, 2)
    fp_kernel(const double2* __restrict__ U, int64_t P, int M1, const double2* __restrict__ twS,
              const double2* __restrict__ lo, const double2* __restrict__ hi, double2* G) {
  constexpr int VS = vstride<M2>();
  extern __shared__ __align__(16) double2 smv[];  // 2 kRT vectors
  const int M = M1 * M2;
  const int64_t p = blockIdx.y;
  const int r0 = blockIdx.x * kRT;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp w: spectra rows r0 + w of curve 1 (vector w) and of curve 2 (vector kRT + w)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double2* u = U + (h ? P + p : p) * (int64_t)M + (int64_t)(r0 + w) * M2;
    double2* x = smv + (h * kRT + w) * VS;
    double2 q[M2 / 32];  // the row's loads in flight before the shared stores
#pragma unroll
    for (int i0 = 0; i0 < M2; i0 += 32) q[i0 / 32] = __ldg(&u[i0 + lane]);
#pragma unroll
    for (int i0 = 0; i0 < M2; i0 += 32) x[padL(i0 + lane)] = q[i0 / 32];
    __syncwarp();
    wfft<M2>(x, twS, 1, lane);
  }
  // product Z1 conj(Z2) (same warp owns both rows), its row FFT, twiddle W_M^{k1 m2}
  double2* x = smv + w * VS;
  const double2* y = smv + (kRT + w) * VS;
#pragma unroll
  for (int i0 = 0; i0 < M2; i0 += 32) x[padL(i0 + lane)] = cmulconj(x[padL(i0 + lane)], y[padL(i0 + lane)]);
  __syncwarp();
  wfft<M2>(x, twS, 1, lane);
  const int k1 = r0 + w;
  double2* g = G + p * (int64_t)M + (int64_t)k1 * M2;
  // W_M^(k1 (i0 + lane)): geometric in i0 (step W_M^(32 k1)), see f1_kernel
  double2 wt = tw_m(lo, hi, k1 * lane);
  const double2 wstep = tw_m(lo, hi, (32 * k1) & (M - 1));
#pragma unroll
  for (int i0 = 0; i0 < M2; i0 += 32) {
    g[i0 + lane] = cmul(x[padL(i0 + lane)], wt);
    wt = cmul(wt, wstep);
  }
}

// Column pass of the correlation transform: F[m2 + M2 m1] (natural order) and
// the per-block max of |F|^2 over m < N. grid (M2 / kCT, P).
template <int M1>
__global__ void __launch_bounds__(kT)
    p2_kernel(const double2* __restrict__ G, int64_t P, int N, int M2, const double2* __restrict__ twS, double2* F,
              double* bmax) {
  constexpr int VS = vstride<M1>();
  __shared__ __align__(16) double2 sm[kCT * VS];
  __shared__ double2 red[64];
  const int M = M1 * M2;
  const int64_t p = blockIdx.y;
  const int c0 = blockIdx.x * kCT;
  const double2* g = G + p * (int64_t)M;
  constexpr int kLd = M1 * kCT / kT;
  double2 q[kLd];  // every load in flight before the shared stores
#pragma unroll
  for (int it = 0; it < kLd; ++it) {
    const int idx = threadIdx.x + it * kT;
    q[it] = __ldg(&g[(int64_t)(idx / kCT) * M2 + c0 + idx % kCT]);
  }
#pragma unroll
  for (int it = 0; it < kLd; ++it) {
    const int idx = threadIdx.x + it * kT;
    sm[(idx % kCT) * VS + padL(idx / kCT)] = q[it];
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  wfft<M1>(sm + w * VS, twS, 1, lane);
  __syncthreads();
  double2* f = F + p * (int64_t)M;
  double mx = -1.0;
#pragma unroll
  for (int it = 0; it < M1 * kCT / kT; ++it) {
    const int idx = threadIdx.x + it * kT;
    const int m1 = idx / kCT, c = idx % kCT;
    const int m = (c0 + c) + M2 * m1;
    const double2 v = sm[c * VS + padL(m1)];
    f[m] = v;
    if (m < N) mx = fmax(mx, fma(v.x, v.x, v.y * v.y));
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) bmax[p * gridDim.x + blockIdx.x] = mx;
}
// Tie-band pick of the four-step layout, one CTA per pair: global max from the
// column-tile maxima, then only tiles whose maximum reaches the band are
// scanned (usually one) for the smallest m with |F_m|^2 >= thr^2; then, in
// warp 0, lpick_kernel's work for the pair (shift, rotation, trace, energy),
// so the candidate never goes through global memory and there is one launch.
template <int M1>
__global__ void __launch_bounds__(kT)
    pick_kernel(const double2* __restrict__ F, int N, int M2, const double* __restrict__ bmax,
                const double* __restrict__ sq1, const double* __restrict__ sq2, const int32_t* bad1,
                const int32_t* bad2, cva_alignment* out, double2* rot) {
  __shared__ double2 red[64];
  __shared__ unsigned s_mask;
  __shared__ double2 s_v;
  const int64_t p = blockIdx.x;
  const int nt = M2 / kCT, M = M1 * M2;  // nt <= 32 column tiles
  const int lane = threadIdx.x & 31;
  // independent loads first: the tile maxima, and (warp 0) the sum |z'|^2 partials
  const double tb = (int)threadIdx.x < nt ? bmax[p * nt + threadIdx.x] : -1.0;
  double s1 = 0.0, s2 = 0.0;
  if (threadIdx.x < 32)
    for (int b = lane; b < nt; b += 32) {
      s1 += sq1[p * nt + b];
      s2 += sq2[p * nt + b];
    }
  const double best2 = block_max(tb, red);
  const double best = sqrt(best2) / (double)M;
  const double thr = best - pf::kTieRelTol * fmax(1.0, fabs(best));
  const double thrM = thr * (double)M;
  const double thr2 = thr > 0.0 ? thrM * thrM : -1.0;
  if (threadIdx.x < 32) {  // tiles whose maximum reaches the band (usually one)
    const unsigned msk = __ballot_sync(0xffffffffu, (int)threadIdx.x < nt && tb >= thr2);
    if (lane == 0) s_mask = msk;
  }
  __syncthreads();
  const double2* f = F + p * (int64_t)M;
  int cand = INT_MAX;
  double2 vc = make_double2(0.0, 0.0);  // F at this thread's candidate
  for (unsigned msk = s_mask; msk; msk &= msk - 1) {
    const int b = __ffs(msk) - 1;
    for (int idx = threadIdx.x; idx < M1 * kCT; idx += kT) {
      const int m = (b * kCT + idx % kCT) + M2 * (idx / kCT);
      if (m < N && m < cand) {
        const double2 v = __ldg(&f[m]);
        if (fma(v.x, v.x, v.y * v.y) >= thr2) {
          cand = m;
          vc = v;
        }
      }
    }
  }
  const int cmin = block_min_int(cand, red);
  if (cand == cmin && cand != INT_MAX) s_v = vc;  // one thread scanned index cmin
  __syncthreads();
  if (threadIdx.x >= 32) return;
  // lpick_kernel's work for pair p (one candidate, nt sum-of-squares partials)
  const int m = isfinite(best) && best2 >= 0.0 ? cmin : INT_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
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
    const double2 v = s_v;
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
}  // namespace fs

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

// Four-step split M = M1 x M2 with M1, M2 in {64, 128, 256} (M1 <= M2); 0 if none.
int four_step_m1_impl(int M) {
  if (M < 4096 || M > 65536) return 0;
  int p = 0;
  while ((1 << p) < M) ++p;
  return 1 << (p / 2);
}

template <int M1>
cudaError_t f1_launch(const double2* z1, const double2* z2, int64_t P, int N, int M2, const FourStepTw& t,
                      const double4* part, int normalize, ln::CurveNorm* norm, int32_t* bad, double2* U, double* q1,
                      double* q2, cudaStream_t s) {
  ln::fs::f1_kernel<M1><<<dim3((unsigned)(M2 / ln::fs::kCT), (unsigned)(2 * P)), ln::fs::kT, 0, s>>>(
      z1, z2, P, N, M2, t.s1, t.lo, t.hi, part, normalize, norm, bad, U, q1, q2);
  return cudaGetLastError();
}
template <int M1>
cudaError_t p2_launch(const double2* G, int64_t P, int N, int M2, const FourStepTw& t, double2* F, double* bmax,
                      cudaStream_t s) {
  ln::fs::p2_kernel<M1><<<dim3((unsigned)(M2 / ln::fs::kCT), (unsigned)P), ln::fs::kT, 0, s>>>(G, P, N, M2, t.s1, F,
                                                                                               bmax);
  return cudaGetLastError();
}
template <int M2>
cudaError_t fp_launch(const double2* U, int64_t P, int M1, const FourStepTw& t, double2* G, cudaStream_t s) {
  const size_t sm = sizeof(double2) * 2 * ln::fs::kRT * ln::fs::vstride<M2>();
  cudaError_t e = cudaFuncSetAttribute((const void*)ln::fs::fp_kernel<M2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  ln::fs::fp_kernel<M2><<<dim3((unsigned)(M1 / ln::fs::kRT), (unsigned)P), ln::fs::kT, sm, s>>>(U, P, M1, t.s2, t.lo,
                                                                                                 t.hi, G);
  return cudaGetLastError();
}

// The three passes of one chunk; F in natural order, bmax / sq partials per tile.
cudaError_t four_step(int M1, const double2* z1, const double2* z2, int64_t P, int N, const FourStepTw& t,
                      const double4* part, int normalize, ln::CurveNorm* norm, int32_t* bad, double2* U, double2* G,
                      double2* F, double* q1, double* q2, double* bmax, cudaStream_t s) {
  const int M = pf::fft_len(N), M2 = M / M1;
  cudaError_t e;
  switch (M1) {
    case 64: e = f1_launch<64>(z1, z2, P, N, M2, t, part, normalize, norm, bad, U, q1, q2, s); break;
    case 128: e = f1_launch<128>(z1, z2, P, N, M2, t, part, normalize, norm, bad, U, q1, q2, s); break;
    default: e = f1_launch<256>(z1, z2, P, N, M2, t, part, normalize, norm, bad, U, q1, q2, s); break;
  }
  if (e != cudaSuccess) return e;
  switch (M2) {
    case 64: e = fp_launch<64>(U, P, M1, t, G, s); break;
    case 128: e = fp_launch<128>(U, P, M1, t, G, s); break;
    default: e = fp_launch<256>(U, P, M1, t, G, s); break;
  }
  if (e != cudaSuccess) return e;
  switch (M1) {
    case 64: return p2_launch<64>(G, P, N, M2, t, F, bmax, s);
    case 128: return p2_launch<128>(G, P, N, M2, t, F, bmax, s);
    default: return p2_launch<256>(G, P, N, M2, t, F, bmax, s);
  }
}

}  // namespace

size_t large_workspace_bytes(int64_t chunk, int N) {
  const Layout L = layout(N);
  const size_t seq = sizeof(double2) * (size_t)L.M;
  return 4 * seq * (size_t)chunk + 4096                                        // spectra ping-pong
         + 2 * sizeof(ln::CurveNorm) * (size_t)chunk                           // norms
         + 2 * sizeof(double4) * (size_t)(chunk * ln::kStatBlocks)             // stat partials
         + 2 * sizeof(double) * (size_t)(chunk * (L.sqn > L.M / 8 ? L.sqn : L.M / 8))  // |z'|^2 partials
         + 2 * sizeof(int32_t) * (size_t)chunk                                 // bad flags
         + sizeof(double2) * (size_t)chunk                                     // rotations
         + (sizeof(double) + sizeof(int)) * (size_t)(chunk * (L.nblk + L.M / 8)) + 4096;  // argmax partials
}

int64_t large_chunk_pairs(int N) {
  // ~96 MB working set: 4 spectra of 16 M bytes per pair at N = 65536
  const int M = pf::fft_len(N);
  const int64_t per = 4 * (int64_t)sizeof(double2) * M;
  int64_t c = (96ll << 20) / per;
  return c < 1 ? 1 : c;
}

int four_step_m1(int M) { return four_step_m1_impl(M); }

cudaError_t launch_large_align(const double2* c1, const double2* c2, int64_t pairs, int N, int normalize,
                               const double2* tw, const FourStepTw* fst, cva_alignment* out, double2* aligned,
                               void* ws, int64_t chunk, cudaStream_t s) {
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
  ln::CurveNorm* nn = (ln::CurveNorm*)take(sizeof(ln::CurveNorm) * 2 * chunk);   // curve 1s then curve 2s
  double4* spp = (double4*)take(sizeof(double4) * 2 * chunk * ln::kStatBlocks);
  const int sqcap = sqn > M / 8 ? sqn : M / 8;
  double* q1 = (double*)take(sizeof(double) * chunk * sqcap);
  double* q2 = (double*)take(sizeof(double) * chunk * sqcap);
  int32_t* bb = (int32_t*)take(sizeof(int32_t) * 2 * chunk);
  double2* rot = (double2*)take(sizeof(double2) * chunk);
  double* bmax = (double*)take(sizeof(double) * chunk * (nblk + M / 8));
  int* bcand = (int*)take(sizeof(int) * chunk * nblk);
  const int fm1 = fst ? four_step_m1_impl(M) : 0;
  cudaError_t e = cudaSuccess;
  for (int64_t p0 = 0; p0 < pairs && e == cudaSuccess; p0 += chunk) {
    const int64_t P = pairs - p0 < chunk ? pairs - p0 : chunk;
    const double2* z1 = c1 + p0 * N;
    const double2* z2 = c2 + p0 * N;
    ln::CurveNorm *n1 = nn, *n2 = nn + P;
    int32_t *b1 = bb, *b2 = bb + P;
    ln::stats_partial<<<dim3(ln::kStatBlocks, (unsigned)(2 * P)), ln::kT, 0, s>>>(z1, N, spp, z2, P);
    double2* F = nullptr;
    const int nbmax = nblk, nsq = sqn;
    if (fm1) {  // four-step: U = A|B (2P sequences, adjacent), G = C, F = D; f1 forms the norms
      e = four_step(fm1, z1, z2, P, N, *fst, spp, normalize, nn, bb, A, C, D, q1, q2, bmax, s);
      if (e != cudaSuccess) break;
      const int M2 = M / fm1;
      switch (fm1) {  // argmax + pick in one kernel
        case 64: ln::fs::pick_kernel<64><<<(unsigned)P, ln::kT, 0, s>>>(D, N, M2, bmax, q1, q2, b1, b2, out + p0, rot); break;
        case 128: ln::fs::pick_kernel<128><<<(unsigned)P, ln::kT, 0, s>>>(D, N, M2, bmax, q1, q2, b1, b2, out + p0, rot); break;
        default: ln::fs::pick_kernel<256><<<(unsigned)P, ln::kT, 0, s>>>(D, N, M2, bmax, q1, q2, b1, b2, out + p0, rot); break;
      }
      if (aligned)
        ln::aligned_kernel<<<dim3((unsigned)((N + 4 * ln::kT - 1) / (4 * ln::kT)), (unsigned)P), ln::kT, 0, s>>>(
            z2, N, n2, out + p0, rot, aligned + p0 * N);
      e = cudaGetLastError();
      continue;
    } else {
      ln::stats_final<<<(unsigned)((2 * P + 7) / 8), 256, 0, s>>>(spp, 2 * P, N, normalize, nn, bb);
      double2 *Z1 = nullptr, *Z2 = nullptr;
      e = fft_many<ln::kLoadA>(z1, nullptr, A, B, M, N, tw, n1, P, q1, s, &Z1);
      if (e == cudaSuccess) e = fft_many<ln::kLoadB>(z2, nullptr, C, D, M, N, tw, n2, P, q2, s, &Z2);
      if (e != cudaSuccess) break;
      double2* fa = (Z1 == A) ? B : A;  // free buffers for the correlation transform
      double2* fb = (Z2 == C) ? D : C;
      e = fft_many<ln::kProduct>(Z1, Z2, fa, fb, M, N, tw, nullptr, P, nullptr, s, &F);
      if (e != cudaSuccess) break;
      ln::lmax_kernel<<<dim3((unsigned)nblk, (unsigned)P), ln::kT, 0, s>>>(F, M, N, bmax);
    }
    ln::lcand_kernel<<<dim3((unsigned)nblk, (unsigned)P), ln::kT, 0, s>>>(F, M, N, bmax, nbmax, bcand);
    ln::lpick_kernel<<<(unsigned)((P + 7) / 8), 256, 0, s>>>(F, M, N, bcand, nblk, q1, q2, nsq, b1, b2, P, out + p0,
                                                             rot);
    if (aligned)
      ln::aligned_kernel<<<dim3((unsigned)((N + 4 * ln::kT - 1) / (4 * ln::kT)), (unsigned)P), ln::kT, 0, s>>>(
          z2, N, n2, out + p0, rot, aligned + p0 * N);
    e = cudaGetLastError();
  }
  return e;
}

namespace ln {
__global__ void broadcast_kernel(const double2* __restrict__ c, int64_t n, int64_t copies, double2* __restrict__ out) {
  const int64_t total = n * copies;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = c[i % n];
}
}  // namespace ln

// out[k * n + l] = c[l], k < copies (one row of an all-pairs matrix as a pair batch)
cudaError_t launch_broadcast_curve(const double2* c, int64_t n, int64_t copies, double2* out, cudaStream_t s) {
  const int64_t total = n * copies;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
  ln::broadcast_kernel<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, s>>>(c, n, copies, out);
  return cudaGetLastError();
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
