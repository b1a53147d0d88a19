// All-pairs alignment with spectrum reuse (BASELINE config C2: 2048 curves,
// N = 512, every ordered pair (i, j) -> align_fft(curve_i, curve_j)).
//
// Reference: the matrix cells of distance_matrix call align_fft per pair
// (proj/src/elastic.cpp:176-236 via run_align, :51-53), recomputing both
// curves' spectra for every cell (proj/src/rigid_align.cpp:147-183). Here:
//   spectra_kernel   each curve's spectra once: ZA_i = FFT([z_i, 0...]) (row
//                    role) and ZB_j = FFT([z_j, z_j, 0...]) (column role; the
//                    same array when N is a power of two), plus s_i = |z_i|^2.
//   allpairs_kernel  one warp per (i, j): the product ZA_i conj(ZB_j) is formed
//                    in registers inside the first radix-8 pass of an in-place
//                    warp FFT (no block barriers), then a shuffle argmax with
//                    the reference's tie band. A CTA owns kRowTile rows whose
//                    spectra sit in shared memory; each warp keeps its column's
//                    spectrum in registers across those rows.
// Output per cell: energy (f64), shift (i32), theta (f64): 20 B.
#include <cuda_runtime.h>

#include <climits>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "fft.cuh"
#include "pairfft.cuh"

namespace cva {
namespace ap {

constexpr int kWarps = 8;
// 8 rows per CTA, one CTA of 8 warps per SM with up to 255 registers: each
// warp keeps its column's spectrum in registers across the rows (one L1 read
// per column instead of one per cell; the kernel is bound by L1 / shared
// wavefronts). 2 CTAs of 128 registers spilled that copy (9.9 ms); with it
// re-read per cell from L1: 8.85 ms; this: 8.55 ms (C2 step).
#ifndef CVA_AP_ROWS
#define CVA_AP_ROWS 8
#endif
constexpr int kRowTile = CVA_AP_ROWS;
#ifndef CVA_AP_ZC_REG
#define CVA_AP_ZC_REG 1
#endif
#ifndef CVA_AP_TW_REG
#define CVA_AP_TW_REG 0
#endif
#ifndef CVA_AP_MINB
#define CVA_AP_MINB 1
#endif
// twiddles W^3, W^5, W^6, W^7 of the radix-8 passes 2 and 3 formed from
// W^1, W^2, W^4 (3 shared reads per butterfly instead of 7; the kernel is
// bound by shared / L1 wavefronts)
#ifndef CVA_AP_TW_DERIVE
#define CVA_AP_TW_DERIVE 1
#endif
// w[0..6] = W^1..W^7 of one butterfly from the [r - 1][stride] table column
template <int kStride>
__device__ __forceinline__ void tw8(const double2 (*t)[kStride], int col, double2 (&w)[7]) {
#if CVA_AP_TW_DERIVE
  w[0] = t[0][col];
  w[1] = t[1][col];
  w[3] = t[3][col];
  w[2] = cmul(w[0], w[1]);
  w[4] = cmul(w[0], w[3]);
  w[5] = cmul(w[1], w[3]);
  w[6] = cmul(w[2], w[3]);
#else
#pragma unroll
  for (int r = 0; r < 7; ++r) w[r] = t[r][col];
#endif
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 3); }

// ------------------------------------------------------------ spectra

// Two curves per CTA (one per 128-thread half). M = fft_len(N).
__global__ void __launch_bounds__(256) spectra_kernel(const double2* __restrict__ curves, int64_t count,
                                                      int N, const double2* __restrict__ tw,
                                                      double2* za, double2* zb, double* ss) {
  extern __shared__ __align__(16) char smem[];
  const int M = pf::fft_len(N);
  const int NP = pf::padded_len(M);
  const int grp = threadIdx.x / 128, g = threadIdx.x % 128;
  const int64_t c = 2 * (int64_t)blockIdx.x + grp;
  double2* B0 = reinterpret_cast<double2*>(smem) + grp * 2 * NP;
  double2* B1 = B0 + NP;
  auto sync = [grp]() { pf::named_sync(1 + grp, 128); };
  const bool live = c < count;
  const double2* z = curves + (live ? c : 0) * N;
  for (int role = 0; role < (M == N ? 1 : 2); ++role) {
    const int lim = role == 0 ? N : 2 * N;
    double acc = 0.0;
    auto load = [&](int i) {
      if (i >= lim) return make_double2(0.0, 0.0);
      const double2 q = z[i < N ? i : i - N];
      if (i < N) acc = fma(q.x, q.x, fma(q.y, q.y, acc));
      return q;
    };
    const double2* X = pf::group_fft<128>(load, B0, B1, M, tw, g, sync);
    if (live) {
      double2* dst = (role == 0 ? za : zb) + c * M;
      for (int k = g; k < M; k += 128) dst[k] = X[pf::pad(k)];
      if (role == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        __shared__ double part[8];
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
        sync();
        if (g == 0) ss[c] = part[grp * 4] + part[grp * 4 + 1] + part[grp * 4 + 2] + part[grp * 4 + 3];
      }
    }
    sync();
  }
}

// ------------------------------------------------------------ pair FFT

// One in-place radix-R Stockham pass over a warp's padded buffer (M points,
// nb = M / R butterflies, B = nb / 32 per lane). Values of the butterflies are
// taken from / left in v[][] (registers).
template <int M, int R>
__device__ __forceinline__ void warp_compute(double2 (&v)[M / R / 32][R], int Ns, int lane,
                                             const double2* __restrict__ tw) {
  constexpr int nb = M / R, B = nb / 32;
  const int tws = M / (Ns * R);
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = lane + 32 * b;
    const int jm = j & (Ns - 1);
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], __ldg(&tw[r * jm * tws]));
    }
    dft_r<R>(v[b]);
  }
}

template <int M, int R>
__device__ __forceinline__ void warp_store(const double2 (&v)[M / R / 32][R], double2* buf, int Ns,
                                           int lane) {
  constexpr int nb = M / R, B = nb / 32;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = lane + 32 * b;
    const int jm = j & (Ns - 1);
    const int base = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pad(base + r * Ns)] = v[b][r];
  }
}

template <int M, int R>
__device__ __forceinline__ void warp_load(double2 (&v)[M / R / 32][R], const double2* buf, int lane) {
  constexpr int nb = M / R, B = nb / 32;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = lane + 32 * b;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = buf[pad(j + r * nb)];
  }
}

// C2 all-pairs for M = N = 512 (three radix-8 passes, 2 butterflies per lane).
constexpr int kM = 512;
constexpr int kR = 8;
constexpr int kB = kM / kR / 32;  // 2
constexpr int kNB = kM / kR;      // 64

__global__ void __launch_bounds__(kWarps * 32, CVA_AP_MINB)
    allpairs_kernel(const double2* __restrict__ za, const double2* __restrict__ zb,
                    const double* __restrict__ ss, int64_t count, int64_t row_begin, int64_t row_end,
                    int64_t col_chunk, const double2* __restrict__ tw, double* energy,
                    int32_t* shift, double2* dm) {
  extern __shared__ __align__(16) char smem[];
  double2* rows = reinterpret_cast<double2*>(smem);  // kRowTile x kM spectra
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* buf = rows + kRowTile * kM + warp * pf::padded_len(kM);
  const int64_t i0 = row_begin + (int64_t)blockIdx.x * kRowTile;
  const int nrows = (int)min((int64_t)kRowTile, row_end - i0);
  for (int k = threadIdx.x; k < nrows * kM; k += blockDim.x)
    rows[k] = za[(i0 + k / kM) * kM + (k % kM)];
  __syncthreads();
  const double invN = 1.0 / (double)kM;
  // twiddles of passes 2 and 3 in shared memory, laid out [r - 1][jm] so a
  // warp's reads are consecutive (pass 2: jm = lane & 7; pass 3: jm = lane + 32 b)
  __shared__ double2 s_t2[kR - 1][8], s_t3[kR - 1][64];
  for (int k = threadIdx.x; k < (kR - 1) * 72; k += blockDim.x) {
    const int r = k / 72 + 1, q = k % 72;
    if (q < 8)
      s_t2[r - 1][q] = __ldg(&tw[r * q * (kM / (8 * kR))]);
    else
      s_t3[r - 1][q - 8] = __ldg(&tw[r * (q - 8) * (kM / (64 * kR))]);
  }
  __syncthreads();
#if CVA_AP_TW_REG
  // this lane's pass-2 / pass-3 twiddles in registers (the same for every cell)
  double2 t2r[kR - 1], t3r[kB][kR - 1];
#pragma unroll
  for (int r = 1; r < kR; ++r) {
    t2r[r - 1] = s_t2[r - 1][lane & 7];
#pragma unroll
    for (int b = 0; b < kB; ++b) t3r[b][r - 1] = s_t3[r - 1][lane + 32 * b];
  }
#endif
  const int64_t j_begin = (int64_t)blockIdx.y * col_chunk;
  const int64_t j_end = min(count, j_begin + col_chunk);
  for (int64_t j = j_begin + warp; j < j_end; j += kWarps) {
    const double2* zc = zb + j * kM;
    const double sj = __ldg(&ss[j]);
#if CVA_AP_ZC_REG
    // the column spectrum in registers across the CTA's rows (one L1 read per column)
    double2 cz[kB][kR];
#pragma unroll
    for (int b = 0; b < kB; ++b)
#pragma unroll
      for (int r = 0; r < kR; ++r) cz[b][r] = __ldg(&zc[lane + 32 * b + r * kNB]);
#endif
    for (int rr = 0; rr < nrows; ++rr) {
      const double2* zr = rows + rr * kM;
      double2 v[kB][kR];
      // pass 1 (Ns = 1): P = ZA_i conj(ZB_j) formed on load
#pragma unroll
      for (int b = 0; b < kB; ++b)
#pragma unroll
        for (int r = 0; r < kR; ++r)
#if CVA_AP_ZC_REG
          v[b][r] = cmulconj(zr[lane + 32 * b + r * kNB], cz[b][r]);
#else
          v[b][r] = cmulconj(zr[lane + 32 * b + r * kNB], __ldg(&zc[lane + 32 * b + r * kNB]));
#endif
      warp_compute<kM, kR>(v, 1, lane, tw);
      warp_store<kM, kR>(v, buf, 1, lane);
      __syncwarp();
      warp_load<kM, kR>(v, buf, lane);
      __syncwarp();
#if !CVA_AP_TW_REG
      double2 w2[7];
      tw8<8>(s_t2, lane & 7, w2);
#endif
#pragma unroll
      for (int b = 0; b < kB; ++b) {
#pragma unroll
        for (int r = 1; r < kR; ++r)
#if CVA_AP_TW_REG
          v[b][r] = cmul(v[b][r], t2r[r - 1]);
#else
          v[b][r] = cmul(v[b][r], w2[r - 1]);
#endif
        dft_r<kR>(v[b]);
      }
      warp_store<kM, kR>(v, buf, 8, lane);
      __syncwarp();
      warp_load<kM, kR>(v, buf, lane);
#pragma unroll
      for (int b = 0; b < kB; ++b) {
#if CVA_AP_TW_REG
#pragma unroll
        for (int r = 1; r < kR; ++r) v[b][r] = cmul(v[b][r], t3r[b][r - 1]);
#else
        double2 w3[7];
        tw8<64>(s_t3, lane + 32 * b, w3);
#pragma unroll
        for (int r = 1; r < kR; ++r) v[b][r] = cmul(v[b][r], w3[r - 1]);
#endif
        dft_r<kR>(v[b]);
      }
      // last pass output index of v[b][r]: base + r * 64 with base = j (Ns = 64 = nb)
      // |D_m| = |F_m| / N; band test on squared magnitudes (see pairfft.cuh)
      double best2 = -1.0;
#pragma unroll
      for (int b = 0; b < kB; ++b)
#pragma unroll
        for (int r = 0; r < kR; ++r) best2 = fmax(best2, fma(v[b][r].x, v[b][r].x, v[b][r].y * v[b][r].y));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best2 = fmax(best2, __shfl_xor_sync(0xffffffffu, best2, o));
      const double best = sqrt(best2) * invN;
      const double thr = best - pf::kTieRelTol * fmax(1.0, fabs(best));
      const double thrN = thr * (double)kM;
      const double thr2 = thr > 0.0 ? thrN * thrN : -1.0;
      // each lane's smallest qualifying index (m = lane + 32 b + 64 r grows with
      // (r, b)) and its value; the warp minimum's owner lane reports
      int cand = INT_MAX;
      double2 fc = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < kR; ++r)
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const bool hit = fma(v[b][r].x, v[b][r].x, v[b][r].y * v[b][r].y) >= thr2;
          if (cand == INT_MAX && hit) {
            cand = lane + 32 * b + r * 64;
            fc = v[b][r];
          }
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
      const int m = cand;
      const int64_t cell = (i0 + rr - row_begin) * count + j;
      if (m != INT_MAX && lane == (m & 31)) {
        const double tr = sqrt(fma(fc.x, fc.x, fc.y * fc.y)) * invN;
        double e = invN * (__ldg(&ss[i0 + rr]) + sj) - 2.0 * invN * tr;
        if (e < 0.0) e = 0.0;
        energy[cell] = e;
        shift[cell] = m;
        dm[cell] = fc;  // theta = arg conj(F_m) in a coalesced pass (theta_kernel)
      }
      if (m == INT_MAX && lane == 0) {  // non-finite correlation
        energy[cell] = __longlong_as_double(0x7ff8000000000000ULL);
        shift[cell] = 0;
        dm[cell] = make_double2(__longlong_as_double(0x7ff8000000000000ULL), 0.0);
      }
      __syncwarp();
    }
  }
}

// theta per cell from the winning correlation value (one full warp of cells at
// a time instead of one lane per cell inside allpairs_kernel): degenerate
// (F_m = 0) -> 0, non-finite -> NaN (rigid_align.cpp:86-88, :83).
__global__ void theta_kernel(const double2* __restrict__ dm, int64_t cells, double* theta) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const double2 f = dm[c];
  theta[c] = (f.x == 0.0 && f.y == 0.0) ? 0.0 : atan2(-f.y, f.x);
}

}  // namespace ap

size_t allpairs_spectra_smem(int N) { return 4 * sizeof(double2) * (size_t)pf::padded_len(pf::fft_len(N)); }

cudaError_t launch_spectra(const double2* curves, int64_t count, int N, const double2* tw, double2* za,
                           double2* zb, double* ss, cudaStream_t s) {
  const size_t sm = allpairs_spectra_smem(N);
  cudaError_t e = cudaFuncSetAttribute((const void*)ap::spectra_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  ap::spectra_kernel<<<(unsigned)((count + 1) / 2), 256, sm, s>>>(curves, count, N, tw, za, zb, ss);
  return cudaGetLastError();
}

bool allpairs_fast_supported(int N) { return N == ap::kM; }

size_t allpairs_scratch_cells(int64_t rows, int64_t count) { return sizeof(double2) * (size_t)(rows * count); }

cudaError_t launch_allpairs(const double2* za, const double2* zb, const double* ss, int64_t count,
                            int64_t row_begin, int64_t row_end, const double2* tw, double* energy,
                            int32_t* shift, double* theta, double2* dm, cudaStream_t s) {
  const size_t sm = sizeof(double2) * (size_t)(ap::kRowTile * ap::kM + ap::kWarps * pf::padded_len(ap::kM));
  cudaError_t e = cudaFuncSetAttribute((const void*)ap::allpairs_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int64_t rows = row_end - row_begin;
  const unsigned gx = (unsigned)((rows + ap::kRowTile - 1) / ap::kRowTile);
  // split the columns so that the grid covers the machine a few times over
  int64_t splits = 1;
  while (gx * splits < 4 * 148 * 2 && count / (splits * 2) >= 64) splits *= 2;
  const int64_t chunk = (count + splits - 1) / splits;
  dim3 grid(gx, (unsigned)splits);
  ap::allpairs_kernel<<<grid, ap::kWarps * 32, sm, s>>>(za, zb, ss, count, row_begin, row_end, chunk, tw,
                                                         energy, shift, dm);
  const int64_t cells = rows * count;
  ap::theta_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, s>>>(dm, cells, theta);
  return cudaGetLastError();
}

}  // namespace cva
