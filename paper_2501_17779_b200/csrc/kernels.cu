// sm_100a kernels of the curve-alignment hot path and their host launchers.
//
//   tw_init_kernel                     twiddle table w_N^k = exp(-2 pi i k / N) (sincospi)
//   preprocess_resample_kernel         resample -> center -> normalize (curve.cpp:93-97), one
//                                      curve per CTA in shared memory (raw curves the v2
//                                      resampler of fused.cu does not hold, up to ~4.6 K nodes)
//   preprocess_resample_global_kernel  the same on per-CTA global slabs (any node count)
//   preprocess_center_kernel           center -> normalize (resample=false)
//
// The alignment itself runs in fused.cu / largen.cu / allpairs.cu.
#include <cuda_runtime.h>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "fft.cuh"
#include "kernels.h"
#include "pairfft.cuh"
#include "spline.cuh"

namespace cva {

constexpr int kThreads = 256;
constexpr int kRedSlots = 64;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

__global__ void tw_init_kernel(double2* tw, int N) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < N) {
    double s, c;
    // exp(-2 pi i k / N) = cospi(2k/N) - i sinpi(2k/N); 2k/N exact for N = 2^p
    sincospi(2.0 * (double)k / (double)N, &s, &c);
    tw[k] = make_double2(c, -s);
  }
}

// Layout checks (N = 1024: plan 8, 8, 8, 2 for 128 threads and for one warp,
// tables of 7 x 8, 7 x 64 and 1 x 512 entries after the W_N table; 256 threads:
// radix 8 only with CVA_R8_MIN <= 4).
static_assert(pf::ptw_off<128>(1024, 8) == 1024 && pf::ptw_off<128>(1024, 64) == 1024 + 56 &&
                  pf::ptw_off<128>(1024, 512) == 1024 + 56 + 448,
              "pass table offsets, 128-thread plan");
#if CVA_R8_MIN <= 4  // all three plans are 8, 8, 8, 2 at N = 1024: one shared set of tables
static_assert(pf::ptw_off<256>(1024, 8) == 1024 && pf::ptw_off_warp(1024, 512) == 1024 + 56 + 448 &&
                  pf::ptw_len(1024) == 3 * 1016,
              "pass table offsets, 256-thread and one-warp plans");
#else  // 256 threads: radix 4 x 5 (3 x 4, 3 x 16, 3 x 64, 3 x 256 entries)
static_assert(pf::ptw_off<256>(1024, 4) == 1024 + 1016 && pf::ptw_off_warp(1024, 8) == 1024,
              "pass table offsets, 256-thread and one-warp plans");
#endif

// Pass twiddle tables after the length-N table (layout: pairfft.cuh ptw_off),
// copied from it entry by entry. One CTA; N <= 2048.
__global__ void ptw_fill_kernel(double2* tw, int N) {
  for (int h = 0; h < 3; ++h) {  // 128-thread, 256-thread, one-warp plans
    int off = h == 0 ? pf::ptw_off<128>(N, 1) : h == 1 ? pf::ptw_off<256>(N, 1) : pf::ptw_off_warp(N, 1);
    for (int Ns = 1; Ns < N;) {
      const int R = h == 0 ? pf::plan_radix<128>(N, Ns) : h == 1 ? pf::plan_radix<256>(N, Ns)
                                                                 : pf::plan_radix_warp(N, Ns);
      if (Ns > 1) {
        const int tws = N / (Ns * R);
        for (int k = threadIdx.x; k < (R - 1) * Ns; k += blockDim.x) tw[off + k] = tw[(k / Ns + 1) * (k % Ns) * tws];
        off += (R - 1) * Ns;
      }
      Ns *= R;
    }
  }
}

__device__ __forceinline__ void load_curve(const double2* __restrict__ g, double2* sm, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = __ldg(&g[i]);
}

__device__ __forceinline__ int block_any_nonfinite(const double2* sm, int n, double2* red) {
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 p = sm[i];
    bad |= !(isfinite(p.x) && isfinite(p.y));
  }
  return block_or(bad, red);
}

// Shared-memory layout for resampling one curve of up to nmax raw nodes.
struct ResampleSmem {
  double2* xy;      // nmax
  double* s;        // nmax + 1 (padded to even)
  double2* m;       // nmax
  ChunkEnds* ends;  // kThreads
  static __host__ __device__ size_t bytes(int nmax) {
    return sizeof(double2) * (size_t)nmax + sizeof(double) * (size_t)((nmax + 2) & ~1) +
           sizeof(double2) * (size_t)nmax + sizeof(ChunkEnds) * kThreads;
  }
  __device__ void carve(char* base, int nmax) {
    xy = reinterpret_cast<double2*>(base);
    s = reinterpret_cast<double*>(xy + nmax);
    m = reinterpret_cast<double2*>(s + ((nmax + 2) & ~1));
    ends = reinterpret_cast<ChunkEnds*>(m + nmax);
  }
};

// raw curve (global, n nodes) -> preprocess(raw, n_out, true) in out_sm.
// Returns block-uniform status.
__device__ inline int block_resample_preprocess(const double2* __restrict__ raw, int n, int n_out,
                                                const ResampleSmem& R, double2* out_sm,
                                                double2* red, bool center_normalize = true,
                                                double* cpv_g = nullptr) {
  if (n < 4 || n_out < 8) return kInvalid;  // validate_curve(c, 4), n_out >= 8 (curve.cpp:68-69)
  load_curve(raw, R.xy, n);
  __syncthreads();
  int bad = block_any_nonfinite(R.xy, n, red);
  if (bad) return kInvalid;
  block_arc_length(R.xy, n, R.s, red, &bad);
  if (bad) return kInvalid;
  block_spline_solve(R.s, R.xy, R.m, n, R.ends, red, cpv_g);
  block_spline_eval(R.s, R.xy, R.m, n, n_out, out_sm);
  if (center_normalize) block_center_normalize(out_sm, n_out, red, &bad);
  return bad ? kInvalid : kOk;
}

__device__ inline void fill_nan(double2* g, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) g[i] = make_double2(qnan(), qnan());
}

// ------------------------------------------------------------------ kernels

__global__ void __launch_bounds__(kThreads)
    preprocess_resample_kernel(const double2* __restrict__ pts, const int64_t* __restrict__ off,
                               int nmax, int n_out, int center_normalize,
                               double2* __restrict__ out, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smem_raw[];
  __shared__ double2 red[kRedSlots];
  ResampleSmem R;
  R.carve(smem_raw, nmax);
  double2* obuf = reinterpret_cast<double2*>(smem_raw + ResampleSmem::bytes(nmax));
  const int64_t c = blockIdx.x;
  const int64_t b0 = off[c];
  const int n = (int)(off[c + 1] - b0);
  // a curve above the caller's max_n_in would overrun the carved arrays: invalid
  const int st = n > nmax ? kInvalid : block_resample_preprocess(pts + b0, n, n_out, R, obuf, red, center_normalize != 0);
  double2* o = out + c * n_out;
  if (st == kOk) {
    for (int i = threadIdx.x; i < n_out; i += blockDim.x) o[i] = obuf[i];
  } else {
    fill_nan(o, n_out);
  }
  if (status && threadIdx.x == 0) status[c] = st;
}

// The same resample -> center -> normalize for raw curves too long for shared
// memory (any n >= 4, any n_out >= 8): the solver's arrays live in a per-CTA
// slab of global memory (L2-resident: 48 B per raw node) and the samples are
// written straight to `out`. A grid-stride loop over curves reuses the slabs.
__global__ void __launch_bounds__(kThreads)
    preprocess_resample_global_kernel(const double2* __restrict__ pts, const int64_t* __restrict__ off,
                                      int64_t curves, int nmax, int n_out, int center_normalize,
                                      double2* __restrict__ out, int32_t* __restrict__ status, char* slab,
                                      size_t slab_bytes) {
  __shared__ double2 red[kRedSlots];
  char* base = slab + (size_t)blockIdx.x * slab_bytes;
  ResampleSmem R;
  R.carve(base, nmax);
  double* cpv = reinterpret_cast<double*>(base + ResampleSmem::bytes(nmax));
  for (int64_t c = blockIdx.x; c < curves; c += gridDim.x) {
    const int64_t b0 = off[c];
    const int n = (int)(off[c + 1] - b0);
    double2* o = out + c * n_out;
    const int st = n > nmax ? kInvalid : block_resample_preprocess(pts + b0, n, n_out, R, o, red,
                                                                   center_normalize != 0, cpv);
    if (st != kOk) fill_nan(o, n_out);
    if (status && threadIdx.x == 0) status[c] = st;
    __syncthreads();  // the slab is reused by the next curve
  }
}

// center + normalize in place in global memory (no resampling; any n >= 3).
__global__ void __launch_bounds__(kThreads)
    preprocess_center_kernel(const double2* __restrict__ pts, const int64_t* __restrict__ off,
                             double2* __restrict__ out, int32_t* __restrict__ status) {
  __shared__ double2 red[kRedSlots];
  const int64_t c = blockIdx.x;
  const int64_t b0 = off[c];
  const int n = (int)(off[c + 1] - b0);
  const double2* in = pts + b0;
  double2* o = out + b0;
  int bad = n < 3;  // validate_curve(c) default min_nodes = 3 (curve.hpp:29)
  if (!bad) {
    double2 acc = make_double2(0, 0);
    int nf = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double2 q = __ldg(&in[i]);
      nf |= !(isfinite(q.x) && isfinite(q.y));
      acc = cadd(acc, q);
    }
    bad = block_or(nf, red);
    acc = block_sum2(acc, red);
    const double invn = 1.0 / (double)n;
    const double2 g = make_double2(invn * acc.x, invn * acc.y);
    double len = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double2 p0 = csub(__ldg(&in[i]), g), p1 = csub(__ldg(&in[i + 1 == n ? 0 : i + 1]), g);
      const double dx = p1.x - p0.x, dy = p1.y - p0.y;
      len += sqrt(fma(dx, dx, dy * dy));
    }
    len = block_sum(len, red);
    bad |= !(len > 0.0);
    if (!bad) {
      const double sc = 1.0 / len;
      for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = cscale(csub(__ldg(&in[i]), g), sc);
    }
  }
  if (bad) fill_nan(o, n > 0 ? n : 0);
  if (status && threadIdx.x == 0) status[c] = bad ? kInvalid : kOk;
}

// ------------------------------------------------------------ host launchers

size_t resample_smem_bytes(int nmax, int n_out) {
  return ResampleSmem::bytes(nmax) + sizeof(double2) * (size_t)n_out;
}

static cudaError_t set_smem(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t launch_tw_init(double2* tw, int N, cudaStream_t s) {
  tw_init_kernel<<<(N + 255) / 256, 256, 0, s>>>(tw, N);
  if (twiddle_extra(N)) ptw_fill_kernel<<<1, 256, 0, s>>>(tw, N);  // after the table (same stream)
  return cudaGetLastError();
}

int twiddle_extra(int N) {
  return (N >= 4 && N <= 4096 && (N & (N - 1)) == 0) ? pf::ptw_len(N) : 0;
}

cudaError_t launch_preprocess_resample(const double2* pts, const int64_t* off, int64_t curves,
                                       int nmax, int n_out, int center_normalize, double2* out,
                                       int32_t* status, cudaStream_t s) {
  const size_t sm = resample_smem_bytes(nmax, n_out);
  cudaError_t e = set_smem((const void*)preprocess_resample_kernel, sm);
  if (e != cudaSuccess) return e;
  preprocess_resample_kernel<<<(unsigned)curves, kThreads, sm, s>>>(pts, off, nmax, n_out,
                                                                     center_normalize, out, status);
  return cudaGetLastError();
}

cudaError_t launch_preprocess_center(const double2* pts, const int64_t* off, int64_t curves,
                                     double2* out, int32_t* status, cudaStream_t s) {
  preprocess_center_kernel<<<(unsigned)curves, kThreads, 0, s>>>(pts, off, out, status);
  return cudaGetLastError();
}

int max_chunked_nodes() { return kThreads * kMaxChunk; }

size_t resample_global_slab_bytes(int nmax) {
  return (ResampleSmem::bytes(nmax) + sizeof(double) * (size_t)nmax + 255) & ~size_t(255);
}
int resample_global_grid(int64_t curves) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)(curves < 4 * (int64_t)sms ? curves : 4 * (int64_t)sms);
}
cudaError_t launch_preprocess_resample_global(const double2* pts, const int64_t* off, int64_t curves, int nmax,
                                              int n_out, int center_normalize, double2* out, int32_t* status,
                                              void* slab, cudaStream_t s) {
  const int grid = resample_global_grid(curves);
  if (grid == 0) return cudaSuccess;
  preprocess_resample_global_kernel<<<grid, kThreads, 0, s>>>(pts, off, curves, nmax, n_out, center_normalize, out,
                                                              status, (char*)slab,
                                                              resample_global_slab_bytes(nmax));
  return cudaGetLastError();
}

}  // namespace cva
