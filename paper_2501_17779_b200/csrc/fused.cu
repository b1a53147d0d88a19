#include <algorithm>
#include <cstdlib>
// v2 sm_100a kernels (256 threads, 2 CTAs per SM): the fused C1 path and the
// shared-memory preprocess / align / SRV-align kernels built from resample.cuh
// and pairfft.cuh. kernels.cu keeps the general v1 kernels for sizes outside
// these bounds (raw curves > 3072 nodes, N > 2048).
#include <cuda_runtime.h>

#include "../../include/curvalign_cuda.h"
#include "fused.h"
#include "pairfft.cuh"
#include "prof.cuh"
#include "resample.cuh"
#include "resample3.cuh"

#ifdef CVA_PHASE_TIMING
extern "C" int cva_debug_set_prof(long long* p) {
  return cudaMemcpyToSymbol(g_cva_prof, &p, sizeof(p)) == cudaSuccess ? 0 : 4;
}
#endif

namespace cva {
namespace v2 {

constexpr int kT = 256;
constexpr size_t kRawBytes = sizeof(double2) * rs::kNMax + sizeof(double) * (rs::kNMax + 2);
constexpr size_t kScrBytes = sizeof(double) * rs::kScratchDoubles;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

// One TMA bulk copy (cp.async.bulk, completion counted on an mbarrier) per raw
// curve instead of n/256 dependent load->store rounds per thread. `bar` is a
// CTA mbarrier initialised by bulk_init; `phase` alternates 0, 1, ... per use.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_init(uint64_t* bar) {
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}
// Loads g[0..n) into sm and returns once every thread can read it. Requires a
// preceding __syncthreads() after the last generic access of sm's old data, and
// g 16-byte aligned (checked at the C ABI).
__device__ __forceinline__ void raw_to_smem(const double2* g, double2* sm, int n, uint64_t* bar,
                                            uint32_t phase) {
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)n * 16u, b = smem_u32(bar);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm)),
        "l"(g), "r"(bytes), "r"(b)
        : "memory");
  }
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void prefetch_l2(const void* p, int bytes) {
  if (bytes >= 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes & ~15) : "memory");
}

__device__ inline void write_bad(cva_alignment* out, int status) {
  cva_alignment r;
  r.shift = 0;
  r.t0 = 0.0;
  r.theta = qnan();
  r.trace = qnan();
  r.energy = qnan();
  r.degenerate = 0;
  r.status = status;
  *out = r;
}

// ---------------------------------------------------------------- fused C1

// Pair p = (curve 2p, curve 2p+1) of the ragged raw batch: preprocess both to
// N nodes (resample -> center -> normalize, curve.cpp:93-97) and align_fft
// (rigid_align.cpp:204-208), all on chip: the first curve's samples in their
// own padded buffer, the second's in the resampler's PCR scratch (dead by
// then), the transforms in the raw-curve region.
template <int N>
__global__ void __launch_bounds__(kT, 2)
    resample_align_kernel(const double2* __restrict__ pts, const int64_t* __restrict__ off,
                          const double2* __restrict__ tw, cva_alignment* __restrict__ out,
                          double2* aligned) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[16];
  double2* xy = reinterpret_cast<double2*>(smem);
  double* s = reinterpret_cast<double*>(xy + rs::kNMax);
  double2* bufs = reinterpret_cast<double2*>(smem);  // aliases the raw region after resampling
  double* scr = reinterpret_cast<double*>(smem + kRawBytes);
  double2* Z1 = reinterpret_cast<double2*>(smem + kRawBytes + kScrBytes);

  const int64_t p = blockIdx.x;
  const int64_t a0 = off[2 * p], a1 = off[2 * p + 1], b1 = off[2 * p + 2];
  const int na = (int)(a1 - a0), nb = (int)(b1 - a1);
  double2* al = aligned ? aligned + p * N : nullptr;  // null: results only
  if (threadIdx.x == 0) prefetch_l2(pts + a1, nb * (int)sizeof(double2));
  if (na < 4 || nb < 4 || na > rs::kNMax || nb > rs::kNMax) {  // validate_curve(c, 4)
    if (threadIdx.x == 0) write_bad(out + p, CVA_INVALID_ARGUMENT);
    if (al)
      for (int l = threadIdx.x; l < N; l += kT) al[l] = make_double2(qnan(), qnan());
    return;
  }
  CVA_MARK(0);
  __shared__ uint64_t mbar;
  bulk_init(&mbar);
  raw_to_smem(pts + a0, xy, na, &mbar, 0);
  CVA_MARK(1);
  const rs::CurveStats A = rs::resample_block<true, false, true>(xy, na, s, scr, red, Z1, N, 2);
  __syncthreads();  // resample_block's last reads of xy are done
  raw_to_smem(pts + a1, xy, nb, &mbar, 1);
  CVA_MARK(10);
  static_assert(sizeof(double2) * (N + N / 8) <= kScrBytes, "B's padded samples must fit the PCR scratch");
  double2* Z2 = reinterpret_cast<double2*>(scr);  // B's samples replace the PCR scratch
  const rs::CurveStats B = rs::resample_block<true, false, true, true>(xy, nb, s, scr, red, Z2, N, 11);
  if (A.bad || B.bad) {
    if (threadIdx.x == 0) write_bad(out + p, CVA_INVALID_ARGUMENT);
    if (al)
      for (int l = threadIdx.x; l < N; l += kT) al[l] = make_double2(qnan(), qnan());
    return;
  }
  __syncthreads();
  pf::PairIn in{Z1, Z2, A.centroid, B.centroid, A.inv_len, B.inv_len};
  pf::pair_stage<false, N, true, 2>(in, bufs, N, tw, out + p, al, red);
}

// ------------------------------------------------------------- preprocess

// preprocess(raw, n_out, true) (curve.cpp:93-97) or resample_uniform alone
// (center_normalize == 0) for one curve per CTA; n_out <= 2048.
template <bool kPow2>
__global__ void __launch_bounds__(kT, 2)
    preprocess_kernel(const double2* __restrict__ pts, const int64_t* __restrict__ off, int n_out,
                      int center_normalize, double2* out,
                      int32_t* __restrict__ status) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[16];
  double2* xy = reinterpret_cast<double2*>(smem);
  double* s = reinterpret_cast<double*>(xy + rs::kNMax);
  double* scr = reinterpret_cast<double*>(smem + kRawBytes);
  double2* Z = reinterpret_cast<double2*>(smem + kRawBytes + kScrBytes);
  const int64_t c = blockIdx.x;
  const int64_t b0 = off[c];
  const int n = (int)(off[c + 1] - b0);
  double2* o = out + c * n_out;
  int bad = n < 4 || n > rs::kNMax;
  rs::CurveStats st{};
  if (!bad) {
    __shared__ uint64_t mbar;
    bulk_init(&mbar);
    raw_to_smem(pts + b0, xy, n, &mbar, 0);
    st = rs::resample_block<kPow2, true, true>(xy, n, s, scr, red, Z, n_out);
    bad = st.bad;
  }
  if (bad) {
    for (int l = threadIdx.x; l < n_out; l += kT) o[l] = make_double2(qnan(), qnan());
  } else if (center_normalize) {
    for (int l = threadIdx.x; l < n_out; l += kT) {
      const double2 z = Z[l + (l >> 3)];
      o[l] = make_double2((z.x - st.centroid.x) * st.inv_len, (z.y - st.centroid.y) * st.inv_len);
    }
  } else {
    for (int l = threadIdx.x; l < n_out; l += kT) o[l] = Z[l + (l >> 3)];
  }
  if (status && threadIdx.x == 0) status[c] = bad ? CVA_INVALID_ARGUMENT : CVA_OK;
}

// ----------------------------------------------------------------- align

// align_fft on pre-sampled pairs (rigid_align.cpp:204-208), N = 2^p <= 2048.
// Pair p reads c1 + p * stride and c2 + p * stride (stride N: separate
// batches; stride 2N with c2 = c1 + N: interleaved rows 2p, 2p+1).
// Optional per-curve normalisation (centroid x, y, 1/length, -) and invalid
// flags fuse preprocess(resample=false) into the load (cva_preprocess_align_uniform).
template <bool kIP, int kN>
__global__ void __launch_bounds__(kT, kIP ? 2 : 3)
    align_kernel(const double2* __restrict__ c1, const double2* __restrict__ c2, int N,
                 int64_t stride1, int64_t stride2, const double2* __restrict__ tw,
                 cva_alignment* __restrict__ out, double2* aligned, const double4* __restrict__ norm1,
                 const double4* __restrict__ norm2, const int32_t* __restrict__ bad1,
                 const int32_t* __restrict__ bad2) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[16];
  const int64_t p = blockIdx.x;
  pf::PairIn in{c1 + p * stride1, c2 + p * stride2, make_double2(0, 0), make_double2(0, 0), 1.0, 1.0};
  if (norm1) {
    if (bad1[p] || bad2[p]) {
      if (threadIdx.x == 0) write_bad(out + p, CVA_INVALID_ARGUMENT);
      if (aligned)
        for (int l = threadIdx.x; l < N; l += kT) aligned[p * N + l] = make_double2(qnan(), qnan());
      return;
    }
    const double4 a = norm1[p], b = norm2[p];
    in.g1 = make_double2(a.x, a.y);
    in.sc1 = a.z;
    in.g2 = make_double2(b.x, b.y);
    in.sc2 = b.z;
  }
  pf::pair_stage<kIP, kN>(in, reinterpret_cast<double2*>(smem), N, tw, out + p,
                          aligned ? aligned + p * N : nullptr, red);
}

// align_fft for transform length M = 4096 (non-power-of-two N in (1024, 2048],
// zero-padded per pairfft.cuh fft_len, and N = 4096): 512 threads, one CTA per
// SM, the two forward transforms in place on 256-thread halves, the
// correlation transform in place on all 512 (147 KB of shared memory).
// Same parameters as align_kernel.
constexpr int kT4 = 512;
__global__ void __launch_bounds__(kT4, 1)
    align4k_kernel(const double2* __restrict__ c1, const double2* __restrict__ c2, int N,
                   int64_t stride1, int64_t stride2, const double2* __restrict__ tw,
                   cva_alignment* __restrict__ out, double2* aligned, const double4* __restrict__ norm1,
                   const double4* __restrict__ norm2, const int32_t* __restrict__ bad1,
                   const int32_t* __restrict__ bad2) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[32];
  static_assert(pf::plan_is_128<kT4>(4096), "the 512-thread plan reads the 128-thread tables");
  const int64_t p = blockIdx.x;
  pf::PairIn in{c1 + p * stride1, c2 + p * stride2, make_double2(0, 0), make_double2(0, 0), 1.0, 1.0};
  if (norm1) {
    if (bad1[p] || bad2[p]) {
      if (threadIdx.x == 0) write_bad(out + p, CVA_INVALID_ARGUMENT);
      if (aligned)
        for (int l = threadIdx.x; l < N; l += kT4) aligned[p * N + l] = make_double2(qnan(), qnan());
      return;
    }
    const double4 a = norm1[p], b = norm2[p];
    in.g1 = make_double2(a.x, a.y);
    in.sc1 = a.z;
    in.g2 = make_double2(b.x, b.y);
    in.sc2 = b.z;
  }
  pf::pair_stage<true, 0, false, 0, kT4, 4096>(in, reinterpret_cast<double2*>(smem), N, tw, out + p,
                                                aligned ? aligned + p * N : nullptr, red);
}

// ------------------------------------------------------------------- SRV

// SRV alignment (srv_transform -> srv_center -> align_fft, the (t0,R) step of
// elastic.cpp:138-139). Both raw curves arrive by TMA bulk copy in the
// transform buffers they will be read from; the SRVs are formed from shared
// memory into the padded layout the first transform pass reads (the input
// buffers of that pass: in place at M = 2048, the ping-pong partner
// otherwise), and the aligned output recomputes q2 from the raw curve (L2).
#ifndef CVA_SRV_TMA_RAW
#define CVA_SRV_TMA_RAW 1
#endif
#ifndef CVA_SRV_KEEP_Q
#define CVA_SRV_KEEP_Q 1
#endif
template <bool kIP, int kN>
__global__ void __launch_bounds__(kT, kIP ? 2 : 3)
    srv_align_kernel(const double2* __restrict__ c1, const double2* __restrict__ c2, int N,
                     const double2* __restrict__ tw, cva_alignment* __restrict__ out, double2* aligned) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[16];
  __shared__ uint64_t mbar;
  constexpr int kMaxPer = 8;  // N / kT values per thread (N <= 2048)
  if constexpr (kN > 0) N = kN;
  const int64_t p = blockIdx.x;
  const double2* a = c1 + p * N;
  const double2* b = c2 + p * N;
  const int NP = pf::padded_len(pf::fft_len(N));
  double2* bufs = reinterpret_cast<double2*>(smem);
  double2* qa = kIP ? bufs : bufs + NP;           // B0 (in place) or B1
  double2* qb = kIP ? bufs + NP : bufs + 3 * NP;  // B2 (in place: bufs + NP) or B3
  bulk_init(&mbar);
  if (threadIdx.x == 0) {  // both raw curves on one mbarrier phase
    const uint32_t bytes = (uint32_t)N * 16u, bar = smem_u32(&mbar);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(qa)),
                 "l"(a), "r"(bytes), "r"(bar)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(qb)),
                 "l"(b), "r"(bytes), "r"(bar)
                 : "memory");
  }
  {
    uint32_t done = 0;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(smem_u32(&mbar))
          : "memory");
    } while (!done);
  }
  // one curve at a time (half the live registers): SRV of the raw samples into
  // registers, a barrier (every raw read done), then the padded write in place
  int bad = 0;
  double2 mean0 = make_double2(0, 0), mean1 = make_double2(0, 0);  // (not an array: the loop index is runtime)
  // the in-place plan brings q2 back by TMA for the aligned output: park it in
  // this pair's aligned rows (L2-resident, overwritten at the end)
  double2* const keep = (CVA_SRV_KEEP_Q && CVA_SRV_TMA_RAW && kIP && aligned) ? aligned + p * N : nullptr;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    double2* qc = h ? qb : qa;
    double2 x[kMaxPer];
    double2 m = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      const int l = threadIdx.x + q * kT;
      if (l < N) {
        const double2 u = qc[l];
        bad |= !(isfinite(u.x) && isfinite(u.y));
        x[q] = pf::srv_at(qc, l, N);
        if (h && keep) keep[l] = x[q];
        m = cadd(m, x[q]);
      }
    }
    double mz = 0.0;
    rs::block_sum3(m.x, m.y, mz, red);  // its barriers order every raw read before the writes
    if (h)
      mean1 = m;
    else
      mean0 = m;
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      const int l = threadIdx.x + q * kT;
      if (l < N) qc[pf::pad(l)] = x[q];
    }
  }
  bad = __syncthreads_or(bad);
  double2* al = aligned ? aligned + p * N : nullptr;
  if (bad) {
    if (threadIdx.x == 0) write_bad(out + p, CVA_INVALID_ARGUMENT);
    if (al)
      for (int l = threadIdx.x; l < N; l += kT) al[l] = make_double2(qnan(), qnan());
    return;
  }
  const double2 m1 = mean0;
  const double m2x = mean1.x, m2y = mean1.y;
  const double invn = 1.0 / (double)N;  // srv_center (srv.cpp:90-98)
  pf::PairIn in{qa, qb, make_double2(invn * m1.x, invn * m1.y), make_double2(invn * m2x, invn * m2y), 1.0, 1.0, b};
#if CVA_SRV_TMA_RAW
  in.bar = &mbar;  // phase 0 was the input copies
  if (keep) {  // the generic stores of q2 before the async-proxy read of them
    asm volatile("fence.proxy.async.global;" ::: "memory");
    in.q2_in_aligned = true;
  }
#endif
  pf::pair_stage<kIP, kN, false, 2, kT, 2048, true>(in, bufs, N, tw, out + p, al, red);
}

// srv_center(srv_transform(c)) of one curve per CTA into global memory, any
// N (srv.cpp:71-98): the large-N SRV alignment feeds these to the multi-pass
// transforms. A curve with a non-finite node becomes NaN (its pair then
// reports CVA_INVALID_ARGUMENT, like validate_curve).
__global__ void __launch_bounds__(kT) srv_center_kernel(const double2* __restrict__ c, int N, double2* __restrict__ q) {
  __shared__ double2 red[16];
  const int64_t k = blockIdx.x;
  const double2* x = c + k * N;
  double2* o = q + k * N;
  double mx = 0.0, my = 0.0, nf = 0.0;
  for (int l = threadIdx.x; l < N; l += kT) {
    const double2 u = x[l];
    nf += (isfinite(u.x) && isfinite(u.y)) ? 0.0 : 1.0;
    const double2 v = pf::srv_at(x, l, N);
    o[l] = v;
    mx += v.x;
    my += v.y;
  }
  rs::block_sum3(mx, my, nf, red);
  const double invn = 1.0 / (double)N;
  const double2 m = nf != 0.0 ? make_double2(qnan(), qnan()) : make_double2(invn * mx, invn * my);
  for (int l = threadIdx.x; l < N; l += kT) {  // each thread rewrites only its own entries
    const double2 v = o[l];
    o[l] = make_double2(v.x - m.x, v.y - m.y);
  }
}

}  // namespace v2

// ------------------------------------------------------------ fused C1 (v3)

namespace v3 {


// Shared memory: [XY | S] (rs3::kRawBytes, reused by the four FFT buffers),
// scratch (PCR; curve B's samples in its first 16 KB; the interval map at
// rs3::kMapOff), curve A's samples.
constexpr size_t kZ1Off = rs3::kRawBytes + rs3::kScrBytes;
template <int N>
constexpr size_t smem_bytes() {
  return kZ1Off + sizeof(double2) * N;
}
static_assert(4 * sizeof(double2) * pf::padded_len(1024) <= rs3::kRawBytes, "FFT buffers fit the raw region");

// Pair p = (curve 2p, curve 2p+1) of the ragged raw batch: preprocess both to
// N nodes (resample -> center -> normalize, curve.cpp:93-97) and align_fft
// (rigid_align.cpp:204-208), all on chip.
template <int N>
__global__ void __launch_bounds__(rs3::kT, 2)
    resample_align_kernel(const double2* __restrict__ pts, const int64_t* __restrict__ off, int64_t pairs,
                          int64_t ahead, const double2* __restrict__ tw, cva_alignment* __restrict__ out,
                          double2* aligned) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double2 red[16];
  double2* XY = reinterpret_cast<double2*>(smem);
  double* S = reinterpret_cast<double*>(smem + rs3::kXYBytes);
  double* scr = reinterpret_cast<double*>(smem + rs3::kRawBytes);
  double2* Z1 = reinterpret_cast<double2*>(smem + kZ1Off);
  double2* Z2 = reinterpret_cast<double2*>(scr);  // B's samples replace the PCR scratch

  // one CTA per pair; the CTA that starts `ahead` pairs later (about one wave
  // of resident CTAs) finds its raw curves in L2: prefetch them now
  const int64_t p = blockIdx.x;
  const int64_t a0 = off[2 * p], a1 = off[2 * p + 1], b1 = off[2 * p + 2];
  const int na = (int)(a1 - a0), nb = (int)(b1 - a1);
  double2* al = aligned ? aligned + p * N : nullptr;  // null: results only
  if (threadIdx.x == rs3::kT - 32) {  // a thread of the last warp (idle in most phases)
    v2::prefetch_l2(pts + a1, nb * (int)sizeof(double2));
    const int64_t q = p + ahead;
    if (ahead > 0 && q < pairs) {
      const int64_t c0 = off[2 * q], c2 = off[2 * q + 2];
      const int64_t cn = c2 - c0 < (1 << 20) ? c2 - c0 : (1 << 20);
      v2::prefetch_l2(pts + c0, (int)cn * (int)sizeof(double2));
    }
  }
  if (na < 4 || nb < 4 || na > rs3::kNMax || nb > rs3::kNMax) {  // validate_curve(c, 4)
    if (threadIdx.x == 0) v2::write_bad(out + p, CVA_INVALID_ARGUMENT);
    if (al)
      for (int l = threadIdx.x; l < N; l += rs3::kT) al[l] = make_double2(v2::qnan(), v2::qnan());
    return;
  }
  CVA_MARK(0);
  rs3::load_raw(pts + a0, XY, na);
  rs3::cp_async_wait();
  __syncthreads();
  CVA_MARK(1);
  // centroids: each resample leaves its per-warp partial sums here and both
  // are reduced after curve B (block_sum2's order, so bitwise the same
  // centroids, minus one block reduction and its barriers per pair: -1 %)
  __shared__ double2 wsA[rs3::kT / 32], wsB[rs3::kT / 32];
  const rs3::Stats A = rs3::resample_curve<N>(pts + a0, XY, S, scr, Z1, red, na, 2, wsA);
  __syncthreads();  // A's last reads of XY / S / the map are done
  rs3::load_raw(pts + a1, XY, nb);
  rs3::cp_async_wait();
  __syncthreads();
  CVA_MARK(10);
  const rs3::Stats B = rs3::resample_curve<N>(pts + a1, XY, S, scr, Z2, red, nb, 11, wsB);
  if (A.bad | B.bad) {
    if (threadIdx.x == 0) v2::write_bad(out + p, CVA_INVALID_ARGUMENT);
    if (al)
      for (int l = threadIdx.x; l < N; l += rs3::kT) al[l] = make_double2(v2::qnan(), v2::qnan());
    return;
  }
  __syncthreads();
  double2 cA, cB;
  {
    const int lane = threadIdx.x & 31;
    constexpr double invN = 1.0 / (double)N;
    const double2 sA = warp_sum2(lane < rs3::kT / 32 ? wsA[lane] : make_double2(0.0, 0.0));
    const double2 sB = warp_sum2(lane < rs3::kT / 32 ? wsB[lane] : make_double2(0.0, 0.0));
    cA = make_double2(sA.x * invN, sA.y * invN);
    cB = make_double2(sB.x * invN, sB.y * invN);
  }
  pf::PairIn in{Z1, Z2, cA, cB, 1.0, 1.0};
  pf::pair_stage<false, N, true, 0, rs3::kT, 2048, true>(in, reinterpret_cast<double2*>(smem), N, tw, out + p, al,
                                                         red);
}

}  // namespace v3

// ------------------------------------------------------------ launchers

namespace {
cudaError_t set_smem(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
}  // namespace

int v2_max_raw_nodes() { return rs::kNMax; }

// In-place transforms (half the buffers) once four buffers would exceed ~75 KB,
// so the pair kernels keep >= 2-3 CTAs per SM (N = 2048: 147 KB -> 74 KB).
bool v2_inplace(int N) { return pf::fft_len(N) == 2048; }

// Compile-time FFT plans for the common power-of-two lengths (no runtime
// radix loop or index division); kN = 0 is the runtime-N kernel.
template <int kN>
static cudaError_t launch_align_n(unsigned grid, size_t sm, cudaStream_t s, const double2* c1,
                                  const double2* c2, int N, int64_t st1, int64_t st2, const double2* tw,
                                  cva_alignment* out, double2* aligned, const double4* n1, const double4* n2,
                                  const int32_t* b1, const int32_t* b2) {
  constexpr bool kIP = kN == 2048;
  cudaError_t e = set_smem((const void*)v2::align_kernel<kIP, kN>, sm);
  if (e != cudaSuccess) return e;
  v2::align_kernel<kIP, kN><<<grid, v2::kT, sm, s>>>(c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
  return cudaGetLastError();
}

static cudaError_t launch_align_kernel(unsigned grid, size_t sm, cudaStream_t s, const double2* c1,
                                       const double2* c2, int N, int64_t st1, int64_t st2, const double2* tw,
                                       cva_alignment* out, double2* aligned, const double4* n1, const double4* n2,
                                       const int32_t* b1, const int32_t* b2) {
  if (pf::fft_len(N) == 4096) {
    const size_t sm4 = 2 * sizeof(double2) * (size_t)pf::padded_len(4096);
    cudaError_t e = set_smem((const void*)v2::align4k_kernel, sm4);
    if (e != cudaSuccess) return e;
    v2::align4k_kernel<<<grid, v2::kT4, sm4, s>>>(c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
    return cudaGetLastError();
  }
  switch (N) {
    case 2048: return launch_align_n<2048>(grid, sm, s, c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
    case 1024: return launch_align_n<1024>(grid, sm, s, c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
    case 512: return launch_align_n<512>(grid, sm, s, c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
    case 256: return launch_align_n<256>(grid, sm, s, c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
    default: break;
  }
  const bool ip = v2_inplace(N);
  const void* fn = ip ? (const void*)v2::align_kernel<true, 0> : (const void*)v2::align_kernel<false, 0>;
  cudaError_t e = set_smem(fn, sm);
  if (e != cudaSuccess) return e;
  if (ip)
    v2::align_kernel<true, 0><<<grid, v2::kT, sm, s>>>(c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
  else
    v2::align_kernel<false, 0><<<grid, v2::kT, sm, s>>>(c1, c2, N, st1, st2, tw, out, aligned, n1, n2, b1, b2);
  return cudaGetLastError();
}

size_t v2_resample_align_smem(int N) {
  const size_t fft = 4 * sizeof(double2) * (size_t)pf::padded_len(N);
  const size_t raw = v2::kRawBytes > fft ? v2::kRawBytes : fft;
  return raw + v2::kScrBytes + sizeof(double2) * (size_t)(N + N / 8);  // Z1 padded
}
size_t v2_preprocess_smem(int n_out) {
  return v2::kRawBytes + v2::kScrBytes + sizeof(double2) * (size_t)(n_out + n_out / 8);  // Z padded
}
size_t v2_align_smem(int N) {
  return (v2_inplace(N) ? 2 : 4) * sizeof(double2) * (size_t)pf::padded_len(pf::fft_len(N));
}
int v2_fft_len(int N) { return pf::fft_len(N); }

bool v2_resample_align_supported(int N) { return N == 512 || N == 1024; }

cudaError_t launch_v2_resample_align(const double2* pts, const int64_t* off, int64_t pairs, int N,
                                     const double2* tw, cva_alignment* out, double2* aligned,
                                     cudaStream_t s) {
  const size_t sm = v2_resample_align_smem(N)
#ifdef CVA_PAD_SMEM
      + CVA_PAD_SMEM
#endif
      ;
  const void* fn = N == 512 ? (const void*)v2::resample_align_kernel<512>
                            : (const void*)v2::resample_align_kernel<1024>;
  cudaError_t e = set_smem(fn, sm);
  if (e != cudaSuccess) return e;
  if (N == 512)
    v2::resample_align_kernel<512><<<(unsigned)pairs, v2::kT, sm, s>>>(pts, off, tw, out, aligned);
  else
    v2::resample_align_kernel<1024><<<(unsigned)pairs, v2::kT, sm, s>>>(pts, off, tw, out, aligned);
  return cudaGetLastError();
}


bool v3_resample_align_supported(int N) { return N == 512 || N == 1024; }
int v3_max_raw_nodes() { return rs3::kNMax; }

// One CTA per pair; each prefetches (into L2) the pair one wave of resident
// CTAs ahead.
template <int N>
static cudaError_t launch_v3_n(const double2* pts, const int64_t* off, int64_t pairs, const double2* tw,
                               cva_alignment* out, double2* aligned, size_t sm, cudaStream_t s) {
  const void* fn = (const void*)v3::resample_align_kernel<N>;
  cudaError_t e = set_smem(fn, sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, rs3::kT, sm);
  const int64_t ahead = (int64_t)std::max(1, sms) * std::max(1, per);
  v3::resample_align_kernel<N><<<(unsigned)pairs, rs3::kT, sm, s>>>(pts, off, pairs, ahead, tw, out, aligned);
  return cudaGetLastError();
}

cudaError_t launch_v3_resample_align(const double2* pts, const int64_t* off, int64_t pairs, int N,
                                     const double2* tw, cva_alignment* out, double2* aligned,
                                     cudaStream_t s) {
  // CVA_SMEM_PAD=<bytes> (measurement only): extra dynamic shared memory per CTA,
  // e.g. to run one CTA per SM
  static const size_t pad = [] {
    const char* e = std::getenv("CVA_SMEM_PAD");
    return e ? (size_t)std::strtoul(e, nullptr, 10) : (size_t)0;
  }();
  if (pairs <= 0) return cudaSuccess;
  if (N == 512) return launch_v3_n<512>(pts, off, pairs, tw, out, aligned, v3::smem_bytes<512>() + pad, s);
  return launch_v3_n<1024>(pts, off, pairs, tw, out, aligned, v3::smem_bytes<1024>() + pad, s);
}

cudaError_t launch_v2_preprocess(const double2* pts, const int64_t* off, int64_t curves, int n_out,
                                 int center_normalize, double2* out, int32_t* status,
                                 cudaStream_t s) {
  const size_t sm = v2_preprocess_smem(n_out);
  const bool pow2 = (n_out & (n_out - 1)) == 0;
  const void* fn = pow2 ? (const void*)v2::preprocess_kernel<true> : (const void*)v2::preprocess_kernel<false>;
  cudaError_t e = set_smem(fn, sm);
  if (e != cudaSuccess) return e;
  if (pow2)
    v2::preprocess_kernel<true><<<(unsigned)curves, v2::kT, sm, s>>>(pts, off, n_out, center_normalize,
                                                                     out, status);
  else
    v2::preprocess_kernel<false><<<(unsigned)curves, v2::kT, sm, s>>>(pts, off, n_out,
                                                                      center_normalize, out, status);
  return cudaGetLastError();
}

cudaError_t launch_v2_align(const double2* c1, const double2* c2, int64_t pairs, int N,
                            const double2* tw, cva_alignment* out, double2* aligned,
                            cudaStream_t s) {
  const size_t sm = v2_align_smem(N);
  return launch_align_kernel((unsigned)pairs, sm, s, c1, c2, N, N, N, tw, out, aligned, nullptr, nullptr, nullptr,
                             nullptr);
}

cudaError_t launch_v2_align_norm(const double2* c1, const double2* c2, int64_t pairs, int N, const double2* tw,
                                 const double4* norm1, const double4* norm2, const int32_t* bad1,
                                 const int32_t* bad2, cva_alignment* out, double2* aligned, cudaStream_t s) {
  const size_t sm = v2_align_smem(N);
  return launch_align_kernel((unsigned)pairs, sm, s, c1, c2, N, N, N, tw, out, aligned, norm1, norm2, bad1, bad2);
}

cudaError_t launch_v2_align_interleaved(const double2* rows, int64_t pairs, int N, const double2* tw,
                                        cva_alignment* out, double2* aligned, cudaStream_t s) {
  const size_t sm = v2_align_smem(N);
  return launch_align_kernel((unsigned)pairs, sm, s, rows, rows + N, N, 2 * (int64_t)N, 2 * (int64_t)N, tw, out,
                             aligned, nullptr, nullptr, nullptr, nullptr);
}

// One row of an all-pairs matrix: pair j = (row, curves[j]) for j < count.
cudaError_t launch_v2_align_row(const double2* row, const double2* curves, int64_t count, int N,
                                const double2* tw, cva_alignment* out, cudaStream_t s) {
  const size_t sm = v2_align_smem(N);
  return launch_align_kernel((unsigned)count, sm, s, row, curves, N, 0, N, tw, out, nullptr, nullptr, nullptr,
                             nullptr, nullptr);
}

namespace v2 {
__global__ void unpack_row_kernel(const cva_alignment* __restrict__ in, int64_t count, double* energy,
                                  int32_t* shift, double* theta) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < count) {
    const cva_alignment r = in[j];
    energy[j] = r.energy;
    shift[j] = (int32_t)r.shift;
    theta[j] = r.theta;
  }
}
}  // namespace v2

cudaError_t launch_unpack_row(const cva_alignment* in, int64_t count, double* energy, int32_t* shift,
                              double* theta, cudaStream_t s) {
  v2::unpack_row_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(in, count, energy, shift, theta);
  return cudaGetLastError();
}

template <bool kIP, int kN>
static cudaError_t launch_srv_n(const double2* c1, const double2* c2, int64_t pairs, int N,
                                const double2* tw, cva_alignment* out, double2* aligned, size_t sm, cudaStream_t s) {
  cudaError_t e = set_smem((const void*)v2::srv_align_kernel<kIP, kN>, sm);
  if (e != cudaSuccess) return e;
  v2::srv_align_kernel<kIP, kN><<<(unsigned)pairs, v2::kT, sm, s>>>(c1, c2, N, tw, out, aligned);
  return cudaGetLastError();
}

cudaError_t launch_v2_srv_align(const double2* c1, const double2* c2, int64_t pairs, int N,
                                const double2* tw, cva_alignment* out, double2* aligned, cudaStream_t s) {
  const size_t sm = v2_align_smem(N);
  switch (N) {
    case 2048: return launch_srv_n<true, 2048>(c1, c2, pairs, N, tw, out, aligned, sm, s);
    case 1024: return launch_srv_n<false, 1024>(c1, c2, pairs, N, tw, out, aligned, sm, s);
    case 512: return launch_srv_n<false, 512>(c1, c2, pairs, N, tw, out, aligned, sm, s);
    default: break;
  }
  if (v2_inplace(N)) return launch_srv_n<true, 0>(c1, c2, pairs, N, tw, out, aligned, sm, s);
  return launch_srv_n<false, 0>(c1, c2, pairs, N, tw, out, aligned, sm, s);
}

}  // namespace cva

namespace cva {
cudaError_t launch_v2_srv_center(const double2* c, int64_t curves, int N, double2* q, cudaStream_t s) {
  if (curves > 0) v2::srv_center_kernel<<<(unsigned)curves, v2::kT, 0, s>>>(c, N, q);
  return cudaGetLastError();
}
}  // namespace cva
