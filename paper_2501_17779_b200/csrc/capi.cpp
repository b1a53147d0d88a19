#include <cstdlib>
// extern "C" entry points of libcurvalign_cuda.so (declared in include/curvalign_cuda.h).
//
// Host-side validation mirrors the reference's std::invalid_argument checks
// (proj/src/rigid_align.cpp:18-21, proj/src/curve.cpp:10-15, :68-69,
// proj/src/srv.cpp:72); data-dependent failures are reported per pair by the
// kernels. There is no CPU fallback: without a CUDA device every compute entry
// point fails with CVA_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <climits>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/curvalign_cuda.h"
#include "elastic.h"
#include "fused.h"
#include "kernels.h"
#include "largen.h"

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

// Curve buffers are read and written as double2 (16 B): device pointers must
// be 16-byte aligned (cudaMalloc'd arrays and whole-point offsets are).
bool a16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
int misaligned(const char* what) {
  return fail(CVA_INVALID_ARGUMENT, std::string(what) +
                                        ": curve buffers must be 16-byte aligned (interleaved x, y doubles)");
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(CVA_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}


// Twiddle tables w_N^k, one per (device, N), built once and kept for the process.
std::mutex g_tw_mu;
std::map<std::pair<int, int>, double2*> g_tw;

int get_twiddles(int n, cudaStream_t stream, const double2** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(g_tw_mu);
  auto it = g_tw.find({dev, n});
  if (it != g_tw.end()) {
    *out = it->second;
    return CVA_OK;
  }
  double2* tw = nullptr;
  e = cudaMalloc(&tw, sizeof(double2) * (size_t)(n + cva::twiddle_extra(n)));
  if (e != cudaSuccess) return fail(CVA_BAD_ALLOC, "twiddle table allocation failed");
  e = cva::launch_tw_init(tw, n, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    cudaFree(tw);
    return cuda_fail(e, "twiddle init");
  }
  g_tw[{dev, n}] = tw;
  *out = tw;
  return CVA_OK;
}

int require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(CVA_CUDA_ERROR, "no CUDA device available");
  return CVA_OK;
}

int smem_limit() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

// FFT sizes the shared-memory kernels cover in this build.
// Shared-memory pair kernels: power-of-two N <= 2048, other N zero-padded to a
// power of two M >= 2N (pairfft.cuh), so N <= 1024. Larger N: largen.cu.
constexpr int64_t kMaxLargeN = 1 << 22;

bool small_fft(int64_t n) { return n <= 2048 && cva::v2_fft_len((int)n) <= 2048; }
// the pair-alignment kernels (launch_v2_align*): shared-memory transforms up to
// M = 2048, and the 512-thread in-place kernel for M = 4096
bool pair_fft(int64_t n) { return small_fft(n) || (n <= 4096 && cva::v2_fft_len((int)n) == 4096); }

int check_fft_size(int64_t n) {
  if (n < 4) return fail(CVA_INVALID_ARGUMENT, "align: need at least 4 nodes");
  if (n > kMaxLargeN) return fail(CVA_UNSUPPORTED, "align: N beyond 4M nodes");
  return CVA_OK;
}


// Stream-ordered scratch (cudaMallocAsync on the call's stream, freed after the
// kernels on the same stream): safe for concurrent calls on different streams.
// Scratch comes from this library's own stream-ordered pool per device (freed
// blocks stay cached up to kPoolKeep bytes; the process-wide default pool and
// its release threshold are left to the application).
constexpr uint64_t kPoolKeep = uint64_t(2) << 30;
std::mutex g_pool_mu;
std::map<int, cudaMemPool_t> g_pools;

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    auto it = g_pools.find(dev);
    if (it == g_pools.end()) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pool, &props);
      if (e != cudaSuccess) return e;
      uint64_t thr = kPoolKeep;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      g_pools[dev] = pool;
    } else {
      pool = it->second;
    }
  }
  return cudaMallocFromPoolAsync(p, bytes ? bytes : 16, pool, s);
}

int64_t host_max_n(const int64_t* offsets, int64_t curves) {
  int64_t m = 0;
  for (int64_t c = 0; c < curves; ++c) m = std::max(m, offsets[c + 1] - offsets[c]);
  return m;
}

int device_max_n(const int64_t* d_offsets, int64_t curves, cudaStream_t s, int64_t* out) {
  std::vector<int64_t> h((size_t)curves + 1);
  cudaError_t e = cudaMemcpyAsync(h.data(), d_offsets, sizeof(int64_t) * h.size(),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "offsets D2H");
  *out = host_max_n(h.data(), curves);
  return CVA_OK;
}

int finish(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return cuda_fail(e, what);
  return CVA_OK;
}

// General resampler for raw curves the v2 kernel does not hold: the v1
// shared-memory kernel when the curve and its solver arrays fit shared memory,
// else the same solver on per-CTA global slabs (any n_in, any n_out).
int resample_general(const double* points, const int64_t* offsets, int64_t curves, int nmax, int64_t n_out,
                     int center_normalize, double* out, int32_t* status, cudaStream_t s) {
  const size_t smem = cva::resample_smem_bytes(nmax, (int)n_out);
  if (nmax <= cva::max_chunked_nodes() && smem <= (size_t)smem_limit())
    return finish(cva::launch_preprocess_resample((const double2*)points, offsets, curves, nmax, (int)n_out,
                                                  center_normalize, (double2*)out, status, s),
                  "preprocess launch");
  void* slab = nullptr;
  const size_t bytes = cva::resample_global_slab_bytes(nmax) * (size_t)cva::resample_global_grid(curves);
  if (scratch_alloc(&slab, bytes, s) != cudaSuccess) return fail(CVA_BAD_ALLOC, "resample slab allocation failed");
  cudaError_t e = cva::launch_preprocess_resample_global((const double2*)points, offsets, curves, nmax, (int)n_out,
                                                         center_normalize, (double2*)out, status, slab, s);
  cudaFreeAsync(slab, s);
  return finish(e, "preprocess (global slab) launch");
}

#ifndef CVA_LARGE_TWO_STREAMS
#define CVA_LARGE_TWO_STREAMS 1
#endif

// This host thread's side stream on the current device (non-blocking, kept).
cudaStream_t side_stream() {
  thread_local std::map<int, cudaStream_t> streams;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto it = streams.find(dev);
  if (it != streams.end()) return it->second;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  streams[dev] = st;
  return st;
}

int large_align(const double* c1, const double* c2, int64_t pairs, int64_t n, int normalize,
                cva_alignment* out, double* aligned, const double2* tw, cudaStream_t s) {
  // four-step twiddle tables (sub-transform lengths and the two-level W_M)
  cva::FourStepTw fst{};
  const int M = cva::v2_fft_len((int)n), m1 = cva::four_step_m1(M);
  if (m1) {
    fst.lo = tw;
    if (int rc = get_twiddles(m1, s, &fst.s1)) return rc;
    if (int rc = get_twiddles(M / m1, s, &fst.s2)) return rc;
    if (int rc = get_twiddles(M / 256, s, &fst.hi)) return rc;
  }
  // Chunks of pairs alternate between the caller's stream and a side stream
  // (forked / joined with events), each with its own workspace: the small
  // tail kernels of chunk c (candidate / pick / aligned output, a few dozen
  // CTAs) run under the transforms of chunk c + 1. Two chunks in flight share
  // the L2, so each is half the single-stream chunk.
  const int64_t full = cva::large_chunk_pairs((int)n);
  const bool two = CVA_LARGE_TWO_STREAMS && pairs > full / 2 && full >= 2;
  const int64_t chunk = std::min<int64_t>(pairs, two ? std::max<int64_t>(1, full / 2) : full);
  void* ws[2] = {nullptr, nullptr};
  for (int i = 0; i < (two ? 2 : 1); ++i)
    if (scratch_alloc(&ws[i], cva::large_workspace_bytes(chunk, (int)n), s) != cudaSuccess) {
      if (ws[0]) cudaFreeAsync(ws[0], s);
      return fail(CVA_BAD_ALLOC, "large-N workspace allocation failed");
    }
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaError_t e = cudaSuccess;
  if (two) {
    side = side_stream();
    if (!side || cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&join, cudaEventDisableTiming) != cudaSuccess) {
      e = cudaErrorUnknown;
    } else {
      e = cudaEventRecord(fork, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
    }
  }
  for (int64_t p0 = 0, c = 0; p0 < pairs && e == cudaSuccess; p0 += chunk, ++c) {
    const int64_t P = std::min(chunk, pairs - p0);
    const bool alt = two && (c & 1);
    e = cva::launch_large_align((const double2*)c1 + p0 * n, (const double2*)c2 + p0 * n, P, (int)n, normalize, tw,
                                m1 ? &fst : nullptr, out + p0, aligned ? (double2*)aligned + p0 * n : nullptr,
                                ws[alt ? 1 : 0], chunk, alt ? side : s);
  }
  if (two && side) {
    if (e == cudaSuccess) e = cudaEventRecord(join, side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, join, 0);
  }
  if (fork) cudaEventDestroy(fork);
  if (join) cudaEventDestroy(join);
  for (void* w : ws)
    if (w) cudaFreeAsync(w, s);
  return finish(e, "large-N align launch");
}

// v2 shared-memory resampler when the batch fits it, else the general v1 kernel.
int resample_dispatch(const double* points, const int64_t* offsets, int64_t curves,
                      int64_t max_n_in, int64_t n_out, int center_normalize, double* out,
                      int32_t* status, cudaStream_t s) {
  const int nmax = (int)std::max<int64_t>(max_n_in, 4);
  if (nmax <= cva::v2_max_raw_nodes() && n_out <= 2048)
    return finish(cva::launch_v2_preprocess((const double2*)points, offsets, curves, (int)n_out,
                                            center_normalize, (double2*)out, status, s),
                  "preprocess launch");
  return resample_general(points, offsets, curves, nmax, n_out, center_normalize, out, status, s);
}

// RAII device buffer for the *_host entry points.
// Scratch of the synchronous *_host entry points: stream-ordered on the calling
// host thread's default stream (cudaStreamPerThread), so concurrent callers
// (the reference's distance_matrix pattern, elastic.cpp:196-234) neither
// serialise on the legacy stream nor hit cudaFree's device-wide sync.
const cudaStream_t kHostStream = cudaStreamPerThread;
struct DevBuf {
  void* p = nullptr;
  cudaError_t alloc(size_t bytes) { return scratch_alloc(&p, bytes, kHostStream); }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, kHostStream);
  }
};

}  // namespace

// CVA_FUSED=v2 selects the round-2 fused C1 kernel (A/B measurements).
static bool use_v2_fused() {
  static const bool v2 = [] {
    const char* e = std::getenv("CVA_FUSED");
    return e != nullptr && std::strcmp(e, "v2") == 0;
  }();
  return v2;
}

extern "C" {

int cva_abi_version(void) { return CVA_ABI_VERSION; }

const char* cva_last_error(void) { return g_last_error.c_str(); }

int cva_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int64_t cva_max_resample_nodes(void) { return INT32_MAX; }  // beyond shared memory: global slabs

int cva_align_batch(const double* c1, const double* c2, int64_t pairs, int64_t n,
                    cva_alignment* out, double* aligned, void* stream) {
  if (int rc = check_fft_size(n)) return rc;
  if (pairs < 0) return fail(CVA_INVALID_ARGUMENT, "align: negative pair count");
  if (pairs == 0) return CVA_OK;
  if (!c1 || !c2 || !out) return fail(CVA_INVALID_ARGUMENT, "align: null pointer");
  if (!a16(c1) || !a16(c2) || !a16(aligned)) return misaligned("align");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const double2* tw = nullptr;
  if (int rc = get_twiddles(cva::v2_fft_len((int)n), s, &tw)) return rc;
  if (!pair_fft(n)) return large_align(c1, c2, pairs, n, 0, out, aligned, tw, s);
  return finish(cva::launch_v2_align((const double2*)c1, (const double2*)c2, pairs, (int)n, tw,
                                     out, (double2*)aligned, s),
                "align launch");
}

int cva_preprocess_batch(const double* points, const int64_t* offsets, int64_t curves,
                         int64_t max_n_in, int64_t n_out, int resample, double* out,
                         int32_t* status, void* stream) {
  if (curves < 0) return fail(CVA_INVALID_ARGUMENT, "preprocess: negative curve count");
  if (curves == 0) return CVA_OK;
  if (!points || !offsets || !out) return fail(CVA_INVALID_ARGUMENT, "preprocess: null pointer");
  if (!a16(points) || !a16(out)) return misaligned("preprocess");
  if (resample && n_out < 8)
    return fail(CVA_INVALID_ARGUMENT, "resample: need at least 8 output nodes");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (!resample)
    return finish(cva::launch_preprocess_center((const double2*)points, offsets, curves,
                                                (double2*)out, status, s),
                  "preprocess launch");
  if (max_n_in <= 0)
    if (int rc = device_max_n(offsets, curves, s, &max_n_in)) return rc;
  return resample_dispatch(points, offsets, curves, max_n_in, n_out, 1, out, status, s);
}

int cva_resample_batch(const double* points, const int64_t* offsets, int64_t curves,
                       int64_t max_n_in, int64_t n_out, double* out, int32_t* status,
                       void* stream) {
  if (curves < 0) return fail(CVA_INVALID_ARGUMENT, "resample: negative curve count");
  if (curves == 0) return CVA_OK;
  if (!points || !offsets || !out) return fail(CVA_INVALID_ARGUMENT, "resample: null pointer");
  if (!a16(points) || !a16(out)) return misaligned("resample");
  if (n_out < 8) return fail(CVA_INVALID_ARGUMENT, "resample: need at least 8 output nodes");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (max_n_in <= 0)
    if (int rc = device_max_n(offsets, curves, s, &max_n_in)) return rc;
  return resample_dispatch(points, offsets, curves, max_n_in, n_out, 0, out, status, s);
}

int cva_preprocess_align_batch(const double* points, const int64_t* offsets, int64_t pairs,
                               int64_t max_n_in, int64_t n_out, int resample, cva_alignment* out,
                               double* aligned, void* stream) {
  if (pairs < 0) return fail(CVA_INVALID_ARGUMENT, "align: negative pair count");
  if (pairs == 0) return CVA_OK;
  if (!points || !offsets || !out) return fail(CVA_INVALID_ARGUMENT, "align: null pointer");
  if (!a16(points) || !a16(aligned)) return misaligned("preprocess_align");
  if (!resample)
    return fail(CVA_UNSUPPORTED,
                "preprocess_align: resample=0 takes equal-size pairs; use "
                "cva_preprocess_align_uniform");
  if (n_out < 8) return fail(CVA_INVALID_ARGUMENT, "resample: need at least 8 output nodes");
  if (int rc = check_fft_size(n_out)) return rc;
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (max_n_in <= 0)
    if (int rc = device_max_n(offsets, 2 * pairs, s, &max_n_in)) return rc;
  const int nmax = (int)std::max<int64_t>(max_n_in, 4);
  if (!small_fft(n_out)) {
    // beyond the shared-memory transforms: preprocess every curve, split the
    // pairs' rows into two arrays, then the multi-pass alignment (any N)
    const size_t row = sizeof(double2) * (size_t)n_out;
    void* ws = nullptr;
    if (scratch_alloc(&ws, 4 * row * (size_t)pairs, s) != cudaSuccess)
      return fail(CVA_BAD_ALLOC, "scratch allocation failed");
    char* prep = (char*)ws;
    char* ab = prep + 2 * row * (size_t)pairs;
    int rc = resample_dispatch(points, offsets, 2 * pairs, nmax, n_out, 1, (double*)prep, nullptr, s);
    for (int h = 0; h < 2 && rc == CVA_OK; ++h) {
      const cudaError_t e = cudaMemcpy2DAsync(ab + h * row * (size_t)pairs, row, prep + h * row, 2 * row, row,
                                              (size_t)pairs, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "de-interleave");
    }
    if (rc == CVA_OK)
      rc = cva_align_batch((const double*)ab, (const double*)(ab + row * (size_t)pairs), pairs, n_out, out,
                           aligned, stream);
    cudaFreeAsync(ws, s);
    return rc;
  }
  const double2* tw = nullptr;
  if (int rc = get_twiddles(cva::v2_fft_len((int)n_out), s, &tw)) return rc;
  if (nmax <= cva::v3_max_raw_nodes() && cva::v3_resample_align_supported((int)n_out) && !use_v2_fused()) {
    return finish(cva::launch_v3_resample_align((const double2*)points, offsets, pairs, (int)n_out, tw, out,
                                                (double2*)aligned, s),
                  "resample_align launch");
  }
  if (nmax <= cva::v2_max_raw_nodes()) {
    const size_t ab = sizeof(double2) * (size_t)(pairs * n_out);
    if (cva::v2_resample_align_supported((int)n_out)) {
      // fused kernel (aligned may be null: results only)
      return finish(cva::launch_v2_resample_align((const double2*)points, offsets, pairs, (int)n_out, tw, out,
                                                  (double2*)aligned, s),
                    "resample_align launch");
    }
    // other N: preprocess into scratch, then align
    void* ws = nullptr;
    if (scratch_alloc(&ws, 2 * ab, s) != cudaSuccess)
      return fail(CVA_BAD_ALLOC, "scratch allocation failed");
    cudaError_t e = cva::launch_v2_preprocess((const double2*)points, offsets, 2 * pairs,
                                              (int)n_out, 1, (double2*)ws, nullptr, s);
    // pair p = prepared rows 2p, 2p+1: strided views via a second launch on
    // de-interleaved halves is avoided by aligning row pairs in place
    if (e == cudaSuccess)
      e = cva::launch_v2_align_interleaved((const double2*)ws, pairs, (int)n_out, tw, out,
                                           (double2*)aligned, s);
    cudaFreeAsync(ws, s);
    return finish(e, "preprocess+align launch");
  }
  // raw curves beyond the v2 resampler: general resampler into scratch, then align
  void* ws = nullptr;
  if (scratch_alloc(&ws, 2 * sizeof(double2) * (size_t)(pairs * n_out), s) != cudaSuccess)
    return fail(CVA_BAD_ALLOC, "scratch allocation failed");
  if (int rc = resample_general(points, offsets, 2 * pairs, nmax, n_out, 1, (double*)ws, nullptr, s)) {
    cudaFreeAsync(ws, s);
    return rc;
  }
  cudaError_t e = cva::launch_v2_align_interleaved((const double2*)ws, pairs, (int)n_out, tw, out,
                                                   (double2*)aligned, s);
  cudaFreeAsync(ws, s);
  return finish(e, "preprocess+align launch");
}

int cva_preprocess_align_uniform(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                 cva_alignment* out, double* aligned, void* stream) {
  if (n < 4) return fail(CVA_INVALID_ARGUMENT, "align: need at least 4 nodes");
  if (int rc = check_fft_size(n)) return rc;
  if (pairs < 0) return fail(CVA_INVALID_ARGUMENT, "align: negative pair count");
  if (pairs == 0) return CVA_OK;
  if (!c1 || !c2 || !out) return fail(CVA_INVALID_ARGUMENT, "align: null pointer");
  if (!a16(c1) || !a16(c2) || !a16(aligned)) return misaligned("preprocess_align_uniform");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const double2* tw = nullptr;
  if (int rc = get_twiddles(cva::v2_fft_len((int)n), s, &tw)) return rc;
  if (!pair_fft(n)) return large_align(c1, c2, pairs, n, 1, out, aligned, tw, s);
  // shared-memory path: per-curve stats, then the pair kernel normalising on load
  void* ws = nullptr;
  const size_t nb = sizeof(double4) * (size_t)(2 * pairs), bb = sizeof(int32_t) * (size_t)(2 * pairs);
  const size_t sb = cva::curve_stats_workspace(pairs);
  if (scratch_alloc(&ws, nb + bb + sb + 512, s) != cudaSuccess) return fail(CVA_BAD_ALLOC, "scratch allocation failed");
  double4* norm = (double4*)ws;
  int32_t* bad = (int32_t*)((char*)ws + nb);
  void* part = (char*)ws + ((nb + bb + 255) & ~size_t(255));
  cudaError_t e = cva::launch_curve_stats((const double2*)c1, pairs, (int)n, 1, norm, bad, part, s);
  if (e == cudaSuccess) e = cva::launch_curve_stats((const double2*)c2, pairs, (int)n, 1, norm + pairs, bad + pairs, part, s);
  if (e == cudaSuccess)
    e = cva::launch_v2_align_norm((const double2*)c1, (const double2*)c2, pairs, (int)n, tw, norm, norm + pairs, bad,
                                  bad + pairs, out, (double2*)aligned, s);
  cudaFreeAsync(ws, s);
  return finish(e, "preprocess_align_uniform launch");
}

int cva_srv_align_batch(const double* c1, const double* c2, int64_t pairs, int64_t n,
                        cva_alignment* out, double* aligned_q, void* stream) {
  if (n < 8) return fail(CVA_INVALID_ARGUMENT, "curve: too few nodes");  // srv.cpp:72
  if (int rc = check_fft_size(n)) return rc;
  if (pairs < 0) return fail(CVA_INVALID_ARGUMENT, "srv: negative pair count");
  if (pairs == 0) return CVA_OK;
  if (!c1 || !c2 || !out) return fail(CVA_INVALID_ARGUMENT, "srv: null pointer");
  if (!a16(c1) || !a16(c2) || !a16(aligned_q)) return misaligned("srv");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (!small_fft(n)) {  // SRV curves into scratch, then the multi-pass alignment (any N)
    const size_t rows = sizeof(double2) * (size_t)(pairs * n);
    void* ws = nullptr;
    if (scratch_alloc(&ws, 2 * rows, s) != cudaSuccess) return fail(CVA_BAD_ALLOC, "scratch allocation failed");
    double2* q1 = (double2*)ws;
    double2* q2 = q1 + pairs * n;
    cudaError_t e = cva::launch_v2_srv_center((const double2*)c1, pairs, (int)n, q1, s);
    if (e == cudaSuccess) e = cva::launch_v2_srv_center((const double2*)c2, pairs, (int)n, q2, s);
    int rc = e == cudaSuccess ? CVA_OK : cuda_fail(e, "srv launch");
    if (rc == CVA_OK) rc = cva_align_batch((const double*)q1, (const double*)q2, pairs, n, out, aligned_q, stream);
    cudaFreeAsync(ws, s);
    return rc;
  }
  const double2* tw = nullptr;
  if (int rc = get_twiddles(cva::v2_fft_len((int)n), s, &tw)) return rc;
  return finish(cva::launch_v2_srv_align((const double2*)c1, (const double2*)c2, pairs, (int)n, tw, out,
                                         (double2*)aligned_q, s),
                "srv_align launch");
}

int cva_allpairs(const double* curves, int64_t count, int64_t n, int64_t row_begin, int64_t row_end,
                 double* energy, int32_t* shift, double* theta, void* stream) {
  if (int rc = check_fft_size(n)) return rc;
  if (count < 0 || row_begin < 0 || row_end > count || row_begin > row_end)
    return fail(CVA_INVALID_ARGUMENT, "allpairs: bad row range");
  if (row_end == row_begin || count == 0) return CVA_OK;
  if (!curves || !energy || !shift || !theta) return fail(CVA_INVALID_ARGUMENT, "allpairs: null pointer");
  if (!a16(curves)) return misaligned("allpairs");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int M = cva::v2_fft_len((int)n);
  const double2* tw = nullptr;
  if (int rc = get_twiddles(M, s, &tw)) return rc;
  if (!pair_fft(n)) {
    // beyond the shared-memory kernels: each row i is a batch of `count` pairs
    // (curve i, curve j) through the large-N pair path (multi-pass transforms)
    void* ws = nullptr;
    const size_t rep = sizeof(double2) * (size_t)(count * n);
    if (scratch_alloc(&ws, rep + sizeof(cva_alignment) * (size_t)count, s) != cudaSuccess)
      return fail(CVA_BAD_ALLOC, "scratch allocation failed");
    double2* row = (double2*)ws;
    cva_alignment* rec = (cva_alignment*)((char*)ws + rep);
    int rc = CVA_OK;
    for (int64_t i = row_begin; i < row_end && rc == CVA_OK; ++i) {
      const int64_t o = (i - row_begin) * count;
      cudaError_t e = cva::launch_broadcast_curve((const double2*)curves + i * n, n, count, row, s);
      if (e != cudaSuccess) {
        rc = cuda_fail(e, "allpairs broadcast");
        break;
      }
      rc = large_align((const double*)row, curves, count, n, 0, rec, nullptr, tw, s);
      if (rc == CVA_OK) {
        e = cva::launch_unpack_row(rec, count, energy + o, shift + o, theta + o, s);
        if (e != cudaSuccess) rc = cuda_fail(e, "allpairs unpack");
      }
    }
    cudaFreeAsync(ws, s);
    return rc;
  }
  if (cva::allpairs_fast_supported((int)n)) {
    // spectra once per curve (kept L2-resident), then one warp per cell
    void* ws = nullptr;
    const size_t zbytes = sizeof(double2) * (size_t)(count * M);
    const size_t sbytes = (sizeof(double) * (size_t)count + 255) & ~size_t(255);
    const size_t dbytes = cva::allpairs_scratch_cells(row_end - row_begin, count);
    if (scratch_alloc(&ws, zbytes + sbytes + dbytes, s) != cudaSuccess)
      return fail(CVA_BAD_ALLOC, "scratch allocation failed");
    double2* za = (double2*)ws;
    double* ss = (double*)((char*)ws + zbytes);
    double2* dm = (double2*)((char*)ws + zbytes + sbytes);
    cudaError_t e = cva::launch_spectra((const double2*)curves, count, (int)n, tw, za, za, ss, s);
    if (e == cudaSuccess)
      e = cva::launch_allpairs(za, za, ss, count, row_begin, row_end, tw, energy, shift, theta, dm, s);
    cudaFreeAsync(ws, s);
    return finish(e, "allpairs launch");
  }
  // general N: one CTA per cell through the pair kernel, row by row
  void* ws = nullptr;
  if (scratch_alloc(&ws, sizeof(cva_alignment) * (size_t)count, s) != cudaSuccess)
    return fail(CVA_BAD_ALLOC, "scratch allocation failed");
  cudaError_t e = cudaSuccess;
  for (int64_t i = row_begin; i < row_end && e == cudaSuccess; ++i) {
    const int64_t o = (i - row_begin) * count;
    e = cva::launch_v2_align_row((const double2*)curves + i * n, (const double2*)curves, count, (int)n, tw,
                                 (cva_alignment*)ws, s);
    if (e == cudaSuccess) e = cva::launch_unpack_row((const cva_alignment*)ws, count, energy + o, shift + o, theta + o, s);
  }
  cudaFreeAsync(ws, s);
  return finish(e, "allpairs launch");
}

// ------------------------------------------------------------- host entries

// Per-thread, per-device host-path context: grow-only device buffers and
// streams reused across calls (no per-call cudaMalloc of hundreds of MB).
struct HostCtx {
  int dev = -1;
  static constexpr int kStreams = 3;  // H2D, kernels, D2H
#ifndef CVA_HOST_MAX_CHUNKS
#define CVA_HOST_MAX_CHUNKS 16
#endif
#ifndef CVA_HOST_MIN_CHUNK
#define CVA_HOST_MIN_CHUNK 256
#endif
  static constexpr int kMaxChunks = CVA_HOST_MAX_CHUNKS;
  cudaStream_t st[kStreams] = {};
  cudaEvent_t ready = nullptr;
  cudaEvent_t in_done[kMaxChunks] = {}, k_done[kMaxChunks] = {};
  void* buf[4] = {};
  size_t cap[4] = {};
  ~HostCtx() {
    for (void* p : buf)
      if (p) cudaFree(p);
    for (cudaStream_t x : st)
      if (x) cudaStreamDestroy(x);
    if (ready) cudaEventDestroy(ready);
    for (int c = 0; c < kMaxChunks; ++c) {
      if (in_done[c]) cudaEventDestroy(in_done[c]);
      if (k_done[c]) cudaEventDestroy(k_done[c]);
    }
  }
  int init() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return fail(CVA_CUDA_ERROR, "cudaGetDevice failed");
    if (d == dev) return CVA_OK;
    this->~HostCtx();
    new (this) HostCtx();
    dev = d;
    for (auto& x : st)
      if (cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess)
        return fail(CVA_CUDA_ERROR, "stream creation failed");
    if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess)
      return fail(CVA_CUDA_ERROR, "event creation failed");
    for (int c = 0; c < kMaxChunks; ++c)
      if (cudaEventCreateWithFlags(&in_done[c], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&k_done[c], cudaEventDisableTiming) != cudaSuccess)
        return fail(CVA_CUDA_ERROR, "event creation failed");
    return CVA_OK;
  }
  void* get(int i, size_t bytes) {
    if (cap[i] < bytes) {
      if (buf[i]) cudaFree(buf[i]);
      buf[i] = nullptr;
      cap[i] = 0;
      if (cudaMalloc(&buf[i], bytes) != cudaSuccess) return nullptr;
      cap[i] = bytes;
    }
    return buf[i];
  }
};
thread_local HostCtx t_host;

namespace {
// resample: 0 = center+normalize, 1 = resample+center+normalize, 2 = resample only
int preprocess_host_impl(const double* points, const int64_t* offsets, int64_t curves,
                         int64_t n_out, int resample, double* out, int32_t* status) {
  if (curves <= 0) return curves == 0 ? CVA_OK : fail(CVA_INVALID_ARGUMENT, "negative curve count");
  if (int rc = require_device()) return rc;
  const int64_t total = offsets[curves] - offsets[0];
  if (offsets[0] != 0) return fail(CVA_INVALID_ARGUMENT, "offsets[0] must be 0");
  const size_t ib = sizeof(double) * 2 * (size_t)total;
  const size_t ob = resample ? sizeof(double) * 2 * (size_t)(curves * n_out) : ib;
  // the grow-only per-thread buffers of the other host paths (no per-call cudaMalloc)
  if (int rc = t_host.init()) return rc;
  HostCtx& h = t_host;
  void* dp = h.get(0, ib);
  void* doff = h.get(1, sizeof(int64_t) * (curves + 1));
  void* dout = h.get(2, ob);
  void* dst = h.get(3, sizeof(int32_t) * curves);
  if (!dp || !doff || !dout || !dst) return fail(CVA_BAD_ALLOC, "device allocation failed");
  cudaStream_t s = h.st[1];
  auto drain = [&](int rc) {
    cudaStreamSynchronize(s);
    return rc;
  };
  cudaError_t e = cudaMemcpyAsync(dp, points, ib, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(doff, offsets, sizeof(int64_t) * (curves + 1), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return drain(cuda_fail(e, "H2D"));
  const int rc = resample == 2
                     ? cva_resample_batch((const double*)dp, (const int64_t*)doff, curves,
                                          host_max_n(offsets, curves), n_out, (double*)dout,
                                          (int32_t*)dst, s)
                     : cva_preprocess_batch((const double*)dp, (const int64_t*)doff, curves,
                                            host_max_n(offsets, curves), n_out, resample,
                                            (double*)dout, (int32_t*)dst, s);
  if (rc) return drain(rc);
  e = cudaMemcpyAsync(out, dout, ob, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && status)
    e = cudaMemcpyAsync(status, dst, sizeof(int32_t) * curves, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return finish(e, "preprocess_batch_host");
}
}  // namespace

int cva_preprocess_batch_host(const double* points, const int64_t* offsets, int64_t curves,
                              int64_t n_out, int resample, double* out, int32_t* status) {
  return preprocess_host_impl(points, offsets, curves, n_out, resample ? 1 : 0, out, status);
}

int cva_resample_batch_host(const double* points, const int64_t* offsets, int64_t curves,
                            int64_t n_out, double* out, int32_t* status) {
  return preprocess_host_impl(points, offsets, curves, n_out, 2, out, status);
}


// Host-buffer fused path, pipelined in chunks of pairs over three streams:
// all H2D copies back to back on one stream (the step is bound by the host ->
// device link, so it never waits behind a D2H), each chunk's kernel on a
// second stream once its input has landed, each chunk's D2H on a third once
// its kernel is done. Up to 16 chunks of >= 256 pairs keep the un-overlapped
// tail (last chunk's kernel + D2H) small. Pinned host buffers give the
// asynchronous copies; pageable ones still work, with less overlap.
int cva_preprocess_align_batch_host(const double* points, const int64_t* offsets, int64_t pairs,
                                    int64_t n_out, int resample, cva_alignment* out,
                                    double* aligned) {
  if (pairs <= 0) return pairs == 0 ? CVA_OK : fail(CVA_INVALID_ARGUMENT, "negative pair count");
  if (int rc = require_device()) return rc;
  if (offsets[0] != 0) return fail(CVA_INVALID_ARGUMENT, "offsets[0] must be 0");
  if (int rc = t_host.init()) return rc;
  HostCtx& h = t_host;
  const int64_t total = offsets[2 * pairs];
  const size_t ib = sizeof(double2) * (size_t)total;
  const size_t ab = sizeof(double2) * (size_t)(pairs * n_out);
  double2* dp = (double2*)h.get(0, ib);
  int64_t* doff = (int64_t*)h.get(1, sizeof(int64_t) * (size_t)(2 * pairs + 1));
  cva_alignment* dout = (cva_alignment*)h.get(2, sizeof(cva_alignment) * (size_t)pairs);
  double2* dal = aligned ? (double2*)h.get(3, ab) : nullptr;
  if (!dp || !doff || !dout || (aligned && !dal)) return fail(CVA_BAD_ALLOC, "device allocation failed");
  const int64_t max_n = host_max_n(offsets, 2 * pairs);
  // Every exit after the first asynchronous call drains the three streams, so
  // no copy still reads or writes the caller's host buffers after return.
  auto drain = [&](int rc) {
    for (cudaStream_t x : h.st) cudaStreamSynchronize(x);
    return rc;
  };
  cudaError_t e = cudaMemcpyAsync(doff, offsets, sizeof(int64_t) * (size_t)(2 * pairs + 1),
                                  cudaMemcpyHostToDevice, h.st[0]);  // ahead of chunk 0's input
  if (e != cudaSuccess) return drain(cuda_fail(e, "H2D offsets"));
  const int64_t nchunks = std::min<int64_t>(HostCtx::kMaxChunks, std::max<int64_t>(1, pairs / CVA_HOST_MIN_CHUNK));
  const int64_t per = (pairs + nchunks - 1) / nchunks;
  cudaStream_t sin = h.st[0], sk = h.st[1], sout = h.st[2];
  for (int64_t c = 0; c < nchunks; ++c) {  // all input copies first, in order
    const int64_t p0 = c * per, p1 = std::min(pairs, p0 + per);
    if (p0 >= p1) break;
    const int64_t a = offsets[2 * p0], b = offsets[2 * p1];
    e = cudaMemcpyAsync(dp + a, points + 2 * a, sizeof(double2) * (size_t)(b - a), cudaMemcpyHostToDevice, sin);
    if (e == cudaSuccess) e = cudaEventRecord(h.in_done[c], sin);
    if (e != cudaSuccess) return drain(cuda_fail(e, "H2D"));
  }
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t p0 = c * per, p1 = std::min(pairs, p0 + per);
    if (p0 >= p1) break;
    e = cudaStreamWaitEvent(sk, h.in_done[c], 0);
    if (e != cudaSuccess) return drain(cuda_fail(e, "stream wait"));
    // the kernels index points with the absolute offsets; pass this chunk's slice
    if (int rc = cva_preprocess_align_batch((const double*)dp, doff + 2 * p0, p1 - p0, max_n, n_out, resample,
                                            dout + p0, aligned ? (double*)(dal + p0 * n_out) : nullptr, sk))
      return drain(rc);
    e = cudaEventRecord(h.k_done[c], sk);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, h.k_done[c], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out + p0, dout + p0, sizeof(cva_alignment) * (size_t)(p1 - p0), cudaMemcpyDeviceToHost,
                          sout);
    if (e == cudaSuccess && aligned)
      e = cudaMemcpyAsync(aligned + 2 * p0 * n_out, dal + p0 * n_out, sizeof(double2) * (size_t)((p1 - p0) * n_out),
                          cudaMemcpyDeviceToHost, sout);
    if (e != cudaSuccess) return drain(cuda_fail(e, "D2H"));
  }
  cudaError_t first = cudaSuccess;
  for (cudaStream_t x : h.st) {
    e = cudaStreamSynchronize(x);
    if (first == cudaSuccess) first = e;
  }
  return first == cudaSuccess ? CVA_OK : cuda_fail(first, "preprocess_align_batch_host");
}

// Host-buffer all-pairs rows: with the warp-per-cell kernel, spectra once, then
// row chunks whose results go back on a second stream while the next chunk
// computes (grow-only buffers); other sizes in one call.
int cva_allpairs_host(const double* curves, int64_t count, int64_t n, int64_t row_begin,
                      int64_t row_end, double* energy, int32_t* shift, double* theta) {
  if (int rc = check_fft_size(n)) return rc;
  if (count < 0 || row_begin < 0 || row_end > count || row_begin > row_end)
    return fail(CVA_INVALID_ARGUMENT, "allpairs: bad row range");
  if (int rc = require_device()) return rc;
  const int64_t cells = (row_end - row_begin) * count;
  if (cells > 0 && pair_fft(n) && cva::allpairs_fast_supported((int)n)) {
    if (int rc = t_host.init()) return rc;
    HostCtx& h = t_host;
    const int M = cva::v2_fft_len((int)n);
    const int64_t rows = row_end - row_begin;
    const int64_t nchunks = std::min<int64_t>(HostCtx::kMaxChunks, std::max<int64_t>(1, rows / 64));
    const int64_t per = (rows + nchunks - 1) / nchunks;
    double2* dc = (double2*)h.get(0, sizeof(double2) * (size_t)(count * n));
    double* de = (double*)h.get(1, sizeof(double) * (size_t)cells);
    int32_t* dk = (int32_t*)h.get(2, sizeof(int32_t) * (size_t)cells);
    double* dt = (double*)h.get(3, sizeof(double) * (size_t)cells);
    if (!dc || !de || !dk || !dt) return fail(CVA_BAD_ALLOC, "device allocation failed");
    cudaStream_t sk = h.st[1], sout = h.st[2];
    auto drain = [&](int rc) {
      for (cudaStream_t x : h.st) cudaStreamSynchronize(x);
      return rc;
    };
    const double2* tw = nullptr;
    if (int rc = get_twiddles(M, sk, &tw)) return drain(rc);
    const size_t zbytes = sizeof(double2) * (size_t)(count * M);
    const size_t sbytes = (sizeof(double) * (size_t)count + 255) & ~size_t(255);
    void* ws = nullptr;
    if (scratch_alloc(&ws, zbytes + sbytes + cva::allpairs_scratch_cells(per, count), sk) != cudaSuccess)
      return drain(fail(CVA_BAD_ALLOC, "scratch allocation failed"));
    double2* za = (double2*)ws;
    double* ss = (double*)((char*)ws + zbytes);
    double2* dm = (double2*)((char*)ws + zbytes + sbytes);
    cudaError_t e = cudaMemcpyAsync(dc, curves, sizeof(double2) * (size_t)(count * n), cudaMemcpyHostToDevice, sk);
    if (e == cudaSuccess) e = cva::launch_spectra(dc, count, (int)n, tw, za, za, ss, sk);
    for (int64_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
      const int64_t r0 = row_begin + c * per, r1 = std::min(row_end, r0 + per);
      if (r0 >= r1) break;
      const int64_t o = (r0 - row_begin) * count, nc = (r1 - r0) * count;
      e = cva::launch_allpairs(za, za, ss, count, r0, r1, tw, de + o, dk + o, dt + o, dm, sk);
      if (e == cudaSuccess) e = cudaEventRecord(h.k_done[c], sk);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, h.k_done[c], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(energy + o, de + o, sizeof(double) * (size_t)nc, cudaMemcpyDeviceToHost, sout);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(shift + o, dk + o, sizeof(int32_t) * (size_t)nc, cudaMemcpyDeviceToHost, sout);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(theta + o, dt + o, sizeof(double) * (size_t)nc, cudaMemcpyDeviceToHost, sout);
    }
    cudaFreeAsync(ws, sk);
    cudaError_t first = e;
    for (cudaStream_t x : h.st) {
      const cudaError_t f = cudaStreamSynchronize(x);
      if (first == cudaSuccess) first = f;
    }
    return first == cudaSuccess ? CVA_OK : cuda_fail(first, "allpairs_host");
  }
  DevBuf dc, de, dk, dt;
  if (dc.alloc(sizeof(double2) * (size_t)(count * n)) || de.alloc(sizeof(double) * cells) ||
      dk.alloc(sizeof(int32_t) * cells) || dt.alloc(sizeof(double) * cells))
    return fail(CVA_BAD_ALLOC, "device allocation failed");
  cudaStream_t s = kHostStream;
  cudaError_t e = cudaMemcpyAsync(dc.p, curves, sizeof(double2) * (size_t)(count * n), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  if (int rc = cva_allpairs((const double*)dc.p, count, n, row_begin, row_end, (double*)de.p,
                            (int32_t*)dk.p, (double*)dt.p, s))
    return rc;
  e = cudaMemcpyAsync(energy, de.p, sizeof(double) * cells, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(shift, dk.p, sizeof(int32_t) * cells, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(theta, dt.p, sizeof(double) * cells, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return finish(e, "allpairs_host");
}

// Host-buffer paths over pairs of uniform curves (c1, c2: pairs x n each),
// pipelined like cva_preprocess_align_batch_host: every chunk's H2D copies on
// one stream, its kernels on a second once they have landed, its results back
// on a third, with the grow-only per-thread device buffers (no per-call
// cudaMalloc). Chunks of >= ~4 MB of input per curve array; at large N a
// chunk holds whole internal chunks of the L2-chunked path (large_chunk_pairs).
}  // extern "C" (the helper below is a template)
namespace {
template <class Launch>
int uniform_pairs_host(const double* c1, const double* c2, int64_t pairs, int64_t n, cva_alignment* out,
                       double* aligned, Launch launch, const char* what) {
  if (pairs <= 0) return pairs == 0 ? CVA_OK : fail(CVA_INVALID_ARGUMENT, "negative pair count");
  if (int rc = require_device()) return rc;
  if (int rc = t_host.init()) return rc;
  HostCtx& h = t_host;
  const size_t cb = sizeof(double2) * (size_t)(pairs * n);
  double2* d1 = (double2*)h.get(0, cb);
  double2* d2 = (double2*)h.get(1, cb);
  cva_alignment* dout = (cva_alignment*)h.get(2, sizeof(cva_alignment) * (size_t)pairs);
  double2* dal = aligned ? (double2*)h.get(3, cb) : nullptr;
  if (!d1 || !d2 || !dout || (aligned && !dal)) return fail(CVA_BAD_ALLOC, "device allocation failed");
  auto drain = [&](int rc) {
    for (cudaStream_t x : h.st) cudaStreamSynchronize(x);
    return rc;
  };
  const int64_t min_chunk = std::max<int64_t>(1, (int64_t(4) << 20) / (16 * n));
  const int64_t nchunks = std::min<int64_t>(HostCtx::kMaxChunks, std::max<int64_t>(1, pairs / min_chunk));
  int64_t per = (pairs + nchunks - 1) / nchunks;
  if (!pair_fft(n)) {  // whole internal chunks of the large-N path
    const int64_t g = std::max<int64_t>(1, cva::large_chunk_pairs((int)n));
    per = std::min<int64_t>(pairs, (per + g - 1) / g * g);
  }
  cudaStream_t sin = h.st[0], sk = h.st[1], sout = h.st[2];
  cudaError_t e = cudaSuccess;
  int64_t used = 0;
  for (int64_t p0 = 0, c = 0; p0 < pairs; p0 += per, ++c) {  // all input copies first, in order
    const size_t bytes = sizeof(double2) * (size_t)(std::min(per, pairs - p0) * n);
    e = cudaMemcpyAsync(d1 + p0 * n, c1 + 2 * p0 * n, bytes, cudaMemcpyHostToDevice, sin);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d2 + p0 * n, c2 + 2 * p0 * n, bytes, cudaMemcpyHostToDevice, sin);
    if (e == cudaSuccess) e = cudaEventRecord(h.in_done[c], sin);
    if (e != cudaSuccess) return drain(cuda_fail(e, "H2D"));
    used = c + 1;
  }
  for (int64_t c = 0; c < used; ++c) {
    const int64_t p0 = c * per, np = std::min(per, pairs - p0);
    e = cudaStreamWaitEvent(sk, h.in_done[c], 0);
    if (e != cudaSuccess) return drain(cuda_fail(e, "stream wait"));
    if (int rc = launch((const double*)(d1 + p0 * n), (const double*)(d2 + p0 * n), np, n, dout + p0,
                        aligned ? (double*)(dal + p0 * n) : nullptr, sk))
      return drain(rc);
    e = cudaEventRecord(h.k_done[c], sk);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, h.k_done[c], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out + p0, dout + p0, sizeof(cva_alignment) * (size_t)np, cudaMemcpyDeviceToHost, sout);
    if (e == cudaSuccess && aligned)
      e = cudaMemcpyAsync(aligned + 2 * p0 * n, dal + p0 * n, sizeof(double2) * (size_t)(np * n),
                          cudaMemcpyDeviceToHost, sout);
    if (e != cudaSuccess) return drain(cuda_fail(e, "D2H"));
  }
  cudaError_t first = cudaSuccess;
  for (cudaStream_t x : h.st) {
    e = cudaStreamSynchronize(x);
    if (first == cudaSuccess) first = e;
  }
  return first == cudaSuccess ? CVA_OK : cuda_fail(first, what);
}
}  // namespace
extern "C" {

int cva_align_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                         cva_alignment* out, double* aligned) {
  if (int rc = check_fft_size(n)) return rc;
  return uniform_pairs_host(c1, c2, pairs, n, out, aligned, cva_align_batch, "align_batch_host");
}

int cva_preprocess_align_uniform_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                      cva_alignment* out, double* aligned) {
  if (n < 4) return fail(CVA_INVALID_ARGUMENT, "align: need at least 4 nodes");
  if (int rc = check_fft_size(n)) return rc;
  return uniform_pairs_host(c1, c2, pairs, n, out, aligned, cva_preprocess_align_uniform,
                            "preprocess_align_uniform_host");
}

int cva_srv_align_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                             cva_alignment* out, double* aligned_q) {
  if (n < 8) return fail(CVA_INVALID_ARGUMENT, "curve: too few nodes");
  if (int rc = check_fft_size(n)) return rc;
  return uniform_pairs_host(c1, c2, pairs, n, out, aligned_q, cva_srv_align_batch, "srv_align_batch_host");
}

// ------------------------------------------------------------- elastic (SRV) matching

namespace {
int check_elastic(int64_t pairs, int64_t n, int max_slope, const char* what) {
  if (pairs < 0) return fail(CVA_INVALID_ARGUMENT, std::string(what) + ": negative pair count");
  if (n < 8) return fail(CVA_INVALID_ARGUMENT, std::string(what) + ": need at least 8 nodes");  // elastic.cpp:57, srv.cpp:183
  if (max_slope < 1) return fail(CVA_INVALID_ARGUMENT, "dp: max_slope must be >= 1");  // srv.cpp:131
  if (n > 1 << 20 || !cva::elastic_supported((int)n, max_slope))
    return fail(CVA_UNSUPPORTED, std::string(what) +
                                     ": supported sizes are 8 <= n <= 2^20 and max_slope <= 20 (beyond 20 the "
                                     "reference's 8-bit parent indices wrap)");
  return CVA_OK;
}

struct Slab {
  void* p = nullptr;
  cudaStream_t s = kHostStream;
  ~Slab() {
    if (p) cudaFreeAsync(p, s);
  }
};
}  // namespace

int cva_dp_reparam_batch(const double* q1, const double* q2, int64_t pairs, int64_t n, int max_slope,
                         double* gamma, double* energy, int32_t* status, void* stream) {
  if (int rc = check_elastic(pairs, n, max_slope, "dp")) return rc;
  if (pairs == 0) return CVA_OK;
  if (!q1 || !q2 || !gamma || !energy) return fail(CVA_INVALID_ARGUMENT, "dp: null pointer");
  if (!a16(q1) || !a16(q2)) return misaligned("dp");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = cva::elastic_grid(pairs, (int)n, max_slope);
  Slab slab;
  slab.s = s;
  const size_t per = cva::elastic_parent_slab(pairs, (int)n, max_slope);
  if (per && scratch_alloc(&slab.p, per * (size_t)grid, s) != cudaSuccess)
    return fail(CVA_BAD_ALLOC, "dp: parent scratch allocation failed");
  return finish(cva::launch_dp_reparam((const double2*)q1, (const double2*)q2, pairs, (int)n, max_slope,
                                       (uint8_t*)slab.p, grid, gamma, energy, status, s),
                "dp launch");
}

static int elastic_launch(const double* A, const double* B, int64_t pairs, int64_t k, int64_t n, int max_iters,
                          double energy_tol, int max_slope, int use_fft, const cva::ElasticOut& o, cudaStream_t s) {
  const double2* tw = nullptr;  // slab mode aligns by the direct correlation (no transform)
  if (!cva::elastic_slab_mode((int)n, max_slope))
    if (int rc = get_twiddles(cva::v2_fft_len((int)n), s, &tw)) return rc;
  const int grid = cva::elastic_grid(pairs, (int)n, max_slope);
  Slab slab;
  slab.s = s;
  const size_t per = cva::elastic_parent_slab(pairs, (int)n, max_slope);
  if (per && scratch_alloc(&slab.p, per * (size_t)grid, s) != cudaSuccess)
    return fail(CVA_BAD_ALLOC, "elastic: parent scratch allocation failed");
  const cva::ElasticParams prm{max_iters, energy_tol, max_slope, use_fft ? 1 : 0};
  return finish(cva::launch_elastic_approach2((const double2*)A, (const double2*)B, pairs, k, (int)n, prm,
                                              (uint8_t*)slab.p, grid, tw, o, s),
                "elastic launch");
}

int cva_elastic_approach2_batch(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                int max_iters, double energy_tol, int max_slope, double* distance,
                                double* energy, double* t0, double* theta, double* gamma,
                                int32_t* iterations, int32_t* converged, int32_t* status,
                                double* energy_trace, void* stream) {
  return cva_elastic_approach2_batch_ex(c1, c2, pairs, n, max_iters, energy_tol, max_slope, 1, distance, energy,
                                        t0, theta, gamma, iterations, converged, status, energy_trace, stream);
}

int cva_elastic_approach2_batch_ex(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                   int max_iters, double energy_tol, int max_slope, int use_fft,
                                   double* distance, double* energy, double* t0, double* theta, double* gamma,
                                   int32_t* iterations, int32_t* converged, int32_t* status,
                                   double* energy_trace, void* stream) {
  if (int rc = check_elastic(pairs, n, max_slope, "elastic")) return rc;
  if (pairs == 0) return CVA_OK;
  if (!c1 || !c2 || !distance || !energy || !t0 || !theta || !iterations || !converged || !status)
    return fail(CVA_INVALID_ARGUMENT, "elastic: null pointer");
  if (!a16(c1) || !a16(c2)) return misaligned("elastic");
  if (int rc = require_device()) return rc;
  if (max_iters < 0) return fail(CVA_INVALID_ARGUMENT, "elastic: negative max_iters");
  const cva::ElasticOut o{distance, energy, t0, theta, gamma, iterations, converged, status, energy_trace};
  return elastic_launch(c1, c2, pairs, 0, n, max_iters, energy_tol, max_slope, use_fft, o, (cudaStream_t)stream);
}

// Approach 1 keeps per-item results until the per-pair pick. With gamma wanted
// (independent pairs only: distance matrices pass gamma = null), the items'
// gammas would need pairs * n * (n + 1) doubles, so the pairs run in chunks
// whose scratch stays below kA1ScratchCap.
static int approach1_launch(const double* A, const double* B, int64_t pairs, int64_t k, int64_t n, int max_slope,
                            const cva::ElasticOut& o, cudaStream_t s) {
  constexpr size_t kA1ScratchCap = size_t(1) << 30;
  const bool gamma = o.gamma != nullptr;
  int64_t chunk = pairs;
  if (gamma && k == 0) {
    const size_t per_pair = cva::elastic_a1_scratch(1, (int)n, true);
    chunk = std::max<int64_t>(1, std::min<int64_t>(pairs, (int64_t)(kA1ScratchCap / per_pair)));
  }
  const int64_t items = chunk * n;
  const int grid = cva::elastic_items_grid(items, (int)n, max_slope);
  Slab slab, scratch;
  slab.s = scratch.s = s;
  const size_t per = cva::elastic_parent_slab(items, (int)n, max_slope);
  if (per && scratch_alloc(&slab.p, per * (size_t)grid, s) != cudaSuccess)
    return fail(CVA_BAD_ALLOC, "elastic: parent scratch allocation failed");
  if (scratch_alloc(&scratch.p, cva::elastic_a1_scratch(chunk, (int)n, gamma), s) != cudaSuccess)
    return fail(CVA_BAD_ALLOC, "elastic: scratch allocation failed");
  for (int64_t p0 = 0; p0 < pairs; p0 += chunk) {
    const int64_t cp = std::min(chunk, pairs - p0);
    cva::ElasticOut oc = o;
    if (p0) {  // independent pairs: offset inputs and outputs (k == 0 here)
      oc.distance += p0;
      oc.energy += p0;
      oc.t0 += p0;
      oc.theta += p0;
      oc.gamma += p0 * (n + 1);
      oc.iterations += p0;
      oc.converged += p0;
      oc.status += p0;
    }
    const cudaError_t e = cva::launch_elastic_approach1((const double2*)A + p0 * n, (const double2*)B + p0 * n, cp,
                                                        k, (int)n, max_slope, (uint8_t*)slab.p,
                                                        cva::elastic_items_grid(cp * n, (int)n, max_slope),
                                                        scratch.p, oc, s);
    if (e != cudaSuccess) return finish(e, "elastic approach1 launch");
  }
  return finish(cudaSuccess, "elastic approach1 launch");
}

static int check_a1(int64_t n, int64_t n_max) {
  if (n > n_max)  // elastic.cpp:66-69
    return fail(CVA_INVALID_ARGUMENT,
                "approach 1 is O(N^3); node count exceeds the configured limit, use approach 2");
  return CVA_OK;
}

int cva_elastic_approach1_batch(const double* c1, const double* c2, int64_t pairs, int64_t n, int max_slope,
                                int64_t n_max_approach1, double* distance, double* energy, double* t0,
                                double* theta, double* gamma, int32_t* iterations, int32_t* converged,
                                int32_t* status, void* stream) {
  if (int rc = check_elastic(pairs, n, max_slope, "elastic")) return rc;
  if (int rc = check_a1(n, n_max_approach1)) return rc;
  if (pairs == 0) return CVA_OK;
  if (!c1 || !c2 || !distance || !energy || !t0 || !theta || !iterations || !converged || !status)
    return fail(CVA_INVALID_ARGUMENT, "elastic: null pointer");
  if (!a16(c1) || !a16(c2)) return misaligned("elastic");
  if (int rc = require_device()) return rc;
  const cva::ElasticOut o{distance, energy, t0, theta, gamma, iterations, converged, status, nullptr};
  return approach1_launch(c1, c2, pairs, 0, n, max_slope, o, (cudaStream_t)stream);
}

int cva_elastic_distance_matrix(const double* curves, int64_t count, int64_t n, int method, int max_iters,
                                double energy_tol, int max_slope, int64_t n_max_approach1, double* d,
                                void* stream) {
  return cva_elastic_distance_matrix_ex(curves, count, n, method, max_iters, energy_tol, max_slope, 1,
                                        n_max_approach1, d, stream);
}

int cva_elastic_distance_matrix_ex(const double* curves, int64_t count, int64_t n, int method, int max_iters,
                                   double energy_tol, int max_slope, int use_fft, int64_t n_max_approach1,
                                   double* d, void* stream) {
  if (count < 2) return fail(CVA_INVALID_ARGUMENT, "distance_matrix: need at least 2 curves");  // elastic.cpp:181
  if (method != 1 && method != 2) return fail(CVA_INVALID_ARGUMENT, "distance_matrix: method is 1 or 2");
  if (int rc = check_elastic(count * count, n, max_slope, "distance_matrix")) return rc;
  if (!curves || !d) return fail(CVA_INVALID_ARGUMENT, "distance_matrix: null pointer");
  if (!a16(curves)) return misaligned("distance_matrix");
  if (int rc = require_device()) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t pairs = count * count;
  if (method == 1 && n > n_max_approach1) {
    // every cell throws in the reference and becomes NaN (elastic.cpp:210-217)
    const double qnan = std::nan("");
    std::vector<double> h((size_t)pairs, qnan);
    return finish(cudaMemcpyAsync(d, h.data(), sizeof(double) * pairs, cudaMemcpyHostToDevice, s), "fill");
  }
  void* ws = nullptr;
  const size_t per = 3 * sizeof(double) + 3 * sizeof(int32_t);
  if (scratch_alloc(&ws, per * (size_t)pairs + 256, s) != cudaSuccess)
    return fail(CVA_BAD_ALLOC, "scratch allocation failed");
  double* e = (double*)ws;
  cva::ElasticOut o{d, e, e + pairs, e + 2 * pairs, nullptr, (int32_t*)(e + 3 * pairs),
                    (int32_t*)(e + 3 * pairs) + pairs, (int32_t*)(e + 3 * pairs) + 2 * pairs, nullptr};
  const int rc = method == 1 ? approach1_launch(curves, nullptr, pairs, count, n, max_slope, o, s)
                             : elastic_launch(curves, nullptr, pairs, count, n, max_iters, energy_tol, max_slope, use_fft,
                                              o, s);
  cudaFreeAsync(ws, s);
  return rc;
}

int cva_dp_reparam_batch_host(const double* q1, const double* q2, int64_t pairs, int64_t n,
                              int max_slope, double* gamma, double* energy, int32_t* status) {
  if (int rc = check_elastic(pairs, n, max_slope, "dp")) return rc;
  if (pairs == 0) return CVA_OK;
  if (int rc = require_device()) return rc;
  const size_t cb = sizeof(double2) * (size_t)(pairs * n), gb = sizeof(double) * (size_t)(pairs * (n + 1));
  DevBuf d1, d2, dg, de, ds;
  if (d1.alloc(cb) || d2.alloc(cb) || dg.alloc(gb) || de.alloc(sizeof(double) * pairs) ||
      ds.alloc(sizeof(int32_t) * pairs))
    return fail(CVA_BAD_ALLOC, "device allocation failed");
  cudaStream_t s = kHostStream;
  cudaError_t e = cudaMemcpyAsync(d1.p, q1, cb, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d2.p, q2, cb, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  if (int rc = cva_dp_reparam_batch((const double*)d1.p, (const double*)d2.p, pairs, n, max_slope, (double*)dg.p,
                                    (double*)de.p, (int32_t*)ds.p, s))
    return rc;
  e = cudaMemcpyAsync(gamma, dg.p, gb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(energy, de.p, sizeof(double) * pairs, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && status) e = cudaMemcpyAsync(status, ds.p, sizeof(int32_t) * pairs, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return finish(e, "dp_reparam_batch_host");
}

int cva_elastic_approach2_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                     int max_iters, double energy_tol, int max_slope, double* distance,
                                     double* energy, double* t0, double* theta, double* gamma,
                                     int32_t* iterations, int32_t* converged, int32_t* status,
                                     double* energy_trace) {
  return cva_elastic_approach2_batch_ex_host(c1, c2, pairs, n, max_iters, energy_tol, max_slope, 1, distance,
                                             energy, t0, theta, gamma, iterations, converged, status, energy_trace);
}

int cva_elastic_approach2_batch_ex_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                        int max_iters, double energy_tol, int max_slope, int use_fft,
                                        double* distance, double* energy, double* t0, double* theta,
                                        double* gamma, int32_t* iterations, int32_t* converged, int32_t* status,
                                        double* energy_trace) {
  if (int rc = check_elastic(pairs, n, max_slope, "elastic")) return rc;
  if (max_iters < 0) return fail(CVA_INVALID_ARGUMENT, "elastic: negative max_iters");
  if (pairs == 0) return CVA_OK;
  if (int rc = require_device()) return rc;
  const size_t cb = sizeof(double2) * (size_t)(pairs * n), gb = sizeof(double) * (size_t)(pairs * (n + 1));
  const size_t vb = sizeof(double) * pairs, ib = sizeof(int32_t) * pairs;
  const size_t tb = sizeof(double) * (size_t)(pairs * (max_iters + 1));
  DevBuf d1, d2, dv, dg, di, dt;
  if (d1.alloc(cb) || d2.alloc(cb) || dv.alloc(4 * vb) || (gamma && dg.alloc(gb)) || di.alloc(3 * ib) ||
      (energy_trace && dt.alloc(tb)))
    return fail(CVA_BAD_ALLOC, "device allocation failed");
  cudaStream_t s = kHostStream;
  cudaError_t e = cudaMemcpyAsync(d1.p, c1, cb, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d2.p, c2, cb, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  double* v = (double*)dv.p;
  int32_t* iv = (int32_t*)di.p;
  if (int rc = cva_elastic_approach2_batch_ex((const double*)d1.p, (const double*)d2.p, pairs, n, max_iters,
                                              energy_tol, max_slope, use_fft, v, v + pairs, v + 2 * pairs,
                                              v + 3 * pairs, gamma ? (double*)dg.p : nullptr, iv, iv + pairs,
                                              iv + 2 * pairs, energy_trace ? (double*)dt.p : nullptr, s))
    return rc;
  double* hv[4] = {distance, energy, t0, theta};
  for (int k = 0; k < 4 && e == cudaSuccess; ++k)
    if (hv[k]) e = cudaMemcpyAsync(hv[k], v + k * pairs, vb, cudaMemcpyDeviceToHost, s);
  int32_t* hi[3] = {iterations, converged, status};
  for (int k = 0; k < 3 && e == cudaSuccess; ++k)
    if (hi[k]) e = cudaMemcpyAsync(hi[k], iv + k * pairs, ib, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && gamma) e = cudaMemcpyAsync(gamma, dg.p, gb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && energy_trace) e = cudaMemcpyAsync(energy_trace, dt.p, tb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return finish(e, "elastic_approach2_batch_host");
}

int cva_elastic_distance_matrix_host(const double* curves, int64_t count, int64_t n, int method, int max_iters,
                                     double energy_tol, int max_slope, int64_t n_max_approach1, double* d) {
  return cva_elastic_distance_matrix_ex_host(curves, count, n, method, max_iters, energy_tol, max_slope, 1,
                                             n_max_approach1, d);
}

int cva_elastic_distance_matrix_ex_host(const double* curves, int64_t count, int64_t n, int method,
                                        int max_iters, double energy_tol, int max_slope, int use_fft,
                                        int64_t n_max_approach1, double* d) {
  if (count < 2) return fail(CVA_INVALID_ARGUMENT, "distance_matrix: need at least 2 curves");
  if (int rc = check_elastic(count * count, n, max_slope, "distance_matrix")) return rc;
  if (int rc = require_device()) return rc;
  const size_t cb = sizeof(double2) * (size_t)(count * n), db = sizeof(double) * (size_t)(count * count);
  DevBuf dc, dd;
  if (dc.alloc(cb) || dd.alloc(db)) return fail(CVA_BAD_ALLOC, "device allocation failed");
  cudaStream_t s = kHostStream;
  cudaError_t e = cudaMemcpyAsync(dc.p, curves, cb, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  if (int rc = cva_elastic_distance_matrix_ex((const double*)dc.p, count, n, method, max_iters, energy_tol,
                                              max_slope, use_fft, n_max_approach1, (double*)dd.p, s))
    return rc;
  e = cudaMemcpyAsync(d, dd.p, db, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return finish(e, "elastic_distance_matrix_host");
}

int cva_elastic_approach1_batch_host(const double* c1, const double* c2, int64_t pairs, int64_t n,
                                     int max_slope, int64_t n_max_approach1, double* distance, double* energy,
                                     double* t0, double* theta, double* gamma, int32_t* iterations,
                                     int32_t* converged, int32_t* status) {
  if (int rc = check_elastic(pairs, n, max_slope, "elastic")) return rc;
  if (int rc = check_a1(n, n_max_approach1)) return rc;
  if (pairs == 0) return CVA_OK;
  if (int rc = require_device()) return rc;
  const size_t cb = sizeof(double2) * (size_t)(pairs * n), gb = sizeof(double) * (size_t)(pairs * (n + 1));
  const size_t vb = sizeof(double) * pairs, ib = sizeof(int32_t) * pairs;
  DevBuf d1, d2, dv, dg, di;
  if (d1.alloc(cb) || d2.alloc(cb) || dv.alloc(4 * vb) || (gamma && dg.alloc(gb)) || di.alloc(3 * ib))
    return fail(CVA_BAD_ALLOC, "device allocation failed");
  cudaStream_t s = kHostStream;
  cudaError_t e = cudaMemcpyAsync(d1.p, c1, cb, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d2.p, c2, cb, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  double* v = (double*)dv.p;
  int32_t* iv = (int32_t*)di.p;
  if (int rc = cva_elastic_approach1_batch((const double*)d1.p, (const double*)d2.p, pairs, n, max_slope,
                                           n_max_approach1, v, v + pairs, v + 2 * pairs, v + 3 * pairs,
                                           gamma ? (double*)dg.p : nullptr, iv, iv + pairs, iv + 2 * pairs, s))
    return rc;
  double* hv[4] = {distance, energy, t0, theta};
  for (int k = 0; k < 4 && e == cudaSuccess; ++k)
    if (hv[k]) e = cudaMemcpyAsync(hv[k], v + k * pairs, vb, cudaMemcpyDeviceToHost, s);
  int32_t* hi[3] = {iterations, converged, status};
  for (int k = 0; k < 3 && e == cudaSuccess; ++k)
    if (hi[k]) e = cudaMemcpyAsync(hi[k], iv + k * pairs, ib, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && gamma) e = cudaMemcpyAsync(gamma, dg.p, gb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return finish(e, "elastic_approach1_batch_host");
}

}  // extern "C"
