// Pair stage of the alignment on one 256-thread CTA (v2): two concurrent
// forward FFTs (one per 128-thread half, named barriers), the correlation
// spectrum Z1 conj(Z2) fused into the first pass of the third FFT, a
// deterministic two-phase argmax with the reference's tie band, and the
// rotated, shifted aligned curve. Replaces correlation_all_shifts_fft +
// pick_best + optimal_rotation_svd (proj/src/rigid_align.cpp:147-183, :31-61,
// :82-102); the 4 real r2c + 4 real c2r FFTW transforms per pair become 3
// complex transforms on z = x + i y.
#pragma once

#include <climits>

#include "../../include/curvalign_cuda.h"
#include "cva_common.cuh"
#include "fft.cuh"
#include "prof.cuh"

namespace cva {
namespace pf {

constexpr int kT = 256;
constexpr int kHalf = 128;
constexpr double kTieRelTol = 1e-12;  // proj/src/rigid_align.cpp:16

// Shared-memory index with one pad slot every 8 double2 (128 B): Stockham
// stores at stride R (first passes) become bank-conflict free.
__device__ __forceinline__ int pad(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int padded_len(int n) { return n + n / 8; }

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// One Stockham pass (see fft.cuh) reading through a functor (runtime N, Ns).
template <int R, int NT, typename Src>
__device__ __forceinline__ void pass(Src src, double2* dst, int N, int Ns,
                                     const double2* __restrict__ tw, int g) {
  const int nb = N / R;
  const int tws = N / (Ns * R);
  for (int j = g; j < nb; j += NT) {
    double2 v[R];
    const int jm = j & (Ns - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src(j + r * nb);
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[r * jm * tws]));
    }
    dft_r<R>(v);
    const int base = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[pad(base + r * Ns)] = v[dft_slot<R>(r)];
  }
}

// Radix plan: radix 8 while it keeps every thread of the group busy, then 4 / 2
// (1024 points, 128 threads: 8 x 8 x 8 x 2). Radix 16 was measured slower here
// (register spills at the 128-register cap, half the threads idle).
template <int NT>
// CVA_R8_MIN: radix 8 only when every thread has a butterfly (N / NT >= 8).
// With scattered twiddle loads, 4 (radix 8 with half the threads idle in the
// 1024-point correlation transform: 4 passes instead of 5) was 1.4 % faster;
// with the per-pass twiddle tables, 8 is 0.35 % faster.
// Radix 8 for the 256-thread transform too (4: its pass tables are then the
// 128-thread plan's, 16 KB of twiddles per pair instead of 32 KB) measured
// slower in round 3 (align kernel 111 -> 132 us): half the threads idle.
#ifndef CVA_R8_MIN
#define CVA_R8_MIN 8
#endif
// CVA_R16_2048: the 128-thread plan of N = 2048 (16 points per thread: the
// forward transforms of the in-place SRV / N = 2048 pair kernels) is 16, 16, 8
// instead of 8, 8, 8, 4: one in-place pass fewer, same 16 values per thread.
#ifndef CVA_R16_2048
#define CVA_R16_2048 1
#endif
__host__ __device__ constexpr int plan_radix(int N, int Ns) {
  return (CVA_R16_2048 && NT == 128 && N == 2048 && (N / Ns) % 16 == 0)
             ? 16
             : (((N / Ns) % 8 == 0 && N / NT >= CVA_R8_MIN) ? 8 : ((N / Ns) % 4 == 0 ? 4 : 2));
}


// Pass twiddle tables, stored after the length-N table of W_N^k: for every
// pass (R, Ns > 1) of the NT = 128 plan, then of the NT = 256 plan, the
// values W_N^(r jm N/(Ns R)) laid out [r - 1][jm] (copied from the table, so
// bitwise the same values): a warp's twiddle load of one r reads consecutive
// entries (4 lines) instead of entries r*tws apart (up to 8r lines).
template <int NT>
__host__ __device__ constexpr int ptw_until(int N, int Ns_stop) {
  int s = 0;
  for (int Ns = 1; Ns < N && Ns < Ns_stop; Ns *= plan_radix<NT>(N, Ns))
    if (Ns > 1) s += (plan_radix<NT>(N, Ns) - 1) * Ns;
  return s;
}
// One warp per transform (largen.cu four-step sub-transforms): radix 8 while
// every lane has a butterfly, then 4 / 2.
__host__ __device__ constexpr int plan_radix_warp(int N, int Ns) {
  return ((N / Ns) % 8 == 0 && N / 8 >= 32) ? 8 : ((N / Ns) % 4 == 0 ? 4 : 2);
}
__host__ __device__ constexpr int ptw_until_warp(int N, int Ns_stop) {
  int s = 0;
  for (int Ns = 1; Ns < N && Ns < Ns_stop; Ns *= plan_radix_warp(N, Ns))
    if (Ns > 1) s += (plan_radix_warp(N, Ns) - 1) * Ns;
  return s;
}
// layout after the length-N table: [128-thread plan][256-thread plan][warp plan];
// a plan equal to an earlier one (same radix sequence) reads that one's tables
// (its own region is left unused).
__host__ __device__ constexpr bool plan256_is_128(int N) {
  for (int Ns = 1; Ns < N; Ns *= plan_radix<128>(N, Ns))
    if (plan_radix<128>(N, Ns) != plan_radix<256>(N, Ns)) return false;
  return true;
}
__host__ __device__ constexpr bool planwarp_is_128(int N) {
  for (int Ns = 1; Ns < N; Ns *= plan_radix<128>(N, Ns))
    if (plan_radix<128>(N, Ns) != plan_radix_warp(N, Ns)) return false;
  return true;
}
__host__ __device__ constexpr int ptw_len(int N) {
  return ptw_until<128>(N, N) + ptw_until<256>(N, N) + ptw_until_warp(N, N);
}
template <int NT>
__host__ __device__ constexpr bool plan_is_128(int N) {
  for (int Ns = 1; Ns < N; Ns *= plan_radix<128>(N, Ns))
    if (plan_radix<128>(N, Ns) != plan_radix<NT>(N, Ns)) return false;
  return true;
}
// NT = 512 (the M = 4096 pair kernel) reads the 128-thread plan's tables, which
// its radix sequence must equal (checked where it is used)
template <int NT>
__host__ __device__ constexpr int ptw_off(int N, int Ns) {
  return NT == 256 && !plan256_is_128(N) ? N + ptw_until<128>(N, N) + ptw_until<256>(N, Ns)
                                         : N + ptw_until<128>(N, Ns);
}
__host__ __device__ constexpr int ptw_off_warp(int N, int Ns) {
  return planwarp_is_128(N) ? N + ptw_until<128>(N, Ns)
                            : N + ptw_until<128>(N, N) + ptw_until<256>(N, N) + ptw_until_warp(N, Ns);
}


// Twiddles of one butterfly, v[r] *= W^(r e) for r = 1 .. R-1, where the pass
// table holds W^(r e) at pt[(r - 1) Ns + jm]. With CVA_TW_DERIVE (default)
// only r = 1, 2, 4 are read and W^3 = W^1 W^2, W^5 = W^1 W^4, W^6 = W^2 W^4,
// W^7 = W^3 W^4 are formed by products of table values (at most two
// roundings from sincospi-exact entries, no recurrence): 3 L1 reads per
// radix-8 butterfly instead of 7, 2 instead of 3 for radix 4 (the pass
// tables were the top L1 consumer of the transforms: C4 539.9 -> 521.6 us,
// C1 349.7 -> 347.0 us; profiles/r4_c1_variants.txt). CVA_TW_DERIVE=0 reads
// every twiddle.
#ifndef CVA_TW_DERIVE
#define CVA_TW_DERIVE 1
#endif
#ifndef CVA_TW_DERIVE16
#define CVA_TW_DERIVE16 1
#endif
template <int R>
__device__ __forceinline__ void twiddle(double2 (&v)[R], const double2* __restrict__ pt, int Ns, int jm) {
#if CVA_TW_DERIVE
  if constexpr (R == 8) {
    const double2 w1 = __ldg(&pt[jm]), w2 = __ldg(&pt[Ns + jm]), w4 = __ldg(&pt[3 * Ns + jm]);
    const double2 w3 = cmul(w1, w2);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    v[4] = cmul(v[4], w4);
    v[5] = cmul(v[5], cmul(w1, w4));
    v[6] = cmul(v[6], cmul(w2, w4));
    v[7] = cmul(v[7], cmul(w3, w4));
  } else if constexpr (R == 16 && CVA_TW_DERIVE16) {
    const double2 w1 = __ldg(&pt[jm]), w2 = __ldg(&pt[Ns + jm]), w4 = __ldg(&pt[3 * Ns + jm]),
                  w8 = __ldg(&pt[7 * Ns + jm]);
    const double2 w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    v[4] = cmul(v[4], w4);
    v[5] = cmul(v[5], w5);
    v[6] = cmul(v[6], w6);
    v[7] = cmul(v[7], w7);
    v[8] = cmul(v[8], w8);
    v[9] = cmul(v[9], cmul(w1, w8));
    v[10] = cmul(v[10], cmul(w2, w8));
    v[11] = cmul(v[11], cmul(w3, w8));
    v[12] = cmul(v[12], cmul(w4, w8));
    v[13] = cmul(v[13], cmul(w5, w8));
    v[14] = cmul(v[14], cmul(w6, w8));
    v[15] = cmul(v[15], cmul(w7, w8));
  } else if constexpr (R == 4) {
    const double2 w1 = __ldg(&pt[jm]), w2 = __ldg(&pt[Ns + jm]);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], cmul(w1, w2));
  } else
#endif
  {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&pt[(r - 1) * Ns + jm]));
  }
}

// Compile-time pass: N, Ns, the butterfly count per thread and every index
// stride are constants.
template <int R, int NT, int N, int Ns, typename Src>
__device__ __forceinline__ void pass_ct(Src src, double2* dst, const double2* __restrict__ tw, int g) {
  static_assert(NT == 128 || NT == 256, "pass twiddle tables exist for the 128- and 256-thread plans");
  constexpr int nb = N / R;
  const double2* __restrict__ pt = tw + ptw_off<NT>(N, Ns);  // this pass's [r - 1][jm] table
#pragma unroll
  for (int j0 = 0; j0 < nb; j0 += NT) {
    const int j = j0 + g;
    if (nb % NT == 0 || j < nb) {
      double2 v[R];
      const int jm = j & (Ns - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = src(j + r * nb);
      if (Ns > 1) twiddle<R>(v, pt, Ns, jm);
      dft_r<R>(v);
      const int base = (j - jm) * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) dst[pad(base + r * Ns)] = v[dft_slot<R>(r)];
    }
  }
}

// Forward FFT of compile-time length N by NT threads, first pass through src,
// ping-ponging dst/other. Returns the buffer holding the spectrum.
// (kStop: stop before the pass whose Ns is kStop; the default runs all passes)
template <int NT, int N, int Ns = 1, int kStop = N, typename Src, typename Sync>
__device__ __forceinline__ double2* group_fft_ct(Src src, double2* dst, double2* other,
                                                 const double2* __restrict__ tw, int g, Sync sync) {
  constexpr int R = plan_radix<NT>(N, Ns);
  pass_ct<R, NT, N, Ns>(src, dst, tw, g);
  sync();
  CVA_MARK(40 + (NT == 256 ? 8 : 0) + (Ns == 1 ? 0 : Ns == 8 ? 1 : Ns == 64 ? 2 : Ns == 512 ? 3 : Ns == 4 ? 4 : Ns == 16 ? 5 : Ns == 256 ? 6 : 7));
  if constexpr (Ns * R < N && Ns * R < kStop) {
    auto next = [dst](int i) { return dst[pad(i)]; };
    return group_fft_ct<NT, N, Ns * R, kStop>(next, other, dst, tw, g, sync);
  } else {
    return dst;
  }
}

// Forward FFT of length N (power of two) by NT threads (index g), first pass
// reading through src0, then ping-ponging b0 -> b1 -> b0 ... Returns the
// buffer holding the spectrum. sync() is the group barrier.
template <int NT, typename Src, typename Sync>
__device__ inline double2* group_fft(Src src0, double2* b0, double2* b1, int N,
                                     const double2* __restrict__ tw, int g, Sync sync) {
  int Ns = 1;
  double2* dst = b0;
  double2* other = b1;
  bool first = true;
  const int maxR = N / NT >= 8 ? 8 : 4;
  while (Ns < N) {
    const int rem = N / Ns;
    const int R = (rem % 8 == 0 && maxR >= 8) ? 8 : (rem % 4 == 0 ? 4 : 2);
    if (first) {
      if (R == 8) pass<8, NT>(src0, dst, N, Ns, tw, g);
      else if (R == 4) pass<4, NT>(src0, dst, N, Ns, tw, g);
      else pass<2, NT>(src0, dst, N, Ns, tw, g);
      first = false;
    } else {
      const double2* in = other;
      auto src = [in](int i) { return in[pad(i)]; };
      if (R == 8) pass<8, NT>(src, dst, N, Ns, tw, g);
      else if (R == 4) pass<4, NT>(src, dst, N, Ns, tw, g);
      else pass<2, NT>(src, dst, N, Ns, tw, g);
    }
    sync();
    Ns *= R;
    double2* t = dst;
    dst = other;
    other = t;
  }
  return other;  // last written
}

// In-place variant (one buffer per transform; used where shared memory binds,
// M = 2048): the pass sequence is fixed at compile time (8, 8, 8, 4) so every
// register index is static. Each pass loads all of a thread's butterflies
// (<= 16 values) into registers, syncs, then transforms and stores in place.
template <int R, int NT, int M, int Ns, typename Src, typename Sync>
__device__ __forceinline__ void pass_ip(Src src, double2* buf, const double2* __restrict__ tw, int g,
                                        Sync sync) {
  constexpr int nb = M / R;
  constexpr int B = nb / NT;  // butterflies per thread
  static_assert(B >= 1 && B * R <= 16, "in-place pass keeps <= 16 values per thread");
  // the 8, 8, 8, 4 sequence is also the 128- and 256-thread plan of M = 2048,
  // so the pass twiddle tables of ptw_off apply
  static_assert(R == plan_radix<NT>(M, Ns), "in-place sequence must match the table plan");
  static_assert(NT == 128 || NT == 256 || plan_is_128<NT>(M), "pass twiddle tables exist for this plan");
  const double2* __restrict__ pt = tw + ptw_off<NT>(M, Ns);
  double2 v[B][R];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = g + b * NT;
    const int jm = j & (Ns - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = src(j + r * nb);
    if (Ns > 1) twiddle<R>(v[b], pt, Ns, jm);
  }
  sync();
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = g + b * NT;
    const int jm = j & (Ns - 1);
    dft_r<R>(v[b]);
    const int base = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pad(base + r * Ns)] = v[b][dft_slot<R>(r)];
  }
  sync();
}

// In-place transform of compile-time length M by NT threads with the table
// plan (plan_radix<NT>): M = 2048 gives 8, 8, 8, 4, M = 4096 8, 8, 8, 8.
template <int NT, int M, int Ns = 1, int kStop = M, typename Src, typename Sync>
__device__ __forceinline__ void fft_ip_ct(Src src, double2* buf, const double2* __restrict__ tw, int g, Sync sync) {
  constexpr int R = plan_radix<NT>(M, Ns);
  pass_ip<R, NT, M, Ns>(src, buf, tw, g, sync);
  if constexpr (Ns * R < M && Ns * R < kStop) {
    auto next = [buf](int i) { return buf[pad(i)]; };
    fft_ip_ct<NT, M, Ns * R, kStop>(next, buf, tw, g, sync);
  }
}

// ---- last forward pass fused into the first pass of the correlation transform
// The correlation transform's first pass (Ns = 1, radix Rc, butterfly j reads
// k = j + nbC r) needs exactly the outputs of the forward transforms' last
// butterflies jb = j + nbC b (b < B), whose outputs are X[jb + NsF r'] (k's
// r = b + B r'). So thread j runs those B radix-Rf butterflies of both curves
// from the penultimate spectra, forms conj-products, and does its radix-Rc
// butterfly: one shared-memory round trip of 2 N points and a barrier fewer.
template <int NT>
__host__ __device__ constexpr int last_pass_ns(int N) {
  int Ns = 1;
  while (Ns * plan_radix<NT>(N, Ns) < N) Ns *= plan_radix<NT>(N, Ns);
  return Ns;
}
#ifndef CVA_FUSE_LAST
#define CVA_FUSE_LAST 1
#endif
template <int NTf, int NTc, int N>
struct FusePlan {
  static constexpr int NsF = last_pass_ns<NTf>(N);
  static constexpr int Rf = N / NsF;
  static constexpr int Rc = plan_radix<NTc>(N, 1);
  static constexpr int nbC = N / Rc;
  static constexpr int B = NsF >= nbC ? NsF / nbC : 0;
  static constexpr bool ok = CVA_FUSE_LAST && NsF > 1 && B >= 1 && NsF % nbC == 0 && Rc == Rf * B && nbC <= NTc;
};
// v[0 .. Rc) of correlation butterfly j (j < nbC): products of the forward
// spectra finished from Y1 / Y2 (penultimate Stockham buffers, padded), scaled
// by s12 when kScale; returned before the radix-Rc DFT.
template <int NTf, int NTc, int N, bool kScale>
__device__ __forceinline__ void fused_first_inputs(const double2* Y1, const double2* Y2, double s12,
                                                   const double2* __restrict__ tw, int j,
                                                   double2 (&v)[FusePlan<NTf, NTc, N>::Rc]) {
  using P = FusePlan<NTf, NTc, N>;
  const double2* __restrict__ ptf = tw + ptw_off<NTf>(N, P::NsF);  // the forward last pass's table
#pragma unroll
  for (int b = 0; b < P::B; ++b) {
    const int jb = j + P::nbC * b;  // forward-last butterfly (jm = jb: jb < NsF)
    double2 a[P::Rf], c[P::Rf];
#pragma unroll
    for (int r = 0; r < P::Rf; ++r) {
      a[r] = Y1[pad(jb + r * P::NsF)];
      c[r] = Y2[pad(jb + r * P::NsF)];
    }
    twiddle<P::Rf>(a, ptf, P::NsF, jb);
    twiddle<P::Rf>(c, ptf, P::NsF, jb);
    dft_r<P::Rf>(a);
    dft_r<P::Rf>(c);
#pragma unroll
    for (int r = 0; r < P::Rf; ++r) {
      const double2 x = cmulconj(a[dft_slot<P::Rf>(r)], c[dft_slot<P::Rf>(r)]);
      v[b + P::B * r] = kScale ? cscale(x, s12) : x;
    }
  }
}

template <int NT, typename Src, typename Sync>
__device__ inline void fft2048_ip(Src src0, double2* buf, const double2* __restrict__ tw, int g, Sync sync) {
  auto src = [buf](int i) { return buf[pad(i)]; };
  pass_ip<8, NT, 2048, 1>(src0, buf, tw, g, sync);
  pass_ip<8, NT, 2048, 8>(src, buf, tw, g, sync);
  pass_ip<8, NT, 2048, 64>(src, buf, tw, g, sync);
  pass_ip<4, NT, 2048, 512>(src, buf, tw, g, sync);
}

// ---- the correlation transform's last pass into registers
// Its butterfly j = g + b NT (Ns = N / R >= NT, jm = j) writes outputs
// k = j + r Ns = g + NT (b + B r): thread g ends up holding exactly the bins
// k = g + q NT the argmax reads, so they stay in registers (fv[q]) and F is
// never stored or re-read. CVA_REG_LAST=0 keeps the stored spectrum.
#ifndef CVA_REG_LAST
#define CVA_REG_LAST 1
#endif
template <int NT, int N>
struct RegLastPlan {
  static constexpr int Ns = last_pass_ns<NT>(N);
  static constexpr int R = N / Ns;
  static constexpr int B = Ns >= NT ? Ns / NT : 0;
  static constexpr bool ok = CVA_REG_LAST && Ns > 1 && B >= 1 && Ns % NT == 0;
};
template <int NT, int N, int kMax>
__device__ __forceinline__ void last_pass_regs(const double2* src, const double2* __restrict__ tw, int g,
                                               double2 (&fv)[kMax]) {
  using P = RegLastPlan<NT, N>;
  static_assert(P::B * P::R <= kMax, "bins per thread");
  const double2* __restrict__ pt = tw + ptw_off<NT>(N, P::Ns);
#pragma unroll
  for (int b = 0; b < P::B; ++b) {
    const int j = g + b * NT;
    double2 v[P::R];
#pragma unroll
    for (int r = 0; r < P::R; ++r) v[r] = src[pad(j + r * P::Ns)];
    twiddle<P::R>(v, pt, P::Ns, j);
    dft_r<P::R>(v);
#pragma unroll
    for (int r = 0; r < P::R; ++r) fv[b + P::B * r] = v[dft_slot<P::R>(r)];
  }
}

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

struct PairIn {
  const double2* z1;  // curve 1 samples (shared or global), uncentered
  const double2* z2;  // curve 2 samples (global or shared), uncentered
  double2 g1, g2;     // centroids subtracted on load
  double sc1, sc2;    // scale applied after centering (1 for already-normalized input)
  // optional: the raw curve whose SRV z2 holds (global memory); the aligned
  // output then recomputes z2[j] = srv_at(srv2, j) because z2 was overwritten
  const double2* srv2 = nullptr;
  // optional (with srv2, in-place M = 2048 with the fused first pass): a CTA
  // mbarrier initialised for one arrival whose next phase is 1; the raw curve
  // srv2 is then copied back into curve 2's transform buffer by TMA once that
  // buffer is dead, and the aligned output reads it from shared memory
  uint64_t* bar = nullptr;
  // optional (with bar): q2 = SRV(curve 2) already sits in `aligned` (natural
  // order, written by the caller before the transforms); the TMA then brings
  // q2 itself back and the aligned output does not recompute it
  bool q2_in_aligned = false;
};

// q_l = d_l / sqrt(|d_l|), d_l = (N/2)(c[l+1] - c[l-1]); 0 if |d_l| < 1e-8 N (srv.cpp:71-88)
// (MUFU-seeded sqrt / reciprocal with one correction step, <= 1 ulp each: the
// IEEE sqrt and division slow paths were a visible share of the C4 kernel)
#ifndef CVA_SRV_RSQ2
#define CVA_SRV_RSQ2 1
#endif
// refined reciprocal square root (MUFU seed + one third-order step, ~2^-56)
__device__ __forceinline__ double rsqrt_ref(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x * r, r, 1.0);
  return fma(r * e, fma(0.375, e, 0.5), r);
}
__device__ __forceinline__ double2 srv_at(const double2* c, int l, int N) {
  const double nn = (double)N;
  const double2 nx = c[l + 1 == N ? 0 : l + 1], pv = c[l == 0 ? N - 1 : l - 1];
  const double2 d = make_double2((nn / 2.0) * (nx.x - pv.x), (nn / 2.0) * (nx.y - pv.y));
#if CVA_SRV_RSQ2
  // q = d |d|^(-1/2) from two refined rsqrts: |d| = x rsqrt(x), then
  // rsqrt(|d|) (each <= ~1 ulp; 9 FP64 operations fewer than sqrt, sqrt and
  // a reciprocal). x = 0 gives |d| = NaN, which the threshold test maps to 0
  // like the reference's |d| = 0 < 1e-8 N.
  const double x = fma(d.x, d.x, d.y * d.y);
  const double mag = x * rsqrt_ref(x);
  if (!(mag >= 1e-8 * nn)) return make_double2(0.0, 0.0);
  const double r = rsqrt_ref(mag);
#else
  const double mag = fsqrt(fma(d.x, d.x, d.y * d.y));
  if (mag < 1e-8 * nn) return make_double2(0.0, 0.0);
  const double r = frcp(fsqrt(mag));
#endif
  return make_double2(r * d.x, r * d.y);
}

// 1 / polygon length (curve.cpp:17-25) of each curve, measured by the pair
// stage while it loads the samples (kLenOnLoad); {NaN, NaN} flags a bad pair.
struct PairScale {
  double sc1, sc2;
};

// FFT length for N data points: N itself when N is a power of two, else the
// smallest power of two M >= 2N. In the padded case the circular correlation
// of length N is the first N lags of the length-M circular correlation of
// a = [z1, 0...] and b = [z2, z2, 0...]: for m < N and l < N, l + m < 2N <= M,
// so no term wraps and b_{l+m} = z2_{(l+m) mod N}. This gives any N >= 4 (the
// reference's FFTW path accepts any length) with power-of-two
// transforms only.
__host__ __device__ inline int fft_len(int N) {
  if ((N & (N - 1)) == 0) return N;
  int M = 1;
  while (M < 2 * N) M <<= 1;
  return M;
}

// Runs the pair stage. bufs: 4 * padded_len(M) double2 of shared memory (distinct from
// the inputs), M = fft_len(N), tw the length-M twiddle table. out: this pair's
// result (written by thread 0). aligned: this pair's aligned curve (may alias
// in.z2: all reads happen before any write). red: >= kCT / 16 double2 shared.
// Requires blockDim.x == kCT (256, or 512 for the in-place M = 4096 kernel),
// N >= 4, M <= 2048 (M = kIPM with kInPlace).
// kInPlace: 2 * padded_len(M) buffers instead of 4; requires M == 2048.
// kN: compile-time N (a power of two) or 0 for a runtime N.
// kLenOnLoad: in.sc1 / in.sc2 are ignored; each curve's polygon length is
// summed while its samples are loaded for the first FFT pass (the transforms
// run on the centered, unscaled curves) and the scales 1/len are applied to
// the correlation spectrum, the energies and the aligned curve. A length that
// is not finite and > 0 marks the pair invalid (preprocess: curve.cpp:41-48).
// kPad: 1 = in.z1 is shared memory in the padded layout z1[l + (l >> 3)]
// (the resampler's and the transform buffers' layout); 2 = in.z1 and in.z2 both.
// kDirectOut: `aligned` never aliases in.z2 (shared z2 or srv2, global output),
// so the aligned curve is written as it is formed (no register copy, no barrier).
// Compile-time plans (kN > 0 or kInPlace) run the forward transforms up to
// their last pass, fuse that pass into the correlation transform's first
// (FusePlan), and keep the correlation's last-pass bins in registers for the
// argmax (RegLastPlan); runtime-N out-of-place plans run every pass through
// shared memory.
template <bool kInPlace = false, int kN = 0, bool kLenOnLoad = false, int kPad = 0, int kCT = kT, int kIPM = 2048,
          bool kDirectOut = false>
__device__ inline void pair_stage(const PairIn& in, double2* bufs, int N,
                                  const double2* __restrict__ tw, cva_alignment* out,
                                  double2* aligned, double2* red) {
  const int t = threadIdx.x;
  constexpr int kH = kCT / 2;  // threads per forward transform
  const int grp = t / kH, g = t % kH;
  if constexpr (kN > 0) N = kN;
  const int M = kN > 0 ? kN : fft_len(N);
  const int NP = padded_len(M);
  double2* B0 = bufs;
  double2* B1 = bufs + NP;
  double2* B2 = bufs + (kInPlace ? 1 : 2) * NP;
  double2* B3 = bufs + 3 * NP;

  // ---- two forward transforms of the normalized curves (normalization fused into the load)
  double ss = 0.0;   // sum |z'|^2 of this group's curve (rigid_align.cpp:23-27)
  double len = 0.0;  // kLenOnLoad: this thread's share of the polygon length
  double2* X;
  {
    const double2* src = grp == 0 ? in.z1 : in.z2;
    const double2 c = grp == 0 ? in.g1 : in.g2;
    const double sc = kLenOnLoad ? 1.0 : (grp == 0 ? in.sc1 : in.sc2);
    // group 0: a = [z1, 0...]; group 1: b = [z2, z2, 0...] (M == N: plain z)
    const int lim = (grp == 0 || M == N) ? N : 2 * N;
    auto load = [&](int i) {
      if (i >= lim) return make_double2(0.0, 0.0);
      const int k = i < N ? i : i - N;
      const bool padded = kPad == 2 || (kPad == 1 && grp == 0);
      const double2 q = src[padded ? k + (k >> 3) : k];
      const double2 z = make_double2((q.x - c.x) * sc, (q.y - c.y) * sc);
      if (i < N) {
        ss = fma(z.x, z.x, fma(z.y, z.y, ss));
        if constexpr (kLenOnLoad) {  // edge (k, k+1) of the closed polygon (curve.cpp:17-25)
          const int k1 = k + 1 == N ? 0 : k + 1;
          const double2 o = src[padded ? k1 + (k1 >> 3) : k1];
          const double dx = o.x - q.x, dy = o.y - q.y;
          const double e2 = fma(dx, dx, dy * dy);
          const double e = fsqrt_nb(e2);  // branch-free; a zero edge adds 0
          len += e2 == 0.0 ? 0.0 : e;  // NaN / inf edges propagate (flagged below)
        }
      }
      return z;
    };
    auto sync = [grp]() { named_sync(1 + grp, kH); };
    if constexpr (kInPlace) {
      constexpr int stop = FusePlan<kH, kCT, kIPM>::ok ? FusePlan<kH, kCT, kIPM>::NsF : kIPM;
      fft_ip_ct<kH, kIPM, 1, stop>(load, grp == 0 ? B0 : B2, tw, g, sync);
      X = grp == 0 ? B0 : B2;
    } else {
      if constexpr (kN > 0) {
        constexpr int stop = FusePlan<kH, kCT, (kN > 0 ? kN : 2)>::ok ? FusePlan<kH, kCT, (kN > 0 ? kN : 2)>::NsF : kN;
        X = group_fft_ct<kH, kN, 1, stop>(load, grp == 0 ? B0 : B2, grp == 0 ? B1 : B3, tw, g, sync);
      } else {
        X = group_fft<kH>(load, grp == 0 ? B0 : B2, grp == 0 ? B1 : B3, M, tw, g, sync);
      }
    }
  }
  PairScale psc{in.sc1, in.sc2};
  if constexpr (kLenOnLoad) {
    __shared__ double s_len[kCT / 32];
    len = warp_sum(len);
    if ((t & 31) == 0) s_len[t >> 5] = len;
    __syncthreads();
    double l1 = 0.0, l2 = 0.0;
#pragma unroll
    for (int w = 0; w < kCT / 64; ++w) {
      l1 += s_len[w];
      l2 += s_len[kCT / 64 + w];
    }
    if (!(l1 > 0.0) || !isfinite(l1) || !(l2 > 0.0) || !isfinite(l2)) {  // curve.cpp:44-46
      if (t == 0) {
        cva_alignment r;
        r.shift = 0;
        r.t0 = 0.0;
        r.theta = r.trace = r.energy = qnan();
        r.degenerate = 0;
        r.status = CVA_INVALID_ARGUMENT;
        *out = r;
      }
      if (aligned != nullptr) {
        __syncthreads();  // in.z2 may alias `aligned`
        for (int l = t; l < N; l += kCT) aligned[l] = make_double2(qnan(), qnan());
      }
      return;
    }
    psc.sc1 = 1.0 / l1;
    psc.sc2 = 1.0 / l2;
  } else {
    __syncthreads();
  }
  CVA_MARK(20);
  // ---- D_m = sum_l conj(z1_l) z2_{l+m} = IDFT(conj Z1 . Z2)_m = conj(FFT(Z1 conj Z2)_m) / N
  auto sync_all = []() { __syncthreads(); };
  const double2* F = nullptr;
  constexpr int kMaxPer = kInPlace ? 8 : 4;  // N <= 2048 in-place, N <= 1024 otherwise
  constexpr int kNc = kInPlace ? kIPM : (kN > 0 ? kN : 2);  // compile-time transform length (if any)
  constexpr bool kRegLast = (kInPlace || kN > 0) && FusePlan<kH, kCT, kNc>::ok && RegLastPlan<kCT, kNc>::ok &&
                            RegLastPlan<kCT, kNc>::Ns >= FusePlan<kH, kCT, kNc>::Rc;
  double2 fv[kMaxPer];  // kRegLast: bins t + q kCT of the correlation spectrum
  if constexpr (kInPlace) {
    const double2* X1 = B0;
    const double2* X2 = B2;
    const double s12 = kLenOnLoad ? psc.sc1 * psc.sc2 : 1.0;
    auto prod = [X1, X2, s12](int k) {
      const double2 v = cmulconj(X1[pad(k)], X2[pad(k)]);
      return kLenOnLoad ? cscale(v, s12) : v;
    };
    using FP = FusePlan<kH, kCT, kIPM>;
    if constexpr (FP::ok) {  // in place: every load of the fused pass, a barrier, the stores
      double2 v[FP::Rc];
      if (t < FP::nbC) fused_first_inputs<kH, kCT, kIPM, kLenOnLoad>(X1, X2, s12, tw, t, v);
      sync_all();
      if (kDirectOut && t == 0 && in.srv2 && in.bar && aligned != nullptr) {
        // B2 is dead from here on: the raw curve 2 comes back into it under
        // the remaining passes (its SRV is recomputed for the aligned output)
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(in.bar));
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(B2));
        const uint32_t bytes = (uint32_t)N * 16u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         dst),
                     "l"(in.q2_in_aligned ? (const double2*)aligned : in.srv2), "r"(bytes), "r"(b)
                     : "memory");
      }
      if (t < FP::nbC) {
        dft_r<FP::Rc>(v);
#pragma unroll
        for (int r = 0; r < FP::Rc; ++r) B0[pad(t * FP::Rc + r)] = v[dft_slot<FP::Rc>(r)];
      }
      sync_all();
      auto next = [B0](int i) { return B0[pad(i)]; };
      if constexpr (kRegLast) {  // all passes but the last in place, the last into registers
        if constexpr (FP::Rc < RegLastPlan<kCT, kIPM>::Ns)
          fft_ip_ct<kCT, kIPM, FP::Rc, RegLastPlan<kCT, kIPM>::Ns>(next, B0, tw, t, sync_all);
        last_pass_regs<kCT, kIPM>(B0, tw, t, fv);
      } else {
        fft_ip_ct<kCT, kIPM, FP::Rc>(next, B0, tw, t, sync_all);
      }
    } else {
      fft_ip_ct<kCT, kIPM>(prod, B0, tw, t, sync_all);
    }
    F = B0;
  } else {
    // group 0's result is B0 or B1, group 1's is B2 or B3 (same pass count)
    const bool in0 = (X == B0 || X == B2);
    const double2* X1 = in0 ? B0 : B1;
    const double2* X2 = in0 ? B2 : B3;
    double2* F0 = in0 ? B1 : B0;
    double2* F1 = in0 ? B3 : B2;
    const double s12 = kLenOnLoad ? psc.sc1 * psc.sc2 : 1.0;
    auto prod = [X1, X2, s12](int k) {
      const double2 v = cmulconj(X1[pad(k)], X2[pad(k)]);
      return kLenOnLoad ? cscale(v, s12) : v;
    };
    if constexpr (kN > 0) {
      using FP = FusePlan<kH, kCT, (kN > 0 ? kN : 2)>;
      if constexpr (FP::ok) {
        if (t < FP::nbC) {
          double2 v[FP::Rc];
          fused_first_inputs<kH, kCT, kN, kLenOnLoad>(X1, X2, s12, tw, t, v);
          dft_r<FP::Rc>(v);
#pragma unroll
          for (int r = 0; r < FP::Rc; ++r) F0[pad(t * FP::Rc + r)] = v[dft_slot<FP::Rc>(r)];
        }
        sync_all();
        if constexpr (kRegLast) {  // all passes but the last, then the last into registers
          const double2* P = F0;
          if constexpr (FP::Rc < RegLastPlan<kCT, kNc>::Ns) {
            auto next = [F0](int i) { return F0[pad(i)]; };
            P = group_fft_ct<kCT, kN, FP::Rc, RegLastPlan<kCT, kNc>::Ns>(next, F1, F0, tw, t, sync_all);
          }
          last_pass_regs<kCT, kNc>(P, tw, t, fv);
        } else if constexpr (FP::Rc < kN) {
          auto next = [F0](int i) { return F0[pad(i)]; };
          F = group_fft_ct<kCT, kN, FP::Rc>(next, F1, F0, tw, t, sync_all);
        } else {
          F = F0;
        }
      } else {
        F = group_fft_ct<kCT, kN>(prod, F0, F1, tw, t, sync_all);
      }
    } else {
      F = group_fft<kCT>(prod, F0, F1, M, tw, t, sync_all);
    }
  }

  CVA_MARK(21);
  // ---- tie-broken argmax of |D_m| (rigid_align.cpp:31-47): max, then smallest index in band
  // |D_m| = |F_m| / M. The max and the band test run on squared magnitudes,
  // each thread's |F|^2 values read once into registers; the band threshold is
  // formed exactly as the reference does (on |D|).
  const double invN = 1.0 / (double)N;  // h = 1/N (rigid_align.cpp:56)
  const double invM = 1.0 / (double)M;  // D_m = conj(F_m) / M
  // CVA_MAG_REREAD=1 recomputes the magnitudes from shared memory for the band
  // test instead of holding them in registers across the block reduction:
  // measured 0.5 % slower (C1 351.2 -> 352.9 us, C4 0.549 -> 0.553 ms).
#ifndef CVA_MAG_REREAD
#define CVA_MAG_REREAD 0
#endif
  double best2 = -1.0;
#if !CVA_MAG_REREAD
  double mag2[kMaxPer];
#endif
#pragma unroll
  for (int q = 0; q < kMaxPer; ++q) {
    const int k = t + q * kCT;
#if !CVA_MAG_REREAD
    mag2[q] = -1.0;
#endif
    if (k < N) {
      const double2 f = kRegLast ? fv[q] : F[pad(k)];
      const double m2 = fma(f.x, f.x, f.y * f.y);
#if !CVA_MAG_REREAD
      mag2[q] = m2;
#endif
      best2 = fmax(best2, m2);
    }
  }
  // block max of best2 and sums of s1 / s2 in one exchange
  const int lane = t & 31, wid = t >> 5;
  double s1 = grp == 0 ? ss : 0.0, s2 = grp == 1 ? ss : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    best2 = fmax(best2, __shfl_xor_sync(0xffffffffu, best2, o));
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    red[wid] = make_double2(best2, s1);
    red[kCT / 32 + wid].x = s2;
  }
  __syncthreads();
  best2 = -1.0;
  s1 = s2 = 0.0;
#pragma unroll
  for (int w = 0; w < kCT / 32; ++w) {
    best2 = fmax(best2, red[w].x);
    s1 += red[w].y;
    s2 += red[kCT / 32 + w].x;
  }
  if constexpr (kLenOnLoad) {  // sums of |z - c|^2 -> of |(z - c) / len|^2
    s1 *= psc.sc1 * psc.sc1;
    s2 *= psc.sc2 * psc.sc2;
  }
  const double best = sqrt(best2) * invM;  // NaN if the correlation is not finite
  const double thr = best - kTieRelTol * fmax(1.0, fabs(best));
  const double thrM = thr * (double)M;
  const double thr2 = thr > 0.0 ? thrM * thrM : -1.0;  // |F|^2 >= (thr M)^2  <=>  |D| >= thr
  int cand = INT_MAX;
  double2 fc = make_double2(0.0, 0.0);  // kRegLast: F at this thread's candidate
#pragma unroll
  for (int q = kMaxPer - 1; q >= 0; --q) {
    const int k = t + q * kCT;
#if CVA_MAG_REREAD
    if (k < N) {
      const double2 f = kRegLast ? fv[q] : F[pad(k)];
      if (fma(f.x, f.x, f.y * f.y) >= thr2) {  // smallest k of this thread
        cand = k;
        fc = f;
      }
    }
#else
    if (mag2[q] >= thr2 && k < N) {  // smallest k of this thread
      cand = k;
      if constexpr (kRegLast) fc = fv[q];
    }
#endif
  }
  const int cand_t = cand;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
  __shared__ int s_cand[kCT / 32];
  __shared__ double2 s_fc[kRegLast ? kCT / 32 : 1];
  if constexpr (kRegLast) {  // the warp's candidate bin travels with its index
    const unsigned own = __ballot_sync(0xffffffffu, cand_t == cand && cand != INT_MAX);
    const int src = own ? __ffs(own) - 1 : 0;
    const double fx = __shfl_sync(0xffffffffu, fc.x, src), fy = __shfl_sync(0xffffffffu, fc.y, src);
    if (lane == 0) s_fc[wid] = make_double2(fx, fy);
  }
  if (lane == 0) s_cand[wid] = cand;
  __syncthreads();
  int m = INT_MAX, wm = 0;
#pragma unroll
  for (int w = 0; w < kCT / 32; ++w)
    if (s_cand[w] < m) {
      m = s_cand[w];
      wm = w;
    }
  const bool ok = isfinite(best) && best2 >= 0.0 && m != INT_MAX;
  // rotation straight from D_m: (cos, sin) = (Re D, Im D) / |D| (every thread)
  double2 rot = make_double2(qnan(), qnan());
  double trace = 0.0;
  double2 fm = make_double2(0.0, 0.0);
  if (ok) {
    fm = kRegLast ? s_fc[wm] : F[pad(m)];
    const double a2 = fma(fm.x, fm.x, fm.y * fm.y);
    trace = sqrt(a2) * invM;
    if (a2 > 0.0) {
      const double ia = 1.0 / sqrt(a2);
      rot = make_double2(fm.x * ia, -fm.y * ia);
    } else {
      rot = make_double2(1.0, 0.0);  // degenerate: theta = 0 (rigid_align.cpp:86-88)
    }
  }

  // ---- aligned[l] = R(theta) z2'[(l + m) mod N]  (geometry.hpp:70-73; elastic.cpp:80)
  if (kDirectOut && aligned != nullptr) {
    const double2 c = in.g2;
    const double sc = psc.sc2;
    const int mm = ok ? m : 0;
    const double2* raw2 = in.srv2;
    if constexpr (kInPlace && FusePlan<kH, kCT, kIPM>::ok) {
      if (in.srv2 && in.bar) {  // the copy issued after the fused first pass (phase 1)
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(in.bar));
        uint32_t done = 0;
        do {
          asm volatile(
              "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n selp.u32 %0, 1, 0, p;\n}"
              : "=r"(done)
              : "r"(b)
              : "memory");
        } while (!done);
        raw2 = B2;
      }
    }
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      const int j = t + q * kCT;
      if (j < N) {
        const double2 z = in.srv2 ? (raw2 == B2 && in.q2_in_aligned ? B2[j] : srv_at(raw2, j, N))
                                  : in.z2[kPad == 2 ? j + (j >> 3) : j];
        const double2 pz = make_double2((z.x - c.x) * sc, (z.y - c.y) * sc);
        int l = j - mm;
        if (l < 0) l += N;
        aligned[l] = make_double2(fma(rot.x, pz.x, rot.y * pz.y), fma(-rot.y, pz.x, rot.x * pz.y));
      }
    }
  } else if (aligned != nullptr) {
    double2 v[kMaxPer];
    const double2 c = in.g2;
    const double sc = psc.sc2;
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      const int j = t + q * kCT;
      if (j < N) {
        const double2 z = in.srv2 ? srv_at(in.srv2, j, N) : in.z2[kPad == 2 ? j + (j >> 3) : j];
        const double2 p = make_double2((z.x - c.x) * sc, (z.y - c.y) * sc);
        v[q] = make_double2(fma(rot.x, p.x, rot.y * p.y), fma(-rot.y, p.x, rot.x * p.y));
      }
    }
    __syncthreads();  // in.z2 may alias `aligned`
    const int mm = ok ? m : 0;
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      const int j = t + q * kCT;
      if (j < N) {
        int l = j - mm;
        if (l < 0) l += N;
        aligned[l] = v[q];
      }
    }
  }
  if (t == 0) {
    cva_alignment r;
    if (!ok) {
      r.shift = 0;
      r.t0 = 0.0;
      r.theta = qnan();
      r.trace = qnan();
      r.energy = qnan();
      r.degenerate = 0;
      r.status = CVA_INVALID_ARGUMENT;  // non-finite correlation (rigid_align.cpp:83)
    } else {
      const int degenerate = trace == 0.0;
      double e = invN * (s1 + s2) - 2.0 * invN * trace;  // rigid_align.cpp:56-59
      if (e < 0.0) e = 0.0;
      r.shift = m;
      r.t0 = (double)m / (double)N;  // rigid_align.cpp:52
      r.theta = degenerate ? 0.0 : atan2(-fm.y, fm.x);  // arg D_m
      r.trace = trace;
      r.energy = e;
      r.degenerate = degenerate;
      r.status = CVA_OK;
    }
    *out = r;
  }
  CVA_MARK(23);
}

}  // namespace pf
}  // namespace cva
