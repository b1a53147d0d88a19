// Optional per-phase cycle stamps (build with -DCVA_PHASE_TIMING; used by
// tools/phase_timing.py, never in the shipped library). Thread 0 of each CTA
// records clock64() at phase boundaries into g_cva_prof[blockIdx.x * 64 + k].
#pragma once

#ifdef CVA_PHASE_TIMING
static __device__ long long* g_cva_prof = nullptr;
#define CVA_MARK(k)                                                        \
  do {                                                                     \
    if (threadIdx.x == 0 && g_cva_prof) g_cva_prof[blockIdx.x * 64 + (k)] = clock64(); \
  } while (0)
#else
#define CVA_MARK(k) \
  do {              \
  } while (0)
#endif
