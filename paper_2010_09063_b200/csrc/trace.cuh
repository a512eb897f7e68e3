// Device-side phase timestamps for kernel tuning (build with PGB_TRACE=1,
// see build.py). Thread 0 of a CTA writes %globaltimer (ns) into a slot of a
// host-provided buffer; compiled out entirely in normal builds.
#pragma once

#ifdef PGB_TRACE
namespace pgb {
__device__ unsigned long long* g_trace = nullptr;
}
#define PGB_MARK(slot)                                                           \
  do {                                                                           \
    if (::pgb::g_trace && threadIdx.x == 0) {                                    \
      unsigned long long t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
      ::pgb::g_trace[(slot)] = t_;                                               \
    }                                                                            \
  } while (0)
// timestamp from thread `tid` (no-op unless it reaches the mark)
#define PGB_MARK_T(slot, tid)                                                    \
  do {                                                                           \
    if (::pgb::g_trace && threadIdx.x == (tid)) {                                \
      unsigned long long t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
      ::pgb::g_trace[(slot)] = t_;                                               \
    }                                                                            \
  } while (0)
// After a __syncthreads(): BAR.SYNC does not block at issue (the wait is
// deferred to the next dependent instruction), so a timestamp taken right
// after it records the barrier's issue, not its release. A second barrier
// blocks until the first has released.
#define PGB_MARK_BAR(slot) \
  do {                     \
    __syncthreads();       \
    PGB_MARK(slot);        \
  } while (0)
#else
#define PGB_MARK_T(slot, tid) \
  do {                        \
  } while (0)
#define PGB_MARK_BAR(slot) \
  do {                     \
  } while (0)
#define PGB_MARK(slot) \
  do {                 \
  } while (0)
#endif

// slot layout: aggregate CTA b phase p -> kTraceAgg + 8b + p;
//              fused MNIST CTA b phase p -> kTraceFused + 32b + p
#define PGB_TRACE_AGG 0
#define PGB_TRACE_FUSED 40000
#define PGB_FUSED_SLOTS 32
#define PGB_TRACE_SLOTS (40000 + PGB_FUSED_SLOTS * 4096)
