// trace.cuh -- debug-only per-CTA phase timestamps (make trace -> libhybrid_cuda_trace.so,
// tools/trace_amf.py).  Each translation unit that includes it gets its own buffer and exports its
// reader; no effect in normal builds.
#pragma once
#include <cstdint>

namespace hyb {
namespace {
#ifdef HYB_TRACE
// Debug builds only (make trace): per-CTA phase timestamps, read back with hyb_trace_read.
__device__ unsigned long long g_trace[2 * 1024 * 16];
__device__ __forceinline__ void trace_mark(int kid, int slot) {
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[(kid * 1024 + blockIdx.x) * 16 + slot] = t;
    }
}
#ifndef HYB_TRACE_MASK
#define HYB_TRACE_MASK 3
#endif
#define TRACE(kid, slot)                                  \
    do {                                                  \
        if ((HYB_TRACE_MASK >> (kid)) & 1) trace_mark(kid, slot); \
    } while (0)
#else
#define TRACE(kid, slot) \
    do {                 \
    } while (0)
#endif
}  // namespace
}  // namespace hyb
