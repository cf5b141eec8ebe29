// trace.h -- profiling builds only (-DKB_TRACE): per-CTA phase timestamps
// (globaltimer, ns) written by thread 0 of each CTA, one table per translation
// unit, read back through kpme_debug_trace_<unit>(kernel, out[4096][10]).
// Slot 9 holds the SM the CTA ran on. Default builds compile every macro to nothing.
#pragma once
#ifdef KB_TRACE
#include <cuda_runtime.h>
namespace kb_trace_ns {
constexpr int kKernels = 4, kCtas = 4096, kSlots = 10;
static __device__ unsigned long long table[kKernels][kCtas][kSlots];
__device__ __forceinline__ void mark(int k, int slot) {
    if (threadIdx.x == 0 && blockIdx.x < kCtas) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        table[k][blockIdx.x][slot] = t;
        if (slot == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            table[k][blockIdx.x][kSlots - 1] = sm;
        }
    }
}
__device__ __forceinline__ void put(int k, int slot, unsigned long long v) {
    if (threadIdx.x == 0 && blockIdx.x < kCtas) table[k][blockIdx.x][slot] = v;
}
}  // namespace kb_trace_ns
#define TRACE_MARK(k, slot) kb_trace_ns::mark(k, slot)
// warp-0 cycle accounting inside a phase
#define TRACE_CLK(t) long long t = clock64()
#define TRACE_ACC(acc, a, b) acc += (b) - (a)
#define TRACE_DECL(acc) long long acc = 0
#define TRACE_PUT(k, slot, v) kb_trace_ns::put(k, slot, (unsigned long long)(v))
#define TRACE_PTR(acc) (&acc)
#define TRACE_READER(unit)                                                                              \
    extern "C" __attribute__((visibility("default"))) int kpme_debug_trace_##unit(int k,               \
                                                                                  unsigned long long* out) { \
        const size_t bytes = sizeof(unsigned long long) * kb_trace_ns::kCtas * kb_trace_ns::kSlots;      \
        return (int)cudaMemcpyFromSymbol(out, kb_trace_ns::table, bytes, bytes * (size_t)k);             \
    }
#else
#define TRACE_MARK(k, slot)
#define TRACE_CLK(t)
#define TRACE_ACC(acc, a, b)
#define TRACE_DECL(acc)
#define TRACE_PUT(k, slot, v)
#define TRACE_PTR(acc) nullptr
#define TRACE_READER(unit)
#endif
