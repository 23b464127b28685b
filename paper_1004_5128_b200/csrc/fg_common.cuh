// Error plumbing, launch constants, bounds checks and PTX helpers shared by every kernel.
// Part of the single translation unit csrc/fg_kernels.cu (included there in order).
#ifndef FG_COMMON_CUH
#define FG_COMMON_CUH

#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point, no -lcuda)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/fgb200.h"
#include "fg_schedule.cuh"

namespace {

thread_local std::string g_last_error;
thread_local int64_t g_launches = 0;  // kernels this thread has launched (fg_kernel_launches)

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return FG_OK;
    return fail(FG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Device-side bounds checks (FG_CHECKS builds only; compute-sanitizer is closed
// on the GPU pool): every global index a kernel derives from its launch
// arguments — history slice, partial-sum row, coefficient row, tensor-map
// coordinate, step column, ψ index — is checked against the buffer it
// addresses, and a violation traps with file/line (scripts/checked_suite.sh runs
// the GPU tests against that build).
#ifdef FG_CHECKS
#define FG_DCHECK(cond)                                                                                   \
    do {                                                                                                  \
        if (!(cond)) {                                                                                    \
            printf("FG_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x,  \
                   (int)threadIdx.x, #cond);                                                              \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define FG_DCHECK(cond) ((void)0)
#endif

constexpr int kThreads = 256;   // 8 warps
#ifndef FG_STEP_MINB
#define FG_STEP_MINB 4
#endif
constexpr int kMinBlocks = FG_STEP_MINB;   // resident CTAs per SM the register budget targets
constexpr int kVec = 2;         // doubles per thread per slice (one 128-bit load)
constexpr int kUnroll = 8;      // slices in flight per thread
constexpr int kChunk = 1024;    // schedule entries staged in shared memory at once
constexpr int kMaxPasses = 32;  // tiles per CTA in persistent mode (dynamic smem)
#ifndef FG_MAX_TBLOCK
#define FG_MAX_TBLOCK 128
#endif
constexpr int kMaxTBlock = FG_MAX_TBLOCK;  // largest temporal-blocking factor (> 32: itemized stages only)
constexpr int kMaxSub = 16;      // most sub-blocks per temporal block (plan->subblock)
constexpr int kMaxDenseTBlock = 32;  // largest factor of the dense block kernel
constexpr int kCoefRow = 36;    // doubles per row of plan->blkcoef_dev (>= kMaxDenseTBlock + 4)

// ---------------------------------------------------------------- PTX helpers ---

// History slices: read once per step, never in L1 (.cg keeps the load coherent at
// L2, which the persistent kernel needs because slices are written mid-launch).
__device__ __forceinline__ double2 ld_stream(const double* p) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ double2 ld_cg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }

__device__ __forceinline__ void st_pair(double* p, double a, double b) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// L2 eviction-priority hints.  The block stage streams the history through L2
// (evict_first); what the latency-bound step chain reads next — the fields, the
// newest history slices, the block's partial sums — is written evict_last so it
// is still in L2 when read (misses would queue behind the stream in HBM).
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t l2_policy_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void st_pair_hint(double* p, double a, double b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b), "l"(pol) : "memory");
}

__device__ __forceinline__ void st_hint1(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ double2 ld_cg2_hint(const double* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Split grid barrier.  arrive: every thread's writes of this CTA are released
// (bar.sync + gpu-scope fence by the arriving thread); wait: acquire, then the
// CTA proceeds.  The counter is monotonic within a launch (reset before it).
__device__ __forceinline__ void grid_arrive(unsigned long long* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
    }
}

__device__ __forceinline__ void grid_wait(const unsigned long long* bar, unsigned long long target) {
    if (threadIdx.x == 0) {
        while (ld_acquire(bar) < target) __nanosleep(40);
        __threadfence();
    }
    __syncthreads();
}

}  // namespace

#endif  // FG_COMMON_CUH
