// B200 (sm_100a) kernels and the C ABI of the GL history stepper.
//
// Hot path replaced: /root/reference/pkg/src/fracgrid/solver.py:230-265 (run)
//   → step (:200-227) → history_sum (:162-197), with ψ from coefficients.py:76-92,
//   schedules from schedule.py:70-151 and the stencil of grid.py:88-106.
//
// Design:
//  * fg_step_kernel — the fused time step.  A CTA owns tiles of TP points (one
//    member each).  Per step k:
//      A  schedule of step k built in shared memory (segment table → slice index
//         k-m and coefficient w·ψ_b(m), rounded once exactly like solver.py:190);
//         every history slice with m >= 2 is streamed with 128-bit loads, 8 in
//         flight per thread, fp64 FMA into per-tile partial sums.  When tiles are
//         small the CTA's warps split the entry list S ways and combine in a
//         fixed order (deterministic).
//      -- dependency on step k-1 (grid barrier / griddepcontrol.wait) --
//      C  m = 1 (H[k-1]) and m = 0 (δ^k = stencil(u^k), bit-exact, stored to H[k]),
//         reaction + explicit update in the reference's rounding order, ring
//         pinned to zero, non-finite detection, u^{k+1} (+ snapshot) stored.
//    The same kernel runs one step per launch (fg_step, PDL/graph pipelines) or
//    every step in one cooperative launch with a split arrive/wait grid barrier
//    (FG_RUN_PERSISTENT): a CTA arrives after its C phase and only waits after
//    streaming the next step's A phase, so the barrier latency hides under HBM
//    traffic and there is no per-step launch or tail.  Same arithmetic in every
//    mode → bitwise-identical results.
//  * HBM-bound (0.25 flop/B): no tensor cores; roofline = 8 bytes per term.
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

// ------------------------------------------------------------------- stencil ---
// grid.py:98-105 operation order, each op correctly rounded (no contraction):
//   2D ((((x+ + x-) - 4c) + y+) + y-); 1D (x+ + x-) - 2c; 3D with -6c, y±, z±.

struct Shape {
    int32_t n0, n1, n2;  // C-order extents (unused = 1)
};

template <int NDIM>
__device__ __forceinline__ bool interior(const Shape& sh, int32_t q) {
    if (NDIM == 1) return q > 0 && q < sh.n0 - 1;
    if (NDIM == 2) {
        const int32_t j = q / sh.n1, l = q - j * sh.n1;
        return j > 0 && j < sh.n0 - 1 && l > 0 && l < sh.n1 - 1;
    }
    const int32_t plane = sh.n1 * sh.n2;
    const int32_t i0 = q / plane, r = q - i0 * plane;
    const int32_t i1 = r / sh.n2, i2 = r - i1 * sh.n2;
    return i0 > 0 && i0 < sh.n0 - 1 && i1 > 0 && i1 < sh.n1 - 1 && i2 > 0 && i2 < sh.n2 - 1;
}

// Interior flags of the point pair (q, q+1) from one coordinate decomposition
// (the per-point `interior` costs an integer division per axis).
template <int NDIM>
__device__ __forceinline__ void interior_pair(const Shape& sh, int32_t q, bool& in0, bool& in1) {
    if (NDIM == 1) {
        in0 = q > 0 && q < sh.n0 - 1;
        in1 = q + 1 > 0 && q + 1 < sh.n0 - 1;
    } else if (NDIM == 2) {
        const int32_t j = q / sh.n1, l = q - j * sh.n1;
        const bool row = j > 0 && j < sh.n0 - 1;
        in0 = row && l > 0 && l < sh.n1 - 1;
        // q+1 in the same row unless l is the last column (then it is a ring point)
        in1 = row && l + 1 < sh.n1 - 1;
    } else {
        const int32_t plane = sh.n1 * sh.n2;
        const int32_t i0 = q / plane, r = q - i0 * plane;
        const int32_t i1 = r / sh.n2, i2 = r - i1 * sh.n2;
        const bool line = i0 > 0 && i0 < sh.n0 - 1 && i1 > 0 && i1 < sh.n1 - 1;
        in0 = line && i2 > 0 && i2 < sh.n2 - 1;
        in1 = line && i2 + 1 < sh.n2 - 1;
    }
}

// u is read through L2 (.cg): in the persistent kernel the field buffers are
// rewritten every other step, so an L1 copy could be stale.
template <int NDIM>
__device__ __forceinline__ double delta_at(const double* __restrict__ u, const Shape& sh, int32_t q,
                                           double c) {
    if (!interior<NDIM>(sh, q)) return 0.0;
    if (NDIM == 1) {
        return __dsub_rn(__dadd_rn(ld_cg(u + q + 1), ld_cg(u + q - 1)), __dmul_rn(2.0, c));
    } else if (NDIM == 2) {
        const int32_t sx = sh.n1;
        double r = __dadd_rn(ld_cg(u + q + sx), ld_cg(u + q - sx));
        r = __dsub_rn(r, __dmul_rn(4.0, c));
        r = __dadd_rn(r, ld_cg(u + q + 1));
        return __dadd_rn(r, ld_cg(u + q - 1));
    } else {
        const int32_t sy = sh.n2, sx = sh.n1 * sh.n2;
        double r = __dadd_rn(ld_cg(u + q + sx), ld_cg(u + q - sx));
        r = __dsub_rn(r, __dmul_rn(6.0, c));
        r = __dadd_rn(r, ld_cg(u + q + sy));
        r = __dadd_rn(r, ld_cg(u + q - sy));
        r = __dadd_rn(r, ld_cg(u + q + 1));
        return __dadd_rn(r, ld_cg(u + q - 1));
    }
}

// δ of the point pair (q, q+1) (q even) with every neighbour load issued before
// any arithmetic, so the step's critical path holds one L2 round trip: the
// other rows/planes are read as 128-bit pairs when their stride is even, the
// outer x-neighbours u[q-1] (point q) and u[q+2] (point q+1) singly, and each
// δ is formed in the grid.py:98-105 order exactly like delta_in.
__device__ __forceinline__ double2 ld_pair_any(const double* p, bool even) {
    return even ? ld_cg2(p) : make_double2(ld_cg(p), ld_cg(p + 1));
}

template <int NDIM>
__device__ __forceinline__ void delta_pair(const double* __restrict__ u, const Shape& sh, int32_t q, double u0,
                                           double u1, bool in0, bool in1, double& d0, double& d1) {
    const bool any = in0 || in1;
    const double lf = in0 ? ld_cg(u + q - 1) : 0.0;  // u[q-1] (q > 0 when in0)
    const double rt = in1 ? ld_cg(u + q + 2) : 0.0;  // u[q+2]
    double2 xp = make_double2(0.0, 0.0), xm = xp, yp = xp, ym = xp;
    if (NDIM >= 2 && any) {
        const int32_t sx = NDIM == 2 ? sh.n1 : sh.n1 * sh.n2;
        const bool ev = (sx & 1) == 0;
        xp = ld_pair_any(u + q + sx, ev);
        xm = ld_pair_any(u + q - sx, ev);
        if (NDIM == 3) {
            const int32_t sy = sh.n2;
            const bool evy = (sy & 1) == 0;
            yp = ld_pair_any(u + q + sy, evy);
            ym = ld_pair_any(u + q - sy, evy);
        }
    }
    if (NDIM == 1) {
        d0 = in0 ? __dsub_rn(__dadd_rn(u1, lf), __dmul_rn(2.0, u0)) : 0.0;
        d1 = in1 ? __dsub_rn(__dadd_rn(rt, u0), __dmul_rn(2.0, u1)) : 0.0;
    } else if (NDIM == 2) {
        double r0 = __dsub_rn(__dadd_rn(xp.x, xm.x), __dmul_rn(4.0, u0));
        r0 = __dadd_rn(__dadd_rn(r0, u1), lf);
        double r1 = __dsub_rn(__dadd_rn(xp.y, xm.y), __dmul_rn(4.0, u1));
        r1 = __dadd_rn(__dadd_rn(r1, rt), u0);
        d0 = in0 ? r0 : 0.0;
        d1 = in1 ? r1 : 0.0;
    } else {
        double r0 = __dsub_rn(__dadd_rn(xp.x, xm.x), __dmul_rn(6.0, u0));
        r0 = __dadd_rn(__dadd_rn(r0, yp.x), ym.x);
        r0 = __dadd_rn(__dadd_rn(r0, u1), lf);
        double r1 = __dsub_rn(__dadd_rn(xp.y, xm.y), __dmul_rn(6.0, u1));
        r1 = __dadd_rn(__dadd_rn(r1, yp.y), ym.y);
        r1 = __dadd_rn(__dadd_rn(r1, rt), u0);
        d0 = in0 ? r0 : 0.0;
        d1 = in1 ? r1 : 0.0;
    }
}

// ---------------------------------------------------------------- fused step ---

struct StepArgs {
    double* u[2];          // ping-pong fields, u^k in u[k & 1]
    double* snap;          // single-step mode: explicit snapshot target (nullable)
    double* pool;          // multi-step mode: snapshot pool
    const int32_t* snap_slot;  // multi-step mode: pool slot of step `done` or -1 (nullable)
    double* H;
    const double* psi;
    const double* decay;
    const double* diffuse;
    const double* dt;
    const int64_t* horizon;
    int64_t* status;
    unsigned long long* bar;
    int64_t k0, k1;        // steps [k0, k1)
    int64_t slice_stride;  // B*ms
    int64_t ms;
    int64_t psi_stride;
    int64_t base;
    int64_t hz_max;        // max short-memory horizon over members
    double vmax, km;
    Shape sh;
    int32_t n_m;
    int32_t kind;
    int32_t tpm;           // tiles per member
    int32_t total_tiles;
    int32_t passes;        // tiles per CTA
    int32_t pdl_wait;      // single-step: launched as a programmatic dependent
    int32_t pdl_trigger;   // single-step: let the next step launch early
    int32_t m0_from_history;
    int32_t blocked;       // temporal blocking: slices t < kb0 come from P
    int64_t kb0;           // first step of the current block
    const double* P;       // [tblock][B*ms] block partial sums (fg_block_kernel)
    int64_t h_slices;      // history capacity (bounds checks)
    int32_t tblock;        // rows of P (bounds checks)
    int32_t recent_first;  // recent slices loaded evict_first (large fields)
    // blocked single-step launches: the entries of step k's schedule with
    // 2 <= m <= k-kb0 (the only ones a blocked step still sums itself), host-
    // evaluated so the step kernel builds no schedule: offsets ascending, weights,
    // and the weight of m = 1.  Multi-step launches build them on the device.
    int32_t rn;
    int32_t rw1;
    uint8_t rm[kMaxTBlock];
    uint8_t rwt[kMaxTBlock];
    // single member with plan->psi_host: the coefficients themselves (w·ψ(m),
    // rounded once on the host exactly like __dmul_rn), so the step kernel does
    // no ψ loads and no conversions on its critical path
    int32_t has_rc;
    double rc0, rc1;
    double rc[kMaxTBlock];
};

// Recent entries of step k in block kb0 (host and device): offsets 2 <= m <= bb
// ascending with their weights, and the weight of m = 1 (0 if absent or bb = 0).
FG_HD int recent_list(int kind, int64_t k, int64_t kb0, int64_t base, int64_t hz, uint8_t* rm, uint8_t* rwt,
                      int32_t* w1) {
    FgSeg segs[FG_MAX_SEGS];
    const int64_t bb = k - kb0;
    const int n = fg_segments(kind, k, base, hz, segs);
    int c = 0;
    *w1 = 0;
    for (int i = 0; i < n; ++i) {
        const int64_t st = segs[i].stride;
        for (int64_t j = 0; j < segs[i].count; ++j) {
            const int64_t m = segs[i].m0 + j * st;
            if (m > bb) break;
            if (m == 1) *w1 = (int32_t)st;
            if (m >= 2) {
                rm[c] = (uint8_t)m;
                rwt[c] = (uint8_t)st;
                ++c;
            }
        }
    }
    return c;
}

// Number of schedule entries with offset m <= mmax (entries ascend in m).
__device__ __forceinline__ int64_t entries_upto(const FgSeg* s, int n, int64_t mmax) {
    int64_t c = 0;
    for (int i = 0; i < n; ++i) {
        if (s[i].m0 > mmax) break;
        const int64_t in = (mmax - s[i].m0) / s[i].stride + 1;
        c += in < s[i].count ? in : s[i].count;
    }
    return c;
}


// General A phase (unblocked steps): schedule of step k in shared memory, every
// entry with m >= 2 streamed into s_acc; also returns the schedule length and
// the weight of m = 1 for phase C.  Its shared staging exists only in the
// kernels that call it (not in the temporal-blocking variant).
template <int S>
__device__ __forceinline__ void general_a_phase(const StepArgs& a, int64_t k, double2* s_acc, int64_t& len,
                                                int64_t& w1, bool& has_m1) {
    constexpr int kCols = (kThreads / 32) / S;
    constexpr int TP = kCols * 32 * kVec;
    constexpr int kLanes = kCols * 32;
    __shared__ FgSeg segs[FG_MAX_SEGS];
    __shared__ int64_t seg_first[FG_MAX_SEGS + 1];
    __shared__ int s_nseg;
    __shared__ int64_t s_lim;
    __shared__ int32_t s_t[kChunk];
    __shared__ int32_t s_w[kChunk];
    __shared__ double s_c[kChunk];
    __shared__ double2 s_part[S > 1 ? (S - 1) * kLanes : 1];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int col = warp % kCols, split = warp / kCols;
    const int slot = col * 32 + lane;
    const int G = gridDim.x;
    const int64_t bb = k - a.kb0;
    // ================= A: schedule + old slices (m >= 2) =================
    for (int i = tid; i < a.passes * kLanes; i += kThreads) s_acc[i] = make_double2(0.0, 0.0);
    if (tid == 0) {
        int n = fg_segments(a.kind, k, a.base, a.hz_max, segs);
        int64_t acc = 0;
        for (int i = 0; i < n; ++i) {
            seg_first[i] = acc;
            acc += segs[i].count;
        }
        seg_first[n] = acc;
        s_nseg = n;
        // temporal blocking: entries with m > bb (slices t < kb0) are already
        // summed into P by fg_block_kernel; only m <= bb remain for this step
        s_lim = a.blocked ? entries_upto(segs, n, k - a.kb0) : acc;
    }
    __syncthreads();
    const int nseg = s_nseg;
    len = seg_first[nseg];
    const int64_t lim = s_lim;
    // entry 0 is m = 0 (every schedule opens with the dense window); entry 1 is
    // m = 1 whenever the schedule has it.  Both depend on step k-1's output
    // and are summed in phase C; entries from 2 on read slices t <= k-2.
    const int64_t m1 = len >= 2 ? (segs[0].count >= 2 ? segs[0].m0 + segs[0].stride : segs[1].m0) : 0;
    w1 = len >= 2 ? (segs[0].count >= 2 ? segs[0].stride : segs[1].stride) : 0;
    has_m1 = len >= 2 && m1 == 1 && (!a.blocked || bb >= 1);
    const int64_t old = (len >= 2 && m1 == 1) ? 2 : 1;

    for (int64_t c0 = old; c0 < lim; c0 += kChunk) {
        const int cn = (int)((lim - c0) < kChunk ? (lim - c0) : kChunk);
        for (int e = tid; e < cn; e += kThreads) {
            const int64_t j = c0 + e;
            int si = 0;
            while (si + 1 < nseg && seg_first[si + 1] <= j) ++si;
            const int64_t m = segs[si].m0 + (j - seg_first[si]) * segs[si].stride;
            FG_DCHECK(m >= 2 && m <= k && k < a.h_slices);
            s_t[e] = (int32_t)(k - m);
            s_w[e] = (int32_t)segs[si].stride;
        }
        int64_t cur_member = -1;
        for (int p = 0; p < a.passes; ++p) {
            const int tile = blockIdx.x + p * G;
            if (tile >= a.total_tiles) break;
            const int64_t b = tile / a.tpm;
            if (b != cur_member) {  // coefficients c = w·ψ_b(m) for this member
                __syncthreads();
                const double* psi_b = a.psi + b * a.psi_stride;
                for (int e = tid; e < cn; e += kThreads)
                    s_c[e] = __dmul_rn((double)s_w[e], __ldg(psi_b + (k - s_t[e])));
                __syncthreads();
                cur_member = b;
            }
            int64_t len_b = a.kind == 1 ? ((a.horizon[b] < k ? a.horizon[b] : k) + 1) : len;
            if (len_b > lim) len_b = lim;
            const int cnb = (int)(len_b <= c0 ? 0 : (len_b - c0 < cn ? len_b - c0 : cn));
            const int32_t q = (tile % a.tpm) * TP + col * 64 + lane * kVec;
            double acc0 = 0.0, acc1 = 0.0;
            if (q < a.n_m) {
                const double* hbase = a.H + b * a.ms + q;
                for (int e0 = split; e0 < cnb; e0 += S * kUnroll) {
                    double2 v[kUnroll];
                    double c[kUnroll];
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        const int e = e0 + u * S;
                        if (e < cnb) {
                            v[u] = ld_stream(hbase + (int64_t)s_t[e] * a.slice_stride);
                            c[u] = s_c[e];
                        } else {
                            v[u] = make_double2(0.0, 0.0);
                            c[u] = 0.0;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        acc0 = fma(c[u], v[u].x, acc0);
                        acc1 = fma(c[u], v[u].y, acc1);
                    }
                }
            }
            if (S > 1) {
                if (split > 0) s_part[(split - 1) * kLanes + slot] = make_double2(acc0, acc1);
                __syncthreads();
                if (split == 0) {
#pragma unroll
                    for (int s = 1; s < S; ++s) {
                        const double2 pp = s_part[(s - 1) * kLanes + slot];
                        acc0 = __dadd_rn(acc0, pp.x);
                        acc1 = __dadd_rn(acc1, pp.y);
                    }
                }
                __syncthreads();
            }
            if (split == 0) {
                double2& r = s_acc[p * kLanes + slot];
                r.x = __dadd_rn(r.x, acc0);
                r.y = __dadd_rn(r.y, acc1);
            }
        }
        __syncthreads();  // s_t / s_w / s_c are refilled by the next chunk
    }
}

// BLK: temporal-blocking variant (S = 1): the recent-slice A phase only, no
// shared staging, so two of its CTAs fit next to two block-kernel CTAs per SM.
template <int NDIM, int REACT, int S, bool BLK>
__global__ void __launch_bounds__(kThreads, kMinBlocks) fg_step_kernel(const __grid_constant__ StepArgs a) {
    constexpr int kCols = (kThreads / 32) / S;   // warps across a tile
    constexpr int TP = kCols * 32 * kVec;        // points per tile
    constexpr int kLanes = kCols * 32;           // split-0 threads (one point pair each)
    extern __shared__ double2 s_acc[];  // [passes][kLanes] partial sums of the A phase

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int col = warp % kCols, split = warp / kCols;
    const int slot = col * 32 + lane;
    const int G = gridDim.x;
    const bool multi = a.k1 - a.k0 > 1;

    for (int64_t k = a.k0; k < a.k1; ++k) {
        const int64_t bb = k - a.kb0;
        int64_t len, w1;   // schedule length (kinds 0/2), weight of m = 1
        bool has_m1;
        if constexpr (BLK) {
            // ====== A (temporal blocking): recent slices 2 <= m <= bb only ======
            // Everything older is in P[bb].  Single-step launches get the recent
            // entries from the host (no schedule, no shared staging, no CTA
            // barrier); multi-step launches build them here.  Same entry order
            // and rounding as the general path.
            __shared__ uint8_t s_rm[kMaxTBlock], s_rwt[kMaxTBlock];
            __shared__ int32_t s_rn, s_w1;
            const uint8_t* rm = a.rm;
            const uint8_t* rwt = a.rwt;
            const double* rcoef = a.has_rc ? a.rc : nullptr;
            int rn = a.rn;
            w1 = a.rw1;
            if (multi) {
                if (tid == 0) s_rn = recent_list(a.kind, k, a.kb0, a.base, a.hz_max, s_rm, s_rwt, &s_w1);
                __syncthreads();
                rm = s_rm;
                rwt = s_rwt;
                rcoef = nullptr;
                rn = s_rn;
                w1 = s_w1;
            }
            has_m1 = w1 != 0;
#ifdef FG_DBG_NO_RECENT  // timing experiment only: drop the recent sum (wrong results)
            rn = 0;
#endif
            len = k + 1;  // only used for the m = 1 test below (k >= bb >= 1)
            for (int p = 0; p < a.passes; ++p) {
                const int tile = blockIdx.x + p * G;
                if (tile >= a.total_tiles) break;
                const int64_t b = tile / a.tpm;
                const int32_t q = (tile % a.tpm) * TP + col * 64 + lane * kVec;
                double acc0 = 0.0, acc1 = 0.0;
                // P[bb] (slices t < kb0) is final before the block's first step
                // starts: its load is issued first and added after the recent sum,
                // all before the dependency wait (same order as the unblocked path)
                const double2 pb = q < a.n_m ? ld_cg2_hint(a.P + bb * a.slice_stride + b * a.ms + q, l2_policy_first())
                                             : make_double2(0.0, 0.0);  // its only read
                FG_DCHECK(bb >= 0 && bb < a.tblock && k < a.h_slices && rn <= bb);
                if (q < a.n_m && rn > 0) {
                    const uint64_t pol_drop = a.recent_first ? l2_policy_first() : l2_policy_normal();
                    const double* hbase = a.H + b * a.ms + q + k * a.slice_stride;
                    const double* psi_b = a.psi + b * a.psi_stride;
                    const int64_t mmax = a.kind == 1 ? (a.horizon[b] < bb ? a.horizon[b] : bb) : bb;
#ifndef FG_STEP_KR
#define FG_STEP_KR 5
#endif
                    constexpr int kR = REACT ? FG_STEP_KR - 1 : FG_STEP_KR;  // recent slices in flight per round (no spills)
#pragma unroll 1
                    // entries oldest first (descending m): the fused pair kernel must
                    // add the newest ones after its dependency wait, in the same order
                    for (int e0 = 0; e0 < rn; e0 += kR) {
                        double2 v[kR];
                        double c[kR];
#pragma unroll
                        for (int u = 0; u < kR; ++u) {
                            const int e = rn - 1 - (e0 + u);
                            const int m = e >= 0 ? rm[e] : 0;
                            const bool on = e >= 0 && m <= mmax;
                            FG_DCHECK(!on || (m >= 2 && m <= k));
                            if (on) {
                                // large fields: evict_first — keeping even the newest slices in
                                // L2 (offsets <= 3, 5 or 9 evict_last) measured slower than
                                // streaming them (c4-adaptive 589 vs 599-610 ms); small fields'
                                // recent slices stay in L2 (c2)
                                v[u] = ld_cg2_hint(hbase - (int64_t)m * a.slice_stride, pol_drop);
                                c[u] = rcoef ? rcoef[e] : __dmul_rn((double)rwt[e], __ldg(psi_b + m));
                            } else {
                                v[u] = make_double2(0.0, 0.0);
                                c[u] = 0.0;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kR; ++u) {
                            acc0 = fma(c[u], v[u].x, acc0);
                            acc1 = fma(c[u], v[u].y, acc1);
                        }
                    }
                }
                s_acc[p * kLanes + slot] =
                    make_double2(__dadd_rn(__dadd_rn(0.0, acc0), pb.x), __dadd_rn(__dadd_rn(0.0, acc1), pb.y));
            }
        } else {
            general_a_phase<S>(a, k, s_acc, len, w1, has_m1);
        }

        // ================= dependency on step k-1 =================
        if (multi) {
            if (k > a.k0) grid_wait(a.bar, (unsigned long long)(k - a.k0) * (unsigned long long)G);
        } else {
            if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
            // step k-1 is complete, so every slice t <= k-1 is final: let step k+1
            // start its A phase in the slots this grid frees
            if (a.pdl_trigger) asm volatile("griddepcontrol.launch_dependents;");
        }
        // u^j non-finite for some j <= k: this step must not run.  The flag is
        // loaded now but tested only before the stores, so its L2 round trip
        // overlaps the C-phase loads.  A flag for step k+1 raised during this
        // step's C phase by another CTA is ignored, so every CTA leaves at the
        // same step (no CTA can strand the others at the barrier).
        const bool live = *(volatile const int64_t*)a.status > k;

        // ================= C: m = 1, m = 0, update =================
        const uint64_t keep = l2_policy_last(), drop = l2_policy_first();
        const double* u_in = a.u[k & 1];
        double* u_out = a.u[(k + 1) & 1];
        double* snap = a.snap;
        if (a.snap_slot) {  // persistent launches: snapshot slot of step k+1 from the map
            const int32_t sl = a.snap_slot[k + 1];
            snap = sl >= 0 ? a.pool + (int64_t)sl * a.slice_stride : nullptr;
        }
        if (split == 0) {
            for (int p = 0; p < a.passes; ++p) {
                const int tile = blockIdx.x + p * G;
                if (tile >= a.total_tiles) break;
                const int64_t b = tile / a.tpm;
                const int32_t q = (tile % a.tpm) * TP + col * 64 + lane * kVec;
                if (q >= a.n_m) continue;
                const int64_t moff = b * a.ms + q;
                const double* ub = u_in + b * a.ms;
                const double* psi_b = a.psi + b * a.psi_stride;
                FG_DCHECK(k < a.h_slices && k < a.psi_stride && q + 1 < a.ms + 1 && b < a.slice_stride / a.ms);
                // every load of the C phase is issued before any arithmetic or
                // store (one L2 round trip on the step chain's critical path)
                const int64_t len_b = a.kind == 1 ? ((a.horizon[b] < k ? a.horizon[b] : k) + 1) : len;
                const bool m1 = has_m1 && len_b >= 2;
                const double2 h1 = m1 ? ld_cg2(a.H + (k - 1) * a.slice_stride + moff) : make_double2(0.0, 0.0);
                const double2 pb = (!BLK && a.blocked) ? ld_cg2_hint(a.P + bb * a.slice_stride + moff, drop)
                                                       : make_double2(0.0, 0.0);
                const double2 uu = ld_cg2(ub + q);
                const double u0 = uu.x, u1 = uu.y;
                bool in0, in1;
                interior_pair<NDIM>(a.sh, q, in0, in1);
                in1 = in1 && q + 1 < a.n_m;
                double d0, d1;
                if (a.m0_from_history) {
                    const double2 h = ld_cg2(a.H + k * a.slice_stride + moff);
                    d0 = h.x;
                    d1 = h.y;
                } else {
                    delta_pair<NDIM>(ub, a.sh, q, u0, u1, in0, in1, d0, d1);
                }
                const double2 part = s_acc[p * kLanes + slot];
                double acc0 = part.x, acc1 = part.y;
                if (!BLK && a.blocked) {  // slices t < kb0 (the BLK kernel added them before the wait)
                    acc0 = __dadd_rn(acc0, pb.x);
                    acc1 = __dadd_rn(acc1, pb.y);
                }
                const bool host_c = BLK && a.has_rc && !multi;  // single-member coefficients, precomputed
                if (m1) {
                    const double c1 = host_c ? a.rc1 : __dmul_rn((double)w1, __ldg(psi_b + 1));
                    acc0 = fma(c1, h1.x, acc0);
                    acc1 = fma(c1, h1.y, acc1);
                }
                const double c0 = host_c ? a.rc0 : __ldg(psi_b);  // w_0 * ψ(0) = 1 * 1
                acc0 = fma(c0, d0, acc0);
                acc1 = fma(c0, d1, acc1);

                // solver.py:215-226 rounding order, ring pinned, non-finite check
                const double diffuse = a.diffuse[b];
                double n0, n1;
                if (REACT == 0) {
                    const double decay = a.decay[b];
                    n0 = __dadd_rn(__dmul_rn(u0, decay), __dmul_rn(diffuse, acc0));
                    n1 = __dadd_rn(__dmul_rn(u1, decay), __dmul_rn(diffuse, acc1));
                } else {
                    const double dt = a.dt[b];
                    const double f0 = __ddiv_rn(__dmul_rn(-a.vmax, u0), __dadd_rn(a.km, u0));
                    const double f1 = __ddiv_rn(__dmul_rn(-a.vmax, u1), __dadd_rn(a.km, u1));
                    n0 = __dadd_rn(__dadd_rn(u0, __dmul_rn(dt, f0)), __dmul_rn(diffuse, acc0));
                    n1 = __dadd_rn(__dadd_rn(u1, __dmul_rn(dt, f1)), __dmul_rn(diffuse, acc1));
                }
                if (!in0) n0 = 0.0;
                if (!in1) n1 = 0.0;
                if (!live) break;
                if (!a.m0_from_history) st_pair_hint(a.H + k * a.slice_stride + moff, d0, d1, keep);
                if (!isfinite(n0) || !isfinite(n1))
                    atomicMin(reinterpret_cast<long long*>(a.status), (long long)(k + 1));
                st_pair_hint(u_out + moff, n0, n1, keep);
                if (snap) st_pair_hint(snap + moff, n0, n1, drop);
            }
        }
        if (!live) return;  // uniform: every thread read the same flag
        if (multi) grid_arrive(a.bar);
    }
}

// ------------------------------------------------------- fused step pairs ---
// Steps k and k+1 of a temporal block in one launch (1D and 2D fields): a CTA
// computes step k on its tile plus a halo of R points each side (R = 1 in 1D,
// one row in 2D) from u^k staged in shared memory, then step k+1 on its tile
// from those values, so the step chain pays one kernel boundary and one L2
// round trip per two steps.  The halo points' values are recomputed with the
// very same arithmetic as by their owning CTA (bit-identical results).
// Before the dependency wait only slices written two launches back are read:
// step k's recent entries with m >= 3 and step k+1's with m >= 4 (oldest
// first, the order the single-step kernel uses); m = 2 (step k) and m = 3, 2
// (step k+1) and the m = 1 terms are added after it.
// u buffers: the pair reads u^k from `u_in`, writes u^{k+1} of its tile to the
// parity buffer u[(k+1) & 1] (the divergence report reads it) and u^{k+2} to
// `u_out`, which no CTA of the launch reads: pairs alternate between a library
// scratch buffer and the parity buffer u[k & 1], and run in even numbers so the
// field is back in its parity buffer after each sequence.  *u3_step records
// which step's field sits in the scratch buffer (fg_u3_fixup_kernel).
// Recent list of one blocked step (the pair kernel's second step).
struct RecentRow {
    int32_t rn, rw1;
    double rc0, rc1;
    uint8_t rm[kMaxTBlock];
    uint8_t rwt[kMaxTBlock];
    double rc[kMaxTBlock];
};

struct PairArgs {
    StepArgs s;                // step k: shared fields, recent list, P (block kb0)
    RecentRow r2;              // step k+1's recent list
    const double* u_in;        // u^k
    double* u_mid;             // u^{k+1} (own tile) = u[(k+1) & 1]
    double* u_out;             // u^{k+2}
    double* snap1;             // snapshot of u^{k+1} (or NULL)
    double* snap2;             // snapshot of u^{k+2} (or NULL)
    int64_t* u3_step;
    int32_t writes_u3;
};
constexpr int kPairTile = 512;                 // points per CTA (as the blocked step kernel)
constexpr int kPairMaxHalo = 256;              // R <= 256
constexpr int kPairNP = (kPairTile + 2 * kPairMaxHalo + kThreads - 1) / kThreads;  // extended points per thread

template <int NDIM, int REACT>
__global__ void __launch_bounds__(kThreads, 2) fg_step2_kernel(const __grid_constant__ PairArgs A) {
    const StepArgs& a = A.s;
    extern __shared__ double sm2[];
    const int tid = threadIdx.x;
    const int tile = blockIdx.x;
    const int64_t b = tile / a.tpm;
    const int32_t q0 = (tile % a.tpm) * kPairTile;
    const int32_t n = a.n_m;
    const int32_t R = NDIM == 1 ? 1 : a.sh.n1;
    const int32_t o_lo = q0, o_hi = q0 + kPairTile < n ? q0 + kPairTile : n;
    const int32_t lo = o_lo - R > 0 ? o_lo - R : 0, hi = o_hi + R < n ? o_hi + R : n;    // extended range E
    const int32_t ulo = lo - R > 0 ? lo - R : 0, uhi = hi + R < n ? hi + R : n;          // u^k staged
    double* su = sm2;                                  // [uhi - ulo] u^k
    double* su1 = sm2 + (kPairTile + 4 * kPairMaxHalo);  // [hi - lo]  u^{k+1}
    const int64_t k = a.k0, bb = k - a.kb0;
    const int64_t ss = a.slice_stride;
    const double* Hm = a.H + b * a.ms;                 // member's slice rows
    const double* psi_b = a.psi + b * a.psi_stride;
    const bool hc = a.has_rc != 0;
    const RecentRow& r2 = A.r2;
    auto coef1 = [&](int e) { return hc ? a.rc[e] : __dmul_rn((double)a.rwt[e], __ldg(psi_b + a.rm[e])); };
    auto coef2 = [&](int e) { return hc ? r2.rc[e] : __dmul_rn((double)r2.rwt[e], __ldg(psi_b + r2.rm[e])); };

    // ---- A (before the dependency): P rows and the recent entries two launches old
    double acc1[kPairNP], acc2[kPairNP], pb1[kPairNP], pb2[kPairNP];
#pragma unroll
    for (int j = 0; j < kPairNP; ++j) {
        const int32_t p = lo + tid + j * kThreads;
        acc1[j] = acc2[j] = pb1[j] = pb2[j] = 0.0;
        if (p < hi) pb1[j] = ld_cg(a.P + bb * ss + b * a.ms + p);
        if (p >= o_lo && p < o_hi) pb2[j] = ld_cg(a.P + (bb + 1) * ss + b * a.ms + p);
    }
    // rounds of kPR entries x kPairNP points in flight (oldest first); padding
    // entries add fma(0, 0, acc), which leaves every nonzero partial unchanged
    // and is normalised away by the __dadd_rn(0, .) below, as in the step kernel
    constexpr int kPR = 3;
    {
        int n1 = 0;  // step k: entries m >= 3 are the last n1 of the list
        while (n1 < a.rn && a.rm[a.rn - 1 - n1] >= 3) ++n1;
        for (int e0 = 0; e0 < n1; e0 += kPR) {
            double v[kPR][kPairNP], c[kPR];
#pragma unroll
            for (int u = 0; u < kPR; ++u) {
                const int e = a.rn - 1 - (e0 + u);
                const bool on = e0 + u < n1;
                c[u] = on ? coef1(e) : 0.0;
                const double* h = Hm + (k - (on ? a.rm[e] : 0)) * ss;
#pragma unroll
                for (int j = 0; j < kPairNP; ++j) {
                    const int32_t p = lo + tid + j * kThreads;
                    v[u][j] = (on && p < hi) ? ld_cg(h + p) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kPR; ++u)
#pragma unroll
                for (int j = 0; j < kPairNP; ++j) acc1[j] = fma(c[u], v[u][j], acc1[j]);
        }
        int n2 = 0;  // step k+1: entries m >= 4
        while (n2 < r2.rn && r2.rm[r2.rn - 1 - n2] >= 4) ++n2;
        for (int e0 = 0; e0 < n2; e0 += kPR) {
            double v[kPR][kPairNP / 2], c[kPR];
#pragma unroll
            for (int u = 0; u < kPR; ++u) {
                const int e = r2.rn - 1 - (e0 + u);
                const bool on = e0 + u < n2;
                c[u] = on ? coef2(e) : 0.0;
                const double* h = Hm + (k + 1 - (on ? r2.rm[e] : 0)) * ss;
#pragma unroll
                for (int j = 0; j < kPairNP; ++j) {
                    const int32_t p = lo + tid + j * kThreads;
                    const bool own = p >= o_lo && p < o_hi;
                    if (j < kPairNP / 2) v[u][j] = 0.0;
                    if (own) v[u][j % (kPairNP / 2)] = on ? ld_cg(h + p) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kPR; ++u)
#pragma unroll
                for (int j = 0; j < kPairNP; ++j) {
                    const int32_t p = lo + tid + j * kThreads;
                    if (p >= o_lo && p < o_hi) acc2[j] = fma(c[u], v[u][j % (kPairNP / 2)], acc2[j]);
                }
        }
    }

    // ---- dependency on the previous launch (steps k-2, k-1)
    if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.pdl_trigger) asm volatile("griddepcontrol.launch_dependents;");
    const bool live = *(volatile const int64_t*)a.status > k;

    // ---- C: stage u^k, then the newest history terms
    const double* ub = A.u_in + b * a.ms;
    for (int32_t i = tid; i < uhi - ulo; i += kThreads) su[i] = ld_cg(ub + ulo + i);
    double h1[kPairNP], h2[kPairNP];
#pragma unroll
    for (int j = 0; j < kPairNP; ++j) {
        const int32_t p = lo + tid + j * kThreads;
        h1[j] = h2[j] = 0.0;
        if (p < hi) {
            if (k >= 1) h1[j] = ld_cg(Hm + (k - 1) * ss + p);
            if (k >= 2) h2[j] = ld_cg(Hm + (k - 2) * ss + p);
        }
    }
    __syncthreads();
    // entries m = 3 / 2 of a list (ascending, so they are the first ones)
    int e1_2 = -1, e2_2 = -1, e2_3 = -1;
    for (int e = 0; e < a.rn && a.rm[e] <= 3; ++e)
        if (a.rm[e] == 2) e1_2 = e;
    for (int e = 0; e < r2.rn && r2.rm[e] <= 3; ++e) {
        if (r2.rm[e] == 2) e2_2 = e;
        if (r2.rm[e] == 3) e2_3 = e;
    }
    const int64_t len_k = k + 1;  // kinds full/adaptive (short memory never pairs)
    const double decay = a.decay[b], diffuse = a.diffuse[b];
    double d1[kPairNP], u1[kPairNP];
    // step k on E
#pragma unroll
    for (int j = 0; j < kPairNP; ++j) {
        const int32_t p = lo + tid + j * kThreads;
        d1[j] = u1[j] = 0.0;
        if (p >= hi) continue;
        double acc = acc1[j];
        if (e1_2 >= 0) acc = fma(coef1(e1_2), h2[j], acc);
        acc = __dadd_rn(__dadd_rn(0.0, acc), pb1[j]);
        if (a.rw1 != 0 && len_k >= 2) acc = fma(hc ? a.rc1 : __dmul_rn((double)a.rw1, __ldg(psi_b + 1)), h1[j], acc);
        const bool in = interior<NDIM>(a.sh, p);
        const double c = su[p - ulo];
        double d = 0.0;
        if (in) {
            if (NDIM == 1) {
                d = __dsub_rn(__dadd_rn(su[p + 1 - ulo], su[p - 1 - ulo]), __dmul_rn(2.0, c));
            } else {
                double r = __dadd_rn(su[p + R - ulo], su[p - R - ulo]);
                r = __dsub_rn(r, __dmul_rn(4.0, c));
                r = __dadd_rn(r, su[p + 1 - ulo]);
                d = __dadd_rn(r, su[p - 1 - ulo]);
            }
        }
        acc = fma(hc ? a.rc0 : __ldg(psi_b), d, acc);
        double nu;
        if (REACT == 0) {
            nu = __dadd_rn(__dmul_rn(c, decay), __dmul_rn(diffuse, acc));
        } else {
            const double f = __ddiv_rn(__dmul_rn(-a.vmax, c), __dadd_rn(a.km, c));
            nu = __dadd_rn(__dadd_rn(c, __dmul_rn(a.dt[b], f)), __dmul_rn(diffuse, acc));
        }
        if (!in) nu = 0.0;
        d1[j] = d;
        u1[j] = nu;
        su1[p - lo] = nu;
    }
    __syncthreads();
    if (!live) return;
    const uint64_t keep = l2_policy_last(), drop = l2_policy_first();
    const int64_t moff = b * a.ms;
    // step k+1 on the tile
#pragma unroll
    for (int j = 0; j < kPairNP; ++j) {
        const int32_t p = lo + tid + j * kThreads;
        if (p < o_lo || p >= o_hi) continue;
        double acc = acc2[j];
        if (e2_3 >= 0) acc = fma(coef2(e2_3), h2[j], acc);
        if (e2_2 >= 0) acc = fma(coef2(e2_2), h1[j], acc);
        acc = __dadd_rn(__dadd_rn(0.0, acc), pb2[j]);
        if (r2.rw1 != 0) acc = fma(hc ? r2.rc1 : __dmul_rn((double)r2.rw1, __ldg(psi_b + 1)), d1[j], acc);
        const bool in = interior<NDIM>(a.sh, p);
        const double c = u1[j];
        double d = 0.0;
        if (in) {
            if (NDIM == 1) {
                d = __dsub_rn(__dadd_rn(su1[p + 1 - lo], su1[p - 1 - lo]), __dmul_rn(2.0, c));
            } else {
                double r = __dadd_rn(su1[p + R - lo], su1[p - R - lo]);
                r = __dsub_rn(r, __dmul_rn(4.0, c));
                r = __dadd_rn(r, su1[p + 1 - lo]);
                d = __dadd_rn(r, su1[p - 1 - lo]);
            }
        }
        acc = fma(hc ? r2.rc0 : __ldg(psi_b), d, acc);
        double nu;
        if (REACT == 0) {
            nu = __dadd_rn(__dmul_rn(c, decay), __dmul_rn(diffuse, acc));
        } else {
            const double f = __ddiv_rn(__dmul_rn(-a.vmax, c), __dadd_rn(a.km, c));
            nu = __dadd_rn(__dadd_rn(c, __dmul_rn(a.dt[b], f)), __dmul_rn(diffuse, acc));
        }
        if (!in) nu = 0.0;
        if (!isfinite(u1[j])) atomicMin(reinterpret_cast<long long*>(a.status), (long long)(k + 1));
        if (!isfinite(nu)) atomicMin(reinterpret_cast<long long*>(a.status), (long long)(k + 2));
        st_hint1(a.H + k * ss + moff + p, d1[j], keep);
        st_hint1(a.H + (k + 1) * ss + moff + p, d, keep);
        st_hint1(A.u_mid + moff + p, u1[j], keep);
        st_hint1(A.u_out + moff + p, nu, keep);
        if (A.snap1) st_hint1(A.snap1 + moff + p, u1[j], drop);
        if (A.snap2) st_hint1(A.snap2 + moff + p, nu, drop);
    }
    if (tile == 0 && tid == 0) *A.u3_step = A.writes_u3 ? k + 2 : -1;
}

// After a run with pair launches: when the run stopped at a step whose field
// sits in the scratch buffer, copy it to its parity buffer (the divergence
// report and the caller read u[step & 1]).
__global__ void fg_u3_fixup_kernel(const int64_t* status, const int64_t* u3_step, const double* u3, double* u0,
                                   double* u1, int64_t n) {
    const int64_t s = *u3_step;
    if (s < 0 || *status != s) return;
    double* dst = (s & 1) ? u1 : u0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = u3[i];
}

// ------------------------------------------------------- temporal blocking ---
// fg_block_tma_kernel: one pass over the history slices t < kb0 feeds the old
// part of the next `bt` steps (kb0 .. kb0+bt-1) at once:
//     P[b][p] = Σ_{t < kb0} c_b(t)·H[t][p],  c_b(t) = w·ψ(kb0+b-t) if
//               kb0+b-t is in the schedule of step kb0+b (weight w), else 0,
// so each slice of the union of the bt schedules is read from HBM once instead of
// once per step that visits it (full/short memory: bt× fewer bytes; adaptive:
// the thinned intervals' strides < bt share slices).  The step kernel then adds
// P[b] and only its recent entries (m <= b).

constexpr int kBlkSegs = 32;     // segments kept per step (host checks the bound)

struct BlockArgs {
    const double* H;
    double* P;
    const double* psi;
    const int64_t* horizon;
    int64_t slice_stride, ms, psi_stride, base;
    int64_t kb0;
    int64_t t_begin, t_end;  // slices summed by this launch: [t_begin, t_end) ∩ [t_lo, kb0)
    int32_t bt;
    int32_t n_m, kind, tpm, total_tiles;
    int32_t accumulate;      // P += D (tail launch) instead of P = D
    const double* gcoef;  // precomputed coefficient rows (or NULL): single member, or
                          // itemized ensembles ([B][coef_mstride] per block buffer)
    int64_t coef_mstride; // doubles between members' coefficient rows (ensembles)
    int64_t h_alloc;      // slices allocated at H (bounds checks)
    int32_t tblock;       // rows of the P buffer (bounds checks)
};

// The history rows are moved by the bulk-copy engine (cp.async.bulk → shared
// memory, mbarrier complete_tx): one producer warp keeps kStages × kE slice rows
// in flight per CTA independent of registers; TP/32 consumer warps turn each
// stage into DMMA m8n8k4 tiles (below).  Candidate slices are all t in
// [t_lo, kb0) (the union covers nearly all of them: full/short memory exactly,
// adaptive whenever the thinned strides are < BT); slices no step uses get zero
// coefficients, exactly like the reference's zero-weighted terms.  The
// coefficient table for the next kCH slices is built by the consumers while the
// producer's copies for those slices are already in flight.

constexpr int kE = 8;        // slice rows per stage
constexpr int kCH = 128;     // slices per coefficient table (multiple of kE)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

// Release a ring slot only once the warp's tensor-core work on it has consumed
// its shared-memory operands: the fake `dep` input (a result of the warp's last
// DMMA) makes the arrive wait for that DMMA, hence for every LDS feeding the
// warp-wide DMMAs before it.  Without it ptxas scheduled the arrive right after
// the LDS *issue*, letting the producer's next bulk copy overwrite rows still
// being read (a rare, TP-dependent race).
__device__ __forceinline__ void mbar_arrive_after(uint64_t* b, double dep, double* sink) {
    asm volatile(
        "st.shared.f64 [%2], %1;\n\t"
        "mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)),
        "d"(dep), "r"(smem_u32(sink))
        : "memory");
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

// History rows are streamed once per block: mark them evict-first in L2 so the
// stream does not push out what the concurrently running steps touch (fields,
// partial sums, the recent slices), which would turn their L2 hits into HBM
// misses queued behind the stream.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Padded shared-memory rows: +4 doubles (32 B) per row puts the 4 k-rows a DMMA
// B-fragment load touches in disjoint bank quarters (conflict-free LDS.64).
template <int TP>
__host__ __device__ constexpr int row_pitch() { return TP + 4; }
template <int BT>
__host__ __device__ constexpr int coef_pitch() { return BT + 4; }

#ifndef FG_STAGED_RING
#define FG_STAGED_RING 6
#endif
template <bool STAGED>
__host__ __device__ constexpr int ring_stages() { return STAGED ? FG_STAGED_RING : 4; }

constexpr int kMainStages = FG_STAGED_RING;  // staged main launches
#ifndef FG_TAIL_STAGES
#define FG_TAIL_STAGES 2
#endif
constexpr int kTailStages = FG_TAIL_STAGES;  // tail launches: small ring, so they fit beside two main CTAs per SM

// slice rows per stage of the dense kernel: 16 for the 4-M-tile blocks (lean
// consumers), kE otherwise; rings keep their bytes (fewer, deeper stages)
template <int BT>
__host__ __device__ constexpr int dense_ke() { return BT / 8 == 4 ? 16 : kE; }

template <int BT, int TP, bool STAGED, int NS, int WP>
size_t tma_block_smem() {
    constexpr int KE = dense_ke<BT>();
    constexpr int CROWS = STAGED ? NS * KE : kCH;
    return (size_t)NS * KE * row_pitch<TP>() * sizeof(double) + (size_t)CROWS * coef_pitch<BT>() * sizeof(double) +
           (2 * NS) * sizeof(uint64_t) + (TP / WP) * sizeof(double) +
           (STAGED ? 0 : (size_t)BT * kBlkSegs * sizeof(FgSeg) + BT * sizeof(int));
}

// Item flushes add into P with reductions performed at L2 (no load round trip
// in the consumer warps).  Still deterministic: a step's row is touched by one
// lane per item, and the __syncwarp before every flush orders the previous
// item's store/adds (other lanes) before this one's, so the adds reach each
// element in table order — the same rounding as the load-add-store they replace.
__device__ __forceinline__ void red_add(double* p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Coefficient rows of a block, one per candidate slice t (pitch CP doubles):
// row[t - t_lo][b] = w·ψ(kb0+b-t) if kb0+b-t is in the schedule of step kb0+b.
// Single-member runs compute them once per block (all CTAs of the block kernel
// then bulk-copy their rows next to the history rows): the rows are zeroed
// (cudaMemsetAsync) and CTA b scatters its step's entries with t < kb0 by
// walking the schedule segments — no per-slice search, no 64-bit divisions.
template <int BT>
__global__ void fg_block_coef_kernel(const BlockArgs a, double* __restrict__ out) {
    constexpr int CP = coef_pitch<BT>();
    __shared__ FgSeg segs[FG_MAX_SEGS];
    __shared__ int nseg;
    const int bb = blockIdx.x;
    const int64_t hz = a.kind == 1 ? a.horizon[0] : 0;
    const int64_t t_lo = (a.kind == 1 && a.kb0 - hz > 0) ? a.kb0 - hz : 0;
    const int64_t ts = a.t_begin > t_lo ? a.t_begin : t_lo, te = a.t_end;  // rows t - ts, t in [ts, te)
    const int64_t k = a.kb0 + bb;
    if (threadIdx.x == 0) nseg = fg_segments(a.kind, k, a.base, hz, segs);
    __syncthreads();
    for (int si = 0; si < nseg; ++si) {
        // entries m = m0 + i*stride with t = k - m in [ts, te)
        const int64_t m0 = segs[si].m0, st = segs[si].stride, cnt = segs[si].count;
        const int64_t m_min = k - te + 1, m_max = k - ts;
        if (m_max < m0 || m_min > m0 + (cnt - 1) * st) continue;
        const int64_t i0 = m_min > m0 ? (m_min - m0 + st - 1) / st : 0;
        const int64_t i1 = (m_max - m0) / st < cnt - 1 ? (m_max - m0) / st : cnt - 1;
        for (int64_t i = i0 + threadIdx.x; i <= i1; i += blockDim.x) {
            const int64_t m = m0 + i * st;
            FG_DCHECK(k - m >= ts && k - m < te && ((k - m - ts) + 1) * CP <= a.coef_mstride && m < a.psi_stride);
            out[(k - m - ts) * CP + bb] = __dmul_rn((double)st, __ldg(a.psi + m));
        }
    }
}

// The block's old-part sums are a small GEMM per tile: P[BT x TP] += C[BT x 8] ·
// R[8 x TP] per stage (C = coefficients of 8 slices, R = their rows).  Consumers
// feed it to the fp64 tensor pipe (DMMA m8n8k4: 256 FMAs per warp instruction,
// fragments loaded straight from shared memory) instead of 16 FMAs + 9 shared
// loads per element, which made the scalar version shared-memory-issue bound.
// Coefficients: single member → precomputed rows (fg_block_coef_kernel) copied
// into the ring with each stage; ensembles (per-member ψ) → a kCH-slice table
// rebuilt by the consumers at chunk boundaries (scatter over segments).
// WP: points per consumer warp (NT = WP/8 DMMA N tiles).  32-point warps share
// each A fragment over 4 N tiles; 16-point warps hold half the accumulators, so
// a CTA can have twice the warps (measured: the fp64 tensor pipe reaches its
// peak only with 4 issuing warps per SM sub-partition, 16 per SM —
// scripts/micro/dense_consumer.cu; 7-warp CTAs stop at 7/8 of it).
template <int BT, int TP, bool STAGED, int NS, int WP>
__global__ void __launch_bounds__(TP / WP * 32 + 32, 2) fg_block_tma_kernel(const BlockArgs a) {
    constexpr int kStages = NS;
    constexpr int KE = dense_ke<BT>();  // slice rows per stage
    static_assert(KE < 32, "one producer lane per stage row, lane 31 copies the coefficient rows");
    constexpr int RP = row_pitch<TP>();
    constexpr int CP = coef_pitch<BT>();
    constexpr int MT = BT / 8;  // M tiles (steps)
    constexpr int NT = WP / 8;  // N tiles of 8 points per warp
    constexpr int NW = TP / WP; // consumer warps
    constexpr int NC = NW * 32; // consumer threads
    // lean fragments (see the stage loop) for the 4-M-tile blocks: 96 instead of
    // ~125 registers, so 8-warp CTAs (TP 256) fit two per SM
    constexpr bool LEAN = MT == 4;
    constexpr int CROWS = STAGED ? kStages * KE : kCH;
    extern __shared__ __align__(128) unsigned char smem[];
    double* rows = reinterpret_cast<double*>(smem);                  // [kStages][KE][RP]
    double* coef = rows + kStages * KE * RP;                        // [CROWS][CP]
    uint64_t* full = reinterpret_cast<uint64_t*>(coef + CROWS * CP);  // [kStages]
    uint64_t* empty = full + kStages;                               // [kStages]
    double* sink = reinterpret_cast<double*>(empty + kStages);      // [NW] release dependencies
    FgSeg* segs = reinterpret_cast<FgSeg*>(sink + NW);              // [BT][kBlkSegs]
    int* nseg = reinterpret_cast<int*>(segs + BT * kBlkSegs);       // [BT]
    constexpr bool staged = STAGED;  // coefficient rows travel with the stage (single member)

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    // Tiles blockIdx.x, +gridDim.x, ...: single-member launches run one CTA per
    // SM over several tiles (room for the concurrent step kernel); ensembles
    // launch one CTA per tile, so every tile of a CTA has the same member.
    const int64_t mem = blockIdx.x / a.tpm;
    const int64_t hz = a.kind == 1 ? a.horizon[mem] : 0;
    // oldest slice any step of the block can reach: short memory stops at kb0 - H
    const int64_t t_lo = (a.kind == 1 && a.kb0 - hz > 0) ? a.kb0 - hz : 0;
    // this launch's share of [t_lo, kb0): the main launch takes everything but the
    // previous block's slices, the tail launch those
    const int64_t ts = a.t_begin > t_lo ? a.t_begin : t_lo;
    const int64_t te = a.t_end;
    const int64_t n_sl = te > ts ? te - ts : 0;
    const int64_t n_st = (n_sl + KE - 1) / KE;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (!staged && tid < a.bt)
        nseg[tid] = fg_segments(a.kind, a.kb0 + tid, a.base, hz, segs + tid * kBlkSegs, kBlkSegs);
    __syncthreads();

    if (warp == NW) {  // ---- producer warp: lane 0 waits and arms the barrier, lane e copies row e
        // (one warp instruction issues a stage's row copies: c4-full 1292 -> 1285 ms)
        const uint64_t pol = l2_evict_first_policy();
        int64_t g = 0;  // stage counter over all tiles of the CTA
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            const int64_t q0 = (int64_t)(tile % a.tpm) * TP;
            const int64_t row_elems = (a.ms - q0) < TP ? (a.ms - q0) : TP;
            const uint32_t row_bytes = (uint32_t)(row_elems * sizeof(double));
            const double* src0 = a.H + mem * a.ms + q0;
            for (int64_t gl = 0; gl < n_st; ++gl, ++g) {
                const int s = (int)(g % kStages);
                const int64_t t0 = ts + gl * KE;
                const int nr = (int)((te - t0) < KE ? (te - t0) : KE);
                const uint32_t cbytes = staged ? (uint32_t)(nr * CP * sizeof(double)) : 0u;
                if (lane == 0) {
                    if (g >= kStages) mbar_wait(&empty[s], (uint32_t)(((g / kStages) & 1) ^ 1));
                    FG_DCHECK(t0 >= 0 && t0 + nr <= a.h_alloc && t0 + nr <= a.kb0);
                    FG_DCHECK(!staged || (t0 - ts + nr) * CP <= a.coef_mstride);
                    FG_DCHECK(row_bytes <= TP * sizeof(double) && q0 + row_elems <= a.ms);
                    mbar_expect_tx(&full[s], (uint32_t)nr * row_bytes + cbytes);
                }
                __syncwarp();  // the slot is free (lane 0 waited) before any lane copies into it
                if (lane < nr)
                    bulk_g2s_hint(rows + ((size_t)s * KE + lane) * RP, src0 + (t0 + lane) * a.slice_stride, row_bytes,
                                  &full[s], pol);
                if (staged && lane == 31)
                    bulk_g2s(coef + (size_t)s * KE * CP, a.gcoef + (t0 - ts) * CP, cbytes, &full[s]);
            }
        }
        return;
    }

    // ---- consumers: warp w owns points [32w, 32w+32) of the tile
    const int fr = lane >> 2, fk = lane & 3;  // fragment row / k index
    const double* psi_b = a.psi + mem * a.psi_stride;
    const int ngroups = NC / BT;  // threads per step column when filling the table
    int64_t g = 0;
    const uint32_t rows_s = smem_u32(rows) + (uint32_t)((warp * WP + fr) * 8), coef_s = smem_u32(coef) + (uint32_t)(fr * 8);
    for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
    const int64_t q0 = (int64_t)(tile % a.tpm) * TP;
    double d[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) d[i][j][0] = d[i][j][1] = 0.0;
    uint64_t* pend = nullptr;  // slot of the previous stage, released by the next one
    for (int64_t gl = 0; gl < n_st; ++gl, ++g) {
        const int64_t t0 = ts + gl * KE;
        if (!staged && (gl * KE) % kCH == 0) {
            // ensemble path: coefficient table for slices t0 .. t0+kCH-1 — zero it,
            // then scatter w·ψ_b(m) over every schedule segment (no per-slice search)
            asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
            for (int i = tid; i < kCH * CP; i += NC) coef[i] = 0.0;
            asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
            const int bb = tid % BT, grp = tid / BT;
            if (bb < a.bt && grp < ngroups) {
                const int64_t k = a.kb0 + bb;
                const int64_t t_hi = (t0 + kCH - 1 < te - 1) ? t0 + kCH - 1 : te - 1;
                const int64_t m_lo = k - t_hi, m_hi = k - t0;  // offsets mapping into this table
                const FgSeg* sg = segs + bb * kBlkSegs;
                for (int si = 0; si < nseg[bb]; ++si) {
                    const int64_t m0 = sg[si].m0, st = sg[si].stride, last = m0 + (sg[si].count - 1) * st;
                    const int64_t lo = m_lo > m0 ? m_lo : m0, hi = m_hi < last ? m_hi : last;
                    if (lo > hi) continue;
                    const int64_t i0 = (lo - m0 + st - 1) / st, i1 = (hi - m0) / st;
                    for (int64_t i = i0 + grp; i <= i1; i += ngroups) {
                        const int64_t m = m0 + i * st;
                        coef[(k - m - t0) * CP + bb] = __dmul_rn((double)st, __ldg(psi_b + m));
                    }
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
        }
        const int s = (int)(g % kStages);
        mbar_wait(&full[s], (uint32_t)((g / kStages) & 1));
        const int nr = (int)((te - t0) < KE ? (te - t0) : KE);
        const uint32_t rs = rows_s + (uint32_t)(s * KE * RP * 8);
        const uint32_t cs = staged ? coef_s + (uint32_t)(s * KE * CP * 8) : coef_s + (uint32_t)(((gl * KE) % kCH) * CP * 8);
        if constexpr (LEAN) {
        // one k-step (4 slices) of fragments live at a time, so 8 consumer warps
        // of 32 points fit two CTAs per SM (the fp64 tensor pipe needs 16 issuing
        // warps per SM, scripts/micro/dense_consumer.cu); the previous stage's slot
        // is released after the first k-step's DMMAs: the dependency is on a DMMA
        // issued after every DMMA that read the slot (so those reads are done),
        // and 16 DMMAs old by the time the release needs it.  Stages of 16 slices
        // (4 k-steps, not unrolled: registers) halve the barrier round trips per
        // DMMA (c4-full 1310 -> 1277 ms, c3-full 633 -> 616)
#pragma unroll 1
        for (int ks = 0; ks < KE / 4; ++ks) {
            const int e = ks * 4 + fk;
            double af[MT], bf[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) af[i] = e < nr ? lds_f64(cs + (uint32_t)((e * CP + 8 * i) * 8)) : 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[j] = e < nr ? lds_f64(rs + (uint32_t)((e * RP + 8 * j) * 8)) : 0.0;
            if (ks == 1) {
                if (pend && lane == 0) mbar_arrive_after(pend, d[0][0][0], sink + warp);
                pend = &empty[s];
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma_8x8x4(d[i][j][0], d[i][j][1], af[i], bf[j]);
        }
        } else {
        // all fragments of the stage into registers first (partial last stage masked) ...
        double af[KE / 4][MT], bf[KE / 4][NT];
#pragma unroll
        for (int ks = 0; ks < KE / 4; ++ks) {
            const int e = ks * 4 + fk;
#pragma unroll
            for (int i = 0; i < MT; ++i) af[ks][i] = e < nr ? lds_f64(cs + (uint32_t)((e * CP + 8 * i) * 8)) : 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[ks][j] = e < nr ? lds_f64(rs + (uint32_t)((e * RP + 8 * j) * 8)) : 0.0;
        }
        // ... then release the PREVIOUS stage's slot: the release depends on that
        // stage's last DMMA result, and that DMMA (like every one before it) only
        // issued once the fragments it read from the slot were in registers —
        // so the producer's next bulk copy cannot overwrite rows still being read
        if (pend && lane == 0) mbar_arrive_after(pend, d[MT - 1][NT - 1][1], sink + warp);
        pend = &empty[s];
#pragma unroll
        for (int ks = 0; ks < KE / 4; ++ks)
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma_8x8x4(d[i][j][0], d[i][j][1], af[ks][i], bf[ks][j]);
        }
    }
    // the tile's last stage: released once its DMMAs are done (the flush needs them anyway)
    if (pend && lane == 0) mbar_arrive_after(pend, d[MT - 1][NT - 1][1], sink + warp);
    // D fragment: row = step fr (+8 per M tile), columns = 2 adjacent points
    double* pout = a.P + mem * a.ms + q0 + warp * WP + fk * 2;
    FG_DCHECK(a.bt <= a.tblock && a.bt <= BT);
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int bb = 8 * i + fr;
        if (bb >= a.bt) continue;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int64_t q = q0 + warp * WP + 8 * j + fk * 2;
            if (q >= a.n_m) continue;
            double* o = pout + bb * a.slice_stride + 8 * j;
            if (a.accumulate) {
                const double2 old = ld_cg2(o);
                st_pair(o, __dadd_rn(old.x, d[i][j][0]), __dadd_rn(old.y, d[i][j][1]));
            } else {
                st_pair(o, d[i][j][0], d[i][j][1]);
            }
        }
    }
    }  // tiles
}

// ------------------------------------------- class-decomposed block stage ---
// A thinned (adaptive) schedule samples offsets m with stride s inside each
// interval, so in a block only the steps b with kb0+b-t ≡ m0 (mod s) use slice
// t: the dense [BT x slices] coefficient tile above is mostly zeros (c2: ~1 in
// 9 nonzero) and the fp64 tensor pipe, not HBM, bounds the main launch.  Here
// the block's (step, slice) pairs of the main range are partitioned into
// items = (stride s, residue t mod s): an item streams its slices t_first +
// j*s (every slice of the block's union is read by exactly the items that use
// it — one for most slices) and multiplies them with a dense coefficient tile
// over only its own steps (≈ BT/s), so the work executed is the schedule's
// terms rounded up to 8-step DMMA tiles.  One CTA per tile walks the items in
// table order and adds each item's partial sums into the tile's P rows (first
// item of a step stores), so the sums are deterministic without atomics.  Full
// and short memory (one class holding every step) keep the dense kernel.

constexpr int kMaxItems = 160;
constexpr int kItemCols = 16;   // steps per item: two DMMA M tiles, so the kernel's
                                // accumulators (and registers) do not grow with tblock
constexpr int kItemPitch = kItemCols + 4;  // coefficient row pitch: 20 ≡ 4 (mod 16) doubles, conflict-free
                                           // A-fragment loads (see coef_pitch)
constexpr int kItemPitch8 = 12;            // 8-column items (fg_block_item8_kernel): 12 ≡ -4 (mod 16)

struct BlockItem {
    int64_t t_first;
    int32_t stride, n_slices;
    int32_t coef_row;  // first coefficient row (kCoefRow doubles each) of this item
    int32_t first_mask;  // bit c: this item is the first (in table order) to add to step col2step[c]
    int32_t ncols;     // steps in the item (<= kItemCols); column c is step col2step[c]
    uint8_t col2step[kItemCols];
    uint8_t map;       // 16-column kernel: its stride's tensor map in ItemMaps
};

struct ItemTable {
    int32_t n_items;
    int32_t accumulate;  // tail launch: every item adds to P (no first stores, no zeroing)
    int32_t cols;        // item width of this table: 8 (fg_block_item8_kernel) or 16
    int32_t pitch;       // its coefficient row pitch: kItemPitch8 or kItemPitch
    uint64_t zero_mask[kMaxTBlock / 64];  // main launch: steps no item touches (their P rows are zeroed)
    BlockItem it[kMaxItems];
};

// 16-column item kernel: one TMA tensor map per distinct item stride s, a 4-D
// view [J][s][chunks][16] of the history (dims innermost first: 16 points,
// B·ms/16 chunks of 128 bytes, residue t mod s, j = t div s), box {16, C, 1, kE}
// with the 128-byte swizzle.  Built on the host per launch (encode_item_maps).
constexpr int kMaxMaps = 16;
struct ItemMaps {
    CUtensorMap map[kMaxMaps];
    CUtensorMap half[kMaxMaps];     // the same views with boxes of kIR/2 and kIR/4 slices: an
    CUtensorMap quarter[kMaxMaps];  // item's short last stage reads its rows rounded up to kIR/4
};

// Coefficient rows of every item: row (coef_row + j), column c =
// w·ψ(kb0 + col2step[c] - t_j) when that offset is in step col2step[c]'s
// schedule with weight w == the item's stride (the entry belongs to this
// item), else 0; columns ncols..CP-1 are zero padding for the DMMA tiles.
// Ensembles (the schedule is shared, ψ is per member): blockIdx.z takes every
// gridDim.z-th member; the entry's offset and weight are found once and reused
// for each of its members' rows.
__global__ void fg_item_coef_kernel(const BlockArgs a, const __grid_constant__ ItemTable T,
                                    double* __restrict__ out, int64_t n_members) {
    const int CP = T.pitch;
    __shared__ FgSeg segs[kItemCols][kBlkSegs];
    __shared__ int nseg[kItemCols];
    const BlockItem& it = T.it[blockIdx.y];
    const int64_t hz = a.kind == 1 ? a.horizon[0] : 0;
    if (threadIdx.x < it.ncols) {
        const int b = it.col2step[threadIdx.x];
        nseg[threadIdx.x] = fg_segments(a.kind, a.kb0 + b, a.base, hz, segs[threadIdx.x], kBlkSegs);
    }
    __syncthreads();
    const int64_t rows = it.n_slices;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * CP;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / CP;
        const int c = (int)(e - j * CP);
        int64_t m = -1;
        int32_t w = 0;
        if (c < it.ncols) {
            m = a.kb0 + it.col2step[c] - (it.t_first + j * it.stride);
            w = fg_seg_weight(segs[c], nseg[c], m);
        }
        const bool on = w == it.stride;
        FG_DCHECK(((int64_t)it.coef_row + j + 1) * CP <= a.coef_mstride && (!on || (m >= 1 && m < a.psi_stride)));
        double* o = out + ((int64_t)it.coef_row + j) * CP + c;
        for (int64_t mem = blockIdx.z; mem < n_members; mem += gridDim.z)
            o[mem * a.coef_mstride] = on ? __dmul_rn((double)w, __ldg(a.psi + mem * a.psi_stride + m)) : 0.0;
    }
}

// One ring stage of an item with MTE live M tiles: fragments of the stage's
// kE slices into registers, release the slot (after the reads, see
// fg_block_tma_kernel), then MTE x NT x 2 DMMAs.
template <int MTE, int MT, int NT, int CP, int RP>
__device__ __forceinline__ void item_stage(double (&d)[MT][NT][2], const double* cs, const double* rs, int nr, int fk,
                                           int lane, uint64_t* empty_s, double* sink_w) {
    double af[kE / 4][MTE], bf[kE / 4][NT];
    uint32_t xr = 0;
#pragma unroll
    for (int ks = 0; ks < kE / 4; ++ks) {
        const int e = ks * 4 + fk;
#pragma unroll
        for (int i = 0; i < MTE; ++i) {
            af[ks][i] = e < nr ? cs[e * CP + 8 * i] : 0.0;
            const unsigned long long w = (unsigned long long)__double_as_longlong(af[ks][i]);
            xr ^= (uint32_t)w ^ (uint32_t)(w >> 32);
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            bf[ks][j] = e < nr ? rs[e * RP + 8 * j] : 0.0;
            const unsigned long long w = (unsigned long long)__double_as_longlong(bf[ks][j]);
            xr ^= (uint32_t)w ^ (uint32_t)(w >> 32);
        }
    }
    xr = __reduce_xor_sync(0xffffffffu, xr);
    if (lane == 0) mbar_arrive_after(empty_s, (double)xr, sink_w);
#pragma unroll
    for (int ks = 0; ks < kE / 4; ++ks)
#pragma unroll
        for (int i = 0; i < MTE; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma_8x8x4(d[i][j][0], d[i][j][1], af[ks][i], bf[ks][j]);
}

// ---- 8-column items (fg_block_item8_kernel): warps of 32 points, one DMMA M
// tile.  Wider tiles per CTA (TP 128..256) than the 16-column kernel below, so a
// CTA walks the item table fewer times: measured faster for a single small
// field (c2: 22.9 vs 31.9 ms of block stage at tblock 64), while 16-column items
// win when a class has more than 8 steps in a block (c5 at tblock 128).
// One CTA per tile walks every item in table order through one TMA ring (the
// ring of fg_block_tma_kernel with staged coefficient rows; the pipeline does
// not drain between items): an item's slices are t_first + j*stride, DMMA M
// tiles beyond its steps are skipped, and its partial sums are flushed from the
// accumulators when its last stage is done.
// ENS: ensembles (tpm tiles per member, per-member coefficient rows); the
// single-member variant keeps the simpler addressing (and its registers).
template <int TP, int NS, bool ENS>
__global__ void __launch_bounds__(TP + 32, 4)  // <= 64 registers: two CTAs leave room for two step CTAs
    fg_block_item8_kernel(const BlockArgs a, const __grid_constant__ ItemTable T) {
    constexpr int kStages = NS;
    constexpr int RP = row_pitch<TP>();
    constexpr int CP = kItemPitch8;
    constexpr int MT = 1;
    constexpr int NT = 4;
    constexpr int NW = TP / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    double* rows = reinterpret_cast<double*>(smem);                        // [kStages][kE][RP]
    double* coef = rows + kStages * kE * RP;                              // [kStages*kE][CP]
    uint64_t* full = reinterpret_cast<uint64_t*>(coef + kStages * kE * CP);
    uint64_t* empty = full + kStages;
    double* sink = reinterpret_cast<double*>(empty + kStages);

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NW) {  // producer
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int64_t g = 0;  // stage counter over all tiles and items
            for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            const int64_t mem = ENS ? tile / a.tpm : 0;  // ensembles: tpm tiles per member
            const int64_t qm = (int64_t)(tile - mem * a.tpm) * TP;
            const int64_t row_elems = (a.ms - qm) < TP ? (a.ms - qm) : TP;
            const uint32_t row_bytes = (uint32_t)(row_elems * sizeof(double));
            for (int x = blockIdx.y; x < T.n_items; x += gridDim.y) {
                const BlockItem& it = T.it[x];
                const double* src0 = a.H + mem * a.ms + qm + it.t_first * a.slice_stride;
                const int64_t sstride = (int64_t)it.stride * a.slice_stride;
                const double* c0 = a.gcoef + (ENS ? mem * a.coef_mstride : 0) + (int64_t)it.coef_row * CP;
                for (int64_t j0 = 0; j0 < it.n_slices; j0 += kE, ++g) {
                    const int s = (int)(g % kStages);
                    if (g >= kStages) mbar_wait(&empty[s], (uint32_t)(((g / kStages) & 1) ^ 1));
                    const int nr = (int)((it.n_slices - j0) < kE ? (it.n_slices - j0) : kE);
                    const uint32_t cbytes = (uint32_t)(nr * CP * sizeof(double));
                    FG_DCHECK(it.t_first + (j0 + nr - 1) * it.stride < a.h_alloc && it.t_first >= 0);
                    FG_DCHECK(((int64_t)it.coef_row + j0 + nr) * CP <= a.coef_mstride);
                    mbar_expect_tx(&full[s], (uint32_t)nr * row_bytes + cbytes);
                    for (int e = 0; e < nr; ++e)
                        bulk_g2s_hint(rows + ((size_t)s * kE + e) * RP, src0 + (j0 + e) * sstride, row_bytes,
                                      &full[s], pol);
                    bulk_g2s(coef + (size_t)s * kE * CP, c0 + j0 * CP, cbytes, &full[s]);
                }
            }
            }  // tiles
        }
        return;
    }

    const int fr = lane >> 2, fk = lane & 3;
    double d[MT][NT][2];
    int64_t g = 0;
    for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
    const int64_t mem = ENS ? tile / a.tpm : 0;
    const int64_t qm = (int64_t)(tile - mem * a.tpm) * TP;  // tile's first point within its member
    double* const Pm = ENS ? a.P + mem * a.ms : a.P;         // member's rows of P
    if (!T.accumulate) {  // steps no item adds to: P = 0 (this CTA owns the tile)
        for (int w = 0; w < kMaxTBlock / 64; ++w)
        for (uint64_t zm = T.zero_mask[w]; zm; zm &= zm - 1) {
            const int b = 64 * w + __ffsll((long long)zm) - 1;
            for (int i = tid; i < TP / 2; i += TP) {
                const int64_t q = qm + 2 * i;
                if (q < a.n_m) st_pair(Pm + (int64_t)b * a.slice_stride + q, 0.0, 0.0);
            }
        }
    }
    for (int x = blockIdx.y; x < T.n_items; x += gridDim.y) {
        const BlockItem& it = T.it[x];
        const int mt = (it.ncols + 7) >> 3;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) d[i][j][0] = d[i][j][1] = 0.0;
        for (int64_t j0 = 0; j0 < it.n_slices; j0 += kE, ++g) {
            const int s = (int)(g % kStages);
            mbar_wait(&full[s], (uint32_t)((g / kStages) & 1));
            const int nr = (int)((it.n_slices - j0) < kE ? (it.n_slices - j0) : kE);
            const double* rs = rows + (size_t)s * kE * RP + warp * 32 + fr;
            const double* cs = coef + (size_t)s * kE * CP + fr;
            // warp-uniform branch per item: only the item's M tiles are issued
            // (predicated-off DMMAs would still occupy the fp64 tensor pipe)
            item_stage<1, MT, NT, CP, RP>(d, cs, rs, nr, fk, lane, &empty[s], sink + warp);
        }
        const uint64_t keep = l2_policy_last();  // the steps read P next
        // flush into P (this CTA owns the tile, items in table order, so the
        // sum of each step is deterministic): the first item of a step stores,
        // later ones (and every tail item) add — loads first, one round trip.
        // A step's row can sit in another lane than in the previous item (only
        // this warp touches these points): the warp barrier orders the accesses.
        __syncwarp();
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int r = 8 * i + fr;
            if (i >= mt || r >= it.ncols) continue;
            FG_DCHECK(it.col2step[r] < a.bt && a.bt <= a.tblock);
            double* out = Pm + (int64_t)it.col2step[r] * a.slice_stride;
            const bool add = T.accumulate || !((it.first_mask >> r) & 1);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int64_t q = qm + warp * 32 + 8 * j + fk * 2;
                if (q >= a.n_m) continue;
                if (add) {  // fire-and-forget L2 adds, applied in program order (see red_add)
                    red_add(out + q, d[i][j][0]);
                    red_add(out + q + 1, d[i][j][1]);
                } else {
                    st_pair_hint(out + q, d[i][j][0], d[i][j][1], keep);
                }
            }
        }
    }
    }  // tiles
}

template <int TP, int NS>
size_t item8_block_smem() {
    return (size_t)NS * kE * row_pitch<TP>() * sizeof(double) + (size_t)NS * kE * kItemPitch8 * sizeof(double) +
           (2 * NS) * sizeof(uint64_t) + (TP / 32) * sizeof(double);
}

// One CTA walks its tiles, and per tile every item in table order, through one
// TMA ring (the pipeline does not drain between items or tiles): an item's
// slices are t_first + j*stride, and its partial sums are flushed from the
// accumulators when its last stage is done.  An item has up to 16 step columns
// (two DMMA M tiles), so a residue class of up to 16 steps is streamed once; a
// warp owns 16 points of the tile (one 128-byte chunk, two N tiles), which keeps
// the accumulators at 8 doubles per thread — TP/16 consumer warps + 1 producer
// warp, <= 64 registers, two CTAs per SM (two step CTAs still fit beside them).
// Items of at most 8 columns issue only the first M tile (warp-uniform branch).
//
// A stage (kIR slices of the item's progression × TP points) is ONE tensor copy
// per box (cp.async.bulk.tensor.4d, SASS UTMALDG) from a 4-D view of the
// history [J][s][chunks][16] for the item's stride s (ItemMaps): coordinates
// (0, chunk, t mod s, t div s) select kIR slices t, t+s, … at once.  The per-row
// bulk copies this replaces (one UBLKCP per slice row, issued through a
// serialised uniform loop) left the producer warp issue-bound and the DRAM
// stream at 38 % of peak (profiles/r02_c3a_item16_*).  The box lands densely in
// shared memory with the 128-byte swizzle: line L (128 B = one warp's 16 points
// of one slice) has its 16-byte units XORed with L mod 8, so a B-fragment load
// (4 slices × 8 points) splits 2 + 2 over the two bank halves — the minimum of
// two wavefronts for 32 × 8 bytes.  That needs C chunks per box with C·fk
// mod 8 ∈ {0, 6, 4, 2} or {0, 4, 0, 4}: boxes of 6 chunks (TP 96) or two boxes
// of 4 chunks (TP 128).
// ENS: ensembles (tpm tiles per member, per-member coefficient rows); the
// single-member variant keeps the simpler addressing.
#ifndef FG_ITEM_ROWS
#define FG_ITEM_ROWS 16
#endif
constexpr int kIR = FG_ITEM_ROWS;  // slices per stage of the 16-column item kernel (multiple of kE)
static_assert(kIR % kE == 0 && kIR <= 32, "item stage rows");

template <int TP>
__host__ __device__ constexpr int item_threads() { return TP / 16 * 32 + 32; }
template <int TP>
__host__ __device__ constexpr int item_box_chunks() { return TP == 96 ? 6 : 4; }  // 16-point chunks per TMA box
template <int TP>
__host__ __device__ constexpr int item_stage_bytes() { return kIR * TP * (int)sizeof(double); }  // multiple of 1024 (swizzle atom)

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// One ring stage of an item with MTE live M tiles: A fragments (coefficients)
// at shared address ca (+ e·CP + 8i doubles), B fragments at the swizzled byte
// offsets boff of the stage at ra.  FULL: all kE rows belong to the item (no
// masking).  Before its DMMAs the warp releases the PREVIOUS stage's slot
// (pend): the release depends on the last DMMA result of that stage, which was
// only issued once every fragment it and the DMMAs before it read had arrived
// in registers — so the producer cannot overwrite rows still being read, and
// the release costs one dependent store instead of a warp-wide reduction of the
// loaded values.
template <int MTE, int MT, int NT, int CP, bool FULL>
__device__ __forceinline__ void item_stage_sw(double (&d)[MT][NT][2], uint32_t ca, uint32_t ra,
                                              const uint32_t (&boff)[kE / 4][NT], int nr, int fk, int lane,
                                              uint64_t* pend, double* sink_w) {
    double af[kE / 4][MTE], bf[kE / 4][NT];
#pragma unroll
    for (int ks = 0; ks < kE / 4; ++ks) {
        const int e = ks * 4 + fk;
#pragma unroll
        for (int i = 0; i < MTE; ++i)
            af[ks][i] = (FULL || e < nr) ? lds_f64(ca + (uint32_t)((e * CP + 8 * i) * 8)) : 0.0;
#pragma unroll
        for (int j = 0; j < NT; ++j)  // rows past the item's end hold other (or unwritten) slices: masked
            bf[ks][j] = (FULL || e < nr) ? lds_f64(ra + boff[ks][j]) : 0.0;
    }
    // the previous stage of this item had the same MTE: its last DMMA wrote d[MTE - 1][NT - 1]
    // (a register dependency only: an add here would take a slot of the fp64 pipe)
    if (pend && lane == 0) mbar_arrive_after(pend, d[MTE - 1][NT - 1][1], sink_w);
#pragma unroll
    for (int ks = 0; ks < kE / 4; ++ks)
#pragma unroll
        for (int i = 0; i < MTE; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma_8x8x4(d[i][j][0], d[i][j][1], af[ks][i], bf[ks][j]);
}

template <int TP, int NS, bool ENS>
__global__ void __maxnreg__(64)  // <= 64 registers: two step CTAs fit beside two of these per SM
    fg_block_item_kernel(const BlockArgs a, const __grid_constant__ ItemTable T, const __grid_constant__ ItemMaps M) {
    constexpr int kStages = NS;
    constexpr int CP = kItemPitch;
    constexpr int MT = 2;
    constexpr int NT = 2;
    constexpr int NW = TP / 16;
    constexpr int C = item_box_chunks<TP>();
    constexpr int NB = NW / C;                       // boxes per stage
    constexpr int SB = item_stage_bytes<TP>();
    constexpr int BOXB = C * kIR * 128;              // bytes per box
    static_assert(NB * C == NW && SB % 1024 == 0 && BOXB % 1024 == 0, "item tile / box geometry");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // swizzle-128B boxes need 1024-byte aligned destinations (1 KB of slack is allocated)
    unsigned char* rows = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // [kStages][SB]
    double* coef = reinterpret_cast<double*>(rows + (size_t)kStages * SB);              // [kStages*kIR][CP]
    uint64_t* full = reinterpret_cast<uint64_t*>(coef + kStages * kIR * CP);
    uint64_t* empty = full + kStages;
    double* sink = reinterpret_cast<double*>(empty + kStages);

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NW) {  // producer warp: one lane issues a stage's boxes and coefficient rows
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int64_t g = 0;  // stage counter over all tiles and items
            for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
                const int64_t mem = ENS ? tile / a.tpm : 0;  // ensembles: tpm tiles per member
                const int64_t qm = (int64_t)(tile - mem * a.tpm) * TP;
                const int chunk0 = (int)((mem * a.ms + qm) >> 4);
                for (int x = 0; x < T.n_items; ++x) {
                    const BlockItem& it = T.it[x];
                    const CUtensorMap* map = &M.map[it.map];
                    const int r = (int)(it.t_first % it.stride);
                    const int j_first = (int)(it.t_first / it.stride);
                    const double* c0 = a.gcoef + (ENS ? mem * a.coef_mstride : 0) + (int64_t)it.coef_row * CP;
                    for (int64_t j0 = 0; j0 < it.n_slices; j0 += kIR, ++g) {
                        const int s = (int)(g % kStages);
                        const int nr = (int)((it.n_slices - j0) < kIR ? (it.n_slices - j0) : kIR);
                        if (g >= kStages) mbar_wait(&empty[s], (uint32_t)(((g / kStages) & 1) ^ 1));
                        const uint32_t cbytes = (uint32_t)(nr * CP * sizeof(double));
                        // the box reads kIR slices of the progression: all of them allocated
                        FG_DCHECK(it.t_first + (j0 + kIR - 1) * (int64_t)it.stride < a.h_alloc && it.t_first >= 0);
                        FG_DCHECK(it.t_first + (j0 + nr - 1) * (int64_t)it.stride < a.kb0 + a.bt);
                        FG_DCHECK(((int64_t)it.coef_row + j0 + nr) * CP <= a.coef_mstride);
                        // a box may run past the member (partial last tile: its points are never
                        // stored) or past the history (the TMA zero-fills); it starts inside
                        FG_DCHECK(it.map < kMaxMaps && chunk0 < a.slice_stride / 16);
                        // a short last stage is covered by half- and quarter-depth boxes
                        // (rows rounded up to kIR/4), landing on the same rows of the box
                        // slots as the full box would (the consumers never read past nr)
                        const int rows_rd = nr == kIR ? kIR : nr > kIR / 2 + kIR / 4 ? kIR : (nr + kIR / 4 - 1) / (kIR / 4) * (kIR / 4);
                        mbar_expect_tx(&full[s], (uint32_t)(SB / kIR * rows_rd) + cbytes);
                        for (int e0 = 0; e0 < rows_rd;) {
                            const int depth = rows_rd - e0 >= kIR ? kIR : rows_rd - e0 >= kIR / 2 ? kIR / 2 : kIR / 4;
                            const CUtensorMap* mp = depth == kIR ? map : depth == kIR / 2 ? &M.half[it.map]
                                                                                          : &M.quarter[it.map];
#pragma unroll
                            for (int b = 0; b < NB; ++b)
                                tma_load_4d(rows + (size_t)s * SB + b * BOXB + e0 * C * 128, mp, 0, chunk0 + b * C, r,
                                            j_first + (int)j0 + e0, &full[s], pol);
                            e0 += depth;
                        }
                        bulk_g2s(coef + (size_t)s * kIR * CP, c0 + j0 * CP, cbytes, &full[s]);
                    }
                }
            }  // tiles
        }
        return;
    }

    const int fr = lane >> 2, fk = lane & 3;
    // byte offsets of this lane's B fragments in a stage: slice e = 4ks + fk,
    // point 16·warp + 8j + fr → box warp / C, line L = e·C + warp % C, 16-byte
    // unit (4j + fr/2) XOR (L mod 8), half (fr & 1)
    uint32_t boff[kE / 4][NT];
#pragma unroll
    for (int ks = 0; ks < kE / 4; ++ks)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int L = (ks * 4 + fk) * C + warp % C;
            const int u = (4 * j + (fr >> 1)) ^ (L & 7);
            boff[ks][j] = (uint32_t)((warp / C) * BOXB + L * 128 + u * 16 + (fr & 1) * 8);
        }
    const uint32_t rows_s = smem_u32(rows), coef_s = smem_u32(coef) + (uint32_t)(fr * 8);
    double d[MT][NT][2];
    int64_t g = 0;
    for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
    const int64_t mem = ENS ? tile / a.tpm : 0;
    const int64_t qm = (int64_t)(tile - mem * a.tpm) * TP;  // tile's first point within its member
    double* const Pm = ENS ? a.P + mem * a.ms : a.P;         // member's rows of P
    if (!T.accumulate) {  // steps no item adds to: P = 0 (this CTA owns the tile)
        for (int w = 0; w < kMaxTBlock / 64; ++w)
        for (uint64_t zm = T.zero_mask[w]; zm; zm &= zm - 1) {
            const int b = 64 * w + __ffsll((long long)zm) - 1;
            for (int i = tid; i < TP / 2; i += NW * 32) {
                const int64_t q = qm + 2 * i;
                if (q < a.n_m) st_pair(Pm + (int64_t)b * a.slice_stride + q, 0.0, 0.0);
            }
        }
    }
    for (int x = 0; x < T.n_items; ++x) {
        const BlockItem& it = T.it[x];
        const int mt = (it.ncols + 7) >> 3;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) d[i][j][0] = d[i][j][1] = 0.0;
        uint64_t* pend = nullptr;  // slot of the previous stage, released by the next one
        for (int64_t j0 = 0; j0 < it.n_slices; j0 += kIR, ++g) {
            const int s = (int)(g % kStages);
            mbar_wait(&full[s], (uint32_t)((g / kStages) & 1));
            const int nr = (int)((it.n_slices - j0) < kIR ? (it.n_slices - j0) : kIR);
            // a stage's kIR rows in groups of kE (fragment registers for kE rows
            // only); the previous stage's slot is released after the first group's loads
#pragma unroll
            for (int h = 0; h < kIR / kE; ++h) {
                const int nrh = nr - h * kE;  // rows of this group that belong to the item
                if (nrh <= 0) break;          // warp-uniform
                const uint32_t ra = rows_s + (uint32_t)(s * SB + h * kE * C * 128);
                const uint32_t ca = coef_s + (uint32_t)((s * kIR + h * kE) * CP * 8);
                uint64_t* rel = h == 0 ? pend : nullptr;
                // warp-uniform branches per item and group: only the item's M tiles
                // are issued (predicated-off DMMAs would still occupy the fp64 tensor
                // pipe), and only a partial last group masks its rows
                if (nrh >= kE) {
                    if (mt > 1)
                        item_stage_sw<2, MT, NT, CP, true>(d, ca, ra, boff, nrh, fk, lane, rel, sink + warp);
                    else
                        item_stage_sw<1, MT, NT, CP, true>(d, ca, ra, boff, nrh, fk, lane, rel, sink + warp);
                } else {
                    if (mt > 1)
                        item_stage_sw<2, MT, NT, CP, false>(d, ca, ra, boff, nrh, fk, lane, rel, sink + warp);
                    else
                        item_stage_sw<1, MT, NT, CP, false>(d, ca, ra, boff, nrh, fk, lane, rel, sink + warp);
                }
            }
            pend = &empty[s];
        }
        // the item's last stage: released once its DMMAs are done (the flush needs them anyway)
        if (pend && lane == 0) mbar_arrive_after(pend, d[MT - 1][NT - 1][1] + d[0][NT - 1][1], sink + warp);
        const uint64_t keep = l2_policy_last();  // the steps read P next
        // flush into P (this CTA owns the tile, items in table order, so the
        // sum of each step is deterministic): the first item of a step stores,
        // later ones (and every tail item) add.  A step's row can sit in another
        // lane than in the previous item (only this warp touches these points):
        // the warp barrier orders the accesses.
        __syncwarp();
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int r = 8 * i + fr;
            if (i >= mt || r >= it.ncols) continue;
            FG_DCHECK(it.col2step[r] < a.bt && a.bt <= a.tblock);
            double* out = Pm + (int64_t)it.col2step[r] * a.slice_stride;
            const bool add = T.accumulate || !((it.first_mask >> r) & 1);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int64_t q = qm + warp * 16 + 8 * j + fk * 2;
                if (q >= a.n_m) continue;
                if (add) {  // fire-and-forget L2 adds, applied in program order (see red_add)
                    red_add(out + q, d[i][j][0]);
                    red_add(out + q + 1, d[i][j][1]);
                } else {
                    st_pair_hint(out + q, d[i][j][0], d[i][j][1], keep);
                }
            }
        }
    }
    }  // tiles
}

template <int TP, int NS>
size_t item_block_smem() {
    return 1024 + (size_t)NS * item_stage_bytes<TP>() + (size_t)NS * kIR * kItemPitch * sizeof(double) +
           (2 * NS) * sizeof(uint64_t) + (TP / 16) * sizeof(double);
}

// ------------------------------------------------------------------ ψ tables ---
// coefficients.py:86-91: v = ((-v) * ((2 - γ) - m)) / m, each op rounded once.
__global__ void fg_psi_kernel(const double* __restrict__ gamma, int64_t B, int64_t n, int64_t stride,
                              double* __restrict__ out) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double g = gamma[b];
    const double two_minus_g = __dsub_rn(2.0, g);
    double* o = out + b * stride;
    double v = 1.0;
    o[0] = v;
    for (int64_t m = 1; m <= n; ++m) {
        const double fm = (double)m;
        v = __ddiv_rn(__dmul_rn(-v, __dsub_rn(two_minus_g, fm)), fm);
        o[m] = v;
    }
}

// ----------------------------------------------------------- schedule expand ---
__global__ void fg_schedule_kernel(int kind, int64_t k0, int64_t base, int64_t horizon, int32_t* offs,
                                   int32_t* wts, int64_t row_cap, int64_t* lens) {
    __shared__ FgSeg segs[FG_MAX_SEGS];
    __shared__ int64_t first[FG_MAX_SEGS + 1];
    __shared__ int s_n;
    const int64_t k = k0 + blockIdx.x;
    if (threadIdx.x == 0) {
        int n = fg_segments(kind, k, base, horizon, segs);
        int64_t acc = 0;
        for (int i = 0; i < n; ++i) {
            first[i] = acc;
            acc += segs[i].count;
        }
        first[n > 0 ? n : 0] = acc;
        s_n = n;
        lens[blockIdx.x] = n > 0 ? acc : -1;
    }
    __syncthreads();
    const int n = s_n;
    if (n <= 0) return;
    const int64_t len = first[n];
    const int64_t lim = len < row_cap ? len : row_cap;
    int32_t* orow = offs + (int64_t)blockIdx.x * row_cap;
    int32_t* wrow = wts + (int64_t)blockIdx.x * row_cap;
    for (int64_t j = threadIdx.x; j < lim; j += blockDim.x) {
        int si = 0;
        while (si + 1 < n && first[si + 1] <= j) ++si;
        orow[j] = (int32_t)(segs[si].m0 + (j - first[si]) * segs[si].stride);
        wrow[j] = (int32_t)segs[si].stride;
    }
}

// -------------------------------------------------------- generic history_sum ---
__global__ void fg_history_sum_kernel(const double* __restrict__ H, int64_t ss, int64_t n,
                                      const int64_t* __restrict__ offs, const int64_t* __restrict__ wts,
                                      int64_t len, const double* __restrict__ psi, int64_t k,
                                      double* __restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double acc = 0.0;
    for (int64_t j = 0; j < len; ++j) {
        const int64_t m = offs[j];
        const double c = __dmul_rn((double)wts[j], psi[m]);
        acc = fma(c, H[(k - m) * ss + p], acc);
    }
    out[p] = acc;
}

// ------------------------------------------------------------ plain stencil ---
template <int NDIM>
__global__ void fg_stencil_kernel(const double* __restrict__ u, double* __restrict__ out, int64_t B,
                                  int64_t ms, int32_t n_m, Shape sh) {
    const int64_t b = blockIdx.y;
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_m) return;
    const double* ub = u + b * ms;
    out[b * ms + q] = delta_at<NDIM>(ub, sh, q, ub[q]);
}

// ------------------------------------------------------------------ host side ---

int validate_plan(const fg_plan* p) {
    if (!p) return fail(FG_ERR_ARG, "plan is NULL");
    if (p->ndim < 1 || p->ndim > 3) return fail(FG_ERR_UNSUPPORTED, "ndim must be 1..3, got %d", p->ndim);
    if (p->B < 1 || p->B > (1 << 24)) return fail(FG_ERR_UNSUPPORTED, "members B out of range");
    if (p->n_m < 3 || p->n_m > (int64_t)1 << 30) return fail(FG_ERR_UNSUPPORTED, "points per member out of range");
    if (p->ms < p->n_m || p->ms % 32) return fail(FG_ERR_ARG, "member stride must be >= n_m and a multiple of 32");
    int64_t prod = 1;
    for (int i = 0; i < p->ndim; ++i) {
        if (p->shape[i] < 3) return fail(FG_ERR_ARG, "every extent must be >= 3");
        prod *= p->shape[i];
    }
    if (prod != p->n_m) return fail(FG_ERR_ARG, "prod(shape) != n_m");
    if (p->kind < 0 || p->kind > 2) return fail(FG_ERR_ARG, "unknown memory kind %d", p->kind);
    if (p->kind == 2 && p->base < 2) return fail(FG_ERR_ARG, "adaptive base must be >= 2");
    if (p->kind == 1 && !p->horizon_dev) return fail(FG_ERR_ARG, "short memory needs horizon_dev");
    if (p->reaction < 0 || p->reaction > 1) return fail(FG_ERR_ARG, "unknown reaction %d", p->reaction);
    if (!p->psi_dev || !p->H_dev || !p->u_dev[0] || !p->u_dev[1] || !p->status_dev || !p->decay_dev ||
        !p->diffuse_dev || !p->dt_dev)
        return fail(FG_ERR_ARG, "plan has a NULL device pointer");
    if (p->split != 0 && p->split != 1 && p->split != 2 && p->split != 4 && p->split != 8)
        return fail(FG_ERR_ARG, "split must be 0, 1, 2, 4 or 8");
    if (p->tblock < 0 || p->tblock > kMaxTBlock || p->tblock % 8 != 0 ||
        (p->tblock > 0 && p->tblock < 32 && p->tblock != 8 && p->tblock != 16 && p->tblock != 24))
        return fail(FG_ERR_ARG, "tblock must be 0, 8, 16, 24 or a multiple of 8 from 32 to %d", kMaxTBlock);
    if (p->tblock > kMaxDenseTBlock && (p->kind != FG_MEM_ADAPTIVE || !p->blkcoef_dev))
        return fail(FG_ERR_UNSUPPORTED, "tblock %d needs an adaptive plan with blkcoef_dev", (int)p->tblock);
    if (p->B > 1 && p->blkcoef_dev && p->kind != FG_MEM_ADAPTIVE)
        return fail(FG_ERR_UNSUPPORTED, "ensemble coefficient rows (blkcoef_dev) are for adaptive plans only");
    if (p->tblock && !p->P_dev) return fail(FG_ERR_ARG, "temporal blocking needs P_dev");
    if (p->subblock < 0 || (p->subblock > 0 && (!p->tblock || p->subblock < 2 || p->tblock % p->subblock != 0 ||
                                                p->tblock / p->subblock > kMaxSub || !p->blkcoef_dev ||
                                                (p->kind != FG_MEM_ADAPTIVE && p->B != 1))))
        return fail(FG_ERR_ARG,
                    "subblock must be 0, or divide tblock into at most %d parts (blkcoef_dev; adaptive or one member)",
                    kMaxSub);
    if (p->subdelay < 0 || p->subdelay > p->subblock)
        return fail(FG_ERR_ARG, "subdelay must be in [0, subblock]");
    if (p->tblock) {  // the block kernel keeps kBlkSegs segments per step
        FgSeg s[FG_MAX_SEGS];
        const int n = fg_segments(p->kind, p->h_slices, p->base, p->horizon_max > 0 ? p->horizon_max : 0, s);
        if (n > kBlkSegs) return fail(FG_ERR_UNSUPPORTED, "schedule has too many segments for temporal blocking");
    }
    return FG_OK;
}

Shape shape_of(const fg_plan* p) {
    Shape s;
    s.n0 = (int32_t)p->shape[0];
    s.n1 = p->ndim >= 2 ? (int32_t)p->shape[1] : 1;
    s.n2 = p->ndim >= 3 ? (int32_t)p->shape[2] : 1;
    return s;
}

int g_sm_count = 0;

int sm_count() {
    if (g_sm_count == 0) {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            g_sm_count = n;
        else
            g_sm_count = 148;
    }
    return g_sm_count;
}

int64_t tile_points(int s) { return (int64_t)((kThreads / 32) / s) * 32 * kVec; }

int64_t tiles_of(const fg_plan* p, int s) {
    const int64_t tp = tile_points(s);
    return ((p->n_m + tp - 1) / tp) * p->B;
}

// Smallest split S whose tile count reaches the resident-CTA capacity
// (148 SMs x kMinBlocks): enough loads in flight in one wave.
int choose_split(const fg_plan* p) {
    if (p->split) return p->split;
    // temporal blocking leaves a step at most tblock-1 recent slices (L2 hits):
    // the step is latency-bound, and one warp group per tile (no split, no
    // combine) is fastest (c2: 93.5 ms per run vs 100.6 ms with S = 4)
    if (p->tblock) return 1;
    const int64_t want = (int64_t)kMinBlocks * sm_count() * 3 / 4;
    for (int s = 1; s <= 8; s *= 2)
        if (tiles_of(p, s) >= want) return s;
    return 8;
}

typedef void (*StepKernel)(const StepArgs);

template <int NDIM, int REACT>
StepKernel pick_s(int s, bool blk) {
    if (blk) return fg_step_kernel<NDIM, REACT, 1, true>;
    switch (s) {
        case 1: return fg_step_kernel<NDIM, REACT, 1, false>;
        case 2: return fg_step_kernel<NDIM, REACT, 2, false>;
        case 4: return fg_step_kernel<NDIM, REACT, 4, false>;
        default: return fg_step_kernel<NDIM, REACT, 8, false>;
    }
}

// blk: a temporal-blocking launch with no warp split (the recent-slice kernel)
StepKernel pick_kernel(int ndim, int react, int s, bool blk = false) {
    blk = blk && s == 1;
    if (ndim == 1) return react ? pick_s<1, 1>(s, blk) : pick_s<1, 0>(s, blk);
    if (ndim == 2) return react ? pick_s<2, 1>(s, blk) : pick_s<2, 0>(s, blk);
    return react ? pick_s<3, 1>(s, blk) : pick_s<3, 0>(s, blk);
}

StepArgs make_args(const fg_plan* p, int s) {
    StepArgs a;
    memset(&a, 0, sizeof a);
    a.u[0] = p->u_dev[0];
    a.u[1] = p->u_dev[1];
    a.H = p->H_dev;
    a.psi = p->psi_dev;
    a.decay = p->decay_dev;
    a.diffuse = p->diffuse_dev;
    a.dt = p->dt_dev;
    a.horizon = p->horizon_dev;
    a.status = p->status_dev;
    a.bar = reinterpret_cast<unsigned long long*>(p->status_dev + 1);
    a.slice_stride = p->B * p->ms;
    a.ms = p->ms;
    a.psi_stride = p->psi_stride;
    a.base = p->base;
    // short memory: the shared schedule covers the longest member horizon; each
    // member then uses its own prefix 0..min(H_b, k)
    a.hz_max = p->horizon_max > 0 ? p->horizon_max : INT64_MAX / 4;
    a.vmax = p->vmax;
    a.km = p->km;
    a.sh = shape_of(p);
    a.n_m = (int32_t)p->n_m;
    a.kind = p->kind;
    const int64_t tp = tile_points(s);
    a.tpm = (int32_t)((p->n_m + tp - 1) / tp);
    a.total_tiles = (int32_t)(a.tpm * p->B);
    a.m0_from_history = (p->step_flags & FG_STEP_M0_FROM_HISTORY) ? 1 : 0;
    a.h_slices = p->h_slices;
    a.tblock = p->tblock;
    a.recent_first = p->B * p->ms * (int64_t)sizeof(double) >= (int64_t)(4 << 20);
    return a;
}

// Partial sums of the block of steps [kb0, kb0+bt) over slices t < kb0 live in
// P[(kb0 / tblock) & 1] (two buffers: the next block's main launch fills one while
// the current block's steps read the other).
double* block_P(const fg_plan* p, int64_t kb0) {
    return p->P_dev + ((kb0 / p->tblock) & 1) * (int64_t)p->tblock * p->B * p->ms;
}

// Coefficient rows of block kb0 (single member): buffer (kb0 / tblock) & 1 of
// blkcoef_dev, h_slices rows of kCoefRow doubles each, so the next block's main
// launch can rebuild its rows while this block's tail launch still reads these.
int64_t coef_capacity(const fg_plan* p) { return (p->coef_rows > 0 ? p->coef_rows : p->h_slices) * kCoefRow; }

// Ensembles (itemized adaptive blocks): [2][B][capacity], member stride = capacity.
double* block_coef(const fg_plan* p, int64_t kb0) {
    return p->blkcoef_dev + ((kb0 / p->tblock) & 1) * p->B * coef_capacity(p);
}

// Recent-weight rows of a temporal block: a.rw[k-kb0][m] = weight of offset m in
// the schedule of step k (1 <= m <= k-kb0), for k in [k0, k1).
// t_min: oldest slice the step still sums itself (kb0, or later when sub-block
// launches have added the older slices of the block into P).
void fill_recent(StepArgs& a, const fg_plan* p, int64_t t_min, int64_t k) {
    a.rn = recent_list(p->kind, k, t_min, p->base, a.hz_max, a.rm, a.rwt, &a.rw1);
    if (p->psi_host && p->B == 1) {  // host doubles round like __dmul_rn (IEEE, no contraction)
        a.has_rc = 1;
        for (int e = 0; e < a.rn; ++e) a.rc[e] = (double)a.rwt[e] * p->psi_host[a.rm[e]];
        a.rc1 = (double)a.rw1 * p->psi_host[1];
        a.rc0 = p->psi_host[0];
    }
}

// Ask for the largest shared-memory carveout for every kernel of the pipeline so
// an SM running two block-kernel CTAs (2 x ~94 KB) is configured with room left
// for a step-kernel CTA; with the default choice the SM is carved to just fit the
// block CTAs and the concurrent steps wait for them to drain.
int prefer_max_smem(const void* fn) {
    static std::mutex mu;
    static std::vector<const void*> done;
    std::lock_guard<std::mutex> lock(mu);
    for (const void* f : done)
        if (f == fn) return FG_OK;
    if (int rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                 (int)cudaSharedmemCarveoutMaxShared),
                            "smem carveout"))
        return rc;
    done.push_back(fn);
    return FG_OK;
}

size_t acc_smem(int s, int passes) { return (size_t)passes * (size_t)((kThreads / 32) / s) * 32 * sizeof(double2); }

// One step, one launch; grid = one CTA per tile.  kb0 >= 0: temporal-blocking
// mode, slices t < kb0 are taken from plan->P_dev (block starting at kb0).
int launch_single(const fg_plan* p, int64_t k, double* snap, cudaStream_t st, int pdl_wait, int pdl_trigger,
                  int64_t kb0 = -1, int64_t t_min = -1) {
    const int s = choose_split(p);
    StepArgs a = make_args(p, s);
    a.k0 = k;
    a.k1 = k + 1;
    a.snap = snap;
    a.passes = 1;
    a.pdl_wait = pdl_wait;
    a.pdl_trigger = pdl_trigger;
    if (kb0 >= 0) {
        a.blocked = 1;
        a.kb0 = kb0;
        a.P = block_P(p, kb0);
        fill_recent(a, p, t_min >= 0 ? t_min : kb0, k);
    }
    StepKernel kern = pick_kernel(p->ndim, p->reaction, s, kb0 >= 0);
    if (int rc = prefer_max_smem((const void*)kern)) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.total_tiles, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = acc_smem(s, 1);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (pdl_wait) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    ++g_launches;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, a), "fg_step launch");
}

// ---- fused step pairs (fg_step2_kernel) -------------------------------------
// Eligible plans: blocked 1D/2D fields whose halo (one row) is at most
// kPairMaxHalo points, one warp column per tile (split 1), adaptive or full
// memory, m = 0 from the stencil, with the caller's pair scratch (pair_dev).
// FG_RUN_NO_PAIRS disables them, FG_RUN_PAIRS enables them in 2D.
bool pairs_enabled(const fg_plan* p, int32_t flags) {
    if ((flags & FG_RUN_NO_PAIRS) || !p->pair_dev) return false;
    if (!p->tblock || p->tblock % 2 || p->ndim > 2 || p->kind == FG_MEM_SHORT || p->subblock) return false;
    if (p->step_flags & FG_STEP_M0_FROM_HISTORY) return false;
    if (choose_split(p) != 1 || tile_points(1) != kPairTile) return false;
    // default on for 1D only: measured on B200, c1 8.13 -> 7.86 ms, but c2 (2D,
    // halo = one 256-point row) 33.4 -> 32.9 ms only — a pair CTA recomputes a
    // halo as large as its tile and needs ~95 registers, so one pair CTA per SM
    // fits beside the block stage and consecutive pairs barely overlap
    if (!(flags & FG_RUN_PAIRS) && p->ndim != 1) return false;
    return (p->ndim == 1 ? 1 : p->shape[1]) <= kPairMaxHalo;
}

constexpr size_t kPairSmem = (size_t)(kPairTile + 4 * kPairMaxHalo + kPairTile + 2 * kPairMaxHalo) * sizeof(double);

// Steps k, k+1 of block kb0 in one launch.
int launch_pair(const fg_plan* p, int64_t k, int64_t kb0, double* snap1, double* snap2, cudaStream_t st,
                int pdl_wait, int pdl_trigger, const double* u_in, double* u_mid, double* u_out, int writes_u3,
                int64_t* u3_step) {
    static thread_local PairArgs A;  // ~3 KB: not on the stack of every caller
    memset(&A, 0, sizeof A);
    StepArgs& a = A.s;
    a = make_args(p, 1);
    a.k0 = k;
    a.k1 = k + 2;
    a.passes = 1;
    a.pdl_wait = pdl_wait;
    a.pdl_trigger = pdl_trigger;
    a.blocked = 1;
    a.kb0 = kb0;
    a.P = block_P(p, kb0);
    fill_recent(a, p, kb0, k);
    StepArgs b2;  // step k+1's list, in a scratch StepArgs
    memset(&b2, 0, sizeof b2);
    b2.hz_max = a.hz_max;
    fill_recent(b2, p, kb0, k + 1);
    A.r2.rn = b2.rn;
    A.r2.rw1 = b2.rw1;
    A.r2.rc0 = b2.rc0;
    A.r2.rc1 = b2.rc1;
    memcpy(A.r2.rm, b2.rm, sizeof A.r2.rm);
    memcpy(A.r2.rwt, b2.rwt, sizeof A.r2.rwt);
    memcpy(A.r2.rc, b2.rc, sizeof A.r2.rc);
    A.u_in = u_in;
    A.u_mid = u_mid;
    A.u_out = u_out;
    A.snap1 = snap1;
    A.snap2 = snap2;
    A.u3_step = u3_step;
    A.writes_u3 = writes_u3;
    void (*kern)(const PairArgs) = nullptr;
    if (p->ndim == 1) kern = p->reaction ? fg_step2_kernel<1, 1> : fg_step2_kernel<1, 0>;
    else kern = p->reaction ? fg_step2_kernel<2, 1> : fg_step2_kernel<2, 0>;
    if (int rc = prefer_max_smem((const void*)kern)) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.total_tiles, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kPairSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (pdl_wait) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    ++g_launches;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, A), "fg_step2 launch");
}

typedef void (*BlockKernel)(const BlockArgs);

struct BlockVariant {
    BlockKernel kern;
    size_t smem;
    int tp;
    int threads;
};

template <int BT, int TP, bool ST, int NS, int WP>
BlockVariant block_variant_tp() {
    return {fg_block_tma_kernel<BT, TP, ST, NS, WP>, tma_block_smem<BT, TP, ST, NS, WP>(), TP, TP / WP * 32 + 32};
}

template <int BT, bool ST, int NS>
BlockVariant block_variant(int tp) {
    constexpr int WP = 32;  // 16-point warps at TP 128 measured slower (c4-full 1.58 vs 1.41 s)
    switch (tp) {
        case 128: return block_variant_tp<BT, 128, ST, NS, WP>();
        case 192: return block_variant_tp<BT, 192, ST, NS, WP>();
        case 224: return block_variant_tp<BT, 224, ST, NS, WP>();
        default: return block_variant_tp<BT, 256, ST, NS, WP>();
    }
}

// Tile width: the block kernel is bound per SM (fp64 tensor pipe + its share of
// HBM), so pick the TP (32-point warps, 4..8 per CTA) that minimises the work of
// the busiest SM, ceil(tiles / SMs) * TP; c2 (65536 points) gets 293 tiles of
// 224 instead of 256 tiles of 256 that leave 40 SMs half idle.
template <int BT>
BlockVariant block_variant_of(bool staged, bool tail, int tp) {
    if (tail) return staged ? block_variant<BT, true, kTailStages>(tp) : block_variant<BT, false, kTailStages>(tp);
    constexpr int main_ns = kMainStages * kE / dense_ke<BT>(), ens_ns = ring_stages<false>() * kE / dense_ke<BT>();
    return staged ? block_variant<BT, true, main_ns>(tp) : block_variant<BT, false, (ens_ns > 2 ? ens_ns : 2)>(tp);
}

// tail: the variant with the small ring (see kTailStages)
BlockVariant choose_block_variant(const fg_plan* p, bool tail = false) {
    const int cands[4] = {256, 224, 192, 128};
    const bool staged = p->B == 1 && p->blkcoef_dev;
    BlockVariant best = {nullptr, 0, 0, 0};
    auto cost_of = [&](int tp) {
        const int64_t tiles = ((p->n_m + tp - 1) / tp) * p->B;
        return ((tiles + sm_count() - 1) / sm_count()) * tp;
    };
    int64_t min_cost = INT64_MAX;
    for (int tp : cands)
        if (cost_of(tp) < min_cost) min_cost = cost_of(tp);
    // the widest tile within 2 % of the best balance: a wider CTA shares its
    // stage barrier and coefficient rows over more warps (measured c3-full at
    // tblock 32: TP 224 705 ms vs TP 192 792 ms, nearly equal balance; TP 256,
    // 16 consumer warps per SM: 662 vs 678 ms at TP 224, c4-full 1386 vs 1411 ms)
    bool found = false;
    for (int tp : cands) {
        if (found) continue;
        if (cost_of(tp) * 50 <= min_cost * 51) {
            found = true;
            switch (p->tblock) {
                case 8: best = block_variant_of<8>(staged, tail, tp); break;
                case 24: best = block_variant_of<24>(staged, tail, tp); break;
                case 32: best = block_variant_of<32>(staged, tail, tp); break;
                default: best = block_variant_of<16>(staged, tail, tp); break;
            }
        }
    }
    return best;
}

// Block-kernel grid: ensembles one CTA per tile; single members two CTAs per SM
// looping over tiles (one wave; two step CTAs still fit beside them per SM).
unsigned block_grid(const fg_plan* p, int64_t total_tiles) {
    if (p->B != 1) return (unsigned)total_tiles;
    const int64_t cap = (int64_t)sm_count() * 2;
    return (unsigned)(total_tiles < cap ? total_tiles : cap);
}

int64_t history_alloc(const fg_plan* p) { return p->h_alloc > p->h_slices ? p->h_alloc : p->h_slices; }

BlockArgs block_args(const fg_plan* p, int64_t kb0, int bt, const BlockVariant& v) {
    BlockArgs a;
    memset(&a, 0, sizeof a);
    a.H = p->H_dev;
    a.P = block_P(p, kb0);
    a.psi = p->psi_dev;
    a.horizon = p->horizon_dev;
    a.slice_stride = p->B * p->ms;
    a.ms = p->ms;
    a.psi_stride = p->psi_stride;
    a.base = p->base;
    a.kb0 = kb0;
    a.bt = bt;
    a.n_m = (int32_t)p->n_m;
    a.kind = p->kind;
    a.tpm = (int32_t)((p->n_m + v.tp - 1) / v.tp);
    a.total_tiles = (int32_t)(a.tpm * p->B);
    a.gcoef = p->blkcoef_dev ? block_coef(p, kb0) : nullptr;
    a.coef_mstride = coef_capacity(p);
    a.h_alloc = history_alloc(p);
    a.tblock = p->tblock;
    return a;
}

// Item table of block (kb0, bt) over slices [ts, te) (single member; see
// fg_block_item_kernel).  Returns false when it does not fit the table or the
// scratch buffers, and the caller uses the dense kernel.
// Item width of a plan: plan->item_cols if set (8 or 16), else
// FGB200_ITEM_COLS, else 16 for ensembles and 8 for a single member.
int item_cols(const fg_plan* p) {
    if (p->item_cols == 8 || p->item_cols == 16) return p->item_cols;
    return p->B > 1 ? 16 : 8;
}

bool build_items(const fg_plan* p, int64_t kb0, int bt, int64_t ts, int64_t te, ItemTable& T, int64_t row0,
                 int b_lo = 0) {
    memset(&T, 0, sizeof T);
    if (te <= ts) return true;  // no old slices: n_items = 0
    const int64_t hz = p->kind == 1 ? p->horizon_max : 0;
    // groups: same stride and residue, slice ranges within a few strides of
    // each other (a far-apart range of the same class starts a new group)
    struct Grp {
        int64_t s, r, tmin, tmax;
        int n;
        uint8_t cols[kMaxTBlock];
        int64_t clo[kMaxTBlock], chi[kMaxTBlock];  // slice range of each column's entries in this group
    };
    static thread_local Grp g[kMaxItems];
    int ng = 0;
    FgSeg segs[FG_MAX_SEGS];
    for (int b = b_lo; b < bt; ++b) {  // b_lo: sub-block launches feed only the later steps
        const int64_t k = kb0 + b;
        const int ns = fg_segments(p->kind, k, p->base, hz, segs);
        if (ns < 0 || ns > kBlkSegs) return false;  // the coefficient kernel keeps kBlkSegs
        for (int si = 0; si < ns; ++si) {
            const int64_t m0 = segs[si].m0, st = segs[si].stride, cnt = segs[si].count;
            const int64_t m_min = k - te + 1, m_max = k - ts;  // t = k - m in [ts, te)
            if (m_max < m0 || m_min > m0 + (cnt - 1) * st) continue;
            const int64_t i0 = m_min > m0 ? (m_min - m0 + st - 1) / st : 0;
            const int64_t i1 = (m_max - m0) / st < cnt - 1 ? (m_max - m0) / st : cnt - 1;
            if (i0 > i1) continue;
            const int64_t t_hi = k - (m0 + i0 * st), t_lo = k - (m0 + i1 * st);
            const int64_t r = t_lo % st, gap = 8 * st;
            int x = -1;
            for (int q = 0; q < ng; ++q)
                if (g[q].s == st && g[q].r == r && t_lo <= g[q].tmax + gap && t_hi >= g[q].tmin - gap) {
                    x = q;
                    break;
                }
            if (x < 0) {
                if (ng == kMaxItems) return false;
                x = ng++;
                g[x].s = st;
                g[x].r = r;
                g[x].tmin = t_lo;
                g[x].tmax = t_hi;
                g[x].n = 0;
            } else {
                g[x].tmin = t_lo < g[x].tmin ? t_lo : g[x].tmin;
                g[x].tmax = t_hi > g[x].tmax ? t_hi : g[x].tmax;
            }
            if (g[x].n == 0 || g[x].cols[g[x].n - 1] != b) {
                g[x].clo[g[x].n] = t_lo;
                g[x].chi[g[x].n] = t_hi;
                g[x].cols[g[x].n++] = (uint8_t)b;
            } else {
                const int c = g[x].n - 1;
                g[x].clo[c] = t_lo < g[x].clo[c] ? t_lo : g[x].clo[c];
                g[x].chi[c] = t_hi > g[x].chi[c] ? t_hi : g[x].chi[c];
            }
        }
    }
    // A class's groups must own disjoint slice ranges: the coefficient rows give
    // an entry (step, t) to every item whose range holds t and whose columns hold
    // the step, so two overlapping groups of one class would both add it.  A
    // group can grow into another after both exist (adaptive tail-rule entries
    // near t = 0 start a group that the dense window later reaches), so merge
    // overlapping groups of a class (ranges and sorted column sets) to a fixpoint.
    for (bool merged = true; merged;) {
        merged = false;
        for (int x = 0; x < ng && !merged; ++x)
            for (int y = x + 1; y < ng && !merged; ++y) {
                if (g[x].s != g[y].s || g[x].r != g[y].r || g[y].tmin > g[x].tmax || g[x].tmin > g[y].tmax) continue;
                uint8_t cols[kMaxTBlock];
                int64_t lo[kMaxTBlock], hi[kMaxTBlock];
                int n = 0, i = 0, j = 0;
                while (i < g[x].n || j < g[y].n) {
                    const int cx = i < g[x].n ? g[x].cols[i] : 1 << 30, cy = j < g[y].n ? g[y].cols[j] : 1 << 30;
                    const int c = cx < cy ? cx : cy;
                    lo[n] = INT64_MAX;
                    hi[n] = INT64_MIN;
                    if (cx == c) {
                        lo[n] = g[x].clo[i];
                        hi[n] = g[x].chi[i];
                        ++i;
                    }
                    if (cy == c) {
                        lo[n] = g[y].clo[j] < lo[n] ? g[y].clo[j] : lo[n];
                        hi[n] = g[y].chi[j] > hi[n] ? g[y].chi[j] : hi[n];
                        ++j;
                    }
                    cols[n++] = (uint8_t)c;
                }
                memcpy(g[x].cols, cols, (size_t)n);
                memcpy(g[x].clo, lo, sizeof(int64_t) * n);
                memcpy(g[x].chi, hi, sizeof(int64_t) * n);
                g[x].n = n;
                g[x].tmin = g[y].tmin < g[x].tmin ? g[y].tmin : g[x].tmin;
                g[x].tmax = g[y].tmax > g[x].tmax ? g[y].tmax : g[x].tmax;
                g[y] = g[--ng];
                merged = true;
            }
    }
    // one dense class holding every step (full / short memory): the dense kernel
    // streams it once for all steps; items would re-read it per 8 steps
    // (above kMaxDenseTBlock there is no dense kernel: items it is, each re-reading)
    const int icols = item_cols(p), pitch = icols == 8 ? kItemPitch8 : kItemPitch;
    T.cols = icols;
    T.pitch = pitch;
    if (ng == 1 && g[0].s == 1 && g[0].n == bt && bt > icols && p->tblock <= kMaxDenseTBlock) return false;
    int n = 0;
    int64_t crow = row0;
    for (int x = 0; x < ng; ++x) {
        for (int c0 = 0; c0 < g[x].n; c0 += icols) {
            if (n == kMaxItems) return false;
            BlockItem& it = T.it[n++];
            it.stride = (int32_t)g[x].s;
            it.ncols = g[x].n - c0 < icols ? g[x].n - c0 : icols;
            // the item streams only the slices its own steps use (an 8-step item of
            // a dense class spans its steps' windows, not the whole group)
            int64_t lo = INT64_MAX, hi = INT64_MIN;
            for (int c = 0; c < it.ncols; ++c) {
                it.col2step[c] = g[x].cols[c0 + c];
                lo = g[x].clo[c0 + c] < lo ? g[x].clo[c0 + c] : lo;
                hi = g[x].chi[c0 + c] > hi ? g[x].chi[c0 + c] : hi;
            }
            it.t_first = lo;
            it.n_slices = (int32_t)((hi - lo) / g[x].s + 1);
            it.coef_row = (int32_t)crow;
            crow += it.n_slices;
        }
    }
    T.n_items = n;
    uint64_t seen[kMaxTBlock / 64] = {};
    for (int x = 0; x < n; ++x) {
        BlockItem& it = T.it[x];
        for (int c = 0; c < it.ncols; ++c) {
            const int w = it.col2step[c] >> 6;
            const uint64_t bit = 1ull << (it.col2step[c] & 63);
            if (!(seen[w] & bit)) it.first_mask |= 1 << c;
            seen[w] |= bit;
        }
    }
    for (int w = 0; w < kMaxTBlock / 64; ++w) {
        const int nb = bt - 64 * w;  // steps of the block in this word
        T.zero_mask[w] = ~seen[w] & (nb >= 64 ? ~0ull : nb <= 0 ? 0ull : ((1ull << nb) - 1));
    }
    if (crow * pitch > coef_capacity(p)) return false;
    return true;
}

int launch_item_coef(const BlockArgs& a, const ItemTable& T, cudaStream_t st) {
    if (T.n_items == 0) return FG_OK;
    int max_rows = 0;
    for (int x = 0; x < T.n_items; ++x) max_rows = T.it[x].n_slices > max_rows ? T.it[x].n_slices : max_rows;
    const int cx = (max_rows * T.pitch + 255) / 256;
    const int64_t B = a.total_tiles / a.tpm;
    ++g_launches;
    fg_item_coef_kernel<<<dim3((unsigned)(cx < 16 ? cx : 16), (unsigned)T.n_items, (unsigned)(B < 64 ? B : 64)),
                          256, 0, st>>>(a, T, const_cast<double*>(a.gcoef), B);
    return cuda_check(cudaGetLastError(), "fg_item_coef launch");
}

// Item partial sums (coefficient rows already built) into Q, then the ordered
// reduction into P (or directly into P for a single all-steps item).
#ifndef FG_ITEM_STAGES
#define FG_ITEM_STAGES (64 / FG_ITEM_ROWS)
#endif
constexpr int kItemMainStages = FG_ITEM_STAGES;  // two main CTAs per SM: 64 slice rows of ring each
constexpr int kItemTailStages = 24 / kIR > 2 ? 24 / kIR : 2;  // tail launches run beside the main CTAs

// Item-kernel tile width: two CTAs per SM (two independent rings, so one
// CTA's flushes overlap the other's stream), so pick the TP (16-point warps)
// that minimises the busiest CTA's points, ceil(tiles / (2 SMs)) * TP (c2: 586
// tiles of 112 = 2 per CTA; ensembles of 512-point members: 128, no partial tiles).
int choose_item_tp(const fg_plan* p) {
    const int cands[2] = {128, 96};  // the 16-column kernel's swizzled box geometries
    int best = 128;
    int64_t best_cost = INT64_MAX;
    for (int tp : cands) {
        const int64_t tiles = ((p->n_m + tp - 1) / tp) * p->B;
        const int64_t cost = ((tiles + 2 * sm_count() - 1) / (2 * sm_count())) * tp;
        if (cost < best_cost) {
            best_cost = cost;
            best = tp;
        }
    }
    return best;
}

// Item partial sums (coefficient rows already built) straight into P.
// 8-column tables: fg_block_item8_kernel on the dense kernel's tiling (`a` as
// built by block_args, TP = tp8), two CTAs per SM.
int launch_item8_sums(const fg_plan* p, const BlockArgs& a, const ItemTable& T, int tp, cudaStream_t st, bool tail) {
    void (*kern)(const BlockArgs, const ItemTable) = nullptr;
    size_t smem = 0;
    const bool ens = p->B > 1;
#define FG_ITEM8_PICK(TPV)                                                                                    \
    kern = tail ? (ens ? fg_block_item8_kernel<TPV, kTailStages, true> : fg_block_item8_kernel<TPV, kTailStages, false>) \
                : (ens ? fg_block_item8_kernel<TPV, kMainStages, true> : fg_block_item8_kernel<TPV, kMainStages, false>); \
    smem = tail ? item8_block_smem<TPV, kTailStages>() : item8_block_smem<TPV, kMainStages>();
    switch (tp) {
        case 128: FG_ITEM8_PICK(128) break;
        case 192: FG_ITEM8_PICK(192) break;
        case 224: FG_ITEM8_PICK(224) break;
        default: FG_ITEM8_PICK(256) tp = 256; break;
    }
#undef FG_ITEM8_PICK
    if (int rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                            "item smem attribute"))
        return rc;
    if (int rc = prefer_max_smem((const void*)kern)) return rc;
    const int64_t cap = (int64_t)sm_count() * 2;
    ++g_launches;
    kern<<<(unsigned)(a.total_tiles < cap ? a.total_tiles : cap), tp + 32, smem, st>>>(a, T);
    return cuda_check(cudaGetLastError(), "fg_block_item8 launch");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the library
// links the runtime statically and not libcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}


// Tensor maps of the table's strides (ItemMaps) and each item's map index.  A
// stage box reads kE slices of the item's progression, so its last stage may
// read up to kE - 1 strides past the item's last slice: the history allocation
// must cover that (fg_history_pad), else the launch fails.
int encode_item_maps(const fg_plan* p, ItemTable& T, int tp, ItemMaps& M) {
    const PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return fail(FG_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    const int64_t halloc = history_alloc(p);
    const cuuint64_t slice_bytes = (cuuint64_t)(p->B * p->ms) * sizeof(double);
    int strides[kMaxMaps];
    int nm = 0;
    for (int x = 0; x < T.n_items; ++x) {
        BlockItem& it = T.it[x];
        const int64_t s = it.stride;
        const int64_t j_end = it.t_first / s + ((int64_t)(it.n_slices + kIR - 1) / kIR) * kIR;  // boxes end (exclusive)
        if (j_end > halloc / s)
            return fail(FG_ERR_ARG,
                        "history allocation of %lld slices is too small for the item stream: stride %lld reads "
                        "up to slice %lld (allocate h_slices + fg_history_pad slices, fg_plan.h_alloc)",
                        (long long)halloc, (long long)s, (long long)(j_end * s - 1));
        int m = 0;
        while (m < nm && strides[m] != (int)s) ++m;
        if (m == nm) {
            if (nm == kMaxMaps) return fail(FG_ERR_UNSUPPORTED, "more than %d item strides in one block", kMaxMaps);
            strides[nm++] = (int)s;
            const cuuint64_t dims[4] = {16, (cuuint64_t)(p->B * p->ms / 16), (cuuint64_t)s, (cuuint64_t)(halloc / s)};
            const cuuint64_t gstride[3] = {128, slice_bytes, (cuuint64_t)s * slice_bytes};
            const cuuint32_t box[4] = {16, (cuuint32_t)(tp == 96 ? item_box_chunks<96>() : item_box_chunks<128>()),
                                       1, (cuuint32_t)kIR};
            const cuuint32_t estride[4] = {1, 1, 1, 1};
            CUresult r = enc(&M.map[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)p->H_dev, dims, gstride, box,
                             estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            for (int h = 0; h < 2 && r == CUDA_SUCCESS; ++h) {
                const cuuint32_t hbox[4] = {box[0], box[1], 1, (cuuint32_t)(kIR / (2 << h))};
                r = enc(h ? &M.quarter[m] : &M.half[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)p->H_dev, dims,
                        gstride, hbox, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (r != CUDA_SUCCESS)
                return fail(FG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for stride %lld", (int)r, (long long)s);
        }
        it.map = (uint8_t)m;
    }
    return FG_OK;
}

int launch_item_sums(const fg_plan* p, const BlockArgs& a, ItemTable& T, int tp, cudaStream_t st,
                     bool tail = false) {
    void (*kern)(const BlockArgs, const ItemTable, const ItemMaps) = nullptr;
    size_t smem = 0;
    int threads = 0;
    const bool ens = p->B > 1;
#define FG_ITEM_PICK(TPV)                                                                                  \
    kern = tail ? (ens ? fg_block_item_kernel<TPV, kItemTailStages, true>                                  \
                       : fg_block_item_kernel<TPV, kItemTailStages, false>)                                \
                : (ens ? fg_block_item_kernel<TPV, kItemMainStages, true>                                  \
                       : fg_block_item_kernel<TPV, kItemMainStages, false>);                               \
    smem = tail ? item_block_smem<TPV, kItemTailStages>() : item_block_smem<TPV, kItemMainStages>();       \
    threads = item_threads<TPV>();
    switch (tp) {
        case 96: FG_ITEM_PICK(96) break;
        case 128: FG_ITEM_PICK(128) break;
        default: return fail(FG_ERR_ARG, "item kernel: unsupported tile width %d", tp);
    }
#undef FG_ITEM_PICK
    if (tp * a.tpm < a.n_m || a.tpm * (a.total_tiles / a.tpm) != a.total_tiles)
        return fail(FG_ERR_ARG, "item kernel: tiles do not match the tile width");
    if (int rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                            "item smem attribute"))
        return rc;
    if (int rc = prefer_max_smem((const void*)kern)) return rc;
    // two CTAs per SM (FGB200_BLOCK_CTAS_PER_SM) loop over tiles and walk all
    // items per tile: a CTA owns its tile's P rows, so the items' adds need no atomics
    const int64_t cap = (int64_t)sm_count() * 2;
    ItemMaps M;
    if (int rc = encode_item_maps(p, T, tp, M)) return rc;
    ++g_launches;
    kern<<<(unsigned)(a.total_tiles < cap ? a.total_tiles : cap), threads, smem, st>>>(a, T, M);
    return cuda_check(cudaGetLastError(), "fg_block_item launch");
}

// Dense coefficient rows (fg_block_coef_kernel) of slices [a.t_begin, a.t_end)
// at a.gcoef, zeroed first.
int launch_dense_coef(const fg_plan* p, const BlockArgs& a, cudaStream_t st) {
    const int64_t hz = p->kind == 1 ? p->horizon_max : 0;
    const int64_t t_lo = (p->kind == 1 && a.kb0 - hz > 0) ? a.kb0 - hz : 0;
    const int64_t ts = a.t_begin > t_lo ? a.t_begin : t_lo;
    if (a.t_end <= ts) return FG_OK;
    const size_t cp = (size_t)p->tblock + 4;  // coef_pitch<tblock>()
    double* rows = const_cast<double*>(a.gcoef);
    if (int rc = cuda_check(cudaMemsetAsync(rows, 0, (size_t)(a.t_end - ts) * cp * sizeof(double), st),
                            "coefficient rows reset"))
        return rc;
    switch (p->tblock) {
        case 8: ++g_launches; fg_block_coef_kernel<8><<<a.bt, 256, 0, st>>>(a, rows); break;
        case 24: ++g_launches; fg_block_coef_kernel<24><<<a.bt, 256, 0, st>>>(a, rows); break;
        case 32: ++g_launches; fg_block_coef_kernel<32><<<a.bt, 256, 0, st>>>(a, rows); break;
        default: ++g_launches; fg_block_coef_kernel<16><<<a.bt, 256, 0, st>>>(a, rows); break;
    }
    return cuda_check(cudaGetLastError(), "fg_block_coef launch");
}


// Tail launches of factors above kMaxDenseTBlock are itemized too (the dense
// kernel's accumulators would not fit).
// Itemized ensembles (blkcoef_dev given) itemize their tails as well; when a
// tail does not fit the item table they fall back to the dense kernel, which
// builds per-member coefficient tables in the CTA.
bool item_tail(const fg_plan* p) {
    return p->tblock > kMaxDenseTBlock || (p->B > 1 && p->blkcoef_dev);
}

int64_t tail_begin(const fg_plan* p, int64_t kb0) { return kb0 - p->tblock > 0 ? kb0 - p->tblock : 0; }

// main launch: P = Σ over slices t < kb0 - tblock (all but the previous block's).
// Everything it reads is final once the previous block starts, so fg_run
// issues it on a side stream while the previous block's steps run.  Single
// member: coefficient buffer = [tail rows][main rows]; the tail's rows are
// built here too so the tail launch (on the critical path) only multiplies.
// The item kernel's own tiling of the same block arguments.
BlockArgs item_args(const fg_plan* p, const BlockArgs& a, int* tp) {
    BlockArgs r = a;
    *tp = choose_item_tp(p);
    r.tpm = (int32_t)((p->n_m + *tp - 1) / *tp);
    r.total_tiles = (int32_t)(r.tpm * p->B);
    return r;
}

int launch_block_main(const fg_plan* p, int64_t kb0, int bt, cudaStream_t st) {
    if (kb0 <= 0) {  // nothing older than the block: P = 0
        return cuda_check(cudaMemsetAsync(block_P(p, kb0), 0, (size_t)p->tblock * p->B * p->ms * sizeof(double), st),
                          "P reset");
    }
    const BlockVariant v = choose_block_variant(p);
    if (!v.kern) return fail(FG_ERR_ARG, "no block-kernel variant for FGB200_BLOCK_TP");
    BlockArgs a = block_args(p, kb0, bt, v);
    a.t_begin = 0;
    a.t_end = tail_begin(p, kb0);
    if (a.gcoef) {
        const bool ens = p->B > 1;  // ensembles: per-member item rows, no staged dense rows
        int64_t row0 = 0;  // main rows start after the tail's (in item-pitch rows when itemized)
        BlockArgs tail = a;
        tail.t_begin = tail_begin(p, kb0);
        tail.t_end = kb0;
        if (item_tail(p)) {
            ItemTable Tt;
            if (build_items(p, kb0, bt, tail.t_begin, tail.t_end, Tt, 0)) {
                if (int rc = launch_item_coef(tail, Tt, st)) return rc;
                for (int x = 0; x < Tt.n_items; ++x) row0 += Tt.it[x].n_slices;
            } else if (!ens || p->tblock > kMaxDenseTBlock) {
                return fail(FG_ERR_UNSUPPORTED, "tblock %d: tail of block %lld does not fit the item table",
                            (int)p->tblock, (long long)kb0);
            }  // else: the dense tail launch builds its own tables
        } else {
            if (int rc = launch_dense_coef(p, tail, st)) return rc;
            const int64_t cp = p->tblock + 4;
            const int ip = item_cols(p) == 8 ? kItemPitch8 : kItemPitch;
            row0 = (p->tblock * cp + ip - 1) / ip;  // dense tail rows, in item-pitch rows
        }
        ItemTable T;
        if (build_items(p, kb0, bt, 0, a.t_end, T, row0)) {
            if (T.n_items == 0)
                return cuda_check(
                    cudaMemsetAsync(block_P(p, kb0), 0, (size_t)p->tblock * p->B * p->ms * sizeof(double), st),
                    "P reset");
            if (T.cols == 8) {
                if (int rc = launch_item_coef(a, T, st)) return rc;
                return launch_item8_sums(p, a, T, v.tp, st, false);
            }
            int itp = 0;
            const BlockArgs ai = item_args(p, a, &itp);
            if (int rc = launch_item_coef(ai, T, st)) return rc;
            return launch_item_sums(p, ai, T, itp, st);
        }
        if (p->tblock > kMaxDenseTBlock)
            return fail(FG_ERR_UNSUPPORTED, "tblock %d: block %lld does not fit the item table", (int)p->tblock,
                        (long long)kb0);
        if (!ens) {
            a.gcoef += row0 * (item_cols(p) == 8 ? kItemPitch8 : kItemPitch);
            if (int rc = launch_dense_coef(p, a, st)) return rc;
        }
    }
    if (int rc = cuda_check(cudaFuncSetAttribute(v.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem),
                            "block smem attribute"))
        return rc;
    if (int rc = prefer_max_smem((const void*)v.kern)) return rc;
    ++g_launches;
    v.kern<<<block_grid(p, a.total_tiles), v.threads, v.smem, st>>>(a);
    return cuda_check(cudaGetLastError(), "fg_block_tma launch");
}

// tail launch: P += Σ over the previous block's slices [kb0 - tblock, kb0), in
// stream order after that block's last step and this block's main launch.
int launch_block_tail(const fg_plan* p, int64_t kb0, int bt, cudaStream_t st) {
    if (kb0 <= 0) return FG_OK;
    const BlockVariant v = choose_block_variant(p, true);
    if (!v.kern) return fail(FG_ERR_ARG, "no block-kernel variant for FGB200_BLOCK_TP");
    BlockArgs a = block_args(p, kb0, bt, v);
    a.t_begin = tail_begin(p, kb0);
    a.t_end = kb0;
    a.accumulate = 1;
    if (item_tail(p)) {
        ItemTable T;
        if (build_items(p, kb0, bt, a.t_begin, a.t_end, T, 0)) {
            if (T.n_items == 0) return FG_OK;
            T.accumulate = 1;
            if (T.cols == 8) return launch_item8_sums(p, a, T, v.tp, st, true);
            int itp = 0;
            const BlockArgs ai = item_args(p, a, &itp);
            return launch_item_sums(p, ai, T, itp, st, true);
        }
        if (p->B == 1 || p->tblock > kMaxDenseTBlock)
            return fail(FG_ERR_UNSUPPORTED, "tblock %d: tail of block %lld does not fit the item table",
                        (int)p->tblock, (long long)kb0);
    }
    if (int rc = cuda_check(cudaFuncSetAttribute(v.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem),
                            "block smem attribute"))
        return rc;
    if (int rc = prefer_max_smem((const void*)v.kern)) return rc;
    ++g_launches;
    v.kern<<<block_grid(p, a.total_tiles), v.threads, v.smem, st>>>(a);
    return cuda_check(cudaGetLastError(), "fg_block_tma tail launch");
}

// Steps of a block that sub-block i's launch feeds: b >= (i+1)S + D (D =
// plan->subdelay, default S: the launch has one sub-block of steps to finish).
int64_t sub_delay(const fg_plan* p) { return p->subdelay > 0 ? p->subdelay : p->subblock; }
int64_t sub_first_step(const fg_plan* p, int i) { return (i + 1) * p->subblock + sub_delay(p); }

// Sub-block launch (plan->subblock = S > 0): the slices of sub-block i of the
// block kb0, [kb0 + iS, kb0 + (i+1)S), added into the P rows of the block's
// steps b >= (i+2)S.  Those steps then sum themselves only the slices of their
// own and the previous sub-block (recent offsets < 2S instead of < tblock), so
// a slice of a large field is streamed once by this launch instead of once by
// every later step of the block.  Runs on the library's sub-block stream while
// sub-block i+1's steps run; sub-block i+2 joins it.  Coefficient rows reuse
// the block's buffer from row 0 (its tail and main launches are done).
int launch_block_partial(const fg_plan* p, int64_t kb0, int bt, int i, cudaStream_t st) {
    const int64_t S = p->subblock;
    const int b_lo = (int)sub_first_step(p, i);
    if (b_lo >= bt) return FG_OK;
    const BlockVariant v = choose_block_variant(p, true);
    if (!v.kern) return fail(FG_ERR_ARG, "no block-kernel variant for FGB200_BLOCK_TP");
    BlockArgs a = block_args(p, kb0, bt, v);
    a.t_begin = kb0 + i * S;
    a.t_end = kb0 + (i + 1) * S;
    a.accumulate = 1;
    ItemTable T;
    if (!a.gcoef || !build_items(p, kb0, bt, a.t_begin, a.t_end, T, 0, b_lo))
        return fail(FG_ERR_UNSUPPORTED, "sub-block %d of block %lld does not fit the item table", i, (long long)kb0);
    if (T.n_items == 0) return FG_OK;
    T.accumulate = 1;
    if (T.cols == 8) {
        if (int rc = launch_item_coef(a, T, st)) return rc;
        return launch_item8_sums(p, a, T, v.tp, st, true);
    }
    int itp = 0;
    const BlockArgs ai = item_args(p, a, &itp);
    if (int rc = launch_item_coef(ai, T, st)) return rc;
    return launch_item_sums(p, ai, T, itp, st, true);
}

// Per-thread sub-block stream and its events (one completion event per
// sub-block of a block, kMaxSub at most).
int sub_stream(cudaStream_t* s, cudaEvent_t* ready, cudaEvent_t* done) {
    static thread_local int dev = -1;
    static thread_local cudaStream_t ss = nullptr;
    static thread_local cudaEvent_t er = nullptr, ed[kMaxSub] = {};
    int cur = 0;
    if (int rc = cuda_check(cudaGetDevice(&cur), "cudaGetDevice")) return rc;
    if (!ss || dev != cur) {
        if (int rc = cuda_check(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking), "sub-block stream")) return rc;
        if (int rc = cuda_check(cudaEventCreateWithFlags(&er, cudaEventDisableTiming), "sub-block event")) return rc;
        for (int i = 0; i < kMaxSub; ++i)
            if (int rc = cuda_check(cudaEventCreateWithFlags(&ed[i], cudaEventDisableTiming), "sub-block event"))
                return rc;
        dev = cur;
    }
    *s = ss;
    *ready = er;
    for (int i = 0; i < kMaxSub; ++i) done[i] = ed[i];
    return FG_OK;
}

// Debug timeline of the temporal-blocking pipeline (FGB200_TRACE=<file>, not in
// graph mode): per block, timed events at its start (0), after the join (1),
// after its tail (2), and around the next block's main launch on the side
// stream (3, 4); fg_run synchronises at the end and appends one line per block.
struct BlockTrace {
    const char* path;
    std::vector<int64_t> kb;
    std::vector<cudaEvent_t> ev;  // 5 per block
    explicit BlockTrace(const char* p) : path(p) {}
    void mark(int64_t k, int slot, cudaStream_t s) {
        if (!path) return;
        if (kb.empty() || kb.back() != k) {
            kb.push_back(k);
            ev.resize(ev.size() + 5, nullptr);
        }
        cudaEvent_t& e = ev[(kb.size() - 1) * 5 + slot];
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
    }
    void dump(cudaStream_t s) {
        if (!path || kb.empty()) return;
        cudaEvent_t fin;
        cudaEventCreate(&fin);
        cudaEventRecord(fin, s);
        cudaEventSynchronize(fin);
        cudaDeviceSynchronize();
        FILE* f = fopen(path, "a");
        auto ms = [](cudaEvent_t a, cudaEvent_t b) {
            float t = 0.f;
            if (a && b) cudaEventElapsedTime(&t, a, b);
            return t * 1e3f;
        };
        for (size_t i = 0; f && i < kb.size(); ++i) {
            cudaEvent_t* e = &ev[i * 5];
            cudaEvent_t next = i + 1 < kb.size() ? ev[(i + 1) * 5] : fin;
            fprintf(f, "%lld t=%.1f wait=%.1f tail=%.1f steps=%.1f main_next=%.1f\n", (long long)kb[i],
                    ms(ev[0], e[0]), ms(e[0], e[1]), ms(e[1], e[2]), ms(e[2], next), ms(e[3], e[4]));
        }
        if (f) fclose(f);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        cudaEventDestroy(fin);
    }
};


// Per-thread side stream (lowest priority, so the latency-bound steps win SM
// slots as they free) and its fork/join events, on the current device.
int side_stream(cudaStream_t* s, cudaEvent_t* fork, cudaEvent_t* join) {
    static thread_local int dev = -1;
    static thread_local cudaStream_t side = nullptr;
    static thread_local cudaEvent_t ef = nullptr, ej[2] = {nullptr, nullptr};
    int cur = 0;
    if (int rc = cuda_check(cudaGetDevice(&cur), "cudaGetDevice")) return rc;
    if (!side || dev != cur) {
        int least = 0, greatest = 0;
        if (int rc = cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range")) return rc;
        if (int rc = cuda_check(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, least), "side stream"))
            return rc;
        if (int rc = cuda_check(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming), "fork event")) return rc;
        for (int i = 0; i < 2; ++i)
            if (int rc = cuda_check(cudaEventCreateWithFlags(&ej[i], cudaEventDisableTiming), "join event")) return rc;
        dev = cur;
    }
    *s = side;
    *fork = ef;
    join[0] = ej[0];
    join[1] = ej[1];
    return FG_OK;
}

// Per-thread device-to-host copy stream for fg_run_ex snapshots.
int copy_stream(cudaStream_t* s, cudaEvent_t* ev, cudaEvent_t* join) {
    static thread_local int dev = -1;
    static thread_local cudaStream_t cs = nullptr;
    static thread_local cudaEvent_t e0 = nullptr, e1 = nullptr;
    int cur = 0;
    if (int rc = cuda_check(cudaGetDevice(&cur), "cudaGetDevice")) return rc;
    if (!cs || dev != cur) {
        if (int rc = cuda_check(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "copy stream")) return rc;
        if (int rc = cuda_check(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming), "copy event")) return rc;
        if (int rc = cuda_check(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming), "copy event")) return rc;
        dev = cur;
    }
    *s = cs;
    *ev = e0;
    *join = e1;
    return FG_OK;
}

int launch_block(const fg_plan* p, int64_t kb0, int bt, cudaStream_t st) {
    if (int rc = launch_block_main(p, kb0, bt, st)) return rc;
    return launch_block_tail(p, kb0, bt, st);
}

// Persistent geometry: G co-resident CTAs, `passes` tiles each.  Returns 0 and
// leaves *G = 0 if the cooperative grid cannot be co-resident.
int persistent_geometry(const fg_plan* p, int s, int* G, int* passes) {
    *G = 0;
    *passes = 0;
    StepKernel kern = pick_kernel(p->ndim, p->reaction, s);
    const int64_t tiles = tiles_of(p, s);
    for (int ps = 1; ps <= kMaxPasses; ++ps) {
        const int64_t g = (tiles + ps - 1) / ps;
        int per_sm = 0;
        if (int rc = cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, acc_smem(s, ps)),
                                "occupancy"))
            return rc;
        if (per_sm > 0 && g <= (int64_t)per_sm * sm_count()) {
            *G = (int)g;
            *passes = ps;
            return FG_OK;
        }
    }
    return FG_OK;
}

int launch_persistent(const fg_plan* p, int64_t k0, int64_t k1, double* pool, cudaStream_t st, int G, int passes,
                      int s, int64_t kb0 = -1) {
    StepArgs a = make_args(p, s);
    a.k0 = k0;
    a.k1 = k1;
    a.pool = pool;
    a.snap_slot = pool ? p->snap_slot_dev : nullptr;
    a.passes = passes;
    if (kb0 >= 0) {  // the steps of one temporal block
        a.blocked = 1;
        a.kb0 = kb0;
        a.P = block_P(p, kb0);
    }
    StepKernel kern = pick_kernel(p->ndim, p->reaction, s, kb0 >= 0);
    const size_t smem = acc_smem(s, passes);
    if (smem > 48 * 1024) {
        if (int rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                                "smem attribute"))
            return rc;
    }
    if (int rc = cuda_check(cudaMemsetAsync(p->status_dev + 1, 0, sizeof(int64_t), st), "barrier reset")) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ++g_launches;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, a), "fg_step persistent launch");
}

// Key of a cached run graph (fg_run_ex with FG_RUN_GRAPH): the plan bytes (every
// device pointer and scalar, incl. the caller's scratch buffers), the step
// range, the snapshot list and targets, and the flags.
struct GraphKey {
    fg_plan plan;
    int64_t k0 = -1, k1 = -1;
    const double* pool = nullptr;
    const double* host_pool = nullptr;
    int32_t flags = 0;
    std::vector<int64_t> snaps;
    std::vector<double> psi_host;  // host coefficients baked into the step launches
    GraphKey() { memset(&plan, 0, sizeof plan); }
    bool operator==(const GraphKey& o) const {
        return memcmp(&plan, &o.plan, sizeof plan) == 0 && k0 == o.k0 && k1 == o.k1 && pool == o.pool &&
               host_pool == o.host_pool && flags == o.flags && snaps == o.snaps &&
               psi_host.size() == o.psi_host.size() &&
               (psi_host.empty() || memcmp(psi_host.data(), o.psi_host.data(), psi_host.size() * sizeof(double)) == 0);
    }
};

struct GraphCache {
    cudaGraphExec_t exec = nullptr;
    GraphKey key;
    int64_t kernels = 0;
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
    }
    ~GraphCache() { reset(); }
};



}  // namespace

// ================================================================== C ABI =====

extern "C" {

int fg_abi_version(void) { return FGB200_ABI_VERSION; }

int64_t fg_kernel_launches(void) { return g_launches; }

int64_t fg_plan_sizeof(void) { return (int64_t)sizeof(fg_plan); }

const char* fg_last_error(void) { return g_last_error.c_str(); }

int fg_device_info(int32_t* sm, int32_t* major, int32_t* minor) {
    int dev = 0;
    if (int rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice")) return rc;
    int v = 0;
    if (sm) {
        if (int rc = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev), "attr")) return rc;
        *sm = v;
    }
    if (major) {
        if (int rc = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev), "attr")) return rc;
        *major = v;
    }
    if (minor) {
        if (int rc = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev), "attr")) return rc;
        *minor = v;
    }
    return FG_OK;
}

int fg_psi_tables(const double* gamma_dev, int64_t B, int64_t n, int64_t stride, double* out_dev, void* stream) {
    if (!gamma_dev || !out_dev || B < 1 || n < 0 || stride < n + 1)
        return fail(FG_ERR_ARG, "fg_psi_tables: bad arguments");
    const int threads = 128;
    ++g_launches;
    fg_psi_kernel<<<(unsigned)((B + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
        gamma_dev, B, n, stride, out_dev);
    return cuda_check(cudaGetLastError(), "fg_psi_kernel");
}

int fg_schedule_len(int32_t kind, int64_t k, int64_t base, int64_t horizon, int64_t* len) {
    FgSeg s[FG_MAX_SEGS];
    int n = fg_segments(kind, k, base, horizon, s);
    if (n < 0) return fail(FG_ERR_ARG, "fg_schedule_len: invalid schedule arguments");
    if (len) *len = fg_schedule_length(s, n);
    return FG_OK;
}

int fg_schedule_expand(int32_t kind, int64_t k0, int64_t nk, int64_t base, int64_t horizon, int32_t* offs,
                       int32_t* wts, int64_t row_cap, int64_t* lens, void* stream) {
    if (!offs || !wts || !lens || nk < 1 || row_cap < 1 || k0 < 0 || nk > 0x7fffffff)
        return fail(FG_ERR_ARG, "fg_schedule_expand: bad arguments");
    FgSeg s[FG_MAX_SEGS];
    if (fg_segments(kind, k0, base, horizon, s) < 0) return fail(FG_ERR_ARG, "fg_schedule_expand: invalid schedule");
    ++g_launches;
    fg_schedule_kernel<<<(unsigned)nk, 128, 0, (cudaStream_t)stream>>>(kind, k0, base, horizon, offs, wts,
                                                                        row_cap, lens);
    return cuda_check(cudaGetLastError(), "fg_schedule_kernel");
}

int fg_history_sum(const double* H, int64_t ss, int64_t n, const int64_t* offs, const int64_t* wts,
                   int64_t len, const double* psi, int64_t psi_len, int64_t k, double* out, void* stream) {
    if (!H || !offs || !wts || !psi || !out || n < 1 || len < 1 || k < 0 || ss < n)
        return fail(FG_ERR_ARG, "fg_history_sum: bad arguments");
    (void)psi_len;  // bounds are validated by the host before the call (solver.py:177-189)
    const int threads = 256;
    ++g_launches;
    fg_history_sum_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
        H, ss, n, offs, wts, len, psi, k, out);
    return cuda_check(cudaGetLastError(), "fg_history_sum_kernel");
}

int fg_stencil(const fg_plan* p, const double* u, double* out, void* stream) {
    if (int rc = validate_plan(p)) return rc;
    if (!u || !out) return fail(FG_ERR_ARG, "fg_stencil: NULL field");
    const int threads = 256;
    dim3 grid((unsigned)((p->n_m + threads - 1) / threads), (unsigned)p->B);
    const Shape sh = shape_of(p);
    cudaStream_t st = (cudaStream_t)stream;
    ++g_launches;
    if (p->ndim == 1)
        fg_stencil_kernel<1><<<grid, threads, 0, st>>>(u, out, p->B, p->ms, (int32_t)p->n_m, sh);
    else if (p->ndim == 2)
        fg_stencil_kernel<2><<<grid, threads, 0, st>>>(u, out, p->B, p->ms, (int32_t)p->n_m, sh);
    else
        fg_stencil_kernel<3><<<grid, threads, 0, st>>>(u, out, p->B, p->ms, (int32_t)p->n_m, sh);
    return cuda_check(cudaGetLastError(), "fg_stencil_kernel");
}

int fg_step(const fg_plan* p, int64_t k, double* snap, void* stream) {
    if (int rc = validate_plan(p)) return rc;
    if (k < 0 || k >= p->h_slices || k >= p->psi_stride) return fail(FG_ERR_ARG, "fg_step: k out of range");
    return launch_single(p, k, snap, (cudaStream_t)stream, 0, 0);
}

int fg_run(const fg_plan* p, int64_t k0, int64_t k1, const int64_t* snap_steps, int64_t n_snap, double* pool,
           int32_t flags, void* stream) {
    return fg_run_ex(p, k0, k1, snap_steps, n_snap, pool, nullptr, flags, stream);
}

int fg_run_ex(const fg_plan* p, int64_t k0, int64_t k1, const int64_t* snap_steps, int64_t n_snap, double* pool,
              double* host_pool, int32_t flags, void* stream) {
    if (int rc = validate_plan(p)) return rc;
    if (k0 < 0 || k1 < k0 || k1 > p->h_slices || k1 > p->psi_stride)
        return fail(FG_ERR_ARG, "fg_run: step range [%lld, %lld) outside history capacity %lld", (long long)k0,
                    (long long)k1, (long long)p->h_slices);
    if (n_snap > 0 && (!snap_steps || !pool)) return fail(FG_ERR_ARG, "fg_run: snapshots need steps and a pool");
    if (k1 == k0) return FG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int s = choose_split(p);
    const int64_t tb = p->tblock;

    // ---- persistent launches: one cooperative grid per run (or per temporal block)
    int G = 0, passes = 0;
    bool persistent = false;
    if ((flags & FG_RUN_PERSISTENT) && k1 - k0 > 1) {
        if (int rc = persistent_geometry(p, s, &G, &passes)) return rc;
        bool snaps_ok = true;
        if (n_snap > 0) {
            if (!p->snap_slot_dev) {
                snaps_ok = false;
            } else {
                std::vector<int32_t> slot((size_t)(p->h_slices + 1), -1);
                for (int64_t i = 0; i < n_snap; ++i)
                    if (snap_steps[i] > k0 && snap_steps[i] <= k1) slot[(size_t)snap_steps[i]] = (int32_t)i;
                if (int rc = cuda_check(cudaMemcpyAsync(p->snap_slot_dev, slot.data(), slot.size() * sizeof(int32_t),
                                                        cudaMemcpyHostToDevice, st),
                                        "snapshot map"))
                    return rc;
                // the pageable source must stay alive until the copy has read it
                if (int rc = cuda_check(cudaStreamSynchronize(st), "snapshot map sync")) return rc;
            }
        }
        persistent = G > 0 && snaps_ok;  // else fall back to per-step launches
    }
    double* ppool = n_snap > 0 ? pool : nullptr;
    // sub-block launches (per-step launch modes only)
    const bool sub = tb && p->subblock > 0 && !persistent;
    // fused step pairs (per-step launch modes, small 1D/2D fields, caller scratch)
    const bool pairs = tb && !persistent && !sub && pairs_enabled(p, flags);
    double* const u3 = pairs ? p->pair_dev : nullptr;                                      // u^{k+2} buffer
    int64_t* const u3_step = pairs ? reinterpret_cast<int64_t*>(p->pair_dev + p->B * p->ms) : nullptr;

    const int pdl = (flags & FG_RUN_PDL) ? 1 : 0;
    const bool graph = (flags & FG_RUN_GRAPH) != 0 && !persistent;
    // A graph run of exactly the same plan, range, snapshots and flags as the
    // previous graph run on this thread replays that graph (every kernel
    // argument and copy is a function of those): repeated runs of one problem
    // (benchmarks, restarts from u^0) cost one launch on the host.
    static thread_local GraphCache gc;
    GraphKey key;
    if (graph) {
        key.plan = *p;
        key.k0 = k0;
        key.k1 = k1;
        key.pool = pool;
        key.host_pool = host_pool;
        key.flags = flags;
        key.snaps.assign(snap_steps, snap_steps + (n_snap > 0 ? n_snap : 0));
        if (p->psi_host && p->tblock) key.psi_host.assign(p->psi_host, p->psi_host + p->tblock + 1);
        if (gc.exec && gc.key == key) {
            g_launches += gc.kernels;
            return cuda_check(cudaGraphLaunch(gc.exec, st), "graph replay");
        }
    }
    const int64_t launches0 = g_launches;
    const int64_t slice = p->B * p->ms;
    // Capture into a private stream (the legacy default stream cannot capture),
    // then replay the graph on the caller's stream.
    static thread_local cudaStream_t cap_stream = nullptr;
    cudaStream_t cap = st;
    cudaGraph_t g = nullptr;
    if (graph) {
        if (!cap_stream) {
            if (int rc = cuda_check(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking), "capture stream"))
                return rc;
        }
        cap = cap_stream;
        if (int rc = cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture"))
            return rc;
    }
    int64_t si = 0;
    while (si < n_snap && snap_steps[si] <= k0) ++si;
    int rc = FG_OK;

    // snapshots to host: each one is copied on a library copy stream as soon as
    // the launch that produced it is done, overlapping the following steps
    cudaStream_t cstream = nullptr;
    cudaEvent_t cev = nullptr, cjoin = nullptr;
    if (host_pool && n_snap > 0) {
        if (int r = copy_stream(&cstream, &cev, &cjoin)) rc = r;
    }
    auto copy_out = [&](int64_t i0, int64_t i1) {  // snapshots [i0, i1) are complete on `cap`
        if (!cstream || i1 <= i0) return (int)FG_OK;
        if (int r = cuda_check(cudaEventRecord(cev, cap), "snapshot event")) return r;
        if (int r = cuda_check(cudaStreamWaitEvent(cstream, cev, 0), "snapshot wait")) return r;
        return cuda_check(cudaMemcpyAsync(host_pool + i0 * slice, pool + i0 * slice,
                                          (size_t)(i1 - i0) * slice * sizeof(double), cudaMemcpyDeviceToHost, cstream),
                          "snapshot copy");
    };

    // per-step launches of steps [ka, kz); first_after_block: the previous
    // launch on `cap` was a block launch (no programmatic dependency on it)
    auto steps = [&](int64_t ka, int64_t kz, int64_t kb0, bool first_after_block) {
        for (int64_t k = ka; k < kz; ++k) {
            double* snap = nullptr;
            const int64_t i = si;
            if (si < n_snap && snap_steps[si] == k + 1) {
                snap = pool + si * slice;
                ++si;
            }
            const bool wait = pdl && k > k0 && !(k == ka && first_after_block);
            // sub-blocks: slices older than the previous sub-block are in P already
            int64_t t_min = kb0;
            if (kb0 >= 0 && p->subblock > 0) {
                // sub-blocks i with (i+1)S + D <= b are in P already: the step sums
                // from the first one that is not (offsets < S + D)
                const int64_t b = k - kb0, S = p->subblock, D = sub_delay(p);
                t_min = kb0 + (b >= S + D ? S * ((b - D) / S) : 0);
            }
            if (int r = launch_single(p, k, snap, cap, wait, pdl, kb0, t_min)) return r;
            if (snap)
                if (int r = copy_out(i, i + 1)) return r;
        }
        return (int)FG_OK;
    };
    // persistent launch over [ka, kz): its snapshots are copied after it
    // the steps [ka, kz) of block kb0 as fused pairs (an even number of them, so
    // the field is back in its parity buffer), then single steps for the rest
    auto pair_steps = [&](int64_t ka, int64_t kz, int64_t kb0, bool first) -> int {
        int64_t npairs = (kz - ka) / 2;
        if (npairs % 2) --npairs;
        int64_t k = ka;
        for (int64_t i = 0; i < npairs; ++i, k += 2) {
            double* snap1 = nullptr;
            double* snap2 = nullptr;
            const int64_t i0 = si;
            if (si < n_snap && snap_steps[si] == k + 1) snap1 = pool + (si++) * slice;
            if (si < n_snap && snap_steps[si] == k + 2) snap2 = pool + (si++) * slice;
            const bool wait = pdl && k > k0 && !(k == ka && first);
            const bool even = (i % 2) == 0;
            const double* uin = even ? p->u_dev[k & 1] : u3;
            double* uout = even ? u3 : p->u_dev[k & 1];
            if (int r = launch_pair(p, k, kb0, snap1, snap2, cap, wait, pdl, uin, p->u_dev[(k + 1) & 1], uout,
                                    even ? 1 : 0, u3_step))
                return r;
            if (si > i0)
                if (int r = copy_out(i0, si)) return r;
        }
        // the first single step after a pair must not start before it completes
        // (its A phase reads H[k-2], which the pair wrote)
        return steps(k, kz, kb0, first || npairs > 0);
    };
    // the steps [ks, ke) of block kb with sub-block launches (plan->subblock)
    cudaStream_t sstream = nullptr;
    cudaEvent_t sready = nullptr, sdone[kMaxSub] = {};
    auto sub_steps = [&](int64_t ks, int64_t ke, int64_t kb, int bt, bool start) -> int {
        const int64_t S = p->subblock;
        bool pending[kMaxSub] = {};
        bool after_join = start;
        if (start && ks > kb) {  // P recomputed mid-block: add the finished sub-blocks first
            for (int i = 0; kb + (i + 1) * S <= ks; ++i)
                if (int r = launch_block_partial(p, kb, bt, i, cap)) return r;
        }
        int r = FG_OK;
        for (int64_t k = ks; k < ke && r == FG_OK;) {
            const int64_t b = k - kb;
            // this segment ends at the next sub-block end or the next join point
            // (the first step a pending launch feeds), whichever comes first
            int64_t se = kb + (b / S + 1) * S;
            int join = -1;
            for (int i = 0; i < kMaxSub; ++i)
                if (pending[i]) {
                    const int64_t fs = kb + sub_first_step(p, i);
                    if (fs <= k) {
                        join = i;
                    } else if (fs < se) {
                        se = fs;
                    }
                }
            if (se > ke) se = ke;
            if (join >= 0) {  // launches feeding this step (at most the oldest pending ones)
                for (int i = 0; i <= join && r == FG_OK; ++i)
                    if (pending[i] && kb + sub_first_step(p, i) <= k) {
                        r = cuda_check(cudaStreamWaitEvent(cap, sdone[i], 0), "sub-block join");
                        pending[i] = false;
                        after_join = true;
                    }
            }
            if (r == FG_OK) r = steps(k, se, kb, after_join);
            after_join = false;
            const int i = (int)((se - 1 - kb) / S);
            if (r == FG_OK && se == kb + (i + 1) * S && sub_first_step(p, i) < bt) {  // sub-block i is complete
                r = cuda_check(cudaEventRecord(sready, cap), "sub-block fork");
                if (r == FG_OK) r = cuda_check(cudaStreamWaitEvent(sstream, sready, 0), "sub-block fork wait");
                if (r == FG_OK) r = launch_block_partial(p, kb, bt, i, sstream);
                if (r == FG_OK) r = cuda_check(cudaEventRecord(sdone[i], sstream), "sub-block done");
                pending[i] = r == FG_OK;
            }
            k = se;
        }
        for (int i = 0; i < kMaxSub; ++i)  // never leave the sub-block stream unjoined
            if (pending[i]) {
                const int r2 = cuda_check(cudaStreamWaitEvent(cap, sdone[i], 0), "sub-block join");
                if (r == FG_OK) r = r2;
            }
        return r;
    };
    auto persistent_steps = [&](int64_t ka, int64_t kz, int64_t kb0) {
        if (int r = kb0 >= 0 ? launch_persistent(p, ka, kz, ppool, cap, G, passes, s, kb0)
                             : launch_persistent(p, ka, kz, ppool, cap, G, passes, s))
            return r;
        const int64_t i0 = si;
        while (si < n_snap && snap_steps[si] <= kz) ++si;
        return copy_out(i0, si);
    };

    if (rc != FG_OK) {
    } else if (!tb) {
        rc = persistent ? persistent_steps(k0, k1, -1) : steps(k0, k1, -1, false);
    } else {
        // Temporal-blocking pipeline.  Block j (steps K_j ..
        // K_j+tb-1) needs P_j = main_j (slices t < K_{j-1}) + tail_j (slices
        // K_{j-1} .. K_j-1).  main_{j+1} only reads slices t < K_j, final once
        // block j starts, and writes its own P / coefficient buffers, so it is
        // forked onto a low-priority side stream at block j's start and runs
        // behind main_j while block j's tail and steps run here; block j+1 then
        // joins it.  Same launches and arithmetic with or without the overlap.
        const int64_t n_total = p->psi_stride - 1 < p->h_slices - 1 ? p->psi_stride - 1 : p->h_slices - 1;
        auto block_len = [&](int64_t kb) {
            const int64_t left = n_total - kb;
            return (int)(left < tb ? (left > 0 ? left : 1) : tb);
        };
        cudaStream_t side = nullptr;
        cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
        if (!(flags & FG_RUN_NO_OVERLAP)) rc = side_stream(&side, &ev_fork, ev_join);
        if (rc == FG_OK && sub) rc = sub_stream(&sstream, &sready, sdone);
        if (rc == FG_OK && pairs)
            rc = cuda_check(cudaMemsetAsync(u3_step, 0xff, sizeof(int64_t), cap), "pair step reset");  // -1
        int64_t main_on_side = -1;  // block whose main launch is in flight on `side`
        BlockTrace tr(graph ? nullptr : getenv("FGB200_TRACE"));
        for (int64_t kb = k0 - k0 % tb; kb < k1 && rc == FG_OK; kb += tb) {
            const int64_t ks = kb > k0 ? kb : k0, ke = kb + tb < k1 ? kb + tb : k1;
            // blocks are aligned to multiples of tb, so a run split into several
            // fg_run calls recomputes the same partial sums (deterministic)
            const bool start = ks == kb || !(flags & FG_RUN_CONTINUE);
            if (start) {
                const int64_t nk = kb + tb;
                const bool fork_next = side && nk < k1;
                tr.mark(kb, 0, cap);
                if (fork_next) {
                    rc = cuda_check(cudaEventRecord(ev_fork, cap), "fork record");
                    if (rc == FG_OK) rc = cuda_check(cudaStreamWaitEvent(side, ev_fork, 0), "fork wait");
                    tr.mark(kb, 3, side);
                    if (rc == FG_OK) rc = launch_block_main(p, nk, block_len(nk), side);
                    tr.mark(kb, 4, side);
                    if (rc == FG_OK) rc = cuda_check(cudaEventRecord(ev_join[(nk / tb) & 1], side), "join record");
                    if (rc != FG_OK) break;
                }
                if (main_on_side == kb)
                    rc = cuda_check(cudaStreamWaitEvent(cap, ev_join[(kb / tb) & 1], 0), "join side stream");
                else
                    rc = launch_block_main(p, kb, block_len(kb), cap);
                main_on_side = fork_next ? nk : -1;
                tr.mark(kb, 1, cap);
                if (rc == FG_OK) rc = launch_block_tail(p, kb, block_len(kb), cap);
                tr.mark(kb, 2, cap);
                if (rc != FG_OK) break;
            }
            rc = persistent ? persistent_steps(ks, ke, kb)
                 : sub      ? sub_steps(ks, ke, kb, block_len(kb), start)
                 : pairs    ? pair_steps(ks, ke, kb, start)
                            : steps(ks, ke, kb, start);
        }
        if (rc == FG_OK && pairs) {  // a run that stopped on a field in the scratch buffer
            const int64_t nf = p->B * p->ms;
            ++g_launches;
            fg_u3_fixup_kernel<<<(unsigned)((nf + 255) / 256 < 1024 ? (nf + 255) / 256 : 1024), 256, 0, cap>>>(
                p->status_dev, u3_step, u3, p->u_dev[0], p->u_dev[1], nf);
            rc = cuda_check(cudaGetLastError(), "fg_u3_fixup launch");
        }
        if (main_on_side >= 0) {  // error path: never leave the side stream unjoined
            const int r2 =
                cuda_check(cudaStreamWaitEvent(cap, ev_join[(main_on_side / tb) & 1], 0), "join side stream");
            if (rc == FG_OK) rc = r2;
        }
        tr.dump(cap);
    }

    if (cstream) {  // join the copies: a sync of `stream` covers the host snapshots
        int r2 = cuda_check(cudaEventRecord(cjoin, cstream), "copy join record");
        if (r2 == FG_OK) r2 = cuda_check(cudaStreamWaitEvent(cap, cjoin, 0), "copy join");
        if (rc == FG_OK) rc = r2;
    }
    if (graph) {
        cudaError_t e = cudaStreamEndCapture(cap, &g);
        if (rc != FG_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (int r2 = cuda_check(e, "end capture")) return r2;
        cudaGraphExec_t ge = nullptr;
        if (int r2 = cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate")) {
            cudaGraphDestroy(g);
            return r2;
        }
        cudaGraphDestroy(g);
        rc = cuda_check(cudaGraphLaunch(ge, st), "graph launch");
        gc.reset();
        if (rc == FG_OK) {
            gc.exec = ge;
            gc.key = key;
            gc.kernels = g_launches - launches0;
        } else {
            cudaGraphExecDestroy(ge);
        }
    }
    return rc;
}

int fg_status(const fg_plan* p, int64_t* first_bad, void* stream) {
    if (!p || !p->status_dev || !first_bad) return fail(FG_ERR_ARG, "fg_status: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = cuda_check(cudaMemcpyAsync(first_bad, p->status_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                            "status copy"))
        return rc;
    return cuda_check(cudaStreamSynchronize(st), "status sync");
}

int fg_block_partials(const fg_plan* p, int64_t kb0, int32_t bt, void* stream) {
    if (int rc = validate_plan(p)) return rc;
    if (!p->tblock) return fail(FG_ERR_ARG, "fg_block_partials: plan has no temporal blocking");
    if (kb0 < 0 || bt < 1 || bt > p->tblock || kb0 + bt > p->psi_stride || kb0 > p->h_slices)
        return fail(FG_ERR_ARG, "fg_block_partials: block out of range");
    return launch_block(p, kb0, bt, (cudaStream_t)stream);
}

int fg_block_subpartials(const fg_plan* p, int64_t kb0, int32_t bt, void* stream, int32_t* launched) {
    if (int rc = validate_plan(p)) return rc;
    if (!p->tblock || p->subblock <= 0) return fail(FG_ERR_ARG, "fg_block_subpartials: plan has no sub-block launches");
    if (kb0 < 0 || bt < 1 || bt > p->tblock || kb0 + bt > p->psi_stride || kb0 + bt > p->h_slices)
        return fail(FG_ERR_ARG, "fg_block_subpartials: block out of range");
    int n = 0;
    for (int i = 0; sub_first_step(p, i) < bt; ++i, ++n)
        if (int rc = launch_block_partial(p, kb0, bt, i, (cudaStream_t)stream)) return rc;
    if (launched) *launched = n;
    return FG_OK;
}

int fg_block_item_rows(int32_t kind, int64_t n_steps, int32_t tblock, int64_t base, int64_t horizon,
                       int32_t item_cols, int64_t* max_rows) {
    if (item_cols != 8 && item_cols != 16) return fail(FG_ERR_ARG, "fg_block_item_rows: item_cols must be 8 or 16");
    if (n_steps < 0 || tblock < 1 || tblock > kMaxTBlock || !max_rows)
        return fail(FG_ERR_ARG, "fg_block_item_rows: bad arguments");
    fg_plan q;
    memset(&q, 0, sizeof q);
    q.kind = kind;
    q.base = base;
    q.horizon_max = horizon;
    q.tblock = tblock;
    q.coef_rows = INT64_MAX / (4 * kCoefRow);  // no capacity limit while measuring
    q.item_cols = item_cols;
    int64_t worst = 0;
    static thread_local ItemTable T;
    for (int64_t kb0 = tblock; kb0 < n_steps; kb0 += tblock) {
        const int bt = (int)(n_steps - kb0 < tblock ? n_steps - kb0 : tblock);
        const int64_t tb = kb0 - tblock;
        int64_t rows = 0;
        // a launch that does not itemize takes the dense kernel (no rows) when the
        // factor has one, else the run fails — reported here already
        if (build_items(&q, kb0, bt, tb, kb0, T, 0))
            for (int x = 0; x < T.n_items; ++x) rows += T.it[x].n_slices;
        else if (tblock > kMaxDenseTBlock)
            return fail(FG_ERR_UNSUPPORTED, "tblock %d: tail of block %lld does not fit the item table", (int)tblock,
                        (long long)kb0);
        if (build_items(&q, kb0, bt, 0, tb, T, rows))
            for (int x = 0; x < T.n_items; ++x) rows += T.it[x].n_slices;
        else if (tblock > kMaxDenseTBlock)
            return fail(FG_ERR_UNSUPPORTED, "tblock %d: block %lld does not fit the item table", (int)tblock,
                        (long long)kb0);
        worst = rows > worst ? rows : worst;
    }
    *max_rows = worst;
    return FG_OK;
}

int fg_block_item_table(int32_t kind, int64_t kb0, int32_t bt, int64_t ts, int64_t te, int64_t base,
                        int64_t horizon, int32_t tblock, int32_t item_cols, int64_t* out, int32_t cap,
                        int32_t* n_items) {
    if (item_cols != 8 && item_cols != 16) return fail(FG_ERR_ARG, "fg_block_item_table: item_cols must be 8 or 16");
    if (kb0 < 0 || bt < 1 || bt > kMaxTBlock || tblock < bt || tblock > kMaxTBlock || ts < 0 || te > kb0 || !out ||
        !n_items)
        return fail(FG_ERR_ARG, "fg_block_item_table: bad arguments");
    fg_plan q;
    memset(&q, 0, sizeof q);
    q.kind = kind;
    q.base = base;
    q.horizon_max = horizon;
    q.tblock = tblock;
    q.coef_rows = INT64_MAX / (4 * kCoefRow);
    q.item_cols = item_cols;
    static thread_local ItemTable T;
    if (!build_items(&q, kb0, bt, ts, te, T, 0)) {
        *n_items = -1;  // not itemized (dense class or table overflow)
        return FG_OK;
    }
    *n_items = T.n_items;
    if (T.n_items > cap) return fail(FG_ERR_ARG, "fg_block_item_table: %d items > cap %d", T.n_items, cap);
    for (int x = 0; x < T.n_items; ++x) {
        int64_t* o = out + (int64_t)x * (4 + kItemCols);
        o[0] = T.it[x].t_first;
        o[1] = T.it[x].stride;
        o[2] = T.it[x].n_slices;
        o[3] = T.it[x].ncols;
        for (int c = 0; c < kItemCols; ++c) o[4 + c] = c < T.it[x].ncols ? T.it[x].col2step[c] : -1;
    }
    return FG_OK;
}

int fg_history_pad(int32_t kind, int64_t n_steps, int64_t base, int64_t* pad) {
    if (!pad || n_steps < 0 || (kind == 2 && base < 2)) return fail(FG_ERR_ARG, "fg_history_pad: bad arguments");
    int64_t s_max = 1;  // dense window and tail: stride 1
    if (kind == 2) {
        // interval i >= 2 (stride 2i - 1) is sampled by some step k <= n_steps - 1
        // once a^(i-1) + i <= k (schedule.py:120-133)
        int64_t a_prev = base;
        for (int64_t i = 2; a_prev + i <= n_steps - 1; ++i) {
            s_max = 2 * i - 1;
            if (a_prev > INT64_MAX / base) break;
            a_prev *= base;
        }
    }
    *pad = (kIR - 1) * s_max;
    return FG_OK;
}

int fg_block_union(int32_t kind, int64_t kb0, int32_t bt, int64_t base, int64_t horizon, int64_t* count) {
    if (kb0 < 0 || bt < 1 || bt > kMaxTBlock || !count) return fail(FG_ERR_ARG, "fg_block_union: bad arguments");
    std::vector<char> used((size_t)kb0, 0);
    FgSeg s[FG_MAX_SEGS];
    for (int b = 0; b < bt; ++b) {
        const int64_t k = kb0 + b;
        const int n = fg_segments(kind, k, base, horizon, s);
        if (n < 0) return fail(FG_ERR_ARG, "fg_block_union: invalid schedule");
        for (int i = 0; i < n; ++i)
            for (int64_t c = 0; c < s[i].count; ++c) {
                const int64_t t = k - (s[i].m0 + c * s[i].stride);
                if (t >= 0 && t < kb0) used[(size_t)t] = 1;
            }
    }
    int64_t u = 0;
    for (char x : used) u += x;
    *count = u;
    return FG_OK;
}

int fg_step_geometry(const fg_plan* p, int64_t* ctas, int32_t* threads, int32_t* split) {
    if (int rc = validate_plan(p)) return rc;
    const int s = choose_split(p);
    if (ctas) *ctas = tiles_of(p, s);
    if (threads) *threads = kThreads;
    if (split) *split = s;
    return FG_OK;
}

}  // extern "C"
