// Stencils, the fused time-step kernel (fg_step_kernel) and fused step pairs (fg_step2_kernel): DESIGN.md §3.4, §3.6.
// Part of the single translation unit csrc/fg_kernels.cu (included there in order).
#ifndef FG_STEP_CUH
#define FG_STEP_CUH

#include "fg_common.cuh"

namespace {

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

    // single-step BLK launches (one tile per CTA) keep the A-phase sum in
    // registers: no dynamic shared memory, so a step CTA fits in the ~3.8 KB two
    // dense block CTAs leave per SM
    double2 part_reg = make_double2(0.0, 0.0);
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
                const double2 sum =
                    make_double2(__dadd_rn(__dadd_rn(0.0, acc0), pb.x), __dadd_rn(__dadd_rn(0.0, acc1), pb.y));
                if (multi)
                    s_acc[p * kLanes + slot] = sum;
                else
                    part_reg = sum;
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
                const double2 part = (BLK && !multi) ? part_reg : s_acc[p * kLanes + slot];
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

}  // namespace

#endif  // FG_STEP_CUH
