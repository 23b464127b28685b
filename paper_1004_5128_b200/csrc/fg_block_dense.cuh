// Temporal blocking, dense block stage (fg_block_tma_kernel: TMA ring + fp64 DMMA consumers): DESIGN.md §3.1, §3.3.
// Part of the single translation unit csrc/fg_kernels.cu (included there in order).
#ifndef FG_BLOCK_DENSE_CUH
#define FG_BLOCK_DENSE_CUH

#include "fg_common.cuh"

namespace {

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
#ifndef FG_TAIL_STAGES
#define FG_TAIL_STAGES 2
#endif
#ifndef FG_DENSE_SOLO
#define FG_DENSE_SOLO 1   // large-field BT = 32 main launches: one CTA per SM, <= 128 registers (0: two 96-register CTAs)
#endif
constexpr int kSoloStages = 4;  // ring of the solo main launch: 4 stages of 16 slices (two CTAs: 3)
template <bool STAGED>
__host__ __device__ constexpr int ring_stages() { return STAGED ? FG_STAGED_RING : 4; }

constexpr int kMainStages = FG_STAGED_RING;  // staged main launches
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
template <int BT, int TP, bool STAGED, int NS, int WP, bool SOLO>
__device__ __forceinline__ void fg_block_tma_body(const BlockArgs& a) {
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
        if constexpr (SOLO) {
        // fragments of k-step ks+1 are loaded before the DMMAs of k-step ks issue
        // (two k-steps live, 110 registers, no spills): the shared-memory latency hides
        // behind the warp's own 16 DMMAs instead of behind other warps
        double af[2][MT], bf[2][NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) af[0][i] = fk < nr ? lds_f64(cs + (uint32_t)((fk * CP + 8 * i) * 8)) : 0.0;
#pragma unroll
        for (int j = 0; j < NT; ++j) bf[0][j] = fk < nr ? lds_f64(rs + (uint32_t)((fk * RP + 8 * j) * 8)) : 0.0;
#pragma unroll
        for (int ks = 0; ks < KE / 4; ++ks) {
            const int cur = ks & 1, nxt = cur ^ 1;
            if (ks + 1 < KE / 4) {
                const int e = (ks + 1) * 4 + fk;
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    af[nxt][i] = e < nr ? lds_f64(cs + (uint32_t)((e * CP + 8 * i) * 8)) : 0.0;
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    bf[nxt][j] = e < nr ? lds_f64(rs + (uint32_t)((e * RP + 8 * j) * 8)) : 0.0;
            }
            if (ks == 1) {
                if (pend && lane == 0) mbar_arrive_after(pend, d[0][0][0], sink + warp);
                pend = &empty[s];
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma_8x8x4(d[i][j][0], d[i][j][1], af[cur][i], bf[cur][j]);
        }
        } else {
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
                // one add per element and launch: an L2 reduction rounds exactly like
                // load-add-store and spares the consumer warp the load round trip
                red_add(o, d[i][j][0]);
                red_add(o + 1, d[i][j][1]);
            } else {
                st_pair(o, d[i][j][0], d[i][j][1]);
            }
        }
    }
    }  // tiles
}

// two CTAs per SM (every dense launch but the large-field main launches below)
template <int BT, int TP, bool STAGED, int NS, int WP>
__global__ void __launch_bounds__(TP / WP * 32 + 32, 2) fg_block_tma_kernel(const BlockArgs a) {
    fg_block_tma_body<BT, TP, STAGED, NS, WP, false>(a);
}

// "Solo" main launch of large single fields at BT = 32: ONE CTA per SM with up to
// 128 registers per thread (ptxas: 110), so the lean consumer loop can keep two k-steps of
// fragments live (software-pipelined, no spills) and the 8 consumer warps issue
// DMMAs without waiting for shared memory; the second CTA's registers are left
// to a step CTA of the block running beside it.
template <int BT, int TP, bool STAGED, int NS, int WP>
__global__ void __maxnreg__(128) fg_block_tma_solo_kernel(const BlockArgs a) {
    fg_block_tma_body<BT, TP, STAGED, NS, WP, true>(a);
}

}  // namespace

#endif  // FG_BLOCK_DENSE_CUH
