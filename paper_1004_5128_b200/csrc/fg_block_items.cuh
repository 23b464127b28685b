// Temporal blocking, itemized block stage for thinned schedules (fg_block_item8_kernel, fg_block_item_kernel): DESIGN.md §3.2.
// Part of the single translation unit csrc/fg_kernels.cu (included there in order).
#ifndef FG_BLOCK_ITEMS_CUH
#define FG_BLOCK_ITEMS_CUH

#include "fg_block_dense.cuh"

namespace {

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

}  // namespace

#endif  // FG_BLOCK_ITEMS_CUH
