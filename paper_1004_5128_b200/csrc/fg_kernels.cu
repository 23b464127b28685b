// B200 (sm_100a) kernels and the C ABI of the GL history stepper — one translation unit.
//
// Hot path replaced: /root/reference/pkg/src/fracgrid/solver.py:230-265 (run)
//   → step (:200-227) → history_sum (:162-197), with ψ from coefficients.py:76-92,
//   schedules from schedule.py:70-151 and the stencil of grid.py:88-106.
//
// Layout:
//   fg_common.cuh       error plumbing, constants, FG_CHECKS bounds checks, PTX helpers
//   fg_schedule.cuh     schedule segments (host + device): full / short / adaptive
//   fg_step.cuh         stencils, fg_step_kernel (one fused time step: recent-slice sum
//                       before the dependency wait, then m = 1, m = 0 = stencil(u^k),
//                       reaction + update in the reference's rounding order), fused pairs
//   fg_block_dense.cuh  temporal blocking, dense stage: TMA ring + fp64 DMMA consumers
//   fg_block_items.cuh  temporal blocking, itemized stage for thinned (adaptive) schedules
//   fg_support.cuh      ψ tables, schedule expansion, standalone history_sum / stencil
//   this file           host side: plan validation, kernel variants, launch pipeline
//                       (PDL step chain, main/tail/sub-block launches, side streams,
//                       graph capture, snapshots) and the C ABI of include/fgb200.h
// A step reads 8 bytes of history per term (0.25 flop/B): unblocked it is HBM-bound;
// the block stages read each old slice once per temporal block and run on the fp64
// tensor pipe (DMMA m8n8k4), so full memory is fp64-bound and adaptive memory HBM-bound.
#include "fg_common.cuh"
#include "fg_step.cuh"
#include "fg_block_dense.cuh"
#include "fg_block_items.cuh"
#include "fg_support.cuh"

namespace {

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
    cfg.dynamicSmemBytes = (kb0 >= 0 && s == 1) ? 0 : acc_smem(s, 1);  // BLK: the sum stays in registers
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
    int per_sm = 2;  // CTAs per SM of a single-member launch (grid cap)
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
    // large single fields, full/short memory at BT = 32: the solo main launch
    // (one CTA per SM, fg_block_tma_solo_kernel) once every SM has several tiles
    if (FG_DENSE_SOLO && !tail && staged && p->tblock == 32 && (p->n_m + 255) / 256 >= 4 * (int64_t)sm_count()) {
        BlockVariant v = {fg_block_tma_solo_kernel<32, 256, true, kSoloStages, 32>,
                          tma_block_smem<32, 256, true, kSoloStages, 32>(), 256, 256 / 32 * 32 + 32};
        v.per_sm = 1;
        return v;
    }
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
unsigned block_grid(const fg_plan* p, int64_t total_tiles, int per_sm = 2) {
    if (p->B != 1) return (unsigned)total_tiles;
    const int64_t cap = (int64_t)sm_count() * per_sm;
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
    v.kern<<<block_grid(p, a.total_tiles, v.per_sm), v.threads, v.smem, st>>>(a);
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
    std::vector<std::pair<int64_t, cudaEvent_t>> sev;  // per-step completion events (FGB200_TRACE_STEPS=1)
    bool per_step = false;
    explicit BlockTrace(const char* p) : path(p) { per_step = p && getenv("FGB200_TRACE_STEPS"); }
    void step_mark(int64_t k, cudaStream_t s) {
        if (!per_step) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        sev.emplace_back(k, e);
    }
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
        for (auto& se : sev) {
            if (f) fprintf(f, "step %lld done t=%.1f\n", (long long)se.first, ms(ev[0], se.second));
            cudaEventDestroy(se.second);
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
    BlockTrace tr(graph || !tb ? nullptr : getenv("FGB200_TRACE"));

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
            if ((k & 3) == 3) tr.step_mark(k, cap);
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
