/*
 * fgb200 — C ABI of the B200-native Grünwald–Letnikov history stepper.
 *
 * Drop-in boundary for the reference hot path
 *   /root/reference/pkg/src/fracgrid/solver.py:230-265  run(config)
 *        → step (solver.py:200-227) → history_sum (solver.py:162-197)
 * plus the helpers that path depends on:
 *   coefficients.py:76-92  build_table (ψ recursion)
 *   schedule.py:70-151     full / short / adaptive memory schedules
 *   grid.py:88-106         five-point stencil (generalised to 1D/3D)
 *
 * The reference is pure Python, so there is no C interface to mirror one-for-one;
 * these entry points are what a ctypes binding inside fracgrid would call (see
 * INTEGRATION.md).  All pointers marked _dev are CUDA device pointers; `stream`
 * is a cudaStream_t passed as void* (NULL = legacy default stream).  No torch
 * types cross this boundary.  Every function returns FG_OK (0) or a negative
 * FG_ERR_* code; fg_last_error() describes the most recent failure on the
 * calling thread.
 */
#ifndef FGB200_H
#define FGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGB200_ABI_VERSION 7

#define FG_OK 0
#define FG_ERR_ARG (-1)         /* invalid argument (maps to ValueError)          */
#define FG_ERR_CUDA (-2)        /* CUDA runtime failure                           */
#define FG_ERR_UNSUPPORTED (-3) /* shape / kind outside what the kernels handle   */

/* "no divergence yet" value of fg_plan.status[0] */
#define FG_NO_BAD_STEP INT64_MAX

enum fg_memory_kind {  /* schedule.py:198-254 strategy tags */
    FG_MEM_FULL = 0,      /* "full"                         */
    FG_MEM_SHORT = 1,     /* "short", horizon floor(L/dt)   */
    FG_MEM_ADAPTIVE = 2   /* "adaptive", integer base a>=2  */
};

enum fg_reaction {
    FG_REACT_LINEAR = 0,     /* u*decay + diffuse*S           (solver.py:215-217) */
    FG_REACT_SATURATING = 1  /* u + dt*f(u) + diffuse*S, f(u) = -vmax*u/(km+u)    */
};

/*
 * Everything one run needs, as plain device pointers and sizes.  The caller
 * (Python host, or any C program) owns every device buffer of a run, scratch
 * included; the library allocates none (it keeps only per-thread streams and
 * events for its side-stream pipelines).  Layout in HBM:
 *   fields   u[2][B][ms]                      fp64, ping-pong by step parity
 *   history  H[h_slices][B][ms]               fp64, slice t = δ^t = stencil(u^t)
 *   ψ        psi[B][psi_stride]               fp64, ψ_b(m), m = 0..n_steps
 * `ms` (member stride) is n_m rounded up to a multiple of 32 elements, so every
 * member of every slice starts on a 256-byte boundary and is read with 128-bit
 * loads.  Padding elements are never part of a result.
 */
typedef struct fg_plan {
    int64_t B;            /* members (independent problems)                       */
    int64_t n_m;          /* points per member = prod(shape)                      */
    int64_t ms;           /* member stride in elements (multiple of 32, >= n_m)   */
    int32_t ndim;         /* 1, 2 or 3                                            */
    int32_t reaction;     /* enum fg_reaction                                     */
    int64_t shape[3];     /* member shape, C order; unused trailing entries = 1   */
    int32_t kind;         /* enum fg_memory_kind                                  */
    int32_t split;        /* 0 = auto; else warps-per-column split of the sum (1,2,4,8) */
    int64_t base;         /* adaptive base a                                      */
    const int64_t* horizon_dev;  /* [B] short-memory floor(L/dt_b), host-evaluated */
    const double* psi_dev;       /* [B][psi_stride]                                */
    int64_t psi_stride;          /* >= n_steps + 1                                 */
    const double* decay_dev;     /* [B] 1 - beta*dt_b (host-evaluated)             */
    const double* diffuse_dev;   /* [B] alpha*dt_b**gamma_b/dx**2 (host-evaluated) */
    const double* dt_dev;        /* [B]                                            */
    double vmax, km;             /* saturating reaction parameters                 */
    double* H_dev;               /* [h_slices][B*ms]                               */
    int64_t h_slices;            /* history capacity (n_steps + 1)                 */
    double* u_dev[2];            /* [B*ms] each                                    */
    int64_t* status_dev;         /* [2]: [0] first non-finite step or FG_NO_BAD_STEP,
                                    [1] grid-barrier counter (library scratch)     */
    int32_t step_flags;          /* FG_STEP_* bits                                 */
    int32_t item_cols;           /* itemized block stage: step columns per item, 8 or 16
                                    (0 = FGB200_ITEM_COLS, else 16 for ensembles, 8 otherwise) */
    int32_t* snap_slot_dev;      /* [h_slices+1] scratch for FG_RUN_PERSISTENT snapshots
                                    (filled by fg_run; NULL if no snapshots)       */
    int64_t horizon_max;         /* host copy of max(horizon_dev) (0 = unknown)    */
    int32_t tblock;              /* temporal blocking factor: 0 (off), 8, 16, 24, 32;
                                    multiples of 8 up to 128 above 32 for adaptive
                                    plans (itemized block stage, blkcoef_dev)     */
    int32_t reserved2;
    double* P_dev;               /* [2][tblock][B*ms] scratch for blocked partial sums:
                                    block kb0 uses buffer (kb0 / tblock) & 1        */
    double* blkcoef_dev;         /* [2][coef_rows][36] scratch, single-member blocking:
                                    block kb0 uses buffer (kb0 / tblock) & 1        */
    const double* psi_host;      /* optional, single member: host copy of psi_dev[0..tblock]
                                    (blocked steps then get their coefficients as
                                    launch parameters); NULL = read psi_dev       */
    int64_t subblock;            /* sub-block launches: S > 0 divides tblock (adaptive,
                                    blkcoef_dev); each finished S-step sub-block's
                                    slices are added into the P rows of the block's
                                    steps two sub-blocks on, so steps sum only
                                    offsets < 2S themselves; 0 = off              */
    int64_t coef_rows;           /* rows per blkcoef buffer (0 = h_slices)          */
    int64_t h_alloc;             /* slices allocated at H_dev (0 = h_slices): the 16-column
                                    itemized block stage reads whole TMA boxes of kE slices
                                    of a strided progression, up to fg_history_pad slices
                                    past the last one it needs (never used in a sum);
                                    a blocked adaptive run with a smaller allocation fails */
    double* pair_dev;            /* [B*ms + 1] caller scratch of fused step pairs (1D/2D
                                    blocked runs): a field buffer, then the int64 step
                                    whose field it holds; NULL disables pairs       */
    int64_t subdelay;            /* sub-block launches: sub-block i feeds the steps b >=
                                    (i+1)*subblock + subdelay (1..subblock; 0 = subblock),
                                    which then sum themselves offsets < subblock + subdelay */
} fg_plan;

/* fg_plan.step_flags: take the m = 0 term from the stored H[k] instead of
 * recomputing stencil(u^k) (the reference's step() sums whatever the history
 * holds, solver.py:214). */
#define FG_STEP_M0_FROM_HISTORY 1

/* ---- library ---------------------------------------------------------------- */
int fg_abi_version(void);
/* sizeof(fg_plan) as compiled into the library (binding layout check). */
int64_t fg_plan_sizeof(void);
const char* fg_last_error(void);
/* Kernels this library has launched from the calling thread so far (graph mode:
 * kernel nodes captured); for launch accounting (bench.py gpu_launches). */
int64_t fg_kernel_launches(void);
/* 0 on success; fills the SM count and compute capability of the current device. */
int fg_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* ---- ψ tables: coefficients.py:76-92, bit-exact ------------------------------
 * out_dev[b*stride + m] = ψ(gamma_dev[b], m) for m = 0..n, one sequential
 * recursion per member with correctly rounded sub/mul/div (no FMA). */
int fg_psi_tables(const double* gamma_dev, int64_t B, int64_t n, int64_t stride,
                  double* out_dev, void* stream);

/* ---- schedules: schedule.py:70-151, bit-exact --------------------------------
 * Host helper: number of (offset, weight) entries of schedule(k). */
int fg_schedule_len(int32_t kind, int64_t k, int64_t base, int64_t horizon, int64_t* len);
/* Device generator: rows i = 0..nk-1 hold schedule(k0 + i); offsets / weights
 * are int32 [nk][row_cap]; lens_dev[i] receives the full length (entries past
 * row_cap are dropped). */
int fg_schedule_expand(int32_t kind, int64_t k0, int64_t nk, int64_t base, int64_t horizon,
                       int32_t* offsets_dev, int32_t* weights_dev, int64_t row_cap,
                       int64_t* lens_dev, void* stream);

/* ---- history_sum: solver.py:162-197 -----------------------------------------
 * out_dev[p] = Σ_j weights[j]*psi[offsets[j]] * H[(k - offsets[j])*slice_stride + p]
 * for p < n.  Offsets / weights are int64 device arrays of length len (any
 * valid MemorySchedule).  FMA accumulation: within 1e-10 of the reference, not
 * bitwise (different reduction order). */
int fg_history_sum(const double* H_dev, int64_t slice_stride, int64_t n,
                   const int64_t* offsets_dev, const int64_t* weights_dev, int64_t len,
                   const double* psi_dev, int64_t psi_len, int64_t k,
                   double* out_dev, void* stream);

/* ---- stencil: grid.py:88-106 (zero output ring, no /dx²), bit-exact ------------
 * out = δ(u) for all B members of the plan's shape; u/out are [B*ms]. */
int fg_stencil(const fg_plan* plan, const double* u_dev, double* out_dev, void* stream);

/* ---- fused step: solver.py:200-227 -------------------------------------------
 * One kernel: δ^k = stencil(u^k) → H[k]; S = Σ_j c_j H[k-m_j] (schedule and
 * c_j = w_j ψ_b(m_j) generated on the device); u^{k+1} = update(u^k, S);
 * boundary pinned to zero; first non-finite step recorded in status_dev[0]
 * (later steps become no-ops).  Reads u_dev[k&1], writes u_dev[(k+1)&1] and,
 * if snap_dev != NULL, a copy of u^{k+1} there. */
int fg_step(const fg_plan* plan, int64_t k, double* snap_dev, void* stream);

/* Steps k0..k1-1 (solver.py:249-256).  snap_steps (host, sorted) lists `done`
 * step numbers whose field is copied to snap_pool_dev + i*B*ms for the i-th
 * entry.  flags:
 *   FG_RUN_PERSISTENT  one cooperative launch runs every step; CTAs own fixed
 *                      tiles and meet at a split arrive/wait grid barrier once
 *                      per step (falls back to per-step launches if the grid
 *                      cannot be co-resident);
 *   FG_RUN_PDL         per-step launches with programmatic dependent launch;
 *   FG_RUN_GRAPH       per-step launches captured into one CUDA graph.
 * All modes produce bitwise-identical results.  With temporal blocking the
 * per-step modes run each block's main block-kernel launch on a library-owned
 * low-priority side stream, forked from and joined back into `stream` inside
 * the call (FG_RUN_NO_OVERLAP keeps them on `stream`; results are unchanged). */
#define FG_RUN_GRAPH 1
#define FG_RUN_PDL 2
#define FG_RUN_PERSISTENT 4
/* Launch-shape options (results are bitwise identical either way):
 *   FG_RUN_NO_OVERLAP  main block-stage launches on `stream`, no side stream;
 *   FG_RUN_NO_PAIRS    no fused step pairs;
 *   FG_RUN_PAIRS       fused step pairs for 2D fields too (default: 1D only);
 *                      pairs need plan->pair_dev. */
#define FG_RUN_NO_OVERLAP 64
#define FG_RUN_NO_PAIRS 128
#define FG_RUN_PAIRS 256
/* Temporal blocking: P_dev already holds the partial sums of the block that
 * contains k0 (this call continues the previous fg_run of the same plan), so a
 * block that started before k0 is not recomputed. */
#define FG_RUN_CONTINUE 16
int fg_run(const fg_plan* plan, int64_t k0, int64_t k1,
           const int64_t* snap_steps, int64_t n_snap, double* snap_pool_dev,
           int32_t flags, void* stream);

/* fg_run plus snapshot streaming: when snap_pool_host (pinned host memory,
 * same layout as snap_pool_dev) is non-NULL, each snapshot is copied there on a
 * library-owned copy stream as soon as the launch that wrote it is done, so the
 * device-to-host traffic overlaps the following steps; the copies are joined
 * into `stream` before the call returns (a sync of `stream` covers them). */
int fg_run_ex(const fg_plan* plan, int64_t k0, int64_t k1,
              const int64_t* snap_steps, int64_t n_snap, double* snap_pool_dev,
              double* snap_pool_host, int32_t flags, void* stream);

/* Stream-synchronous read of status_dev[0] (first non-finite step). */
int fg_status(const fg_plan* plan, int64_t* first_bad_step, void* stream);

/* Slices to allocate at H_dev beyond h_slices (fg_plan.h_alloc = h_slices + pad)
 * for blocked runs of this schedule: the 16-column item stage reads TMA boxes of
 * 8 slices of a stride-s progression, so up to 7 strides past the last slice an
 * item needs (those rows are never summed).  Host-only. */
int fg_history_pad(int32_t kind, int64_t n_steps, int64_t base, int64_t* pad);

/* Host accounting for temporal blocking: number of distinct history slices
 * t < kb0 that the block of steps kb0..kb0+bt-1 reads (the union of their
 * schedules' old parts), i.e. the slices fg_block_kernel streams once. */
int fg_block_union(int32_t kind, int64_t kb0, int32_t bt, int64_t base, int64_t horizon, int64_t* count);
/* Host-only view of the item table the library builds for a temporal block
 * (steps kb0..kb0+bt-1, old slices [ts, te)): 20 int64 per item = t_first,
 * stride, n_slices, ncols, the ncols (<= 16) step columns (padded with -1).  *n_items =
 * -1 when the range is not itemized (one dense class, or the table overflows).
 * Lets tests prove every schedule entry is owned by exactly one item. */
int fg_block_item_table(int32_t kind, int64_t kb0, int32_t bt, int64_t ts, int64_t te, int64_t base,
                        int64_t horizon, int32_t tblock, int32_t item_cols, int64_t* out, int32_t cap,
                        int32_t* n_items);
/* Largest number of item coefficient rows (tail + main; 12 doubles each for
 * 8-column items, 20 for 16-column items) any temporal block of an n_steps run
 * needs: sizes blkcoef_dev for itemized ensembles (coef_rows >= ceil(rows *
 * pitch / 36)).  Host-only, no device work. */
int fg_block_item_rows(int32_t kind, int64_t n_steps, int32_t tblock, int64_t base, int64_t horizon,
                       int32_t item_cols, int64_t* max_rows);

/* Temporal blocking building block (normally driven by fg_run): write into
 * buffer (kb0 / tblock) & 1 of plan->P_dev the partial sums of steps
 * kb0..kb0+bt-1 over history slices t < kb0 (bt <= plan->tblock), as the main
 * launch (t < kb0 - tblock) followed by the tail launch (the rest).  Exposed
 * for testing the block kernel alone. */
int fg_block_partials(const fg_plan* plan, int64_t kb0, int32_t bt, void* stream);
/* The sub-block launches of the same block (plan->subblock = S > 0), one after
 * the other on `stream`: sub-block i's slices [kb0 + iS, kb0 + (i+1)S) added
 * into the P rows of the steps b >= (i+1)S + subdelay.  fg_run issues each one
 * when its sub-block's steps are done; exposed so a measurement can replay a
 * block's whole stage (main + tail + sub-blocks) over a resident history.
 * *launched (optional) receives the number of sub-block launches issued. */
int fg_block_subpartials(const fg_plan* plan, int64_t kb0, int32_t bt, void* stream, int32_t* launched);

/* Launch geometry fg_step would use: CTAs, threads per CTA, split factor. */
int fg_step_geometry(const fg_plan* plan, int64_t* ctas, int32_t* threads, int32_t* split);

#ifdef __cplusplus
}
#endif

#endif /* FGB200_H */
