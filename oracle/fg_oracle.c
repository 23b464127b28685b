/*
 * C restatement of the reference GL history stepper — TEST INFRASTRUCTURE ONLY.
 *
 * Checker / CPU baseline for paper_1004_5128_b200 (see oracle/__init__.py); never
 * linked into the product.  Follows /root/reference/pkg/src/fracgrid/:
 *   coefficients.py:76-92  psi recursion  v = ((-v) * ((2 - g) - m)) / m
 *   schedule.py:70-151     full / short / adaptive schedules (segment form)
 *   solver.py:162-197      history_sum: coeff = w * psi[m] (one rounding);
 *                          contiguous 0..M -> accumulate oldest first,
 *                          otherwise gathered newest first; mul then add (no FMA)
 *   solver.py:200-227      update u*decay + diffuse*S (or the saturating form),
 *                          zero ring, non-finite check, append stencil(next)
 *   grid.py:88-106         stencil operation order (1D/3D in the same pattern)
 *
 * Built with -ffp-contract=off so every product and sum rounds separately, exactly
 * like the NumPy reference; OpenMP parallelises over grid points only, which keeps
 * each point's reduction order sequential and hence the output bitwise identical
 * to oracle/fg_oracle.py (checked by tests/test_oracle_c.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
    int64_t B;          /* members */
    int64_t n_m;        /* points per member (prod(shape)) */
    int32_t ndim;       /* 1..3 */
    int32_t reaction;   /* 0 linear (decay form), 1 saturating */
    int64_t shape[3];   /* shape[0..ndim-1], C order */
    const double* gamma;   /* [B] */
    const double* dt;      /* [B] */
    const double* decay;   /* [B] host-evaluated 1 - beta*dt */
    const double* diffuse; /* [B] host-evaluated alpha*dt**gamma/dx**2 */
    double vmax, km;       /* saturating f(u) = -vmax*u/(km+u) */
    int32_t kind;          /* 0 full, 1 short, 2 adaptive */
    int32_t pad_;
    double param;          /* short: length L; adaptive: base a */
    int64_t n_steps;
} fgo_problem;

typedef struct { int64_t m0, count, stride; } fgo_seg;

int fgo_build_table(double gamma, int64_t n, double* out) {
    if (!(gamma > 0.0 && gamma < 2.0) || n < 0) return -1;
    double v = 1.0;
    out[0] = v;
    for (int64_t m = 1; m <= n; ++m) {
        double fm = (double)m;
        v = ((-v) * ((2.0 - gamma) - fm)) / fm;
        out[m] = v;
    }
    return 0;
}

/* Segments of schedule(k); returns segment count (<= 64) or -1. */
static int segments(int32_t kind, int64_t k, double param, double dt, fgo_seg* s) {
    if (k < 0) return -1;
    if (kind == 0) { s[0] = (fgo_seg){0, k + 1, 1}; return 1; }
    if (kind == 1) {
        double h = floor(param / dt);
        int64_t hz = (h >= (double)k) ? k : (int64_t)h;
        s[0] = (fgo_seg){0, hz + 1, 1};
        return 1;
    }
    int64_t a = (int64_t)param;
    if (a < 2) return -1;
    if (k <= a) { s[0] = (fgo_seg){0, k + 1, 1}; return 1; }
    int n = 0;
    s[n++] = (fgo_seg){0, a + 1, 1};
    int have = 0;
    int64_t last_m = 0, last_i = 0, last_ai = 0;
    int64_t a_prev = a;
    for (int64_t i = 2;; ++i) {
        int64_t start = a_prev + i;
        if (start > k) break;
        int64_t a_i = a_prev * a;
        int64_t stride = 2 * i - 1;
        int64_t hi = a_i < (k - i + 1) ? a_i : (k - i + 1);
        if (hi >= start) {
            int64_t cnt = (hi - start) / stride + 1;
            s[n++] = (fgo_seg){start, cnt, stride};
            have = 1;
            last_m = start + (cnt - 1) * stride;
            last_i = i;
            last_ai = a_i;
        }
        a_prev = a_i;
    }
    int64_t tail = !have ? a + 1 : (k > last_ai ? last_ai + 1 : last_m + last_i);
    if (tail <= k) s[n++] = (fgo_seg){tail, k - tail + 1, 1};
    return n;
}

int64_t fgo_schedule(int32_t kind, int64_t k, double param, double dt,
                     int64_t* offs, int64_t* wts, int64_t cap) {
    fgo_seg s[64];
    int ns = segments(kind, k, param, dt, s);
    if (ns < 0) return -1;
    int64_t len = 0;
    for (int i = 0; i < ns; ++i)
        for (int64_t c = 0; c < s[i].count; ++c) {
            if (len < cap) { offs[len] = s[i].m0 + c * s[i].stride; wts[len] = s[i].stride; }
            ++len;
        }
    return len;
}

static void stencil_member(const fgo_problem* p, const double* u, double* out, int64_t lo, int64_t hi) {
    const int64_t* sh = p->shape;
    for (int64_t q = lo; q < hi; ++q) {
        double r = 0.0;
        if (p->ndim == 1) {
            if (q > 0 && q < sh[0] - 1) r = (u[q + 1] + u[q - 1]) - 2.0 * u[q];
        } else if (p->ndim == 2) {
            int64_t j = q / sh[1], l = q % sh[1];
            if (j > 0 && j < sh[0] - 1 && l > 0 && l < sh[1] - 1) {
                int64_t sx = sh[1];
                r = (((u[q + sx] + u[q - sx]) - 4.0 * u[q]) + u[q + 1]) + u[q - 1];
            }
        } else {
            int64_t sx = sh[1] * sh[2], sy = sh[2];
            int64_t i0 = q / sx, i1 = (q / sy) % sh[1], i2 = q % sh[2];
            if (i0 > 0 && i0 < sh[0] - 1 && i1 > 0 && i1 < sh[1] - 1 && i2 > 0 && i2 < sh[2] - 1)
                r = (((((u[q + sx] + u[q - sx]) - 6.0 * u[q]) + u[q + sy]) + u[q - sy]) + u[q + 1]) + u[q - 1];
        }
        out[q] = r;
    }
}

static int on_ring(const fgo_problem* p, int64_t q) {
    const int64_t* sh = p->shape;
    if (p->ndim == 1) return q == 0 || q == sh[0] - 1;
    if (p->ndim == 2) {
        int64_t j = q / sh[1], l = q % sh[1];
        return j == 0 || j == sh[0] - 1 || l == 0 || l == sh[1] - 1;
    }
    int64_t sx = sh[1] * sh[2], sy = sh[2];
    int64_t i0 = q / sx, i1 = (q / sy) % sh[1], i2 = q % sh[2];
    return i0 == 0 || i0 == sh[0] - 1 || i1 == 0 || i1 == sh[1] - 1 || i2 == 0 || i2 == sh[2] - 1;
}

#define CHUNK 512

/*
 * Run the stepper.  u_io: [B*n_m] initial field in, final field out (on
 * divergence: the rejected non-finite field, so the caller can take its peak).
 * snaps: [n_snap][B*n_m] for the sorted snapshot steps (0 allowed).
 * Returns 0, 1 on divergence (*bad_step = k+1), <0 on bad arguments / OOM.
 */
int fgo_run(const fgo_problem* p, double* u_io, int64_t n_snap, const int64_t* snap_steps,
            double* snaps, int64_t* bad_step, int nthreads, int64_t max_steps, double* elapsed_s) {
    const int64_t B = p->B, nm = p->n_m, N = B * nm, T = p->n_steps;
    int64_t steps = (max_steps >= 0 && max_steps < T) ? max_steps : T;
    if (nthreads > 0) omp_set_num_threads(nthreads);
    double* H = (double*)malloc((size_t)(steps + 1) * (size_t)N * sizeof(double));
    double* tab = (double*)malloc((size_t)B * (size_t)(T + 1) * sizeof(double));
    double* nxt = (double*)malloc((size_t)N * sizeof(double));
    double* u = (double*)malloc((size_t)N * sizeof(double));
    /* per-member expanded schedule (t, coeff) */
    int64_t cap = steps + 1;
    int64_t* tix = (int64_t*)malloc((size_t)B * (size_t)cap * sizeof(int64_t));
    double* cof = (double*)malloc((size_t)B * (size_t)cap * sizeof(double));
    int64_t* len = (int64_t*)malloc((size_t)B * sizeof(int64_t));
    int* contig = (int*)malloc((size_t)B * sizeof(int));
    if (!H || !tab || !nxt || !u || !tix || !cof || !len || !contig) {
        free(H); free(tab); free(nxt); free(u); free(tix); free(cof); free(len); free(contig);
        return -2;
    }
    for (int64_t b = 0; b < B; ++b)
        if (fgo_build_table(p->gamma[b], T, tab + b * (T + 1))) return -1;
    /* first-touch the history in parallel, outside the timed loop (page faults
       taken inside the loop serialise on the address-space lock) */
    {
        const int64_t total = (steps + 1) * N;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < total; i += 512) H[i] = 0.0;
    }
    memcpy(u, u_io, (size_t)N * sizeof(double));
    for (int64_t b = 0; b < B; ++b) stencil_member(p, u + b * nm, H + b * nm, 0, nm);
    int64_t si = 0;
    while (si < n_snap && snap_steps[si] == 0) {
        memcpy(snaps + si * N, u, (size_t)N * sizeof(double));
        ++si;
    }
    int rc = 0;
    double t0 = omp_get_wtime();
    for (int64_t k = 0; k < steps; ++k) {
        /* schedule per member (members differ only through dt for short memory) */
        for (int64_t b = 0; b < B; ++b) {
            fgo_seg s[64];
            int ns = segments(p->kind, k, p->param, p->dt[b], s);
            int64_t n = 0;
            const double* tb = tab + b * (T + 1);
            for (int i = 0; i < ns; ++i)
                for (int64_t c = 0; c < s[i].count; ++c) {
                    int64_t m = s[i].m0 + c * s[i].stride;
                    tix[b * cap + n] = k - m;
                    cof[b * cap + n] = (double)s[i].stride * tb[m];
                    ++n;
                }
            len[b] = n;
            contig[b] = (tix[b * cap + n - 1] == k - (n - 1));  /* offsets 0..n-1 */
        }
        int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
        for (int64_t blk = 0; blk < (N + CHUNK - 1) / CHUNK; ++blk) {
            int64_t g0 = blk * CHUNK, g1 = g0 + CHUNK < N ? g0 + CHUNK : N;
            /* a chunk may straddle members: split it */
            for (int64_t g = g0; g < g1;) {
                int64_t b = g / nm, q0 = g % nm;
                int64_t q1 = q0 + (g1 - g);
                if (q1 > nm) q1 = nm;
                double acc[CHUNK];
                int64_t w = q1 - q0;
                for (int64_t i = 0; i < w; ++i) acc[i] = 0.0;
                const int64_t n = len[b];
                const int64_t* tt = tix + b * cap;
                const double* cc = cof + b * cap;
                if (contig[b]) {
                    for (int64_t j = n - 1; j >= 0; --j) {  /* oldest first */
                        const double c = cc[j];
                        const double* h = H + tt[j] * N + b * nm + q0;
                        for (int64_t i = 0; i < w; ++i) acc[i] = acc[i] + c * h[i];
                    }
                } else {
                    for (int64_t j = 0; j < n; ++j) {       /* newest first */
                        const double c = cc[j];
                        const double* h = H + tt[j] * N + b * nm + q0;
                        for (int64_t i = 0; i < w; ++i) acc[i] = acc[i] + c * h[i];
                    }
                }
                const double* ub = u + b * nm;
                double* nb = nxt + b * nm;
                for (int64_t i = 0; i < w; ++i) {
                    int64_t q = q0 + i;
                    double r;
                    if (p->reaction == 0) {
                        r = ub[q] * p->decay[b] + p->diffuse[b] * acc[i];
                    } else {
                        double f = ((-p->vmax) * ub[q]) / (p->km + ub[q]);
                        r = (ub[q] + p->dt[b] * f) + p->diffuse[b] * acc[i];
                    }
                    if (on_ring(p, q)) r = 0.0;
                    if (!isfinite(r)) bad = 1;
                    nb[q] = r;
                }
                g += w;
            }
        }
        if (bad) {
            *bad_step = k + 1;
            memcpy(u_io, nxt, (size_t)N * sizeof(double));
            rc = 1;
            break;
        }
        double* tmp = u; u = nxt; nxt = tmp;
        {
            const int64_t cpm = (nm + CHUNK - 1) / CHUNK;
#pragma omp parallel for schedule(static)
            for (int64_t blk = 0; blk < B * cpm; ++blk) {
                int64_t b = blk / cpm, q0 = (blk % cpm) * CHUNK;
                int64_t q1 = q0 + CHUNK < nm ? q0 + CHUNK : nm;
                stencil_member(p, u + b * nm, H + (k + 1) * N + b * nm, q0, q1);
            }
        }
        while (si < n_snap && snap_steps[si] == k + 1) {
            memcpy(snaps + si * N, u, (size_t)N * sizeof(double));
            ++si;
        }
    }
    *elapsed_s = omp_get_wtime() - t0;
    if (rc == 0) memcpy(u_io, u, (size_t)N * sizeof(double));
    free(H); free(tab); free(nxt); free(u); free(tix); free(cof); free(len); free(contig);
    return rc;
}

int fgo_max_threads(void) { return omp_get_max_threads(); }
