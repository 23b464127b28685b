// Support kernels: psi tables, schedule expansion, standalone history_sum and stencil: DESIGN.md §3.7.
// Part of the single translation unit csrc/fg_kernels.cu (included there in order).
#ifndef FG_SUPPORT_CUH
#define FG_SUPPORT_CUH

#include "fg_step.cuh"

namespace {

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

}  // namespace

#endif  // FG_SUPPORT_CUH
