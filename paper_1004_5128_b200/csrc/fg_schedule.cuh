// Memory schedules in segment form, shared by host and device code.
//
// Restates /root/reference/pkg/src/fracgrid/schedule.py:
//   full_schedule      :70-76   offsets 0..k, weight 1
//   short_schedule     :79-94   offsets 0..min(floor(L/dt), k), weight 1
//                               (floor(L/dt) is evaluated on the host in Python
//                               exactly as the reference does and passed in)
//   adaptive_schedule  :97-151  dense window 0..a, intervals i>=2 starting at
//                               a^(i-1)+i sampled at stride 2i-1 while
//                               m <= min(a^i, k-i+1), then the dense tail whose
//                               start follows the three-way rule at :137-143.
// In every segment weight == stride (1 for dense runs, 2i-1 for interval i), so
// a segment (m0, count, stride) is the whole description of its entries.
#pragma once

#include <stdint.h>

#define FG_MAX_SEGS 64

struct FgSeg {
    int64_t m0;
    int64_t count;
    int64_t stride;  // also the integer weight
};

#if defined(__CUDACC__)
#define FG_HD __host__ __device__ __forceinline__
#else
#define FG_HD inline
#endif

// Returns the number of segments (>=1) or -1 for invalid arguments.
// `cap` bounds the entries written to s (callers size it; FG_MAX_SEGS suffices
// for every k < 2^62 and base >= 2).
FG_HD int fg_segments(int kind, int64_t k, int64_t base, int64_t horizon, FgSeg* s, int cap = FG_MAX_SEGS) {
    if (k < 0) return -1;
    if (kind == 0) {  // full
        s[0].m0 = 0; s[0].count = k + 1; s[0].stride = 1;
        return 1;
    }
    if (kind == 1) {  // short
        if (horizon < 0) return -1;
        int64_t h = horizon < k ? horizon : k;
        s[0].m0 = 0; s[0].count = h + 1; s[0].stride = 1;
        return 1;
    }
    if (kind != 2 || base < 2) return -1;
    const int64_t a = base;
    if (k <= a) {
        s[0].m0 = 0; s[0].count = k + 1; s[0].stride = 1;
        return 1;
    }
    int n = 0;
    s[n].m0 = 0; s[n].count = a + 1; s[n].stride = 1; ++n;
    bool have = false;
    int64_t last_m = 0, last_i = 0, last_ai = 0;
    int64_t a_prev = a;  // a^(i-1)
    for (int64_t i = 2; n < cap - 1; ++i) {
        const int64_t start = a_prev + i;
        if (start > k) break;
        const int64_t a_i = a_prev * a;
        const int64_t stride = 2 * i - 1;
        const int64_t hi = a_i < (k - i + 1) ? a_i : (k - i + 1);
        if (hi >= start) {
            const int64_t cnt = (hi - start) / stride + 1;
            s[n].m0 = start; s[n].count = cnt; s[n].stride = stride; ++n;
            have = true;
            last_m = start + (cnt - 1) * stride;
            last_i = i;
            last_ai = a_i;
        }
        a_prev = a_i;
    }
    const int64_t tail = !have ? a + 1 : (k > last_ai ? last_ai + 1 : last_m + last_i);
    if (tail <= k) {
        s[n].m0 = tail; s[n].count = k - tail + 1; s[n].stride = 1; ++n;
    }
    return n;
}

FG_HD int64_t fg_schedule_length(const FgSeg* s, int n) {
    int64_t len = 0;
    for (int i = 0; i < n; ++i) len += s[i].count;
    return len;
}

// Weight of offset m in a schedule given as ascending segments (0 if absent).
// A later segment may start inside the stride gap after a segment's last sample
// (the adaptive tail starts at last_m + last_i < last_m + stride), so the range
// test stops at the last sample, not at m0 + count*stride.
FG_HD int32_t fg_seg_weight(const FgSeg* s, int n, int64_t m) {
    for (int i = 0; i < n; ++i) {
        const int64_t d = m - s[i].m0;
        if (d < 0) return 0;
        if (d <= (s[i].count - 1) * s[i].stride) return (d % s[i].stride == 0) ? (int32_t)s[i].stride : 0;
    }
    return 0;
}
