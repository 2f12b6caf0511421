// lifting_group.cuh — 5/3 lifting of one 2^k+1 line spread over G = 8 lanes
// of a warp (an aligned 8-lane segment), for the register-light kernels.
//
// Lane r of the segment holds the E + 1 elements E*r .. E*r + E of the line
// (E = (N-1)/8; the last element of lane r is the first of lane r+1).  Every
// level with stride s < E is lane-local except the update of the two shared
// boundary elements, which needs the detail just across the boundary (one
// shuffle each way); both owners compute the shared element from the same
// operands, so the copies stay identical.  Levels with s >= E act on the
// boundary elements only (y_j = element E*j, j = 0..8; y_8 is lane 7's last)
// and use shuffles with lane stride s / E.
//
// Every output is produced by the same IEEE operations, in the same order,
// as dwt_line_reg / idwt_line_reg (lifting.cuh) and hence the reference
// (wavelet.hpp:48-90): predictions of a level first, then its updates
// (forward); the reverse for the inverse.
#pragma once

#include "lifting.cuh"

namespace wg {

constexpr int kGL = 8;  // lanes per line

// m: the lanes taking part (the caller's 8-lane segment, or the full warp)
__device__ __forceinline__ double seg_up(unsigned m, double x, int d) { return __shfl_up_sync(m, x, d, kGL); }
__device__ __forceinline__ double seg_down(unsigned m, double x, int d) { return __shfl_down_sync(m, x, d, kGL); }
__device__ __forceinline__ double seg_idx(unsigned m, double x, int src) { return __shfl_sync(m, x, src, kGL); }

// The 8-lane segment of the calling lane as a shuffle mask.
__device__ __forceinline__ unsigned seg_mask() { return 0xFFu << (threadIdx.x & 24); }

__device__ __forceinline__ double lift_wr(int k, int half) { return (k == 0 || k == half - 1) ? 0.5 : 0.25; }

// Forward L-level transform.  x: the lane's E + 1 elements; r: lane in the
// segment (0..7).  All 32 lanes of the warp must call it (shuffles).
template <int N, int L>
__device__ __forceinline__ void dwt_line_grp(double (&x)[(N - 1) / kGL + 1], int r, unsigned m = 0xffffffffu) {
    constexpr int E = (N - 1) / kGL;
#pragma unroll
    for (int l = 1; l <= L; ++l) {
        const int s = 1 << (l - 1);
        const int half = ((N - 1) / s) / 2;  // details of this level
        if (s < E) {
            // predictions (lane-local)
#pragma unroll
            for (int o = s; o < E; o += 2 * s) x[o] = lift_pred_fwd(x[o], x[o - s], x[o + s]);
            // interior updates
#pragma unroll
            for (int e = 2 * s; e < E; e += 2 * s) {
                const int k = (E * r + e) / (2 * s);
                x[e] = x[e] + lift_upd(lift_wr(k - 1, half), x[e - s], lift_wr(k, half), x[e + s]);
            }
            // the shared boundary elements: the detail across the boundary
            const double dl = seg_up(m, x[E - s], 1), dr = seg_down(m, x[s], 1);
            const int k0 = (E * r) / (2 * s), k1 = (E * r + E) / (2 * s);
            if (r > 0) x[0] = x[0] + lift_upd(lift_wr(k0 - 1, half), dl, lift_wr(k0, half), x[s]);
            if (r < kGL - 1) x[E] = x[E] + lift_upd(lift_wr(k1 - 1, half), x[E - s], lift_wr(k1, half), dr);
        } else {
            const int t = s / E;  // lane stride; y_j = lane j's x[0], y_8 = lane 7's x[E]
            const double last = seg_idx(m, x[E], kGL - 1);
            {
                const double yl = seg_up(m, x[0], t), yr0 = seg_down(m, x[0], t);
                const double yr = (r + t == kGL) ? last : yr0;
                if ((r % (2 * t)) == t) x[0] = lift_pred_fwd(x[0], yl, yr);
            }
            {
                const double dl = seg_up(m, x[0], t), dr = seg_down(m, x[0], t);
                const int k = r / (2 * t);
                if (r > 0 && (r % (2 * t)) == 0 && r + t < kGL)
                    x[0] = x[0] + lift_upd(lift_wr(k - 1, half), dl, lift_wr(k, half), dr);
            }
            const double nxt = seg_down(m, x[0], 1);
            if (r < kGL - 1) x[E] = nxt;
        }
    }
}

// Inverse L-level transform (in place, interleaved order).
template <int N, int L>
__device__ __forceinline__ void idwt_line_grp(double (&x)[(N - 1) / kGL + 1], int r, unsigned m = 0xffffffffu) {
    constexpr int E = (N - 1) / kGL;
#pragma unroll
    for (int l = L; l >= 1; --l) {
        const int s = 1 << (l - 1);
        const int half = ((N - 1) / s) / 2;
        if (s < E) {
            const double dl = seg_up(m, x[E - s], 1), dr = seg_down(m, x[s], 1);
            const int k0 = (E * r) / (2 * s), k1 = (E * r + E) / (2 * s);
            if (r > 0) x[0] = x[0] - lift_upd(lift_wr(k0 - 1, half), dl, lift_wr(k0, half), x[s]);
            if (r < kGL - 1) x[E] = x[E] - lift_upd(lift_wr(k1 - 1, half), x[E - s], lift_wr(k1, half), dr);
#pragma unroll
            for (int e = 2 * s; e < E; e += 2 * s) {
                const int k = (E * r + e) / (2 * s);
                x[e] = x[e] - lift_upd(lift_wr(k - 1, half), x[e - s], lift_wr(k, half), x[e + s]);
            }
#pragma unroll
            for (int o = s; o < E; o += 2 * s) x[o] = lift_pred_inv(x[o], x[o - s], x[o + s]);
        } else {
            const int t = s / E;
            {
                const double dl = seg_up(m, x[0], t), dr = seg_down(m, x[0], t);
                const int k = r / (2 * t);
                if (r > 0 && (r % (2 * t)) == 0 && r + t < kGL)
                    x[0] = x[0] - lift_upd(lift_wr(k - 1, half), dl, lift_wr(k, half), dr);
            }
            {
                const double last = seg_idx(m, x[E], kGL - 1);
                const double yl = seg_up(m, x[0], t), yr0 = seg_down(m, x[0], t);
                const double yr = (r + t == kGL) ? last : yr0;
                if ((r % (2 * t)) == t) x[0] = lift_pred_inv(x[0], yl, yr);
            }
            const double nxt = seg_down(m, x[0], 1);
            if (r < kGL - 1) x[E] = nxt;
        }
    }
}

// Corner-layout position (wavelet.hpp:102-116) of interleaved index e after
// L levels of a line of N points (runtime e).
template <int N, int L>
__device__ __forceinline__ int corner_pos_rt(int e) {
    if (L == 0) return e;
    if ((e & ((1 << L) - 1)) == 0) return e >> L;
    const int b = __ffs(e) - 1;
    return ((N - 1) >> (b + 1)) + 1 + (e >> (b + 1));
}

// Band index of interleaved index e (0 = sample, 1 + normalised scale).
template <int L>
__device__ __forceinline__ int band_rt(int e) {
    if (L == 0 || (e & ((1 << L) - 1)) == 0) return 0;
    return L - (__ffs(e) - 1);
}

}  // namespace wg
