// lifting.cuh — register-resident 5/3 lifting on one 2^k+1 line (sm_100a).
//
// A thread owns a whole line of N = 2^k + 1 doubles in registers.  All
// indices are compile-time constants (N and the level count L are template
// parameters, every loop is unrolled), so the array lives in registers and a
// multi-level transform is straight-line DADD/DMUL code: no shared-memory
// traffic and no shuffles inside a line.
//
// Naming: registers are kept in the INTERLEAVED (in-place lifting) order.
// After level l (stride s = 2^(l-1)) the coarse values sit at multiples of
// 2s and the level-l details at odd multiples of s.  The reference stores
// the CORNER layout instead (dwt_line, wavelet.hpp:102-116: samples first,
// then detail bands coarse -> fine); corner_pos() maps an interleaved
// register index to its corner-layout position, so converting between the
// two is free register renaming at load/store time.
//
// Bit parity with the reference: every output is produced by the same
// sequence of IEEE operations as dwt_step_1d / idwt_step_1d
// (wavelet.hpp:48-90):
//   detail  d_k = s_{2k+1} - (s_{2k} + s_{2k+2}) / 2.0
//   coarse  c_k = s_{2k} + (w(k-1) d_{k-1} + w(k) d_k),  w = 1/2 at the two
//           boundary details, 1/4 inside (lift_weight, wavelet.hpp:31-33)
// The file is compiled with -fmad=false, so no implicit contraction changes
// the rounding.  Two explicit FMAs are used where the fused product is exact
// (a multiplication by 1/2 or 1/4 is exact for every normal double):
//   d = s_odd - (l + r)/2          == fma(-0.5, l + r, s_odd)
//   w0*d0 + w1*d1 (both exact)     == fma(w0, d0, w1*d1)
// so the results are bit-identical to the reference's separate operations
// (SURVEY A1.2 measured 0 mismatches for the second form).  They could only
// differ if a product underflowed into the subnormal range (|d| < 2^-1020),
// which WG_LIFT_NO_FMA removes at the cost of one instruction per element.
#pragma once

namespace wg {

__host__ __device__ constexpr int ctz_c(int r) {
    int b = 0;
    while (!(r & 1)) {
        r >>= 1;
        ++b;
    }
    return b;
}

// Corner-layout position of interleaved index r after L levels on a line of
// N points (wavelet.hpp:99-101 / CoefficientSet::band :162-170).
template <int N, int L>
__host__ __device__ constexpr int corner_pos(int r) {
    if (L == 0) return r;
    if (r % (1 << L) == 0) return r >> L;
    const int b = ctz_c(r);  // detail of level b+1
    return ((N - 1) >> (b + 1)) + 1 + (r >> (b + 1));
}

// Band index of interleaved index r: 0 = sample, else 1 + normalised scale
// (coarsest detail band = scale 0, CoefficientSet::band wavelet.hpp:162-170).
template <int N, int L>
__host__ __device__ constexpr int band_of_r(int r) {
    if (L == 0 || r % (1 << L) == 0) return 0;
    return L - ctz_c(r);  // level l = b + 1 -> scale L - l -> index L - b
}

// Interleaved index of corner-layout position p (inverse of corner_pos).
template <int N, int L>
__host__ __device__ constexpr int interleaved_of(int p) {
    if (L == 0 || p <= ((N - 1) >> L)) return p << L;
    for (int l = L; l >= 1; --l)
        if (p <= ((N - 1) >> (l - 1))) {
            const int k = p - ((N - 1) >> l) - 1;
            return (2 * k + 1) << (l - 1);
        }
    return -1;
}

// Band index of a corner-layout position p (runtime; rows of a tile).
__host__ __device__ inline int band_of_pos(int n, int L, int p) {
    const int m = n - 1;
    if (L == 0 || p <= (m >> L)) return 0;
    for (int l = L; l >= 1; --l)
        if (p <= (m >> (l - 1))) return 1 + (L - l);
    return 0;
}

__host__ __device__ constexpr double lift_w(int k, int half) {
    return (k == 0 || k == half - 1) ? 0.5 : 0.25;
}

#ifdef WG_LIFT_NO_FMA
__device__ __forceinline__ double lift_pred_fwd(double odd, double l, double r) { return odd - (l + r) / 2.0; }
__device__ __forceinline__ double lift_pred_inv(double odd, double l, double r) { return odd + (l + r) / 2.0; }
__device__ __forceinline__ double lift_upd(double w0, double d0, double w1, double d1) { return w0 * d0 + w1 * d1; }
#else
__device__ __forceinline__ double lift_pred_fwd(double odd, double l, double r) { return __fma_rn(-0.5, l + r, odd); }
__device__ __forceinline__ double lift_pred_inv(double odd, double l, double r) { return __fma_rn(0.5, l + r, odd); }
__device__ __forceinline__ double lift_upd(double w0, double d0, double w1, double d1) {
    return __fma_rn(w0, d0, w1 * d1);
}
#endif

// Forward multi-level transform of v[0..N) in place (interleaved order).
template <int N, int L>
__device__ __forceinline__ void dwt_line_reg(double (&v)[N]) {
#pragma unroll
    for (int l = 1; l <= L; ++l) {
        const int s = 1 << (l - 1);
        const int len = (N - 1) / s + 1;  // signal length at this level
        const int half = (len - 1) / 2;
#pragma unroll
        for (int k = 0; k < half; ++k)
            v[(2 * k + 1) * s] = lift_pred_fwd(v[(2 * k + 1) * s], v[2 * k * s], v[(2 * k + 2) * s]);
#pragma unroll
        for (int k = 1; k < half; ++k)
            v[2 * k * s] = v[2 * k * s] + lift_upd(lift_w(k - 1, half), v[(2 * k - 1) * s], lift_w(k, half),
                                                   v[(2 * k + 1) * s]);
    }
}

// Inverse multi-level transform of v[0..N) in place (interleaved order).
template <int N, int L>
__device__ __forceinline__ void idwt_line_reg(double (&v)[N]) {
#pragma unroll
    for (int l = L; l >= 1; --l) {
        const int s = 1 << (l - 1);
        const int len = (N - 1) / s + 1;
        const int half = (len - 1) / 2;
#pragma unroll
        for (int k = 1; k < half; ++k)
            v[2 * k * s] = v[2 * k * s] - lift_upd(lift_w(k - 1, half), v[(2 * k - 1) * s], lift_w(k, half),
                                                   v[(2 * k + 1) * s]);
#pragma unroll
        for (int k = 0; k < half; ++k)
            v[(2 * k + 1) * s] = lift_pred_inv(v[(2 * k + 1) * s], v[2 * k * s], v[(2 * k + 2) * s]);
    }
}

}  // namespace wg
