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
// IEEE roundings as dwt_step_1d / idwt_step_1d (wavelet.hpp:48-90):
//   detail  d_k = s_{2k+1} - (s_{2k} + s_{2k+2}) / 2.0
//   coarse  c_k = s_{2k} + (w(k-1) d_{k-1} + w(k) d_k),  w = 1/2 at the two
//           boundary details, 1/4 inside (lift_weight, wavelet.hpp:31-33)
// The file is compiled with -fmad=false, so no implicit contraction changes
// the rounding.  Explicit FMAs are used only where every fused product is
// exact (multiplications by 2, 1/2 and 1/4 are exact for normal doubles), so
// each expression still rounds exactly where the reference rounds:
//   d = s_odd - (l + r)/2         == fma(-0.5, l + r, s_odd)
//   w0 d0 + w1 d1                 == 1/4 * (d0 + d1)         (w0 = w1 = 1/4)
//                                 == 1/4 * fma(2, d0, d1)    (w0 = 1/2, w1 = 1/4)
//                                 == 1/2 * (d0 + d1)         (w0 = w1 = 1/2)
//   (the one rounding of the reference's sum is the rounding of the bracket:
//   scaling by a power of two commutes with rounding)
//   c = s + 1/4 * t               == fma(1/4, t, s)           (1/4 t is exact)
// so a predict costs 2 fp64 instructions and an update 2 (3 in the
// reference's own form).  Results could only differ if a product underflowed
// into the subnormal range (|d| < 2^-1020); WG_LIFT_NO_FMA removes even that
// at one more instruction per element.
#pragma once

#include <type_traits>

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

// The update term w(k-1) d0 + w(k) d1 as scale * t (scale a power of two,
// t rounded exactly once); k and half are compile-time after unrolling.
__device__ __forceinline__ double upd_t(int k, int half, double d0, double d1) {
    const double w0 = lift_w(k - 1, half), w1 = lift_w(k, half);
#ifdef WG_LIFT_NO_FMA
    if (w0 == w1) return d0 + d1;
    return w0 > w1 ? 2.0 * d0 + d1 : d0 + 2.0 * d1;
#else
    if (w0 == w1) return d0 + d1;
    return w0 > w1 ? __fma_rn(2.0, d0, d1) : __fma_rn(2.0, d1, d0);
#endif
}
__host__ __device__ constexpr double upd_scale(int k, int half) {
    return lift_w(k - 1, half) < lift_w(k, half) ? lift_w(k - 1, half) : lift_w(k, half);
}

#ifdef WG_LIFT_NO_FMA
__device__ __forceinline__ double lift_pred_fwd(double odd, double l, double r) { return odd - (l + r) / 2.0; }
__device__ __forceinline__ double lift_pred_inv(double odd, double l, double r) { return odd + (l + r) / 2.0; }
__device__ __forceinline__ double lift_upd_fwd(double s, double sc, double t) { return s + sc * t; }
__device__ __forceinline__ double lift_upd_inv(double s, double sc, double t) { return s - sc * t; }
#else
__device__ __forceinline__ double lift_pred_fwd(double odd, double l, double r) { return __fma_rn(-0.5, l + r, odd); }
__device__ __forceinline__ double lift_pred_inv(double odd, double l, double r) { return __fma_rn(0.5, l + r, odd); }
__device__ __forceinline__ double lift_upd_fwd(double s, double sc, double t) { return __fma_rn(sc, t, s); }
__device__ __forceinline__ double lift_upd_inv(double s, double sc, double t) { return __fma_rn(-sc, t, s); }
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
            v[2 * k * s] = lift_upd_fwd(v[2 * k * s], upd_scale(k, half),
                                        upd_t(k, half, v[(2 * k - 1) * s], v[(2 * k + 1) * s]));
    }
}

// Inverse multi-level transform of v[0..N) in place (interleaved order).
// Z: the details of the Z finest levels are known to be +0.0 (the rows /
// columns of a block that CSR-decode to nothing): their update is the
// identity (s - 1/4 (+0 + +0) == s bit for bit, -0.0 and NaN included) and
// their predict d + (l+r)/2 keeps d = +0.0 as a constant operand, so the
// outputs are bit-identical to the full inverse; the detail registers of
// those levels are never read.
template <int N, int L, int Z = 0>
__device__ __forceinline__ void idwt_line_reg(double (&v)[N]) {
#pragma unroll
    for (int l = L; l >= 1; --l) {
        const int s = 1 << (l - 1);
        const int len = (N - 1) / s + 1;
        const int half = (len - 1) / 2;
        if (l > Z) {
#pragma unroll
            for (int k = 1; k < half; ++k)
                v[2 * k * s] = lift_upd_inv(v[2 * k * s], upd_scale(k, half),
                                            upd_t(k, half, v[(2 * k - 1) * s], v[(2 * k + 1) * s]));
#pragma unroll
            for (int k = 0; k < half; ++k)
                v[(2 * k + 1) * s] = lift_pred_inv(v[(2 * k + 1) * s], v[2 * k * s], v[(2 * k + 2) * s]);
        } else {
#pragma unroll
            for (int k = 0; k < half; ++k)
                v[(2 * k + 1) * s] = lift_pred_inv(0.0, v[2 * k * s], v[(2 * k + 2) * s]);
        }
    }
}

// Highest corner-layout position an inverse with Z zero finest levels reads.
__host__ __device__ constexpr int z_top(int N, int Z) { return (N - 1) >> Z; }

// Largest Z (<= L) whose zero-detail levels hold no position above `top`
// (top = -1: nothing stored).
__device__ __forceinline__ int z_of_top(int N, int L, int top) {
    int z = 0;
    while (z < L && top <= ((N - 1) >> (z + 1))) ++z;
    return z;
}

// Dispatch of idwt_line_reg<N, L, Z> on a runtime Z in [0, L].
template <int N, int L, int Z = 0>
__device__ __forceinline__ void idwt_line_z(double (&v)[N], int z) {
    if constexpr (Z < L) {
        if (z == Z) idwt_line_reg<N, L, Z>(v);
        else idwt_line_z<N, L, Z + 1>(v, z);
    } else {
        idwt_line_reg<N, L, L>(v);
    }
}

// f(std::integral_constant<int, Z>{}) for a runtime z in [0, L]: the
// caller's load pattern and transform specialise on Z (no merge of the
// variants' register lines before the consumer).
template <int L, typename F, int Z = 0>
__device__ __forceinline__ void with_z(int z, F&& f) {
    if constexpr (Z < L) {
        if (z == Z) f(std::integral_constant<int, Z>{});
        else with_z<L, F, Z + 1>(z, static_cast<F&&>(f));
    } else {
        f(std::integral_constant<int, L>{});
    }
}

// The same dispatch, handing the result to emit() inside each variant (no
// merge of the variants' register lines before the consumer).
template <int N, int L, typename Emit, int Z = 0>
__device__ __forceinline__ void idwt_line_z_emit(double (&v)[N], int z, Emit&& emit) {
    if constexpr (Z < L) {
        if (z == Z) {
            idwt_line_reg<N, L, Z>(v);
            emit(v);
        } else {
            idwt_line_z_emit<N, L, Emit, Z + 1>(v, z, static_cast<Emit&&>(emit));
        }
    } else {
        idwt_line_reg<N, L, L>(v);
        emit(v);
    }
}

}  // namespace wg
