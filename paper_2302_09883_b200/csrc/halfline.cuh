// halfline.cuh — half-line ownership for 65-point patches (tuning variant,
// selected with WG_HALF_LINES=1; the default full-line kernels measured
// faster in round 1: 7.98 vs 6.62 GLUPS at C2).
//
// With one thread per 65-point line a thread keeps 130 registers of line
// data and an SM holds only ~7-10 warps (patch_phases.cuh).  Here two lanes
// (l and l ^ 16 of one warp) own one line: the lower lane holds logical
// points 0..M and the upper lane points N-1..M mirrored (M = (N-1)/2; the
// midpoint is held by both).  Every lifting level needs one shuffle with the
// partner (the detail on the other side of the midpoint, or the far endpoint
// at the 3-point level of an L = k transform); everything else is local
// registers with compile-time indices.  Each output is computed from the same
// operands as the one-thread lifting (lifting.cuh) and the reference
// (wavelet.hpp:48-90), so results are bit-identical (tests pass with
// WG_HALF_LINES=1).
#pragma once

#include "patch_phases.cuh"

namespace wg {

template <int N>
struct HT {
    static constexpr int M = (N - 1) / 2;  // logical midpoint
    static constexpr int H = M + 1;        // elements per half
    static constexpr int TP = N + 2;       // row pitch (odd)
    static constexpr int TILE = TP * TP;
    __host__ __device__ static constexpr int at(int tr, int tc) { return tr * TP + tc; }
    __host__ __device__ static constexpr int rx(int tr) { return tr * TP; }
    __host__ __device__ static constexpr int cx(int tc) { return tc; }
};

// The two lanes of a line are lane l and l ^ 16 of one warp: a warp holds
// 16 lines, lanes 0-15 their lower halves and lanes 16-31 their upper
// halves, so every half-warp memory phase touches 16 different lines of the
// same half (bank-conflict free like the one-thread-per-line layout).
constexpr int kPairXor = 16;

__device__ __forceinline__ double pair_xchg(double x) {
    return __shfl_xor_sync(__activemask(), x, kPairXor);
}

// thread -> (global line, half) map and its inverse (thread of the lower half)
__device__ __forceinline__ int hl_line(int t) { return (t >> 5) * 16 + (t & 15); }
__device__ __forceinline__ int hl_half(int t) { return (t >> 4) & 1; }
__device__ __forceinline__ int hl_thread(int line) { return (line >> 4) * 32 + (line & 15); }

template <typename T>
__device__ __forceinline__ T hsel(int h, T lo, T hi) {
    return h ? hi : lo;
}

// Lane h = 0 holds logical points 0..M in order (local k = point k); lane
// h = 1 holds points N-1..M MIRRORED (local k = point N-1-k).  Local 0 is
// the line's endpoint and local M the midpoint for both lanes, and the 5/3
// lifting is mirror-symmetric: lift_weight(k) == lift_weight(half-1-k)
// (wavelet.hpp:31-33), the band map satisfies band(r) == band(N-1-r), and
// predict (l + r)/2 and the exact-product update sum are order-independent.
// So both lanes run the SAME straight-line code on their registers; only
// the midpoint update (and the 3-point level of an L = k transform) needs
// the partner's value.
template <int N>
__host__ __device__ constexpr int hglobal(int h, int k) {
    return h ? N - 1 - k : k;
}

// Forward multi-level lifting of the half line v[0..M].
template <int N, int L>
__device__ __forceinline__ void dwt_half(double (&v)[HT<N>::H], int h) {
    constexpr int M = HT<N>::M;
#pragma unroll
    for (int l = 1; l <= L; ++l) {
        const int st = 1 << (l - 1);
        const int len = (N - 1) / st + 1;
        const int half = (len - 1) / 2;
        if (2 * st <= M) {
            const int nd = M / (2 * st);
#pragma unroll
            for (int j = 0; j < nd; ++j)
                v[(2 * j + 1) * st] = lift_pred_fwd(v[(2 * j + 1) * st], v[2 * j * st], v[(2 * j + 2) * st]);
#pragma unroll
            for (int j = 1; j < nd; ++j)
                v[2 * j * st] = v[2 * j * st] +
                                lift_upd(lift_w(j - 1, half), v[(2 * j - 1) * st], lift_w(j, half), v[(2 * j + 1) * st]);
            const double mine = v[M - st];
            const double other = pair_xchg(mine);
            const double dl = h ? other : mine, dr = h ? mine : other;
            v[M] = v[M] + lift_upd(lift_w(nd - 1, half), dl, lift_w(nd, half), dr);
        } else {  // st == M: the 3-point level of an L = k transform
            const double mine = v[0];
            const double other = pair_xchg(mine);
            const double s0 = h ? other : mine, sn = h ? mine : other;
            v[M] = lift_pred_fwd(v[M], s0, sn);
        }
    }
}

template <int N, int L>
__device__ __forceinline__ void idwt_half(double (&v)[HT<N>::H], int h) {
    constexpr int M = HT<N>::M;
#pragma unroll
    for (int l = L; l >= 1; --l) {
        const int st = 1 << (l - 1);
        const int len = (N - 1) / st + 1;
        const int half = (len - 1) / 2;
        if (2 * st <= M) {
            const int nd = M / (2 * st);
#pragma unroll
            for (int j = 1; j < nd; ++j)
                v[2 * j * st] = v[2 * j * st] -
                                lift_upd(lift_w(j - 1, half), v[(2 * j - 1) * st], lift_w(j, half), v[(2 * j + 1) * st]);
            const double mine = v[M - st];
            const double other = pair_xchg(mine);
            const double dl = h ? other : mine, dr = h ? mine : other;
            v[M] = v[M] - lift_upd(lift_w(nd - 1, half), dl, lift_w(nd, half), dr);
#pragma unroll
            for (int j = 0; j < nd; ++j)
                v[(2 * j + 1) * st] = lift_pred_inv(v[(2 * j + 1) * st], v[2 * j * st], v[(2 * j + 2) * st]);
        } else {
            const double mine = v[0];
            const double other = pair_xchg(mine);
            const double s0 = h ? other : mine, sn = h ? mine : other;
            v[M] = lift_pred_inv(v[M], s0, sn);
        }
    }
}

// corner-layout position of local element k of half h
template <int N, int L>
__device__ __forceinline__ int hpos(int h, int k) {
    return hsel(h, corner_pos<N, L>(k), corner_pos<N, L>(N - 1 - k));
}

// ---- tile phases (pair = lanes 2li, 2li+1 of one line) -------------------
// "own" elements: the midpoint (local M) belongs to lane 0 for every write
// and every count.

// ROW phase of the decode for row li.  Every lane of the CTA calls it (it
// contains __syncwarp); inactive lanes pass active = false.
template <int N, int L>
__device__ __forceinline__ bool decode_row_h(double* T, int li, int h, bool active, const DirEntry e,
                                             const unsigned char* store) {
    constexpr int M = HT<N>::M, H = HT<N>::H, TP = HT<N>::TP;
    double* rowp = T + (li + 1) * TP + 1;
    const bool raw = (e.flags & DIR_RAW) != 0 && !(e.flags & DIR_DEAD);
    if (active && !raw) {
#pragma unroll
        for (int k = 0; k < H; ++k)
            if (h == 0 || k < M) rowp[hglobal<N>(h, k)] = 0.0;
    }
    __syncwarp();
    if (active && !(e.flags & DIR_DEAD)) {
        const unsigned char* base = store + e.off;
        if (raw) {
            const double* d = reinterpret_cast<const double*>(base) + (size_t)li * N;
#pragma unroll
            for (int k = 0; k < H; ++k)
                if (h == 0 || k < M) rowp[hglobal<N>(h, k)] = d[hglobal<N>(h, k)];
        } else {
            const double* v = reinterpret_cast<const double*>(base);
            const uint32_t* col = reinterpret_cast<const uint32_t*>(base + 8ull * e.nnz);
            const uint32_t* ro = col + e.nnz;
            const uint32_t k0 = ro[li], k1 = ro[li + 1];
            for (uint32_t kk = k0 + h; kk < k1; kk += 2) rowp[col[kk]] = v[kk];
        }
    }
    __syncwarp();
    if (active && !raw) {
        double x[H];
#pragma unroll
        for (int k = 0; k < H; ++k) x[k] = rowp[hpos<N, L>(h, k)];
        __syncwarp(__activemask());
        idwt_half<N, L>(x, h);
#pragma unroll
        for (int k = 0; k < H; ++k)
            if (h == 0 || k < M) rowp[hglobal<N>(h, k)] = x[k];
    }
    return raw;
}

template <int N>
__device__ __forceinline__ void fill_ghosts_h(double* T, int li, int h, const EdgeSet& e, const PatchPos& pp,
                                              uint32_t q, const ShardGeom& g) {
    using G = HT<N>;
    if (h == 0) {
        T[G::at(li + 1, 0)] = e.colhi[edge_ix(pp.ar, pp.bl, q, g, N) + li];
        T[G::at(0, li + 1)] = e.rowhi[edge_ix(pp.su, pp.b, q, g, N) + li];
        if (li == 0) {
            T[G::at(0, 0)] = e.rowhi[edge_ix(pp.su, pp.bl, q, g, N) + N - 2];
            T[G::at(0, N + 1)] = e.rowhi[edge_ix(pp.su, pp.br, q, g, N) + 1];
        }
    } else {
        T[G::at(li + 1, N + 1)] = e.collo[edge_ix(pp.ar, pp.br, q, g, N) + li];
        T[G::at(N + 1, li + 1)] = e.rowlo[edge_ix(pp.sd, pp.b, q, g, N) + li];
        if (li == 0) {
            T[G::at(N + 1, 0)] = e.rowlo[edge_ix(pp.sd, pp.bl, q, g, N) + N - 2];
            T[G::at(N + 1, N + 1)] = e.rowlo[edge_ix(pp.sd, pp.br, q, g, N) + 1];
        }
    }
}

// COLUMN phase of the decode: column j, inverse along dim 0 -> natural order
template <int N, int L>
__device__ __forceinline__ void decode_col_h(const double* T, int j, int h, bool raw, double (&v)[HT<N>::H]) {
    constexpr int H = HT<N>::H, TP = HT<N>::TP;
    const double* colp = T + TP + j + 1;
    if (raw) {
#pragma unroll
        for (int k = 0; k < H; ++k) v[k] = colp[hglobal<N>(h, k) * TP];
    } else {
#pragma unroll
        for (int k = 0; k < H; ++k) v[k] = colp[hpos<N, L>(h, k) * TP];
        idwt_half<N, L>(v, h);
    }
}

template <int N>
__device__ __forceinline__ void store_col_h(double* T, int j, int h, const double (&v)[HT<N>::H]) {
    constexpr int M = HT<N>::M, H = HT<N>::H, TP = HT<N>::TP;
    double* colp = T + TP + j + 1;
#pragma unroll
    for (int k = 0; k < H; ++k)
        if (h == 0 || k < M) colp[hglobal<N>(h, k) * TP] = v[k];
}

template <int N, int L>
__device__ __forceinline__ void fwd_col_to_tile_h(double* T, int j, int h, double (&v)[HT<N>::H]) {
    constexpr int M = HT<N>::M, H = HT<N>::H, TP = HT<N>::TP;
    dwt_half<N, L>(v, h);
    double* colp = T + TP + j + 1;
#pragma unroll
    for (int k = 0; k < H; ++k)
        if (h == 0 || k < M) colp[hpos<N, L>(h, k) * TP] = v[k];
}

// ROW phase of the compression for row i: forward along dim 1, threshold
// (threshold.hpp:51-86), kept / zeroed counts of the lane's own elements.
template <int N, int L>
__device__ __forceinline__ void fwd_row_threshold_h(const double* T, int i, int h, const double* thr,
                                                    double (&v)[HT<N>::H], unsigned& nz, unsigned& zr) {
    constexpr int M = HT<N>::M, H = HT<N>::H, TP = HT<N>::TP;
    const double* rowp = T + (i + 1) * TP + 1;
#pragma unroll
    for (int k = 0; k < H; ++k) v[k] = rowp[hglobal<N>(h, k)];
    dwt_half<N, L>(v, h);
    const int bi = band_of_pos(N, L, i);
    double trow[L + 1];
#pragma unroll
    for (int bj = 0; bj <= L; ++bj) trow[bj] = thr[bi * (L + 1) + bj];
    nz = 0;
    zr = 0;
#pragma unroll
    for (int k = 0; k < H; ++k) {  // band(k) == band(N-1-k): same threshold for both lanes
        const double x = v[k];
        const bool nzx = x != 0.0;
        const bool kill = fabs(x) < trow[band_of_r<N, L>(k)];
        const bool keep = nzx && !kill;
        v[k] = keep ? x : 0.0;
        const bool own = h == 0 || k < M;
        zr += (own && nzx && kill) ? 1u : 0u;
        nz += (own && keep) ? 1u : 0u;
    }
}

// Ordered CSR write of row i by the lane pair (csr_encode, codec.hpp:37-60).
// In corner order every band is lane 0's elements (ascending k) followed by
// lane 1's (descending k, i.e. ascending position); rowk = entry offset of
// the row inside the block.
template <int N, int L>
__device__ __forceinline__ void write_csr_row_h(unsigned char* base, uint32_t nnz_tot, int i, int h, uint32_t rowk,
                                                const double (&v)[HT<N>::H]) {
    constexpr int M = HT<N>::M, H = HT<N>::H;
    double* vo = reinterpret_cast<double*>(base);
    uint32_t* co = reinterpret_cast<uint32_t*>(base + 8ull * nnz_tot);
    uint32_t* ro = co + nnz_tot;
    unsigned cnt[L + 1];
#pragma unroll
    for (int b = 0; b <= L; ++b) cnt[b] = 0;
#pragma unroll
    for (int k = 0; k < H; ++k)
        cnt[band_of_r<N, L>(k)] += (v[k] != 0.0 && (h == 0 || k < M)) ? 1u : 0u;
    unsigned start[L + 1];
    unsigned acc = rowk;
    const unsigned mask = __activemask();
#pragma unroll
    for (int b = 0; b <= L; ++b) {
        const unsigned other = __shfl_xor_sync(mask, cnt[b], kPairXor);
        const unsigned ca = h ? other : cnt[b], cb = h ? cnt[b] : other;
        // lane 1 fills its chunk from the back: start = last slot of it
        start[b] = h ? acc + ca + cb - 1u : acc;
        acc += ca + cb;
    }
    if (h == 0) {
        if (i == 0) ro[0] = 0;
        ro[i + 1] = acc;
    }
    unsigned rank[L + 1];
#pragma unroll
    for (int b = 0; b <= L; ++b) rank[b] = 0;
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const int b = band_of_r<N, L>(k);
        if (v[k] != 0.0 && (h == 0 || k < M)) {
            const unsigned at = h ? start[b] - rank[b] : start[b] + rank[b];
            vo[at] = v[k];
            co[at] = (uint32_t)hpos<N, L>(h, k);
            ++rank[b];
        }
    }
}

template <int N, int L>
__device__ __forceinline__ void inv_row_to_tile_h(double* T, int i, int h, double (&v)[HT<N>::H]) {
    constexpr int M = HT<N>::M, H = HT<N>::H, TP = HT<N>::TP;
    idwt_half<N, L>(v, h);
    double* rowp = T + (i + 1) * TP + 1;
#pragma unroll
    for (int k = 0; k < H; ++k)
        if (h == 0 || k < M) rowp[hglobal<N>(h, k)] = v[k];
}

// Edge lines of the new state from a column pair (natural order).
template <int N>
__device__ __forceinline__ void write_edges_h(const EdgeSet& e, const PatchPos& pp, uint32_t q, const ShardGeom& g,
                                              int j, int h, const double (&v)[HT<N>::H]) {
    constexpr int M = HT<N>::M, H = HT<N>::H;
    const size_t own = edge_ix((uint32_t)(pp.ar + 1), pp.b, q, g, N);
    (h ? e.rowhi : e.rowlo)[own + j] = v[1];  // logical rows 1 and N-2 are local 1 of each lane
    const size_t oc = edge_ix((uint32_t)pp.ar, pp.b, q, g, N);
    if (j == 1 || j == N - 2) {
        double* dst = (j == 1 ? e.collo : e.colhi) + oc;
#pragma unroll
        for (int k = 0; k < H; ++k)
            if (h == 0 || k < M) dst[hglobal<N>(h, k)] = v[k];
    }
}

template <int N>
__device__ __forceinline__ double col_mass_h(int j, int h, const double (&v)[HT<N>::H]) {
    constexpr int M = HT<N>::M, H = HT<N>::H;
    const double wj = (j == 0 || j == N - 1) ? 0.5 : 1.0;
    double m[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const double wi = k == 0 ? 0.5 : 1.0;  // local 0 is an endpoint for both lanes
        if (h == 0 || k < M) m[k & 3] += (wi * wj) * v[k];
    }
    return (m[0] + m[1]) + (m[2] + m[3]);
}

}  // namespace wg
