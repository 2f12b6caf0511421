// lbm_kernels.cuh — the fused per-patch step for the D2Q9 LBM (9 components).
//
// A 65^2 x 9 fp64 patch is 304 KB and does not fit one SM's shared memory,
// so a CTA works on one patch at a time in three rounds of three
// components (three (N+2)^2 tiles in shared memory) and stages the nine
// N*N population fields in a private scratch block that stays resident in
// L2 (the kernel is persistent: one scratch block per CTA, reused for every
// patch the CTA processes).  Per patch:
//
//   3 rounds: CSR decode + inverse DWT of 3 populations, ghost ring from the
//             edge lines, pull streaming  f_q(x) <- f_q(x - c_q)  -> scratch
//   collide:  BGK on every cell (physics.cuh lbm_collide)      -> scratch
//   3 rounds: forward DWT, threshold, CSR compaction, reconstruction of the
//             kept coefficients -> edge lines + trapezoid mass
//   skip rule on the patch total of zeroed coefficients (pipeline.hpp:243-249)
//
// The D2Q9 scheme is NOT in the reference; its definition
// is shared with oracle/ref_shim.cpp and oracle/wg_oracle.c.
#pragma once

#include "patch_phases.cuh"

namespace wg {

#ifndef WG_LBM_PREFETCH
#define WG_LBM_PREFETCH 1
#endif

#ifndef WG_LBM_CELLS
#define WG_LBM_CELLS 2  // cells per collide iteration
#endif
#ifndef WG_LBM_EXTRA_WARPS
#define WG_LBM_EXTRA_WARPS 1  // 256 threads: the cell phases (stream, collide) get a warp more (+1-2 %)
#endif

#ifndef WG_LBM_SMEM_POPS
#define WG_LBM_SMEM_POPS 0  // 3 measured no faster (C2 7.83 vs 7.86 GLUPS): the L2 scratch is not the bound
#endif

template <int N>
struct LbmLayout {
    static constexpr int TP = N + 2;
    static constexpr int TILE = TP * TP;
    static constexpr int SLOTS = 3;
    static constexpr int NT = ((SLOTS * N + 31) / 32) * 32 + 32 * WG_LBM_EXTRA_WARPS;
    // 3 tiles + the scan buffer: 109.5 KB at N = 65, so two CTAs fit an SM
    // (the per-patch mass reductions reuse the tiles once a patch is done)
    // the first SPOPS populations of the scratch live in shared memory (the
    // rest in the CTA's L2-resident global scratch): 206 KB at N = 65
    static constexpr int SPOPS = (N <= 65) ? WG_LBM_SMEM_POPS : 0;
    static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t)(SLOTS * TILE + SPOPS * N * N) + sizeof(unsigned long long) * NT;
    }
    static constexpr size_t scratch_doubles() { return (size_t)9 * N * N; }
};

// Population q of the per-patch staging (post-stream / post-collide field).
struct LbmScratch {
    double* sm;  // SPOPS populations in shared memory
    double* gl;  // all 9 slots in global memory (the first SPOPS unused)
    int spops, nn;
    __device__ __forceinline__ double* pop(int q) const { return q < spops ? sm + (size_t)q * nn : gl + (size_t)q * nn; }
};

#ifndef WG_LBM_MIN_BLOCKS
#define WG_LBM_MIN_BLOCKS 1
#endif

// decode + pull streaming (3 rounds of 3 populations) then BGK collide, all
// into the scratch S; returns this thread's trapezoid mass partial of the
// collided state.  Uniform: every thread of the CTA calls it.
template <int N, int L>
__device__ __forceinline__ double decode_stream_collide(const StepArgs& a, double* T, const LbmScratch& S, uint32_t p,
                                                        const PatchPos& pp, int s, int li, bool lane_ok) {
    using Lay = LbmLayout<N>;
    constexpr int TP = Lay::TP, NT = Lay::NT, NN = N * N;
    // ROW phase thread mapping: rows interleaved over the 3 slots (thread t
    // takes row t / 3 of slot t % 3), so the coarse rows that hold the few
    // surviving coefficients share warps and the warps of empty detail rows
    // skip their transforms (decode_row)
    const int rs = threadIdx.x % 3, rli = threadIdx.x / 3;
    double* TR = T + (rs - s) * (Lay::TILE);
    for (int rd = 0; rd < 3; ++rd) {
        const int q = 3 * rd + s;
        if (lane_ok) {
#ifdef WG_BOUNDS_CHECK
            {
                const DirEntry e = a.dir_in[(size_t)p * 9 + 3 * rd + rs];
                const uint64_t bytes = (e.flags & DIR_RAW) ? 8ull * N * N : 12ull * e.nnz + 4ull * (N + 1);
                WG_CHECK((e.flags & DIR_DEAD) || e.off + bytes <= a.cap_out, 6);
                WG_CHECK(p < a.g.npatch, 7);
            }
#endif
            decode_row<N, L>(TR, rli, a.dir_in[(size_t)p * 9 + 3 * rd + rs], a.store_in);
            fill_ghosts_lbm<N>(TR, rli, a.ein, pp, 3 * rd + rs, a.g);
        }
        __syncthreads();
        // (threads past the 3 slots have q = 9..11: they must not read — the
        // last patch's q = 9 lies past the end of the directory)
        const bool raw_in = lane_ok && (a.dir_in[(size_t)p * 9 + q].flags & (DIR_RAW | DIR_DEAD)) != 0;
        if (lane_ok && !raw_in) {
            double v[N];
            decode_col<N, L>(T, li, false, v);
            store_col<N>(T, li, v);
        }
        __syncthreads();
        WG_PHASE_MARK(rd == 0 ? 0 : 12);
        if (lane_ok) {  // pull streaming f_q(x) <- f_q(x - c_q), ghost ring included
            const int cx = lbm_cx(q), cy = lbm_cy(q);
            double* Sq = S.pop(q);
            const int j = li;
#pragma unroll 5
            for (int i = 0; i < N; ++i) Sq[i * N + j] = T[(i + 1 - cx) * TP + (j + 1 - cy)];
        }
        __syncthreads();
        WG_PHASE_MARK(1);
    }
    double mfv = 0.0;
    // WG_LBM_CELLS cells per iteration: 9 x that many independent scratch loads in flight
    constexpr int K = WG_LBM_CELLS;
    for (int c0 = threadIdx.x; c0 < NN; c0 += K * NT) {
        double f[K][9];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const int c = c0 + u * NT;
#pragma unroll
            for (int q = 0; q < 9; ++q) f[u][q] = c < NN ? S.pop(q)[c] : 1.0;
        }
#pragma unroll
        for (int u = 0; u < K; ++u) lbm_collide(f[u], a.omega);
        double w[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const int c = c0 + u * NT, i = c / N, j = c - i * N;
            w[u] = ((i == 0 || i == N - 1) ? 0.5 : 1.0) * ((j == 0 || j == N - 1) ? 0.5 : 1.0);
        }
#pragma unroll
        for (int q = 0; q < 9; ++q)
#pragma unroll
            for (int u = 0; u < K; ++u) {
                const int c = c0 + u * NT;
                if (c < NN) {
                    S.pop(q)[c] = f[u][q];
                    mfv += w[u] * f[u][q];
                }
            }
    }
    __syncthreads();
    WG_PHASE_MARK(2);
    return mfv;
}

template <int N, int L, int MODE>
__global__ void __launch_bounds__(LbmLayout<N>::NT, WG_LBM_MIN_BLOCKS) k_lbm_step(const __grid_constant__ StepArgs a) {
    using Lay = LbmLayout<N>;
    constexpr int TP = Lay::TP, TILE = Lay::TILE, NT = Lay::NT, NN = N * N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(tiles + Lay::SLOTS * TILE);
    double* red = tiles;          // per-patch sums: tiles are free by then
    double* red_fv = tiles + NT;
    __shared__ uint64_t slot_off[3];
    __shared__ int slot_ok[3];
    __shared__ ChunkState cs;
    __shared__ DirEntry next_dir[9];
    __shared__ unsigned long long patch_bytes, patch_nnz, patch_zero;
    __shared__ uint32_t comp_nnz[3];

    const int t = threadIdx.x;
    const int s = t / N;
    const int li = t - s * N;
    const bool lane_ok = t < Lay::SLOTS * N;
    const ShardGeom& g = a.g;
    double* T = tiles + (lane_ok ? s : 0) * TILE;
    const LbmScratch S{reinterpret_cast<double*>(inc + NT), a.scratch + (size_t)blockIdx.x * Lay::scratch_doubles(),
                       Lay::SPOPS, NN};

    if (MODE == MODE_DECODE) {
        for (uint32_t p = blockIdx.x; p < g.npatch; p += gridDim.x) {
            for (int rd = 0; rd < 3; ++rd) {
                const int q = 3 * rd + s;
                bool raw_in = false;
                if (lane_ok) raw_in = decode_row<N, L>(T, li, a.dir_in[(size_t)p * 9 + q], a.store_in);
                __syncthreads();
                if (lane_ok) {
                    double v[N];
                    decode_col<N, L>(T, li, raw_in, v);
                    double* out = a.decode_out + ((size_t)p * 9 + q) * TILE;
#pragma unroll
                    for (int i = 0; i < N; ++i) out[(i + 1) * TP + li + 1] = v[i];
                }
                __syncthreads();
            }
        }
        return;
    }

    StepPartial part{0, 0, 0, 0.0, 0.0};
    WG_PHASE_MARK(-1);
    if (t == 0) cs.cur = cs.end = 0;
    for (uint32_t p = blockIdx.x; p < g.npatch; p += gridDim.x) {
        const PatchPos pp = patch_pos(p, g);
        const uint32_t pn = p + gridDim.x;  // this CTA's next patch
        double mfv = 0.0;
        if (t < 9) next_dir[t] = (MODE != MODE_INIT && pn < g.npatch) ? a.dir_in[(size_t)pn * 9 + t] : DirEntry{0, 0u, DIR_DEAD};
        if (MODE == MODE_INIT) {
            // initial state generated on the device (CUDA libm: not bit-pinned
            // to the host IC) for grids whose raw state exceeds the store
            // budget (C4/C5); it enters the store through the same
            // compression cycle as every step
            const int N1 = N - 1;
            for (int c = t; c < NN; c += Lay::NT) {
                const int i = c / N, jj = c - (c / N) * N;
                const uint64_t gi = ((uint64_t)(g.row0 + pp.ar) * N1 + i) % a.ic_period, gj = (uint64_t)pp.b * N1 + jj;
                const double X = (double)gi * a.ic_inv, Y = (double)gj * a.ic_inv;
                const double uy = X <= 0.5 ? a.ic_u0 * tanh(a.ic_kappa * (X - 0.25)) : a.ic_u0 * tanh(a.ic_kappa * (0.75 - X));
                const double ux = a.ic_delta * a.ic_u0 * sin(2.0 * 3.141592653589793 * (Y + 0.25));
                const double usq = ux * ux + uy * uy;
#pragma unroll
                for (int q = 0; q < 9; ++q) S.pop(q)[c] = lbm_feq(q, 1.0, lbm_cu(q, ux, uy), usq);
            }
            __syncthreads();
        } else {
            mfv = decode_stream_collide<N, L>(a, T, S, p, pp, s, li, lane_ok);
        }
        if (WG_LBM_PREFETCH && MODE != MODE_INIT && pn < g.npatch && lane_ok) {  // warm L2 with the next patch's inputs
            for (int q = s; q < 9; q += 3) prefetch_block<N>(a, next_dir[q], li, N);
            prefetch_edges<N>(a, pn, t, Lay::SLOTS * N);
        }
        double m = 0.0;
        bool store_raw = !a.compress;
        // nothing can be zeroed with c == 0 or no transform (threshold.hpp:53):
        // every patch is raw by the skip rule, so no CSR block is written
        // (the coefficients are still transformed and counted for the
        // metrics, pipeline.hpp:234-242)
        const bool cycle = a.thr_any != 0;
        if (a.compress) {
            if (t == 0) {
                patch_bytes = 0;
                patch_nnz = 0;
                patch_zero = 0;
            }
            // ---- per round: forward DWT, threshold, CSR, reconstruction ----
            // written speculatively as compressed: a patch whose cycle zeroed
            // nothing (rare for c > 0) is re-derived and stored raw below,
            // overwriting its directory entries (its CSR blocks are left as
            // unused pool space).
            for (int rd = 0; rd < 3; ++rd) {
                const int q = 3 * rd + s;
                double v[N];
                if (lane_ok) {
                    const int j = li;
#pragma unroll
                    for (int i = 0; i < N; ++i) v[i] = S.pop(q)[i * N + j];
                    fwd_col_to_tile<N, L>(T, j, v);
                }
                __syncthreads();
                WG_PHASE_MARK(3);
                unsigned nz = 0, zr = 0;
                if (lane_ok)
                    fwd_row_threshold<N, L>(T, li, a.thr, v, nz, zr,
                                            MODE == MODE_STEP_LZ ? T + (li + 1) * TP + 1 : nullptr);
                cta_inclusive_scan<NT>(((unsigned long long)zr << 32) | nz, inc);
                if (MODE == MODE_STEP_LZ) tiles_to_dense<N, NT>(tiles, TILE, 3, a.lz_dense + ((size_t)p * 9 + 3 * rd) * NN);
                if (t == 0) {
                    for (int sl = 0; sl < 3; ++sl) {
                        const int qq = 3 * rd + sl;
                        const unsigned long long base = sl == 0 ? 0ull : inc[sl * N - 1];
                        const unsigned long long tot = inc[sl * N + N - 1] - base;
                        const uint32_t snz = (uint32_t)(tot & 0xffffffffu);
                        comp_nnz[sl] = snz;
                        patch_bytes += 12ull * snz + 4ull * (N + 1);
                        patch_nnz += snz;
                        patch_zero += tot >> 32;
                        if (!cycle) {
                            slot_ok[sl] = 0;
                            continue;
                        }
                        const uint64_t off = chunk_alloc(a, cs, round16(12ull * snz + 4ull * (N + 1)));
                        slot_ok[sl] = off != ~0ull;
                        slot_off[sl] = off;
                        a.dir_out[(size_t)p * 9 + qq] = slot_ok[sl] ? DirEntry{off, snz, 0u} : DirEntry{0, 0u, DIR_DEAD};
                    }
                }
                __syncthreads();
                WG_PHASE_MARK(5);
                const bool ok = lane_ok && slot_ok[s];
                if (ok) {
                    const unsigned long long base = s == 0 ? 0ull : inc[s * N - 1];
                    const uint32_t k = (uint32_t)((inc[t] - base) & 0xffffffffu) - nz;
                    WG_CHECK(slot_off[s] + 12ull * comp_nnz[s] + 4ull * (N + 1) <= a.cap_out && k + nz <= comp_nnz[s], 10);
                    write_csr_row<N, L>(a.store_out + slot_off[s], comp_nnz[s], li, k, nz, v);
                    inv_row_to_tile<N, L>(T, li, v, nz);
                }
                __syncthreads();
                WG_PHASE_MARK(6);
                if (ok) {
                    decode_col<N, L>(T, li, false, v);
                    m += col_mass<N>(li, v);
                    store_col<N>(T, li, v);
                }
                __syncthreads();
                if (ok) {  // edges from the tile: no register line live
                    WG_CHECK(edge_ix((uint32_t)(pp.ar + 1), pp.b, 2, g, N) + N <= a.edge_row_elems, 8);
                    WG_CHECK(edge_ix((uint32_t)pp.ar, pp.b, 2, g, N) + N <= a.edge_col_elems, 9);
                    write_edges_lbm_tile<N>(a.eout, pp, q, g, li, T);
                }
                __syncthreads();
                WG_PHASE_MARK(7);
            }
            if (t == 0) {
                part.comp_bytes += patch_bytes;
                part.nnz += patch_nnz;
                part.zeroed += patch_zero;
            }
            // skip rule (pipeline.hpp:243-249): the scratch still holds the
            // collided state bit for bit; the raw store below overwrites the
            // directory entries written by the rounds
            store_raw = patch_zero == 0;
            if (store_raw) m = 0.0;
        }
        if (store_raw) {
            for (int rd = 0; rd < 3; ++rd) {
                const int q = 3 * rd + s;
                if (t == 0) {
                    for (int sl = 0; sl < 3; ++sl) {
                        const int qq = 3 * rd + sl;
                        const uint64_t off = chunk_alloc(a, cs, round16((uint64_t)NN * 8));
                        slot_ok[sl] = off != ~0ull;
                        slot_off[sl] = off;
                        a.dir_out[(size_t)p * 9 + qq] = slot_ok[sl] ? DirEntry{off, 0u, DIR_RAW} : DirEntry{0, 0u, DIR_DEAD};
                    }
                }
                __syncthreads();
                if (lane_ok) {  // through the tile: no register line live
                    const int j = li;
                    double* d = slot_ok[s] ? reinterpret_cast<double*>(a.store_out + slot_off[s]) : nullptr;
#pragma unroll 5
                    for (int i = 0; i < N; ++i) {
                        const double x = S.pop(q)[i * N + j];
                        T[(i + 1) * Lay::TP + j + 1] = x;
                        if (d) d[i * N + j] = x;
                    }
                }
                __syncthreads();
                if (lane_ok) {
                    write_edges_lbm_tile<N>(a.eout, pp, q, g, li, T);
                    m += tile_col_mass<N>(T, li);
                }
                __syncthreads();
            }
        }
        red[t] = m;  // every round / the raw path ended with a barrier: tiles are free
        red_fv[t] = mfv;
        __syncthreads();
        if (t < 32) {
            const double mm = warp_sum_range(red, 0, NT);
            const double mf = warp_sum_range(red_fv, 0, NT);
            if (t == 0) {
                part.mass += mm;
                part.mass_fv += mf;
            }
        }
        __syncthreads();
        WG_PHASE_MARK(9);
    }
    finalize_step(a, part);
    WG_PHASE_MARK(11);
}

}  // namespace wg
