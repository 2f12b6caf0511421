// swe_kernels.cuh — the fused per-patch step for the shallow-water scheme
// (3 components h, hu, hv; exact-Riemann Godunov flux, solver.hpp:74-199).
//
// One launch = one step of run() for Scheme::swe (pipeline.hpp:194-289), with
// the time step kept on the device: every CTA derives dt = cfl dx / vmax,
// clipped to t_end - t, from the clock and the max wave speed of the input
// state (cfl_dt, solver.hpp:242-257 — a max, hence order-independent and
// bit-identical); the launch is a no-op once t >= t_end (pipeline.hpp:194).
// The max wave speed of the output state is accumulated for the next step
// (and all-reduced across shards between steps when world > 1).
//
// Per patch (one CTA, the three components in three slots):
//   decode h, hu, hv (CSR -> inverse DWT) + ghost ring      -> tiles
//   Godunov FV, 4 faces per cell (each face twice, like fv_step) -> scratch
//   forward DWT, threshold, CSR, reconstruction, edges (all 3), mass of h
//   skip rule: nothing zeroed -> the FV output is stored raw (pipeline.hpp:243-249)
//   max wave speed of the stored state (reconstructed or raw)
// The compression stages are bit-exact; the FV differs from the reference
// only where glibc pow(x, 2) (the Newton start, solver.hpp:112) is not the
// correctly rounded square the device uses.
#pragma once

#include "patch_phases.cuh"

namespace wg {

// one warp beyond the 3 x 65 line threads: 256 threads at 2 CTAs/SM (the
// cell-parallel Godunov phase gets them): 5.35 vs 4.84 GLUPS at C3
#ifndef WG_SWE_EXTRA_WARPS
#define WG_SWE_EXTRA_WARPS 1
#endif

template <int N>
struct SweLayout {
    static constexpr int TP = N + 2;
    static constexpr int TILE = TP * TP;
    static constexpr int NT = ((3 * N + 31) / 32) * 32 + 32 * WG_SWE_EXTRA_WARPS;  // extra warps: FV cells
    static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t)(3 * TILE) + sizeof(unsigned long long) * NT;
    }
    static constexpr size_t scratch_doubles() { return (size_t)3 * N * N; }
};

// Skip-rule patches (nothing zeroed, pipeline.hpp:243-249) store the FV
// output raw; a component whose n*n values are bitwise equal (the flat
// regions of the dam break: h = 1 or 2, hu = hv = 0) is stored as a
// constant directory entry (DIR_CONST: the value in the entry, nothing in the
// pool) — the next decode is a fill with the same bits.

#ifndef WG_SWE_MIN_BLOCKS
#define WG_SWE_MIN_BLOCKS 2  // 2 CTAs per SM (spills in the lifting phases, +44% C3)
#endif

// A still-water patch: its three input blocks are constant directory entries
// (h, +0.0, +0.0) and so are those of its four face neighbours (whose edge
// lines, the ghost values, are then these constants too).  Every face then
// carries the same Riemann problem with u* = 0 exactly, the ±x (±y) momentum
// fluxes cancel exactly and the mass fluxes are 0: the FV output equals the
// input bit for bit, its transform has the 5/3 samples h and zero details
// (nothing zeroed: the skip rule stores it raw, i.e. constant entries
// again).  Only patch rows whose neighbours live in this shard qualify.
template <int N, int L>
__device__ __forceinline__ bool swe_still_water(const StepArgs& a, uint32_t p, const PatchPos& pp,
                                                const ShardGeom& g) {
    if (g.world > 1 && (pp.ar == 0 || pp.ar == (int)g.R - 1)) return false;
    const DirEntry* d = a.dir_in;
    const DirEntry e0 = d[(size_t)p * 3], e1 = d[(size_t)p * 3 + 1], e2 = d[(size_t)p * 3 + 2];
    if (!(e0.flags & DIR_CONST) || !(e1.flags & DIR_CONST) || !(e2.flags & DIR_CONST) || e1.off || e2.off)
        return false;
    const double h = __longlong_as_double((long long)e0.off);
    if (!(h > 0.0) || h < a.thr[0]) return false;  // the samples are kept (band 0 x 0)
    const uint32_t up = (uint32_t)((pp.ar + (int)g.R - 1) % (int)g.R) * g.P1 + pp.b;
    const uint32_t dn = (uint32_t)((pp.ar + 1) % (int)g.R) * g.P1 + pp.b;
    const uint32_t nb[4] = {up, dn, (uint32_t)pp.ar * g.P1 + pp.bl, (uint32_t)pp.ar * g.P1 + pp.br};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const DirEntry e = d[(size_t)nb[k] * 3 + q];
            if (!(e.flags & DIR_CONST) || e.off != (q == 0 ? e0.off : 0ull)) return false;
        }
    return true;
}

template <int N, int L, int MODE>
__global__ void __launch_bounds__(SweLayout<N>::NT, WG_SWE_MIN_BLOCKS) k_swe_step(const __grid_constant__ StepArgs a) {
    using Lay = SweLayout<N>;
    constexpr int TP = Lay::TP, TILE = Lay::TILE, NT = Lay::NT, NN = N * N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(tiles + 3 * TILE);
    __shared__ uint64_t slot_off[3];
    __shared__ int slot_ok[3];
    __shared__ uint32_t comp_nnz[3];
    __shared__ int slot_const[3];
    __shared__ unsigned long long patch_bytes, patch_nnz, patch_zero;
    __shared__ ChunkState cs;
    __shared__ double wmax[NT / 32];

    const int t = threadIdx.x;
    const int s = t / N;  // slot == component
    const int li = t - s * N;
    const bool lane_ok = t < 3 * N;
    const ShardGeom& g = a.g;
    double* T = tiles + (lane_ok ? s : 0) * TILE;
    double* S = a.scratch + (size_t)blockIdx.x * Lay::scratch_doubles();

    if (MODE == MODE_DECODE) {
        for (uint32_t p = blockIdx.x; p < g.npatch; p += gridDim.x) {
            bool raw_in = false;
            if (lane_ok) raw_in = decode_row<N, L>(T, li, a.dir_in[(size_t)p * 3 + s], a.store_in);
            __syncthreads();
            if (lane_ok) {
                double v[N];
                decode_col<N, L>(T, li, raw_in, v);
                double* out = a.decode_out + ((size_t)p * 3 + s) * TILE;
#pragma unroll
                for (int i = 0; i < N; ++i) out[(i + 1) * TP + li + 1] = v[i];
            }
            __syncthreads();
        }
        return;
    }

    // the device-side clock (uniform for all CTAs of the launch)
    const SweClock clk = swe_clock(a);
    if (!clk.live) return;        // t >= t_end: the launch is a no-op
    const double r = clk.dt / a.dx;  // solver.hpp:212

    StepPartial part{0, 0, 0, 0.0, 0.0, 0.0};
    double vmax = 0.0;
    // patches are handed out dynamically (the dam break's patches differ in
    // cost by far: flat constant blocks against the front's Riemann solves),
    // the next index fetched while the current patch is decoded
    __shared__ uint32_t p_next;
    __shared__ double red_m[NT / 32], red_f[NT / 32];
    if (t == 0) {
        cs.cur = cs.end = 0;
        p_next = atomicAdd(a.work, 1u);
    }
    __syncthreads();
    WG_PHASE_MARK(-1);
    for (;;) {
        const uint32_t p = p_next;
        if (p >= g.npatch) break;  // uniform
        const PatchPos pp = patch_pos(p, g);
        double m = 0.0, mfv = 0.0;  // the patch's masses (reconstruction, scheme output)
        // still water (swe_still_water, every thread evaluates it: uniform):
        // the cycle's outputs written directly — the same entries, edge
        // lines, counts, masses and wave speed, with the same operations
        if (MODE == MODE_STEP && a.compress && a.thr_any && swe_still_water<N, L>(a, p, pp, g)) {
            __syncthreads();  // every thread has read p
            const DirEntry e0 = a.dir_in[(size_t)p * 3];
            const double h = __longlong_as_double((long long)e0.off);
            if (t == 0) {
                p_next = atomicAdd(a.work, 1u);
#pragma unroll
                for (int sl = 0; sl < 3; ++sl)
                    a.dir_out[(size_t)p * 3 + sl] = DirEntry{sl == 0 ? e0.off : 0ull, 0u, DIR_RAW | DIR_CONST};
                constexpr uint64_t kept = (uint64_t)(((N - 1) >> L) + 1) * (uint64_t)(((N - 1) >> L) + 1);
                part.comp_bytes += 12ull * kept + 3ull * 4ull * (N + 1);  // CSR sizes of (h, 0, 0)
                part.nnz += kept;
            }
            if (lane_ok) {
                double v[N];
#pragma unroll
                for (int i = 0; i < N; ++i) v[i] = s == 0 ? h : 0.0;
                write_edges<N>(a.eout, pp, s, g, li, v);
                if (s == 0) m = col_mass<N>(li, v);
            }
            for (int c = t; c < NN; c += NT) {
                const int i = c / N, j = c - (c / N) * N;
                mfv += (((i == 0 || i == N - 1) ? 0.5 : 1.0) * ((j == 0 || j == N - 1) ? 0.5 : 1.0)) * h;
            }
            if (t < NN) {
                const double cc = sqrt(a.gravity * h);
                const double u = fabs(0.0 / h);
                vmax = fmax(vmax, fmax(u + cc, u + cc));
            }
        } else {
        // ---- decode h, hu, hv + ghost ring --------------------------------
        bool raw_in = false;
        if (lane_ok) {
            raw_in = decode_row<N, L>(T, li, a.dir_in[(size_t)p * 3 + s], a.store_in);
            fill_ghosts<N>(T, li, a.ein, pp, s, g);
        }
        __syncthreads();  // every thread has read p
        if (t == 0) p_next = atomicAdd(a.work, 1u);
        WG_PHASE_MARK(0);
        if (lane_ok && !raw_in) {
            double v[N];
            decode_col<N, L>(T, li, false, v);
            store_col<N>(T, li, v);
        }
        __syncthreads();
        WG_PHASE_MARK(1);
        // ---- Godunov FV (fv_step<SweFlux>, solver.hpp:207-231) -------------
        const double* T0 = tiles;
        const double* T1 = tiles + TILE;
        const double* T2 = tiles + 2 * TILE;
        const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};  // +x, -x, +y, -y
        for (int c = t; c < NN; c += NT) {
            const int i = c / N, j = c - (c / N) * N;
            const int o = (i + 1) * TP + j + 1;
            double w[3] = {T0[o], T1[o], T2[o]};
            double out[3] = {w[0], w[1], w[2]};
            int e = 0;
            double wn[4][3], f[4][3];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int on = o + di[k] * TP + dj[k];
                wn[k][0] = T0[on];
                wn[k][1] = T1[on];
                wn[k][2] = T2[on];
            }
            swe_cell_fluxes(w, wn, a.gravity, f, e);
#pragma unroll
            for (int k = 0; k < 4; ++k)  // directions in order +x, -x, +y, -y (solver.hpp:219-226)
#pragma unroll
                for (int q = 0; q < 3; ++q) out[q] -= r * f[k][q];
            if (e) atomicOr(a.err, e == 1 ? ERR_DOMAIN : ERR_RIEMANN);
#pragma unroll
            for (int q = 0; q < 3; ++q) S[(size_t)q * NN + c] = out[q];
            const double wgt = ((i == 0 || i == N - 1) ? 0.5 : 1.0) * ((j == 0 || j == N - 1) ? 0.5 : 1.0);
            mfv += wgt * out[0];  // global_mass(grid, 0): h only (pipeline.hpp:274)
        }
        __syncthreads();
        WG_PHASE_MARK(2);

        bool store_raw = !a.compress;
        if (a.compress) {
            if (t == 0) {
                patch_bytes = 0;
                patch_nnz = 0;
                patch_zero = 0;
            }
            const bool cycle = a.thr_any != 0;
            double v[N];
            if (lane_ok) {
#pragma unroll
                for (int i = 0; i < N; ++i) v[i] = S[(size_t)s * NN + i * N + li];
                fwd_col_to_tile<N, L>(T, li, v);
            }
            __syncthreads();
            WG_PHASE_MARK(4);
            unsigned nz = 0, zr = 0;
            if (lane_ok)
                fwd_row_threshold<N, L>(T, li, a.thr, v, nz, zr, MODE == MODE_STEP_LZ ? T + (li + 1) * TP + 1 : nullptr);
            cta_inclusive_scan<NT>(((unsigned long long)zr << 32) | nz, inc);
            if (MODE == MODE_STEP_LZ) tiles_to_dense<N, NT>(tiles, TILE, 3, a.lz_dense + (size_t)p * 3 * NN);
            if (t == 0) {
                for (int sl = 0; sl < 3; ++sl) {
                    const unsigned long long base = sl == 0 ? 0ull : inc[sl * N - 1];
                    const unsigned long long tot = inc[sl * N + N - 1] - base;
                    const uint32_t snz = (uint32_t)(tot & 0xffffffffu);
                    comp_nnz[sl] = snz;
                    patch_bytes += 12ull * snz + 4ull * (N + 1);
                    patch_nnz += snz;
                    patch_zero += tot >> 32;
                }
                // skip rule decided before anything is written (pipeline.hpp:243)
                for (int sl = 0; sl < 3; ++sl) {
                    if (!cycle || patch_zero == 0) {
                        slot_ok[sl] = 0;
                        continue;
                    }
                    const uint64_t off = chunk_alloc(a, cs, round16(12ull * comp_nnz[sl] + 4ull * (N + 1)));
                    slot_ok[sl] = off != ~0ull;
                    slot_off[sl] = off;
                    a.dir_out[(size_t)p * 3 + sl] =
                        slot_ok[sl] ? DirEntry{off, comp_nnz[sl], 0u} : DirEntry{0, 0u, DIR_DEAD};
                }
                part.comp_bytes += patch_bytes;
                part.nnz += patch_nnz;
                part.zeroed += patch_zero;
            }
            __syncthreads();
            WG_PHASE_MARK(5);
            store_raw = patch_zero == 0;
            const bool ok = lane_ok && slot_ok[s];
            if (ok) {
                const unsigned long long base = s == 0 ? 0ull : inc[s * N - 1];
                const uint32_t k = (uint32_t)((inc[t] - base) & 0xffffffffu) - nz;
                write_csr_row<N, L>(a.store_out + slot_off[s], comp_nnz[s], li, k, nz, v);
                inv_row_to_tile<N, L>(T, li, v, nz);
            }
            __syncthreads();
            WG_PHASE_MARK(7);
            if (ok) {
                decode_col<N, L>(T, li, false, v);
                write_edges<N>(a.eout, pp, s, g, li, v);
                if (s == 0) m += col_mass<N>(li, v);
            }
            __syncthreads();
            WG_PHASE_MARK(8);
            if (ok) store_col<N>(T, li, v);  // the new state, for the wave speed
            __syncthreads();
            WG_PHASE_MARK(13);
            if (!store_raw) {
                for (int c = t; c < NN; c += NT) {
                    const int o = (c / N + 1) * TP + c - (c / N) * N + 1;
                    const double h = T0[o];
                    if (h <= 0.0) atomicOr(a.err, ERR_DOMAIN);  // cfl_dt, solver.hpp:248
                    const double cc = sqrt(a.gravity * h);
                    const double u = fabs(T1[o] / h), w2 = fabs(T2[o] / h);
                    vmax = fmax(vmax, fmax(u + cc, w2 + cc));
                }
                __syncthreads();  // the next patch's decode overwrites the tiles
                WG_PHASE_MARK(14);
            }
        }
        if (store_raw) {  // raw store of the FV output (skip rule / no_compression)
            // constant components (bitwise) become DIR_CONST entries
            if (t < 3) slot_const[t] = 1;
            __syncthreads();
            if (lane_ok) {
                const unsigned long long c0 = (unsigned long long)__double_as_longlong(S[(size_t)s * NN]);
                bool same = true;
#pragma unroll 5
                for (int i = 0; i < N; ++i)
                    same &= (unsigned long long)__double_as_longlong(S[(size_t)s * NN + i * N + li]) == c0;
                if (!same) slot_const[s] = 0;
            }
            __syncthreads();
            if (t == 0) {
                for (int sl = 0; sl < 3; ++sl) {
                    if (slot_const[sl]) {
                        slot_ok[sl] = 2;
                        a.dir_out[(size_t)p * 3 + sl] =
                            DirEntry{(uint64_t)__double_as_longlong(S[(size_t)sl * NN]), 0u, DIR_RAW | DIR_CONST};
                        continue;
                    }
                    const uint64_t off = chunk_alloc(a, cs, round16((uint64_t)NN * 8));
                    slot_ok[sl] = off != ~0ull;
                    slot_off[sl] = off;
                    a.dir_out[(size_t)p * 3 + sl] = slot_ok[sl] ? DirEntry{off, 0u, DIR_RAW} : DirEntry{0, 0u, DIR_DEAD};
                }
            }
            __syncthreads();
            m = 0.0;
            if (lane_ok) {
                double v[N];
#pragma unroll
                for (int i = 0; i < N; ++i) v[i] = S[(size_t)s * NN + i * N + li];
                if (slot_ok[s] == 1) {
                    double* d = reinterpret_cast<double*>(a.store_out + slot_off[s]);
#pragma unroll
                    for (int i = 0; i < N; ++i) d[i * N + li] = v[i];
                }
                write_edges<N>(a.eout, pp, s, g, li, v);
                if (s == 0) m = col_mass<N>(li, v);
            }
            for (int c = t; c < NN; c += NT) {
                const double h = S[c];
                if (h <= 0.0) atomicOr(a.err, ERR_DOMAIN);
                const double cc = sqrt(a.gravity * h);
                const double u = fabs(S[(size_t)NN + c] / h), w2 = fabs(S[(size_t)2 * NN + c] / h);
                vmax = fmax(vmax, fmax(u + cc, w2 + cc));
            }
            __syncthreads();
            WG_PHASE_MARK(9);
        }
        }  // general path
        // the patch's masses (fixed order: warp trees, then warps in order)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m += __shfl_xor_sync(0xffffffffu, m, o);
            mfv += __shfl_xor_sync(0xffffffffu, mfv, o);
        }
        if ((t & 31) == 0) {
            red_m[t >> 5] = m;
            red_f[t >> 5] = mfv;
        }
        __syncthreads();
        if (t == 0) {
            double sm = 0.0, sf = 0.0;
            for (int w = 0; w < NT / 32; ++w) {
                sm += red_m[w];
                sf += red_f[w];
            }
            a.patch_mass[2 * (size_t)p] = sm;
            a.patch_mass[2 * (size_t)p + 1] = sf;
        }
    }
    if (t != 0) part.comp_bytes = part.nnz = part.zeroed = 0;
    const StepPartial tot = cta_reduce_partial<NT>(part);
    // CTA max of the wave speed (exact: order-independent)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    if ((t & 31) == 0) wmax[t >> 5] = vmax;
    __syncthreads();
    double cta_v = 0.0;
    if (t == 0)
        for (int w = 0; w < NT / 32; ++w) cta_v = fmax(cta_v, wmax[w]);
    finalize_step(a, tot, cta_v, &clk);
    WG_PHASE_MARK(11);
}

}  // namespace wg
