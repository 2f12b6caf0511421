// lbm_group_kernels.cuh — the fused D2Q9 step with register-light lines:
// every line of a tile is transformed by an 8-lane group (lifting_group.cuh),
// so a thread keeps E + 1 = 9 doubles of a line instead of 65 and an SM runs
// 17 warps instead of 7 (k_lbm_step, lbm_kernels.cuh).  Same data flow,
// store layout, skip rule and metrics as k_lbm_step; bit-identical state and
// CSR blocks (the parity tests run it).
//
// A TUNING VARIANT (WG_LBM_LINES=group), not the default: measured at C2 it
// runs 3.7 GLUPS against 7.9 for the one-thread-per-line kernel — it issues
// 2.3x the instructions (82 M vs 35 M per launch: runtime weights and corner
// positions, shuffles, per-slot branches) and the 17 warps raise the issue
// rate only from 0.27 to 0.31 per scheduler (barrier and dependency stalls).
//
// Thread t: group g = t / 8 owns line g (row g or column g) of each of the 3
// slot tiles; lane r = t % 8 owns elements 8r .. 8r+8 of it.  Cell-parallel
// phases (raw copies, streaming, collide, edges) use all threads flat.
#pragma once

#include "lbm_kernels.cuh"
#include "lifting_group.cuh"

namespace wg {

template <int N>
struct GLayout {
    static constexpr int TP = N + 2;
    static constexpr int TILE = TP * TP;
    static constexpr int E = (N - 1) / kGL;
    static constexpr int NT = ((N * kGL + 31) / 32) * 32;  // one 8-lane group per line: 544 at N = 65
    static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t)(3 * TILE) + sizeof(uint32_t) * (size_t)(3 * (3 * N + 1));
    }
    static constexpr size_t scratch_doubles() { return (size_t)9 * N * N; }
};

// Load line elements E*r .. E*r+E of a line whose element e sits at
// base[pos(e) * stride] (pos: corner or natural order).
template <int N, int L, bool CORNER>
__device__ __forceinline__ void grp_load(double (&x)[(N - 1) / kGL + 1], const double* base, int stride, int r) {
    constexpr int E = (N - 1) / kGL;
#pragma unroll
    for (int i = 0; i <= E; ++i) {
        const int e = E * r + i;
        x[i] = base[(CORNER ? corner_pos_rt<N, L>(e) : e) * stride];
    }
}

// Store a line in natural order (each element once: lane r its first E, lane 7 also the last).
template <int N>
__device__ __forceinline__ void grp_store_nat(const double (&x)[(N - 1) / kGL + 1], double* base, int stride, int r) {
    constexpr int E = (N - 1) / kGL;
#pragma unroll
    for (int i = 0; i < E; ++i) base[(E * r + i) * stride] = x[i];
    if (r == kGL - 1) base[(N - 1) * stride] = x[E];
}

template <int N, int L>
__device__ __forceinline__ void grp_store_corner(const double (&x)[(N - 1) / kGL + 1], double* base, int stride,
                                                 int r) {
    constexpr int E = (N - 1) / kGL;
#pragma unroll
    for (int i = 0; i < E; ++i) base[corner_pos_rt<N, L>(E * r + i) * stride] = x[i];
    if (r == kGL - 1) base[corner_pos_rt<N, L>(N - 1) * stride] = x[E];
}

template <int N, int L, int MODE>
__global__ void __launch_bounds__(GLayout<N>::NT, 1) k_lbm_step_g(const __grid_constant__ StepArgs a) {
    using Lay = GLayout<N>;
    constexpr int TP = Lay::TP, TILE = Lay::TILE, NT = Lay::NT, NN = N * N, E = Lay::E;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    uint32_t* rnz = reinterpret_cast<uint32_t*>(tiles + 3 * TILE);  // [3][N] kept coefficients per row
    uint32_t* rzr = rnz + 3 * N;                                     // [3][N] zeroed per row
    uint32_t* roff = rzr + 3 * N;                                    // [3][N + 1] exclusive row offsets
    double* red = tiles;                                             // per-patch sums (tiles free by then)
    double* red_fv = tiles + NT;
    __shared__ uint64_t slot_off[3];
    __shared__ int slot_ok[3];
    __shared__ ChunkState cs;
    __shared__ DirEntry cur_dir[9], next_dir[9];
    __shared__ unsigned long long patch_bytes, patch_nnz, patch_zero;
    __shared__ uint32_t comp_nnz[3];

    const int t = threadIdx.x;
    const int g = t / kGL, r = t % kGL;
    const bool gok = g < N;
    const unsigned sm = seg_mask();
    const ShardGeom& gg = a.g;
    const LbmScratch S{nullptr, a.scratch + (size_t)blockIdx.x * Lay::scratch_doubles(), 0, NN};

    StepPartial part{0, 0, 0, 0.0, 0.0, 0.0};
    if (t == 0) cs.cur = cs.end = 0;
    if (t < 9) next_dir[t] = (MODE != MODE_INIT && blockIdx.x < gg.npatch) ? a.dir_in[(size_t)blockIdx.x * 9 + t]
                                                                           : DirEntry{0, 0u, DIR_DEAD};
    for (uint32_t p = blockIdx.x; p < gg.npatch; p += gridDim.x) {
        const PatchPos pp = patch_pos(p, gg);
        const uint32_t pn = p + gridDim.x;
        __syncthreads();  // next_dir written; the previous patch is done with everything
        if (t < 9) {
            cur_dir[t] = next_dir[t];
            next_dir[t] = (MODE != MODE_INIT && pn < gg.npatch) ? a.dir_in[(size_t)pn * 9 + t] : DirEntry{0, 0u, DIR_DEAD};
        }
        __syncthreads();
        double mfv = 0.0;
        if (MODE == MODE_INIT) {
            const int N1 = N - 1;
            for (int c = t; c < NN; c += NT) {
                const int i = c / N, jj = c - (c / N) * N;
                const uint64_t gi = ((uint64_t)(gg.row0 + pp.ar) * N1 + i) % a.ic_period, gj = (uint64_t)pp.b * N1 + jj;
                const double X = (double)gi * a.ic_inv, Y = (double)gj * a.ic_inv;
                const double uy = X <= 0.5 ? a.ic_u0 * tanh(a.ic_kappa * (X - 0.25)) : a.ic_u0 * tanh(a.ic_kappa * (0.75 - X));
                const double ux = a.ic_delta * a.ic_u0 * sin(2.0 * 3.141592653589793 * (Y + 0.25));
                const double usq = ux * ux + uy * uy;
#pragma unroll
                for (int q = 0; q < 9; ++q) S.pop(q)[c] = lbm_feq(q, 1.0, lbm_cu(q, ux, uy), usq);
            }
            __syncthreads();
        } else {
            for (int rd = 0; rd < 3; ++rd) {
                // ---- decode: raw / lost blocks (whole interior, coalesced) --
                for (int c = t; c < 3 * NN; c += NT) {
                    const int s = c / NN, cc = c - s * NN;
                    const DirEntry e = cur_dir[3 * rd + s];
                    if (e.flags & (DIR_RAW | DIR_DEAD)) {
                        const int i = cc / N, j = cc - i * N;
                        tiles[s * TILE + (i + 1) * TP + j + 1] =
                            (e.flags & DIR_DEAD) ? 0.0 : reinterpret_cast<const double*>(a.store_in + e.off)[cc];
                    }
                }
                // ---- decode: CSR rows (scatter, inverse along dim 1) -------
                if (gok) {
                    for (int s = 0; s < 3; ++s) {
                        const DirEntry e = cur_dir[3 * rd + s];
                        if (e.flags & (DIR_RAW | DIR_DEAD)) continue;
                        const unsigned char* base = a.store_in + e.off;
                        const double* v = reinterpret_cast<const double*>(base);
                        const uint32_t* col = reinterpret_cast<const uint32_t*>(base + 8ull * e.nnz);
                        const uint32_t* ro = col + e.nnz;
                        double* row = tiles + s * TILE + (g + 1) * TP + 1;
                        const uint32_t k0 = ro[g], k1 = ro[g + 1];
                        for (int j = r; j < N; j += kGL) row[j] = 0.0;
                        if (k0 == k1) continue;  // empty row: the inverse is +0.0 everywhere
                        __syncwarp(sm);
                        for (uint32_t k = k0 + r; k < k1; k += kGL) row[col[k]] = v[k];
                        __syncwarp(sm);
                        double x[E + 1];
                        grp_load<N, L, true>(x, row, 1, r);
                        __syncwarp(sm);
                        idwt_line_grp<N, L>(x, r, sm);
                        grp_store_nat<N>(x, row, 1, r);
                    }
                }
                if (MODE == MODE_STEP)  // ghost ring from the neighbours' edge lines
                    for (int c = t; c < 3 * N; c += NT) {
                        const int s = c / N, li = c - s * N;
                        fill_ghosts_lbm<N>(tiles + s * TILE, li, a.ein, pp, 3 * rd + s, gg);
                    }
                __syncthreads();
                // ---- decode: columns (inverse along dim 0) -----------------
                if (gok) {
                    for (int s = 0; s < 3; ++s) {
                        if (cur_dir[3 * rd + s].flags & (DIR_RAW | DIR_DEAD)) continue;
                        double* colp = tiles + s * TILE + TP + g + 1;
                        double x[E + 1];
                        grp_load<N, L, true>(x, colp, TP, r);
                        __syncwarp(sm);
                        idwt_line_grp<N, L>(x, r, sm);
                        grp_store_nat<N>(x, colp, TP, r);
                    }
                }
                __syncthreads();
                if (MODE == MODE_DECODE) {  // the decoded state out (grid buffer layout)
                    for (int c = t; c < 3 * NN; c += NT) {
                        const int s = c / NN, cc = c - s * NN, i = cc / N, j = cc - (cc / N) * N;
                        a.decode_out[((size_t)p * 9 + 3 * rd + s) * TILE + (i + 1) * TP + j + 1] =
                            tiles[s * TILE + (i + 1) * TP + j + 1];
                    }
                    __syncthreads();
                    continue;
                }
                // ---- pull streaming f_q(x) <- f_q(x - c_q) into the scratch -
                for (int c = t; c < 3 * NN; c += NT) {
                    const int s = c / NN, cc = c - s * NN, i = cc / N, j = cc - (cc / N) * N;
                    const int q = 3 * rd + s, cx = lbm_cx(q), cy = lbm_cy(q);
                    S.pop(q)[cc] = tiles[s * TILE + (i + 1 - cx) * TP + (j + 1 - cy)];
                }
                __syncthreads();
            }
            if (MODE == MODE_DECODE) continue;
            // ---- BGK collide (two cells per iteration) ------------------------
            for (int c0 = t; c0 < NN; c0 += 2 * NT) {
                const int c1 = c0 + NT;
                const bool two = c1 < NN;
                double f0[9], f1[9];
#pragma unroll
                for (int q = 0; q < 9; ++q) {
                    f0[q] = S.pop(q)[c0];
                    f1[q] = two ? S.pop(q)[c1] : 1.0;
                }
                lbm_collide(f0, a.omega);
                lbm_collide(f1, a.omega);
                const int i0 = c0 / N, j0 = c0 - i0 * N, i1 = c1 / N, j1 = c1 - i1 * N;
                const double w0 = ((i0 == 0 || i0 == N - 1) ? 0.5 : 1.0) * ((j0 == 0 || j0 == N - 1) ? 0.5 : 1.0);
                const double w1 = ((i1 == 0 || i1 == N - 1) ? 0.5 : 1.0) * ((j1 == 0 || j1 == N - 1) ? 0.5 : 1.0);
#pragma unroll
                for (int q = 0; q < 9; ++q) {
                    S.pop(q)[c0] = f0[q];
                    mfv += w0 * f0[q];
                    if (two) {
                        S.pop(q)[c1] = f1[q];
                        mfv += w1 * f1[q];
                    }
                }
            }
            __syncthreads();
        }
        if (MODE != MODE_INIT && pn < gg.npatch) {  // warm L2 with the next patch's inputs
            if (t < 9 * 32) prefetch_block<N>(a, next_dir[t / 32], t & 31, 32);
            prefetch_edges<N>(a, pn, t, NT);
        }
        // ---- compression rounds (speculatively compressed, as k_lbm_step) --
        double m = 0.0;
        bool store_raw = !a.compress;
        const bool cycle = a.thr_any != 0;
        if (a.compress) {
            if (t == 0) patch_bytes = patch_nnz = patch_zero = 0;
            for (int rd = 0; rd < 3; ++rd) {
                // forward along dim 0: column g from the scratch, corner rows into the tile
                if (gok) {
                    for (int s = 0; s < 3; ++s) {
                        double x[E + 1];
                        grp_load<N, L, false>(x, S.pop(3 * rd + s) + g, N, r);
                        dwt_line_grp<N, L>(x, r, sm);
                        grp_store_corner<N, L>(x, tiles + s * TILE + TP + g + 1, TP, r);
                    }
                }
                __syncthreads();
                // forward along dim 1 + threshold (threshold.hpp:51-86); the
                // kept coefficients back into the row in corner order
                if (gok) {
                    const int bi = band_of_pos(N, L, g);
                    for (int s = 0; s < 3; ++s) {
                        double* row = tiles + s * TILE + (g + 1) * TP + 1;
                        double x[E + 1];
                        grp_load<N, L, false>(x, row, 1, r);
                        dwt_line_grp<N, L>(x, r, sm);
                        unsigned nz = 0, zr = 0;
#pragma unroll
                        for (int i = 0; i <= E; ++i) {
                            const int e = E * r + i;
                            const double xv = x[i];
                            const bool nzx = xv != 0.0;
                            const bool kill = fabs(xv) < a.thr[bi * (L + 1) + band_rt<L>(e)];
                            const bool keep = nzx && !kill;
                            x[i] = keep ? xv : 0.0;  // -0.0 -> +0.0 like the CSR round trip
                            if (i < E || r == kGL - 1) {
                                zr += (nzx && kill) ? 1u : 0u;
                                nz += keep ? 1u : 0u;
                            }
                        }
#pragma unroll
                        for (int o = 1; o < kGL; o <<= 1) {
                            nz += __shfl_xor_sync(sm, nz, o, kGL);
                            zr += __shfl_xor_sync(sm, zr, o, kGL);
                        }
                        if (r == 0) {
                            rnz[s * N + g] = nz;
                            rzr[s * N + g] = zr;
                        }
                        __syncwarp(sm);
                        grp_store_corner<N, L>(x, row, 1, r);
                    }
                }
                __syncthreads();
                // exclusive scan of the row counts per slot (warp s)
                if (t < 96) {
                    const int s = t >> 5, lane = t & 31;
                    uint32_t run = 0;
                    unsigned long long zsum = 0;
                    for (int c = 0; c < N; c += 32) {
                        const int gi = c + lane;
                        uint32_t x = gi < N ? rnz[s * N + gi] : 0u;
                        const uint32_t zx = gi < N ? rzr[s * N + gi] : 0u;
                        uint32_t incl = x;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= o) incl += y;
                        }
                        if (gi < N) roff[s * (N + 1) + gi] = run + incl - x;
                        run += __shfl_sync(0xffffffffu, incl, 31);
                        unsigned long long zz = zx;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, o);
                        zsum += zz;
                    }
                    if (lane == 0) {
                        roff[s * (N + 1) + N] = run;
                        comp_nnz[s] = run;
                        atomicAdd(&patch_zero, zsum);  // 3 adds of integers: order-free
                    }
                }
                __syncthreads();
                if (t == 0) {
                    for (int s = 0; s < 3; ++s) {
                        const uint32_t snz = comp_nnz[s];
                        patch_bytes += 12ull * snz + 4ull * (N + 1);
                        patch_nnz += snz;
                        if (!cycle) {
                            slot_ok[s] = 0;
                            continue;
                        }
                        const uint64_t off = chunk_alloc(a, cs, round16(12ull * snz + 4ull * (N + 1)));
                        slot_ok[s] = off != ~0ull;
                        slot_off[s] = off;
                        a.dir_out[(size_t)p * 9 + 3 * rd + s] = slot_ok[s] ? DirEntry{off, snz, 0u} : DirEntry{0, 0u, DIR_DEAD};
                    }
                }
                __syncthreads();
                // ordered CSR rows (codec.hpp:37-60) + inverse along dim 1
                if (gok) {
                    for (int s = 0; s < 3; ++s) {
                        if (!slot_ok[s]) continue;
                        unsigned char* base = a.store_out + slot_off[s];
                        const uint32_t nnz = comp_nnz[s];
                        double* vo = reinterpret_cast<double*>(base);
                        uint32_t* co = reinterpret_cast<uint32_t*>(base + 8ull * nnz);
                        uint32_t* ro = co + nnz;
                        const uint32_t k0 = roff[s * (N + 1) + g], rn = rnz[s * N + g];
                        if (g == 0 && r == 0) ro[0] = 0;
                        if (r == 0) ro[g + 1] = k0 + rn;
                        double* row = tiles + s * TILE + (g + 1) * TP + 1;
                        if (rn == 0) {  // all coefficients zero: the inverse is +0.0
                            for (int j = r; j < N; j += kGL) row[j] = 0.0;
                            continue;
                        }
                        uint32_t k = k0;
                        for (int c = 0; c < N; c += kGL) {
                            const int pc = c + r;
                            const double val = pc < N ? row[pc] : 0.0;
                            const bool nzv = val != 0.0;
                            const unsigned bal = (__ballot_sync(sm, nzv) >> (t & 24)) & 0xFFu;
                            if (nzv) {
                                const uint32_t at = k + __popc(bal & ((1u << r) - 1u));
                                vo[at] = val;
                                co[at] = (uint32_t)pc;
                            }
                            k += __popc(bal);
                        }
                        double x[E + 1];
                        grp_load<N, L, true>(x, row, 1, r);
                        __syncwarp(sm);
                        idwt_line_grp<N, L>(x, r, sm);
                        grp_store_nat<N>(x, row, 1, r);
                    }
                }
                __syncthreads();
                // reconstruction along dim 0 + mass of the new state
                if (gok) {
                    const double wj = (g == 0 || g == N - 1) ? 0.5 : 1.0;
                    for (int s = 0; s < 3; ++s) {
                        if (!slot_ok[s]) continue;
                        double* colp = tiles + s * TILE + TP + g + 1;
                        double x[E + 1];
                        grp_load<N, L, true>(x, colp, TP, r);
                        __syncwarp(sm);
                        idwt_line_grp<N, L>(x, r, sm);
#pragma unroll
                        for (int i = 0; i <= E; ++i) {
                            const int gi = E * r + i;
                            if (i < E || r == kGL - 1) m += (((gi == 0 || gi == N - 1) ? 0.5 : 1.0) * wj) * x[i];
                        }
                        grp_store_nat<N>(x, colp, TP, r);
                    }
                }
                __syncthreads();
                for (int c = t; c < 3 * N; c += NT) {  // edge lines of the new state
                    const int s = c / N, li = c - s * N;
                    if (slot_ok[s]) write_edges_lbm_tile<N>(a.eout, pp, 3 * rd + s, gg, li, tiles + s * TILE);
                }
                __syncthreads();
            }
            if (t == 0) {
                part.comp_bytes += patch_bytes;
                part.nnz += patch_nnz;
                part.zeroed += patch_zero;
            }
            store_raw = patch_zero == 0;  // skip rule (pipeline.hpp:243-249)
            if (store_raw) m = 0.0;
        }
        if (store_raw) {
            for (int rd = 0; rd < 3; ++rd) {
                if (t == 0) {
                    for (int s = 0; s < 3; ++s) {
                        const uint64_t off = chunk_alloc(a, cs, round16((uint64_t)NN * 8));
                        slot_ok[s] = off != ~0ull;
                        slot_off[s] = off;
                        a.dir_out[(size_t)p * 9 + 3 * rd + s] =
                            slot_ok[s] ? DirEntry{off, 0u, DIR_RAW} : DirEntry{0, 0u, DIR_DEAD};
                    }
                }
                __syncthreads();
                for (int c = t; c < 3 * NN; c += NT) {
                    const int s = c / NN, cc = c - s * NN, i = cc / N, j = cc - (cc / N) * N;
                    const double x = S.pop(3 * rd + s)[cc];
                    tiles[s * TILE + (i + 1) * TP + j + 1] = x;
                    if (slot_ok[s]) reinterpret_cast<double*>(a.store_out + slot_off[s])[cc] = x;
                }
                __syncthreads();
                for (int c = t; c < 3 * N; c += NT) {
                    const int s = c / N, li = c - s * N;
                    write_edges_lbm_tile<N>(a.eout, pp, 3 * rd + s, gg, li, tiles + s * TILE);
                    m += tile_col_mass<N>(tiles + s * TILE, li);
                }
                __syncthreads();
            }
        }
        red[t] = m;
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
    }
    if (MODE == MODE_DECODE) return;
    finalize_step(a, part);
}

}  // namespace wg
