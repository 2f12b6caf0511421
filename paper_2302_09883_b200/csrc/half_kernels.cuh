// half_kernels.cuh — the fused step kernels for 65-point patches with
// half-line ownership (halfline.cuh): k_patch_step_h (FV transport) and
// k_lbm_step_h (D2Q9).  Same algorithm, same outputs and the same one-launch
// step structure as patch_kernels.cuh / lbm_kernels.cuh; two lanes per line
// halve the registers per thread so twice as many warps fit an SM.
#pragma once

#include "halfline.cuh"
#include "lbm_kernels.cuh"

namespace wg {

template <int N, int SLOTS>
struct HLayout {
    static constexpr int TILE = HT<N>::TILE;
    static constexpr int NT = ((SLOTS * N + 15) / 16) * 32;  // 16 lines per warp
    static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t)(SLOTS * TILE) + sizeof(unsigned long long) * NT;
    }
};

// decode (rows + columns) + ghost ring + upwind FV for the lane pair owning
// column li (transport).  Contains barriers: every thread calls it.
template <int N, int L>
__device__ __forceinline__ void decode_and_fv_h(const StepArgs& a, double* T, bool active, const DirEntry e,
                                                const PatchPos& pp, int li, int h, double (&v)[HT<N>::H]) {
    using G = HT<N>;
    constexpr int M = G::M, H = G::H;
    const bool raw_in = decode_row_h<N, L>(T, li, h, active, e, a.store_in);
    if (active) fill_ghosts_h<N>(T, li, h, a.ein, pp, 0, a.g);
    __syncthreads();
    const int j = li;
    if (active) {
        decode_col_h<N, L>(T, j, h, raw_in, v);
        if (!raw_in) store_col_h<N>(T, j, h, v);
    }
    __syncthreads();
    if (active) {
        // lane 0 walks rows 0..M downwards, lane 1 rows N-1..M upwards; the
        // partner supplies the row beyond the midpoint (its local M-1)
        const double across = pair_xchg(v[M - 1]);
        const double outer = T[G::at(h ? N + 1 : 0, j + 1)];  // ghost row 0 / N+1
        double prev = outer;
#pragma unroll
        for (int k = 0; k < H; ++k) {
            const int gi_lo = k, gi_hi = N - 1 - k;
            const double x = v[k];
            const double next = (k == H - 1) ? across : v[k + 1];
            const double xp = h ? prev : next;  // point i+1 (+x)
            const double xm = h ? next : prev;  // point i-1 (-x)
            const double* trow = T + (h ? gi_hi + 1 : gi_lo + 1) * G::TP;
            const double yl = trow[j];
            const double yr = trow[j + 2];
            double out = x;  // solver.hpp:212-226, directions +x, -x, +y, -y
            out -= a.r * flux_upwind(x, xp, a.smax[0], a.smin[0]);
            out -= a.r * flux_upwind(x, xm, a.smax[1], a.smin[1]);
            out -= a.r * flux_upwind(x, yr, a.smax[2], a.smin[2]);
            out -= a.r * flux_upwind(x, yl, a.smax[3], a.smin[3]);
            prev = x;
            v[k] = out;
        }
    }
}

template <int N, int L, int P, int MODE>
__global__ void __launch_bounds__(HLayout<N, P>::NT, 1) k_patch_step_h(const __grid_constant__ StepArgs a) {
    using G = HT<N>;
    using Lay = HLayout<N, P>;
    constexpr int M = G::M, H = G::H, TILE = G::TILE, NT = Lay::NT, LW = 2 * N;  // lanes per slot
    static_assert(P <= 32, "slots are handled by the lanes of warp 0");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(tiles + P * TILE);
    __shared__ DirEntry slot_dir[P], next_dir[P];
    __shared__ uint64_t slot_off[P];
    __shared__ int slot_mode[P];
    __shared__ int any_raw;
    __shared__ ChunkState cs;

    const int t = threadIdx.x;
    const int lane = t & 31;
    const int gl = hl_line(t);
    const int ps = gl / N;
    const int li = gl - ps * N;
    const int h = hl_half(t);
    const bool lane_ok = gl < P * N;
    const ShardGeom& g = a.g;
    double* T = tiles + (lane_ok ? ps : 0) * TILE;
    const int j = li;
    const uint32_t ngroups = (g.npatch + P - 1) / P;
    StepPartial acc{0, 0, 0, 0.0, 0.0};

    if (t == 0) cs.cur = cs.end = 0;
    if (t < P) {
        const uint32_t p0 = blockIdx.x * P + t;
        slot_dir[t] = p0 < g.npatch ? a.dir_in[p0] : DirEntry{0, 0u, DIR_DEAD};
    }
    __syncthreads();

    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const uint32_t p = grp * P + ps;
        const bool valid = lane_ok && p < g.npatch;
        const PatchPos pp = patch_pos(p, g);
        const uint32_t nxt = grp + gridDim.x;
        if (t < P) {
            const uint32_t pn = nxt * P + t;
            next_dir[t] = (nxt < ngroups && pn < g.npatch) ? a.dir_in[pn] : DirEntry{0, 0u, DIR_DEAD};
        }
        const DirEntry myd = lane_ok ? slot_dir[ps] : DirEntry{0, 0u, DIR_DEAD};

        if (MODE == MODE_DECODE) {
            const bool raw_in = decode_row_h<N, L>(T, li, h, valid, myd, a.store_in);
            __syncthreads();
            if (valid) {
                double v[H];
                decode_col_h<N, L>(T, j, h, raw_in, v);
                double* out = a.decode_out + (size_t)p * ((N + 2) * (N + 2));
#pragma unroll
                for (int k = 0; k < H; ++k)
                    if (h == 0 || k < M) out[(hglobal<N>(h, k) + 1) * (N + 2) + j + 1] = v[k];
            }
            __syncthreads();
            if (t < P) slot_dir[t] = next_dir[t];
            __syncthreads();
            continue;
        }

        if (t < P) slot_mode[t] = 2;
        double v[H];
        double m = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
            const bool active = valid && (pass == 0 || slot_mode[ps] == 1);
            decode_and_fv_h<N, L>(a, T, active, myd, pp, li, h, v);
            if (pass == 1) {
                if (active) m = col_mass_h<N>(j, h, v);
                break;
            }
            if (valid) acc.mass_fv += col_mass_h<N>(j, h, v);
            if (nxt < ngroups && lane_ok && nxt * P + ps < g.npatch)
                prefetch_patch<N>(a, nxt * P + ps, next_dir[ps], 0, 2 * li + h, 2 * N);

            unsigned nz = 0, zr = 0;
            if (a.compress) {
                __syncthreads();
                if (valid) fwd_col_to_tile_h<N, L>(T, j, h, v);
                __syncthreads();
                if (valid) fwd_row_threshold_h<N, L>(T, li, h, a.thr, v, nz, zr);
                // per-line totals on the lower-half lane; the upper lane adds 0
                const unsigned long long mine = ((unsigned long long)zr << 32) | nz;
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, mine, kPairXor);
                cta_inclusive_scan<NT>(h ? 0ull : mine + other, inc);
            } else {
                __syncthreads();
            }
            if (t < 32) {
                const uint32_t ps_ = (uint32_t)lane;
                const bool sv = lane < P && grp * P + ps_ < g.npatch;
                unsigned long long base = 0, tot = 0;
                if (sv && a.compress) {
                    base = ps_ == 0 ? 0ull : inc[hl_thread(ps_ * N) - 1];
                    tot = inc[hl_thread(ps_ * N + N - 1)] - base;
                }
                const uint32_t snz = (uint32_t)(tot & 0xffffffffu), szr = (uint32_t)(tot >> 32);
                const int mode = !sv ? 2 : (a.compress && szr != 0 ? 0 : 1);
                const unsigned long long need = mode == 0   ? round16(12ull * snz + 4ull * (N + 1))
                                                : mode == 1 ? round16((unsigned long long)N * N * 8)
                                                            : 0ull;
                unsigned long long ex = need;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long y = __shfl_up_sync(0xffffffffu, ex, o);
                    if (lane >= o) ex += y;
                }
                const unsigned long long total = __shfl_sync(0xffffffffu, ex, 31);
                ex -= need;
                unsigned long long b0 = 0;
                if (lane == 0) b0 = chunk_alloc(a, cs, total);
                b0 = __shfl_sync(0xffffffffu, b0, 0);
                if (sv) {
                    const uint32_t pq = grp * P + ps_;
                    const bool dead = b0 == ~0ull;
                    slot_mode[ps_] = dead ? 2 : mode;
                    slot_off[ps_] = b0 + ex;
                    a.dir_out[pq] = dead ? DirEntry{0, 0u, DIR_DEAD}
                                         : (mode == 0 ? DirEntry{b0 + ex, snz, 0u} : DirEntry{b0 + ex, 0u, DIR_RAW});
                    if (a.compress) {
                        acc.comp_bytes += 12ull * snz + 4ull * (N + 1);
                        acc.nnz += snz;
                        acc.zeroed += szr;
                    }
                }
                const unsigned rawmask = __ballot_sync(0xffffffffu, sv && mode == 1 && b0 != ~0ull);
                if (lane == 0) any_raw = a.compress && rawmask != 0;
            }
            __syncthreads();
            if (!a.compress) break;
            const bool compressed = valid && slot_mode[ps] == 0;
            if (compressed) {
                const unsigned long long base = ps == 0 ? 0ull : inc[hl_thread(ps * N) - 1];
                const int t0 = hl_thread(ps * N + li);
                const uint32_t incl = (uint32_t)((inc[t0] - base) & 0xffffffffu);  // lines <= li
                const uint32_t rowk = incl - (uint32_t)(__shfl_sync(__activemask(), (unsigned)(nz), lane & 15) +
                                                         __shfl_sync(__activemask(), (unsigned)(nz), (lane & 15) | 16));
                const uint32_t snz = (uint32_t)((inc[hl_thread(ps * N + N - 1)] - base) & 0xffffffffu);
                write_csr_row_h<N, L>(a.store_out + slot_off[ps], snz, li, h, rowk, v);
                inv_row_to_tile_h<N, L>(T, li, h, v);
            }
            __syncthreads();
            if (compressed) {
                decode_col_h<N, L>(T, j, h, false, v);
                m = col_mass_h<N>(j, h, v);
                write_edges_h<N>(a.eout, pp, 0, g, j, h, v);
            }
            if (!any_raw) break;
            __syncthreads();
        }
        if (valid && slot_mode[ps] == 1) {
            double* d = reinterpret_cast<double*>(a.store_out + slot_off[ps]);
#pragma unroll
            for (int k = 0; k < H; ++k)
                if (h == 0 || k < M) d[(size_t)hglobal<N>(h, k) * N + j] = v[k];
            write_edges_h<N>(a.eout, pp, 0, g, j, h, v);
            if (!a.compress) m = col_mass_h<N>(j, h, v);
        }
        acc.mass += m;
        __syncthreads();
        if (t < P) slot_dir[t] = next_dir[t];
        __syncthreads();
    }
    if (MODE == MODE_DECODE) return;
    const StepPartial part = cta_reduce_partial<NT>(acc);
    finalize_step(a, part);
}

// ---- D2Q9 -----------------------------------------------------------------

template <int N, int L>
__device__ __forceinline__ double decode_stream_collide_h(const StepArgs& a, double* T, double* S, uint32_t p,
                                                          const PatchPos& pp, int s, int li, int h, bool lane_ok) {
    using G = HT<N>;
    using Lay = HLayout<N, 3>;
    constexpr int M = G::M, H = G::H, NT = Lay::NT, NN = N * N;
    for (int rd = 0; rd < 3; ++rd) {
        const int q = 3 * rd + s;
        const DirEntry e = lane_ok ? a.dir_in[(size_t)p * 9 + q] : DirEntry{0, 0u, DIR_DEAD};
        const bool raw_in = decode_row_h<N, L>(T, li, h, lane_ok, e, a.store_in);
        if (lane_ok) fill_ghosts_h<N>(T, li, h, a.ein, pp, q, a.g);
        __syncthreads();
        if (lane_ok && !raw_in) {
            double v[H];
            decode_col_h<N, L>(T, li, h, false, v);
            store_col_h<N>(T, li, h, v);
        }
        __syncthreads();
        if (lane_ok) {  // pull streaming f_q(x) <- f_q(x - c_q)
            const int cx = lbm_cx(q), cy = lbm_cy(q);
            double* Sq = S + (size_t)q * NN;
            const int j = li;
#pragma unroll 3
            for (int k = 0; k < H; ++k) {
                const int gi = hglobal<N>(h, k);
                if (h == 0 || k < M) Sq[gi * N + j] = T[G::at(gi + 1 - cx, j + 1 - cy)];
            }
        }
        __syncthreads();
    }
    double mfv = 0.0;
    for (int c0 = threadIdx.x; c0 < NN; c0 += 2 * NT) {
        const int c1 = c0 + NT;
        const bool two = c1 < NN;
        double f0[9], f1[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            f0[q] = S[(size_t)q * NN + c0];
            f1[q] = two ? S[(size_t)q * NN + c1] : 1.0;
        }
        lbm_collide(f0, a.omega);
        lbm_collide(f1, a.omega);
        const int i0 = c0 / N, j0 = c0 - i0 * N, i1 = c1 / N, j1 = c1 - i1 * N;
        const double w0 = ((i0 == 0 || i0 == N - 1) ? 0.5 : 1.0) * ((j0 == 0 || j0 == N - 1) ? 0.5 : 1.0);
        const double w1 = ((i1 == 0 || i1 == N - 1) ? 0.5 : 1.0) * ((j1 == 0 || j1 == N - 1) ? 0.5 : 1.0);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            S[(size_t)q * NN + c0] = f0[q];
            mfv += w0 * f0[q];
            if (two) {
                S[(size_t)q * NN + c1] = f1[q];
                mfv += w1 * f1[q];
            }
        }
    }
    __syncthreads();
    return mfv;
}

template <int N, int L, int MODE>
__global__ void __launch_bounds__(HLayout<N, 3>::NT, 1) k_lbm_step_h(const __grid_constant__ StepArgs a) {
    using G = HT<N>;
    using Lay = HLayout<N, 3>;
    constexpr int M = G::M, H = G::H, TILE = G::TILE, NT = Lay::NT, NN = N * N, LW = 2 * N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(tiles + 3 * TILE);
    __shared__ uint64_t slot_off[3];
    __shared__ int slot_ok[3];
    __shared__ uint32_t comp_nnz[3];
    __shared__ unsigned long long patch_bytes, patch_nnz, patch_zero;
    __shared__ ChunkState cs;
    __shared__ DirEntry next_dir[9];

    const int t = threadIdx.x;
    const int gl = hl_line(t);
    const int s = gl / N;
    const int li = gl - s * N;
    const int h = hl_half(t);
    const bool lane_ok = gl < 3 * N;
    const ShardGeom& g = a.g;
    double* T = tiles + (lane_ok ? s : 0) * TILE;
    double* S = a.scratch + (size_t)blockIdx.x * LbmLayout<N>::scratch_doubles();

    if (MODE == MODE_DECODE) {
        for (uint32_t p = blockIdx.x; p < g.npatch; p += gridDim.x) {
            for (int rd = 0; rd < 3; ++rd) {
                const int q = 3 * rd + s;
                const DirEntry e = lane_ok ? a.dir_in[(size_t)p * 9 + q] : DirEntry{0, 0u, DIR_DEAD};
                const bool raw_in = decode_row_h<N, L>(T, li, h, lane_ok, e, a.store_in);
                __syncthreads();
                if (lane_ok) {
                    double v[H];
                    decode_col_h<N, L>(T, li, h, raw_in, v);
                    double* out = a.decode_out + ((size_t)p * 9 + q) * ((N + 2) * (N + 2));
#pragma unroll
                    for (int k = 0; k < H; ++k)
                        if (h == 0 || k < M) out[(hglobal<N>(h, k) + 1) * (N + 2) + li + 1] = v[k];
                }
                __syncthreads();
            }
        }
        return;
    }

    StepPartial part{0, 0, 0, 0.0, 0.0};
    double macc = 0.0, mfacc = 0.0;
    if (t == 0) cs.cur = cs.end = 0;
    for (uint32_t p = blockIdx.x; p < g.npatch; p += gridDim.x) {
        const PatchPos pp = patch_pos(p, g);
        const uint32_t pn = p + gridDim.x;
        if (t < 9) next_dir[t] = pn < g.npatch ? a.dir_in[(size_t)pn * 9 + t] : DirEntry{0, 0u, DIR_DEAD};
        mfacc += decode_stream_collide_h<N, L>(a, T, S, p, pp, s, li, h, lane_ok);
        if (pn < g.npatch && lane_ok)
            for (int q = s; q < 9; q += 3) prefetch_patch<N>(a, pn, next_dir[q], q, 2 * li + h, 2 * N);
        double m = 0.0;
        bool store_raw = !a.compress;
        if (a.compress) {
            if (t == 0) {
                patch_bytes = 0;
                patch_nnz = 0;
                patch_zero = 0;
            }
            const bool cycle = a.thr_any != 0;
            for (int rd = 0; rd < 3; ++rd) {
                const int q = 3 * rd + s;
                double v[H];
                if (lane_ok) {
#pragma unroll
                    for (int k = 0; k < H; ++k) v[k] = S[(size_t)q * NN + hglobal<N>(h, k) * N + li];
                    fwd_col_to_tile_h<N, L>(T, li, h, v);
                }
                __syncthreads();
                unsigned nz = 0, zr = 0;
                if (lane_ok) fwd_row_threshold_h<N, L>(T, li, h, a.thr, v, nz, zr);
                const unsigned long long mine = ((unsigned long long)zr << 32) | nz;
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, mine, kPairXor);
                cta_inclusive_scan<NT>(h ? 0ull : mine + other, inc);
                if (t == 0) {
                    for (int sl = 0; sl < 3; ++sl) {
                        const int qq = 3 * rd + sl;
                        const unsigned long long base = sl == 0 ? 0ull : inc[hl_thread(sl * N) - 1];
                        const unsigned long long tot = inc[hl_thread(sl * N + N - 1)] - base;
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
                const bool ok = lane_ok && slot_ok[s];
                if (ok) {
                    const unsigned long long base = s == 0 ? 0ull : inc[hl_thread(s * N) - 1];
                    const uint32_t incl = (uint32_t)((inc[hl_thread(s * N + li)] - base) & 0xffffffffu);
                    const int ln = t & 31;
                    const uint32_t rowk = incl - (uint32_t)(__shfl_sync(__activemask(), (unsigned)nz, ln & 15) +
                                                            __shfl_sync(__activemask(), (unsigned)nz, (ln & 15) | 16));
                    write_csr_row_h<N, L>(a.store_out + slot_off[s], comp_nnz[s], li, h, rowk, v);
                    inv_row_to_tile_h<N, L>(T, li, h, v);
                }
                __syncthreads();
                if (ok) {
                    decode_col_h<N, L>(T, li, h, false, v);
                    write_edges_h<N>(a.eout, pp, q, g, li, h, v);
                    m += col_mass_h<N>(li, h, v);
                }
                __syncthreads();
            }
            if (t == 0) {
                part.comp_bytes += patch_bytes;
                part.nnz += patch_nnz;
                part.zeroed += patch_zero;
            }
            store_raw = patch_zero == 0;  // skip rule: the scratch holds the collided state
            if (store_raw) m = 0.0;
        }
        if (store_raw) {
            for (int rd = 0; rd < 3; ++rd) {
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
                if (lane_ok) {
                    const int q = 3 * rd + s;
                    double v[H];
#pragma unroll
                    for (int k = 0; k < H; ++k) v[k] = S[(size_t)q * NN + hglobal<N>(h, k) * N + li];
                    if (slot_ok[s]) {
                        double* d = reinterpret_cast<double*>(a.store_out + slot_off[s]);
#pragma unroll
                        for (int k = 0; k < H; ++k)
                            if (h == 0 || k < M) d[hglobal<N>(h, k) * N + li] = v[k];
                    }
                    write_edges_h<N>(a.eout, pp, q, g, li, h, v);
                    m += col_mass_h<N>(li, h, v);
                }
                __syncthreads();
            }
        }
        macc += m;
    }
    part.mass = macc;
    part.mass_fv = mfacc;
    if (t != 0) part.comp_bytes = part.nnz = part.zeroed = 0;
    const StepPartial tot = cta_reduce_partial<NT>(part);
    finalize_step(a, tot);
}

}  // namespace wg
