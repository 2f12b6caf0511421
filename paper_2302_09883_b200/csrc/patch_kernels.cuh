// patch_kernels.cuh — the fused per-patch step for the FV transport scheme.
// ONE kernel launch is the whole step (pipeline.hpp:194-289): for every
// patch
//
//   CSR decode -> inverse DWT (rows, then columns)      [idwt_nd, wavelet.hpp:200-223]
//   ghost ring from the neighbours' edge lines           [sync_ghosts, patchgrid.hpp:131-201]
//   upwind FV update                                     [fv_step, solver.hpp:207-231]
//   forward DWT (columns, then rows)                     [dwt_nd, wavelet.hpp:175-198]
//   threshold + scan-based stream compaction to CSR      [apply_threshold threshold.hpp:51-86,
//                                                         csr_encode codec.hpp:37-60]
//   inverse DWT of the kept coefficients -> edge lines + trapezoid mass
//                                                        [global_mass, patchgrid.hpp:244-266]
//   skip rule: a patch whose cycle zeroed nothing is re-decoded, re-stepped
//   and stored raw, bit-identical to the FV output       [pipeline.hpp:243-249]
//
// and the last CTA reduces the per-CTA partials into the step's MetricsRow.
// The uncompressed patch exists only in shared memory and registers.  CTAs
// are persistent; each owns groups of P patches (P slots, see
// patch_phases.cuh for the ownership model).
#pragma once

#include "patch_phases.cuh"

namespace wg {

template <int N, int P>
struct Layout {
    static constexpr int TP = N + 2;              // tile pitch (odd)
    static constexpr int TILE = TP * TP;
    static constexpr int NT = ((P * N + 31) / 32) * 32;
    static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t)(P * TILE + 2 * NT) + sizeof(unsigned long long) * NT;
    }
};

// decode (rows + columns), ghost ring, upwind FV: returns the FV output
// column j in v (natural order) for an active slot.  Contains 2 barriers.
template <int N, int L>
__device__ __forceinline__ void decode_and_fv(const StepArgs& a, double* T, bool active, const DirEntry e,
                                              const PatchPos& pp, int li, double (&v)[N]) {
    constexpr int TP = N + 2;
    bool raw_in = false;
    if (active) {
        raw_in = decode_row<N, L>(T, li, e, a.store_in);
        fill_ghosts<N>(T, li, a.ein, pp, 0, a.g);
    }
    __syncthreads();
    WG_PHASE_MARK(0);
    const int j = li;
    if (active) {
        decode_col<N, L>(T, j, raw_in, v);
        if (!raw_in) store_col<N>(T, j, v);
    }
    __syncthreads();
    WG_PHASE_MARK(1);
    // upwind FV update of column j (solver.hpp:207-231): directions in the
    // reference order +x, -x, +y, -y (solver.hpp:21-22); x = dim 0 = i.
    // No FMA (-fmad=false): out -= r * Q, Q = wl*max(s,0) + wr*min(s,0).
    if (active) {
        double prev = T[j + 1];                        // ghost row 0
        const double below = T[(N + 1) * TP + j + 1];  // ghost row N+1
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const double x = v[i];
            const double xp = (i == N - 1) ? below : v[i + 1];
            const double yl = T[(i + 1) * TP + j];
            const double yr = T[(i + 1) * TP + j + 2];
            double out = x;
            out -= a.r * flux_upwind(x, xp, a.smax[0], a.smin[0]);
            out -= a.r * flux_upwind(x, prev, a.smax[1], a.smin[1]);
            out -= a.r * flux_upwind(x, yr, a.smax[2], a.smin[2]);
            out -= a.r * flux_upwind(x, yl, a.smax[3], a.smin[3]);
            prev = x;
            v[i] = out;
        }
    }
}

// CTAs per SM the register allocation targets: 2 (spilling ~1 KB) measured
// best for 33-point patches (88 vs 86 GLUPS at 4096^2), 1 (no spills) for
// 65-point patches (75 vs 73)
#ifndef WG_MIN_BLOCKS
#define WG_MIN_BLOCKS(N) ((N) >= 65 ? 1 : 2)
#endif
template <int N, int L, int P, int MODE>
__global__ void __launch_bounds__(Layout<N, P>::NT, WG_MIN_BLOCKS(N))
    k_patch_step(const __grid_constant__ StepArgs a) {
    using Lay = Layout<N, P>;
    constexpr int TP = Lay::TP, TILE = Lay::TILE, NT = Lay::NT;
    static_assert(P <= 32, "slots are handled by the lanes of warp 0");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(tiles + P * TILE + 2 * NT);
    __shared__ DirEntry slot_dir[P], next_dir[P];
    __shared__ uint64_t slot_off[P];
    __shared__ int slot_mode[P];  // 0 compressed, 1 raw (skip rule / no compression), 2 dead
    __shared__ int any_raw;
    __shared__ ChunkState cs;

    const int t = threadIdx.x;
    const int lane = t & 31;
    const int ps = t / N;
    const int li = t - ps * N;
    const bool lane_ok = t < P * N;
    const ShardGeom& g = a.g;
    double* T = tiles + (lane_ok ? ps : 0) * TILE;
    const int j = li;
    const uint32_t ngroups = (g.npatch + P - 1) / P;
    // running partials: every thread its columns' masses, lane s of warp 0
    // the byte/nnz/zeroed counts of slot s (fixed order -> deterministic)
    StepPartial acc{0, 0, 0, 0.0, 0.0, 0.0};
    WG_PHASE_MARK(-1);

    if (t == 0) cs.cur = cs.end = 0;
    if (t < P) {
        const uint32_t p0 = blockIdx.x * P + t;
        slot_dir[t] = p0 < g.npatch ? a.dir_in[p0] : DirEntry{0, 0u, DIR_DEAD};
    }
    __syncthreads();

    // persistent CTAs: patch groups grp, grp + gridDim.x, ... (fixed order)
    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const uint32_t p = grp * P + ps;
        const bool valid = lane_ok && p < g.npatch;
        const PatchPos pp = patch_pos(p, g);
        const uint32_t nxt = grp + gridDim.x;
        if (t < P) {  // the next group's directory entries (latency hidden by this group)
            const uint32_t pn = nxt * P + t;
            next_dir[t] = (nxt < ngroups && pn < g.npatch) ? a.dir_in[pn] : DirEntry{0, 0u, DIR_DEAD};
        }

        if (MODE == MODE_DECODE) {
            bool raw_in = false;
            if (valid) raw_in = decode_row<N, L>(T, li, slot_dir[ps], a.store_in);
            __syncthreads();
            if (valid) {
                double v[N];
                decode_col<N, L>(T, j, raw_in, v);
                if (a.decode_out) {
                    double* out = a.decode_out + (size_t)p * TILE;
#pragma unroll
                    for (int i = 0; i < N; ++i) out[(i + 1) * TP + j + 1] = v[i];
                } else {  // l2 pass: the step's output against exact_transport
                    acc.l2 += col_l2<N>(a, pp, j, v);
                }
            }
            __syncthreads();
            if (t < P) slot_dir[t] = next_dir[t];
            __syncthreads();
            continue;
        }

        if (t < P) slot_mode[t] = 2;
        double v[N];
        double m = 0.0;
        // pass 0 runs the cycle for every slot; pass 1 (only if some slot
        // zeroed nothing: the skip rule, pipeline.hpp:243-249) re-derives
        // the FV output of those slots from the untouched inputs so that it
        // can be stored raw.
        for (int pass = 0; pass < 2; ++pass) {
            const bool active = valid && (pass == 0 || slot_mode[ps] == 1);
            decode_and_fv<N, L>(a, T, active, lane_ok ? slot_dir[ps] : DirEntry{}, pp, li, v);
            if (pass == 1) {
                if (active) m = col_mass<N>(j, v);
                break;
            }
            if (valid) acc.mass_fv += col_mass<N>(j, v);
            WG_PHASE_MARK(2);
            // warm L2 with the next group's inputs while this one computes
            if (nxt < ngroups && lane_ok && nxt * P + ps < g.npatch)
                prefetch_patch<N>(a, nxt * P + ps, next_dir[ps], 0, li, N);

            unsigned nz = 0, zr = 0;
            if (a.compress) {
                // ---- forward DWT along dim 0 (columns) in registers -------
                __syncthreads();  // everyone done reading the state tile
                WG_PHASE_MARK(3);
                if (valid) fwd_col_to_tile<N, L>(T, j, v);
                __syncthreads();
                WG_PHASE_MARK(4);
                // ---- ROW phase: forward DWT along dim 1, threshold, count --
                if (valid)
                    fwd_row_threshold<N, L>(T, li, a.thr, v, nz, zr,
                                            MODE == MODE_STEP_LZ ? T + (li + 1) * TP + 1 : nullptr);
                cta_inclusive_scan<NT>(((unsigned long long)zr << 32) | nz, inc);
                if (MODE == MODE_STEP_LZ)
                    tiles_to_dense<N, NT>(tiles, TILE, (int)min((uint32_t)P, g.npatch - grp * P),
                                          a.lz_dense + (size_t)grp * P * N * N);
                WG_PHASE_MARK(5);
            } else {
                __syncthreads();
            }
            // ---- warp 0, lane s = slot s: modes, one allocation, directory -
            if (t < 32) {
                const uint32_t ps_ = (uint32_t)lane;
                const bool sv = lane < P && grp * P + ps_ < g.npatch;
                unsigned long long base = 0, tot = 0;
                if (sv && a.compress) {
                    base = ps_ == 0 ? 0ull : inc[ps_ * N - 1];
                    tot = inc[ps_ * N + N - 1] - base;
                }
                const uint32_t snz = (uint32_t)(tot & 0xffffffffu), szr = (uint32_t)(tot >> 32);
                const int mode = !sv ? 2 : (a.compress && szr != 0 ? 0 : 1);
                unsigned long long need = mode == 0   ? round16(12ull * snz + 4ull * (N + 1))
                                          : mode == 1 ? round16((unsigned long long)N * N * 8)
                                                      : 0ull;
                unsigned long long ex = need;  // exclusive scan over the lanes
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
                        acc.comp_bytes += 12ull * snz + 4ull * (N + 1);  // CsrBlock::byte_size
                        acc.nnz += snz;
                        acc.zeroed += szr;
                    }
                }
                const unsigned rawmask = __ballot_sync(0xffffffffu, sv && mode == 1 && b0 != ~0ull);
                if (lane == 0) any_raw = a.compress && rawmask != 0;
            }
            __syncthreads();
            WG_PHASE_MARK(6);
            if (!a.compress) break;
            const bool compressed = valid && slot_mode[ps] == 0;
            if (compressed) {
                const unsigned long long base = ps == 0 ? 0ull : inc[ps * N - 1];
                const uint32_t k = (uint32_t)((inc[t] - base) & 0xffffffffu) - nz;
                const uint32_t snz = (uint32_t)((inc[ps * N + N - 1] - base) & 0xffffffffu);
                write_csr_row<N, L>(a.store_out + slot_off[ps], snz, li, k, nz, v);
                inv_row_to_tile<N, L>(T, li, v, nz);  // reconstruction, dim 1 inverse
            }
            __syncthreads();
            WG_PHASE_MARK(7);
            if (compressed) {
                decode_col<N, L>(T, j, false, v);
                m = col_mass<N>(j, v);
                write_edges<N>(a.eout, pp, 0, g, j, v);
            }
            WG_PHASE_MARK(8);
            if (!any_raw) break;
            __syncthreads();
        }

        // ---- raw slots: dense store of the scheme output ------------------
        if (valid && slot_mode[ps] == 1) {
            double* d = reinterpret_cast<double*>(a.store_out + slot_off[ps]);
#pragma unroll
            for (int i = 0; i < N; ++i) d[(size_t)i * N + j] = v[i];
            write_edges<N>(a.eout, pp, 0, g, j, v);
            if (!a.compress) m = col_mass<N>(j, v);
        }
        acc.mass += m;
        __syncthreads();
        if (t < P) slot_dir[t] = next_dir[t];
        __syncthreads();
        WG_PHASE_MARK(9);
    }
    if (MODE == MODE_DECODE) {
        if (!a.decode_out) finalize_l2<NT>(a, acc.l2);
        return;
    }
    const StepPartial part = cta_reduce_partial<NT>(acc);
    WG_PHASE_MARK(10);
    finalize_step(a, part);
    WG_PHASE_MARK(11);
}

}  // namespace wg
