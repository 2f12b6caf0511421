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
__device__ __forceinline__ void decode_and_fv(const StepArgs& a, double* T, bool active, uint32_t p,
                                              const PatchPos& pp, int li, double (&v)[N]) {
    constexpr int TP = N + 2;
    bool raw_in = false;
    if (active) {
        raw_in = decode_row<N, L>(T, li, a.dir_in[p], a.store_in);
        fill_ghosts<N>(T, li, a.ein, pp, 0, a.g);
    }
    __syncthreads();
    const int j = li;
    if (active) {
        decode_col<N, L>(T, j, raw_in, v);
        if (!raw_in) store_col<N>(T, j, v);
    }
    __syncthreads();
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

template <int N, int L, int P, int MODE>
__global__ void __launch_bounds__(Layout<N, P>::NT, 2)
    k_patch_step(const __grid_constant__ StepArgs a) {
    using Lay = Layout<N, P>;
    constexpr int TP = Lay::TP, TILE = Lay::TILE, NT = Lay::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    double* red = tiles + P * TILE;   // per-thread mass partials (after the cycle)
    double* red_fv = red + NT;        // per-thread mass partials (scheme output)
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(red_fv + NT);
    __shared__ uint64_t slot_off[P];
    __shared__ int slot_mode[P];  // 0 compressed, 1 raw (skip rule / no compression), 2 dead
    __shared__ unsigned long long slot_bytes[P], slot_nnz[P], slot_zero[P];
    __shared__ double slot_m[P], slot_mf[P];
    __shared__ int any_raw;

    const int t = threadIdx.x;
    const int ps = t / N;
    const int li = t - ps * N;
    const bool lane_ok = t < P * N;
    const ShardGeom& g = a.g;
    double* T = tiles + (lane_ok ? ps : 0) * TILE;
    const int j = li;
    const uint32_t ngroups = (g.npatch + P - 1) / P;
    StepPartial part{0, 0, 0, 0.0, 0.0};

    // persistent CTAs: patch groups grp, grp + gridDim.x, ... (fixed order)
    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const uint32_t p = grp * P + ps;
        const bool valid = lane_ok && p < g.npatch;
        const PatchPos pp = patch_pos(p, g);

        if (MODE == MODE_DECODE) {
            bool raw_in = false;
            if (valid) raw_in = decode_row<N, L>(T, li, a.dir_in[p], a.store_in);
            __syncthreads();
            if (valid) {
                double v[N];
                decode_col<N, L>(T, j, raw_in, v);
                double* out = a.decode_out + (size_t)p * TILE;
#pragma unroll
                for (int i = 0; i < N; ++i) out[(i + 1) * TP + j + 1] = v[i];
            }
            __syncthreads();
            continue;
        }

        if (t < P) {
            slot_bytes[t] = slot_nnz[t] = slot_zero[t] = 0;
            slot_mode[t] = a.compress ? 2 : 1;  // no_compression: every patch is stored raw
        }
        if (t == 0) any_raw = 0;
        double v[N];
        double m = 0.0;
        // pass 0 runs the cycle for every slot; pass 1 (only if some slot
        // zeroed nothing: the skip rule, pipeline.hpp:243-249) re-derives
        // the FV output of those slots from the untouched inputs so that it
        // can be stored raw.
        for (int pass = 0; pass < 2; ++pass) {
            const bool active = valid && (pass == 0 || slot_mode[ps] == 1);
            decode_and_fv<N, L>(a, T, active, p, pp, li, v);
            if (pass == 1) {
                if (active) m = col_mass<N>(j, v);
                break;
            }
            red_fv[t] = valid ? col_mass<N>(j, v) : 0.0;
            if (!a.compress) {
                m = red_fv[t];
                break;
            }
            // ---- forward DWT along dim 0 (columns) in registers -----------
            __syncthreads();  // everyone done reading the state tile
            if (valid) fwd_col_to_tile<N, L>(T, j, v);
            __syncthreads();

            // ---- ROW phase: forward DWT along dim 1, threshold, count -----
            const int i = li;
            unsigned nz = 0, zr = 0;
            if (valid) fwd_row_threshold<N, L>(T, i, a.thr, v, nz, zr);
            cta_inclusive_scan<NT>(((unsigned long long)zr << 32) | nz, inc);
            unsigned long long slot_base = 0, slot_tot = 0;
            if (lane_ok) {
                slot_base = ps == 0 ? 0ull : inc[ps * N - 1];
                slot_tot = inc[ps * N + N - 1] - slot_base;
            }
            const uint32_t nnz_tot = (uint32_t)(slot_tot & 0xffffffffu);
            const uint32_t zero_tot = (uint32_t)(slot_tot >> 32);
            if (valid && li == 0) {
                slot_bytes[ps] = 12ull * nnz_tot + 4ull * (N + 1);  // CsrBlock::byte_size
                slot_nnz[ps] = nnz_tot;
                slot_zero[ps] = zero_tot;
                if (zero_tot == 0) {  // skip rule: stored raw after pass 1
                    slot_mode[ps] = 1;
                    any_raw = 1;
                } else {
                    const uint64_t bytes = round16(12ull * nnz_tot + 4ull * (N + 1));
                    const uint64_t off = atomicAdd(a.bump_out, (unsigned long long)bytes);
                    if (off + bytes > a.cap_out) {
                        atomicOr(a.err, ERR_STORE_OVERFLOW);
                        a.dir_out[p] = DirEntry{0, 0u, DIR_DEAD};
                        slot_mode[ps] = 2;
                    } else {
                        slot_mode[ps] = 0;
                        slot_off[ps] = off;
                        a.dir_out[p] = DirEntry{off, nnz_tot, 0u};
                    }
                }
            }
            __syncthreads();
            const bool compressed = valid && slot_mode[ps] == 0;
            if (compressed) {
                const uint32_t k = (uint32_t)((inc[t] - slot_base) & 0xffffffffu) - nz;
                write_csr_row<N, L>(a.store_out + slot_off[ps], nnz_tot, i, k, nz, v);
                inv_row_to_tile<N, L>(T, i, v);  // reconstruction, dim 1 inverse
            }
            __syncthreads();
            if (compressed) {
                decode_col<N, L>(T, j, false, v);
                m = col_mass<N>(j, v);
                write_edges<N>(a.eout, pp, 0, g, j, v);
            }
            if (!any_raw) break;
            __syncthreads();
        }

        // ---- raw slots: dense store of the FV output ----------------------
        __syncthreads();
        if (valid && li == 0 && slot_mode[ps] == 1) {
            const uint64_t bytes = round16((uint64_t)N * N * 8);
            const uint64_t off = atomicAdd(a.bump_out, (unsigned long long)bytes);
            if (off + bytes > a.cap_out) {
                atomicOr(a.err, ERR_STORE_OVERFLOW);
                a.dir_out[p] = DirEntry{0, 0u, DIR_DEAD};
                slot_off[ps] = ~0ull;
            } else {
                slot_off[ps] = off;
                a.dir_out[p] = DirEntry{off, 0u, DIR_RAW};
            }
        }
        __syncthreads();
        if (valid && slot_mode[ps] == 1) {
            if (slot_off[ps] != ~0ull) {
                double* d = reinterpret_cast<double*>(a.store_out + slot_off[ps]);
#pragma unroll
                for (int i = 0; i < N; ++i) d[(size_t)i * N + j] = v[i];
            }
            write_edges<N>(a.eout, pp, 0, g, j, v);
        }
        red[t] = m;
        __syncthreads();

        // ---- per-group partial sums (fixed slot order) ---------------------
        const int warp = t >> 5;
        for (int sl = warp; sl < P; sl += NT / 32) {
            const double mm = warp_sum_range(red, sl * N, N);
            const double mf = warp_sum_range(red_fv, sl * N, N);
            if ((t & 31) == 0) {
                slot_m[sl] = mm;
                slot_mf[sl] = mf;
            }
        }
        __syncthreads();
        if (t == 0) {
            for (int sl = 0; sl < P; ++sl) {
                if (grp * P + sl >= g.npatch) break;
                part.comp_bytes += slot_bytes[sl];
                part.nnz += slot_nnz[sl];
                part.zeroed += slot_zero[sl];
                part.mass += slot_m[sl];
                part.mass_fv += slot_mf[sl];
            }
        }
        __syncthreads();
    }
    if (MODE == MODE_DECODE) return;
    finalize_step(a, part);
}

}  // namespace wg
