// patch_kernels.cuh — the fused per-patch step for the FV transport scheme:
// one kernel runs, for every patch,
//
//   CSR decode -> inverse DWT (rows, then columns)      [idwt_nd, wavelet.hpp:200-223]
//   ghost ring from the neighbours' edge lines           [sync_ghosts, patchgrid.hpp:131-201]
//   upwind FV update                                     [fv_step, solver.hpp:207-231]
//   forward DWT (columns, then rows)                     [dwt_nd, wavelet.hpp:175-198]
//   threshold + scan-based stream compaction to CSR      [apply_threshold threshold.hpp:51-86,
//                                                         csr_encode codec.hpp:37-60]
//   skip rule (nothing zeroed -> raw patch)              [pipeline.hpp:243-249]
//   inverse DWT of the kept coefficients -> edge lines + trapezoid mass
//                                                        [global_mass, patchgrid.hpp:244-266]
//
// so the uncompressed patch exists only in shared memory and registers.  A
// CTA owns P patches (P slots); see patch_phases.cuh for the ownership model.
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

template <int N, int L, int P, int MODE>
__global__ void __launch_bounds__(Layout<N, P>::NT)
    k_patch_step(const __grid_constant__ StepArgs a) {
    using Lay = Layout<N, P>;
    constexpr int TP = Lay::TP, TILE = Lay::TILE, NT = Lay::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tiles = reinterpret_cast<double*>(smem_raw);
    double* red = tiles + P * TILE;   // per-thread mass partials (after the cycle)
    double* red_fv = red + NT;        // per-thread mass partials (scheme output)
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(red_fv + NT);
    __shared__ uint64_t slot_off[P];
    __shared__ int slot_mode[P];  // 0 compressed, 1 raw (skip rule), 2 dead slot

    const int t = threadIdx.x;
    const int ps = t / N;
    const int li = t - ps * N;
    const bool lane_ok = t < P * N;
    const ShardGeom& g = a.g;

    // ---- which patch does this slot own -----------------------------------
    uint32_t p = 0;
    bool valid;
    if (MODE == MODE_RAW && a.raw_list) {
        const uint32_t cnt = *a.raw_count;
        if (blockIdx.x * P >= cnt) return;  // whole CTA idle (uniform)
        const uint32_t k = blockIdx.x * P + ps;
        valid = lane_ok && k < cnt;
        p = valid ? a.raw_list[k] : 0;
    } else {
        p = blockIdx.x * P + ps;
        valid = lane_ok && p < g.npatch;
    }
    const PatchPos pp = patch_pos(p, g);
    double* T = tiles + (lane_ok ? ps : 0) * TILE;

    // ---- ROW phase: decode row li, inverse transform along dim 1 ----------
    bool raw_in = false;
    if (valid) {
        raw_in = decode_row<N, L>(T, li, a.dir_in[p], a.store_in);
        if (MODE != MODE_DECODE) fill_ghosts<N>(T, li, a.ein, pp, 0, g);
    }
    __syncthreads();

    // ---- COLUMN phase: inverse transform along dim 0 -> state column li ----
    double v[N];
    const int j = li;
    if (valid) {
        decode_col<N, L>(T, j, raw_in, v);
        if (MODE == MODE_DECODE) {
            double* out = a.decode_out + (size_t)p * TILE;
#pragma unroll
            for (int i = 0; i < N; ++i) out[(i + 1) * TP + j + 1] = v[i];
        } else if (!raw_in) {
            store_col<N>(T, j, v);
        }
    }
    if (MODE == MODE_DECODE) return;
    __syncthreads();

    // ---- upwind FV update of column j (solver.hpp:207-231) ----------------
    // directions in the reference order +x, -x, +y, -y (solver.hpp:21-22);
    // x = dim 0 = i.  No FMA (-fmad=false).
    double mfv = 0.0;
    if (valid) {
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
        mfv = col_mass<N>(j, v);
    }
    red_fv[t] = mfv;

    if (MODE == MODE_RAW) {
        // store the scheme output uncompressed (skip rule / no_compression)
        if (valid && li == 0) {
            const uint64_t bytes = round16((uint64_t)N * N * 8);
            const uint64_t off = atomicAdd(a.bump_out, (unsigned long long)bytes);
            if (off + bytes > a.cap_out) {
                atomicOr(a.err, ERR_STORE_OVERFLOW);
                a.dir_out[p] = DirEntry{0, 0u, DIR_DEAD};
                slot_mode[ps] = 2;
            } else {
                slot_mode[ps] = 1;
                slot_off[ps] = off;
                a.dir_out[p] = DirEntry{off, 0u, DIR_RAW};
            }
        }
        __syncthreads();
        if (valid && slot_mode[ps] == 1) {
            double* d = reinterpret_cast<double*>(a.store_out + slot_off[ps]);
#pragma unroll
            for (int i = 0; i < N; ++i) d[(size_t)i * N + j] = v[i];
        }
        red[t] = mfv;
    } else {
        // ---- forward DWT along dim 0 (columns) in registers ---------------
        __syncthreads();  // everyone done reading the state tile
        if (valid) fwd_col_to_tile<N, L>(T, j, v);
        __syncthreads();

        // ---- ROW phase: forward DWT along dim 1, threshold, count ---------
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
            PatchStats& st = a.stats[p];
            st.comp_bytes = 12ull * nnz_tot + 4ull * (N + 1);  // CsrBlock::byte_size
            st.nnz = nnz_tot;
            st.zeroed = zero_tot;
            if (zero_tot == 0) {  // skip rule: the raw kernel stores the FV output
                const uint32_t k = atomicAdd(a.raw_count, 1u);
                if (k < a.raw_capacity) a.raw_list[k] = p;
                else atomicOr(a.err, ERR_RAW_OVERFLOW);
                slot_mode[ps] = 1;
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
        double m = 0.0;
        if (compressed) {
            decode_col<N, L>(T, j, false, v);
            m = col_mass<N>(j, v);
        }
        red[t] = m;
    }

    // ---- edge lines of the new state (ghost source of the next step) -----
    if (valid && slot_mode[ps] == (MODE == MODE_RAW ? 1 : 0)) write_edges<N>(a.eout, pp, 0, g, j, v);
    __syncthreads();
    // ---- per-patch trapezoid masses (deterministic) ----------------------
    const int warp = t >> 5;
    for (int s = warp; s < P; s += NT / 32) {
        const double mm = warp_sum_range(red, s * N, N);
        const double mf = warp_sum_range(red_fv, s * N, N);
        if ((t & 31) == 0) {
            uint32_t q;
            bool ok;
            if (MODE == MODE_RAW && a.raw_list) {
                const uint32_t k = blockIdx.x * P + s;
                ok = k < *a.raw_count;
                q = ok ? a.raw_list[k] : 0;
            } else {
                q = blockIdx.x * P + s;
                ok = q < g.npatch;
            }
            if (ok && slot_mode[s] != 2) {
                PatchStats& st = a.stats[q];
                if (MODE == MODE_RAW) {
                    st.mass = mm;
                    st.mass_fv = mf;
                    if (!a.raw_list) {  // no_compression: nothing was encoded
                        st.comp_bytes = 0;
                        st.nnz = 0;
                        st.zeroed = 0;
                    }
                } else {
                    st.mass_fv = mf;
                    if (slot_mode[s] == 0) st.mass = mm;
                }
            }
        }
    }
}

}  // namespace wg
