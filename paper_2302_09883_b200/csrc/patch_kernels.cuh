// patch_kernels.cuh — the fused per-patch step for single-component schemes
// (FV transport): one kernel runs, for every patch,
//
//   CSR decode -> inverse DWT (rows, then columns)      [idwt_nd, wavelet.hpp:200-223]
//   ghost ring from the neighbours' edge lines           [sync_ghosts, patchgrid.hpp:131-201]
//   upwind FV update                                     [fv_step, solver.hpp:207-231]
//   forward DWT (columns, then rows)                     [dwt_nd, wavelet.hpp:175-198]
//   threshold + warp-scan stream compaction to CSR       [apply_threshold threshold.hpp:51-86,
//                                                         csr_encode codec.hpp:37-60]
//   skip rule (nothing zeroed -> raw patch)              [pipeline.hpp:243-249]
//   inverse DWT of the kept coefficients -> edge lines + trapezoid mass
//                                                        [global_mass, patchgrid.hpp:244-266]
//
// so the uncompressed patch exists only in shared memory and registers.
//
// Work decomposition: a CTA owns P patches; thread (slot, li) owns line li of
// its patch.  In a ROW phase li is a row, in a COLUMN phase a column; each
// thread keeps its whole line (N doubles) in registers and runs the lifting
// there (lifting.cuh).  Phases exchange data through one (N+2)^2 shared
// tile per patch (odd pitch N+2: conflict-free for both row- and
// column-ownership access patterns).
#pragma once

#include "common.cuh"
#include "lifting.cuh"
#include "physics.cuh"
#include "session.cuh"

namespace wg {

constexpr int kMaxLevels = 8;

struct StepArgs {
    const unsigned char* store_in;
    const DirEntry* dir_in;
    EdgeSet ein;
    unsigned char* store_out;
    DirEntry* dir_out;
    EdgeSet eout;
    PatchStats* stats;
    unsigned long long* bump_out;
    uint64_t cap_out;
    uint32_t* raw_list;   // MODE_RAW: patches to store raw (nullptr = all patches)
    uint32_t* raw_count;
    uint32_t raw_capacity;
    unsigned* err;
    double* decode_out;   // MODE_DECODE: grid buffer (true layout) of this shard
    ShardGeom g;
    double smax[4], smin[4], r;                          // transport faces, dt/dx
    double thr[(kMaxLevels + 1) * (kMaxLevels + 1)];     // T[band_i][band_j]
};

enum { MODE_MAIN = 0, MODE_RAW = 1, MODE_DECODE = 2 };

template <int N, int P>
struct Layout {
    static constexpr int TP = N + 2;              // tile pitch (odd)
    static constexpr int TILE = TP * TP;
    static constexpr int NT = ((P * N + 31) / 32) * 32;
    static constexpr size_t smem_bytes() {
        return sizeof(double) * (size_t)(P * TILE + 2 * NT) + sizeof(unsigned long long) * NT;
    }
};

// Inclusive scan of one u64 per thread over the CTA (warp shuffles + one
// shared pass); result written to inc[threadIdx.x].
template <int NT>
__device__ __forceinline__ void cta_inclusive_scan(unsigned long long x, unsigned long long* inc) {
    __shared__ unsigned long long wtot[NT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wtot[w] = x;
    __syncthreads();
    unsigned long long before = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k)
        if (k < w) before += wtot[k];
    inc[threadIdx.x] = x + before;
    __syncthreads();
}

// Deterministic per-slot sum of red[slot*N .. slot*N+N): one warp per slot,
// fixed lane->element assignment and a fixed shuffle tree.
template <int N, int P, int NT>
__device__ __forceinline__ double slot_sum(const double* red, int slot) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int k = lane; k < N; k += 32) s += red[slot * N + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

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
    const uint32_t P1 = g.P1;
    const int ar = (int)(p / P1);
    const uint32_t b = p % P1;
    double* T = tiles + (lane_ok ? ps : 0) * TILE;

    // ---- ROW phase: decode row li, inverse transform along dim 1 ----------
    bool raw_in = false;
    if (valid) {
        const DirEntry e = a.dir_in[p];
        raw_in = (e.flags & DIR_RAW) != 0;
        const unsigned char* base = a.store_in + e.off;
        double* rowp = T + (li + 1) * TP + 1;
        if (raw_in) {
            const double* d = reinterpret_cast<const double*>(base) + (size_t)li * N;
#pragma unroll 8
            for (int j = 0; j < N; ++j) rowp[j] = d[j];
        } else {
            const double* v = reinterpret_cast<const double*>(base);
            const uint32_t* col = reinterpret_cast<const uint32_t*>(base + 8ull * e.nnz);
            const uint32_t* ro = col + e.nnz;
            const uint32_t k0 = ro[li], k1 = ro[li + 1];
#pragma unroll
            for (int j = 0; j < N; ++j) rowp[j] = 0.0;
            for (uint32_t k = k0; k < k1; ++k) rowp[col[k]] = v[k];
            double x[N];
#pragma unroll
            for (int r = 0; r < N; ++r) x[r] = rowp[corner_pos<N, L>(r)];
            idwt_line_reg<N, L>(x);
#pragma unroll
            for (int j = 0; j < N; ++j) rowp[j] = x[j];
        }
        if (MODE != MODE_DECODE) {
            // ghost ring from the neighbours' reconstructed edge lines
            const uint32_t su = row_slot(ar - 1, g), sd = row_slot(ar + 1, g);
            const uint32_t bl = (b + P1 - 1) % P1, br = (b + 1) % P1;
            T[(li + 1) * TP] = a.ein.colhi[((size_t)ar * P1 + bl) * N + li];
            T[(li + 1) * TP + N + 1] = a.ein.collo[((size_t)ar * P1 + br) * N + li];
            T[li + 1] = a.ein.rowhi[((size_t)su * P1 + b) * N + li];
            T[(N + 1) * TP + li + 1] = a.ein.rowlo[((size_t)sd * P1 + b) * N + li];
            if (li == 0) {
                T[0] = a.ein.rowhi[((size_t)su * P1 + bl) * N + N - 2];
                T[N + 1] = a.ein.rowhi[((size_t)su * P1 + br) * N + 1];
                T[(N + 1) * TP] = a.ein.rowlo[((size_t)sd * P1 + bl) * N + N - 2];
                T[(N + 1) * TP + N + 1] = a.ein.rowlo[((size_t)sd * P1 + br) * N + 1];
            }
        }
    }
    __syncthreads();

    // ---- COLUMN phase: inverse transform along dim 0 -> state column li ----
    double v[N];
    const int j = li;
    if (valid) {
        if (raw_in) {
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = T[(i + 1) * TP + j + 1];
        } else {
#pragma unroll
            for (int r = 0; r < N; ++r) v[r] = T[(corner_pos<N, L>(r) + 1) * TP + j + 1];
            idwt_line_reg<N, L>(v);
            if (MODE != MODE_DECODE) {
#pragma unroll
                for (int i = 0; i < N; ++i) T[(i + 1) * TP + j + 1] = v[i];
            }
        }
        if (MODE == MODE_DECODE) {
            double* out = a.decode_out + (size_t)p * TILE;
#pragma unroll
            for (int i = 0; i < N; ++i) out[(i + 1) * TP + j + 1] = v[i];
        }
    }
    if (MODE == MODE_DECODE) return;
    __syncthreads();

    // ---- upwind FV update of column j (solver.hpp:207-231) ----------------
    // directions in the reference order +x, -x, +y, -y (solver.hpp:21-22);
    // x = dim 0 = i.  No FMA (-fmad=false).
    double mfv = 0.0;
    if (valid) {
        double prev = T[j + 1];                  // ghost row 0
        const double below = T[(N + 1) * TP + j + 1];  // ghost row N+1
        const double wj = (j == 0 || j == N - 1) ? 0.5 : 1.0;
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
            const double wi = (i == 0 || i == N - 1) ? 0.5 : 1.0;
            mfv += (wi * wj) * out;
        }
    }
    red_fv[t] = mfv;

    if (MODE == MODE_RAW) {
        // store the scheme output uncompressed (skip rule / no_compression)
        if (valid && li == 0) {
            const uint64_t bytes = round16((uint64_t)N * N * 8);
            const uint64_t off = atomicAdd(a.bump_out, (unsigned long long)bytes);
            if (off + bytes > a.cap_out) {
                atomicOr(a.err, ERR_STORE_OVERFLOW);
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
        if (valid) dwt_line_reg<N, L>(v);
        __syncthreads();  // everyone done reading the state tile
        if (valid) {
#pragma unroll
            for (int r = 0; r < N; ++r) T[(corner_pos<N, L>(r) + 1) * TP + j + 1] = v[r];
        }
        __syncthreads();

        // ---- ROW phase: forward DWT along dim 1, threshold, count ---------
        const int i = li;
        unsigned nz = 0, zr = 0;
        if (valid) {
#pragma unroll
            for (int jj = 0; jj < N; ++jj) v[jj] = T[(i + 1) * TP + jj + 1];
            dwt_line_reg<N, L>(v);
            const int bi = band_of_pos(N, L, i);
            double trow[L + 1];
#pragma unroll
            for (int bj = 0; bj <= L; ++bj) trow[bj] = a.thr[bi * (L + 1) + bj];
#pragma unroll
            for (int r = 0; r < N; ++r) {
                const double x = v[r];
                const bool nzx = x != 0.0;
                const bool kill = fabs(x) < trow[band_of_r<N, L>(r)];
                zr += (nzx && kill) ? 1u : 0u;
                const bool keep = nzx && !kill;
                v[r] = keep ? x : 0.0;  // also maps -0.0 to +0.0 like the CSR round trip
                nz += keep ? 1u : 0u;
            }
        }
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
            // ordered CSR write of row i (ascending corner-layout columns)
            unsigned char* base = a.store_out + slot_off[ps];
            double* vo = reinterpret_cast<double*>(base);
            uint32_t* co = reinterpret_cast<uint32_t*>(base + 8ull * nnz_tot);
            uint32_t* ro = co + nnz_tot;
            uint32_t k = (uint32_t)((inc[t] - slot_base) & 0xffffffffu) - nz;
            if (i == 0) ro[0] = 0;
            ro[i + 1] = k + nz;
#pragma unroll
            for (int pc = 0; pc < N; ++pc) {
                const double x = v[interleaved_of<N, L>(pc)];
                if (x != 0.0) {
                    vo[k] = x;
                    co[k] = (uint32_t)pc;
                    ++k;
                }
            }
            // reconstruction, dim 1 inverse (the decode of the next step)
            idwt_line_reg<N, L>(v);
#pragma unroll
            for (int jj = 0; jj < N; ++jj) T[(i + 1) * TP + jj + 1] = v[jj];
        }
        __syncthreads();
        double m = 0.0;
        if (compressed) {
#pragma unroll
            for (int r = 0; r < N; ++r) v[r] = T[(corner_pos<N, L>(r) + 1) * TP + j + 1];
            idwt_line_reg<N, L>(v);
            const double wj = (j == 0 || j == N - 1) ? 0.5 : 1.0;
#pragma unroll
            for (int ii = 0; ii < N; ++ii) {
                const double wi = (ii == 0 || ii == N - 1) ? 0.5 : 1.0;
                m += (wi * wj) * v[ii];
            }
        }
        red[t] = m;
    }

    // ---- edge lines of the new state (ghost source of the next step) -----
    const bool write_edges = valid && slot_mode[ps] == (MODE == MODE_RAW ? 1 : 0);
    if (write_edges) {
        const size_t own = ((size_t)(ar + 1) * P1 + b) * N;
        a.eout.rowlo[own + j] = v[1];
        a.eout.rowhi[own + j] = v[N - 2];
        const size_t oc = ((size_t)ar * P1 + b) * N;
        if (j == 1) {
#pragma unroll
            for (int i = 0; i < N; ++i) a.eout.collo[oc + i] = v[i];
        }
        if (j == N - 2) {
#pragma unroll
            for (int i = 0; i < N; ++i) a.eout.colhi[oc + i] = v[i];
        }
    }
    __syncthreads();
    // ---- per-patch trapezoid masses (deterministic) ----------------------
    const int warp = t >> 5;
    for (int s = warp; s < P; s += NT / 32) {
        const double mm = slot_sum<N, P, NT>(red, s);
        const double mf = slot_sum<N, P, NT>(red_fv, s);
        if ((t & 31) == 0) {
            uint32_t ps_patch;
            bool ok;
            if (MODE == MODE_RAW && a.raw_list) {
                const uint32_t k = blockIdx.x * P + s;
                ok = k < *a.raw_count;
                ps_patch = ok ? a.raw_list[k] : 0;
            } else {
                ps_patch = blockIdx.x * P + s;
                ok = ps_patch < g.npatch;
            }
            if (ok && slot_mode[s] != 2) {
                PatchStats& st = a.stats[ps_patch];
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
