// patch_phases.cuh — the phases of the per-patch compression cycle as device
// helpers shared by the transport and D2Q9 kernels.
//
// Ownership model: a "slot" is one (patch, component) tile of (N+2)^2
// doubles in shared memory (odd pitch N+2: conflict-free for both the row-
// and the column-ownership access pattern).  Thread li of a slot owns row li
// in a ROW phase and column li in a COLUMN phase and keeps that whole line
// in registers (double v[N]) while lifting (lifting.cuh).
#pragma once

#include "common.cuh"
#include "lifting.cuh"
#include "physics.cuh"
#include "session.cuh"

namespace wg {

constexpr int kMaxLevels = 8;
constexpr int kMaxN = 65;  // largest patch side of the device session

// ---- phase clocks ---------------------------------------------------------
// Thread 0 of every CTA adds the cycles since its previous mark (the wall time
// of the phase that just ended at a barrier) to a.phase[k] (a 32-entry device
// buffer of the session): the per-phase split of a fused step behind
// RunSummary's dwt / threshold / codec seconds (pipeline.hpp:52-63) and
// tools/phase_profile.py.  One clock read and one reduction per mark.
__device__ __forceinline__ unsigned long long& phase_last() {
    __shared__ unsigned long long last;
    return last;
}
__device__ __forceinline__ void phase_mark(unsigned long long* buf, int k) {
    if (threadIdx.x == 0) {
        const unsigned long long t = clock64();
        if (k >= 0 && buf) atomicAdd(&buf[k], t - phase_last());
        phase_last() = t;
    }
}
#define WG_PHASE_MARK(k) ::wg::phase_mark(a.phase, k)

// ---- optional device bounds checks (debug builds only: -DWG_BOUNDS_CHECK) ---
#ifdef WG_BOUNDS_CHECK
#define WG_CHECK(cond, code)                                                                   \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("WG_CHECK %d failed: block %d thread %d (%s:%d)\n", (code), blockIdx.x,     \
                   threadIdx.x, __FILE__, __LINE__);                                           \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define WG_CHECK(cond, code) ((void)0)
#endif

// Per-CTA partial sums of the step metrics (fixed order inside the CTA).
struct StepPartial {
    unsigned long long comp_bytes, nnz, zeroed;
    double mass, mass_fv;
    double l2;  // transport: sum of squared errors vs exact_transport (l2_error, solver.hpp:293-305)
};

struct StepArgs {
    const unsigned char* store_in;
    const DirEntry* dir_in;
    EdgeSet ein;
    unsigned char* store_out;
    DirEntry* dir_out;
    EdgeSet eout;
    unsigned long long* bump_out;
    unsigned long long* bump_next;  // pool written by the next step: reset by the last CTA
    uint64_t cap_out;
    uint64_t edge_row_elems, edge_col_elems;  // sizes of the edge line arrays (bounds checks)
    uint64_t chunk;                 // per-CTA sub-allocation chunk of the output pool (bytes)
    unsigned* err;
    double* decode_out;   // MODE_DECODE: grid buffer (true layout) of this shard
    double* scratch;      // D2Q9: per-CTA L2-resident staging of 9 N*N fields
    StepPartial* partials;  // [gridDim.x]
    unsigned* done;         // CTA completion counter (last CTA reduces the partials)
    wg_metrics_row* row_out;  // this step's MetricsRow (pipeline.hpp:260-274)
    double* mass_fv_out;      // this step's scheme-output mass (strict mode)
    ShardGeom g;
    int compress;             // 0: RunConfig::no_compression
    int thr_any;              // 0: c == 0 or levels == 0 (nothing can be zeroed)
    uint64_t step;
    double time;
    uint64_t dense_bytes;     // CompressedPatch::dense_bytes summed over the shard
    double smax[4], smin[4], r;                          // transport faces, dt/dx
    double omega;                                        // D2Q9: 1/tau
    double ic_u0, ic_kappa, ic_delta, ic_inv;            // MODE_INIT: shear layer, 1/(nx-1)
    uint64_t ic_period;                                  // MODE_INIT: nx-1 (tiled grids repeat)
    // SWE: the state-dependent time step lives on the device (cfl_dt,
    // solver.hpp:235-258; pipeline.hpp:194-196).  Step k reads the max wave
    // speed of its input state from swe_vmax[k & 1] (all-reduced with MAX
    // across shards by the host between steps when world > 1) and
    // accumulates that of its output state into swe_vmax[(k + 1) & 1].
    double* swe_td;                  // [t, dt of the last step] (nullptr: host dt)
    unsigned long long* swe_vmax;    // [2] max wave speed, bits of a non-negative double
    unsigned long long* swe_steps;   // steps completed on the device
    double t_end, cfl_dx, dx, gravity;
    unsigned long long* phase;       // per-phase cycle sums of thread 0 [32] (phase_mark)
    double* lz_dense;                // Codec::lz: thresholded coefficient arrays [npatch*m][n*n] (else null)
    // transport l2_error diagnostic every step (pipeline.hpp:275-276)
    int l2_on;
    uint64_t l2_nx;
    double l2_scale, l2_dx, l2_alpha, l2_beta;          // area / nx^2, dx, speeds
    double thr[(kMaxLevels + 1) * (kMaxLevels + 1)];     // T[band_i][band_j]
    // trapezoid functional of the inverse transform per corner-layout
    // position (global_mass weights pulled through idwt_line): the mass of a
    // reconstructed block is sum_rc mass_a[r] mass_a[c] C[r][c]
    double mass_a[kMaxN];
    // D2Q9 chunked launches (the streamed first step from a host initial
    // state, chunked decode): this launch handles patches [p_begin, p_end);
    // raw_in (non-null) holds their input in the grid-buffer layout
    // ([patch][m][(n+2)^2], patches from p_begin) instead of the store;
    // decode_out is indexed from p_begin.  The step's partial sums accumulate
    // over the launches: chunk_first starts them, chunk_last reduces them.
    const double* raw_in;
    uint32_t p_begin, p_end;
    int chunk_first, chunk_last;
    // SWE: patches handed out dynamically (work: the launch's patch counter,
    // reset by the last CTA) and the masses kept per patch ([npatch][2]:
    // reconstruction, scheme output), summed by the last CTA in patch order
    // — the step's masses do not depend on which CTA took which patch
    unsigned* work;
    double* patch_mass;
};

// MODE_STEP_LZ: a step that also stages the thresholded coefficient arrays
// for the Codec::lz sizes (a separate instantiation: no cost to MODE_STEP)
enum { MODE_STEP = 0, MODE_INIT = 1, MODE_DECODE = 2, MODE_STEP_LZ = 3 };

struct PatchPos {
    int ar;       // local patch row
    uint32_t b;   // patch column
    uint32_t bl, br;
    uint32_t su, sd;  // edge row slots of the rows above / below
};

__device__ __forceinline__ PatchPos patch_pos(uint32_t p, const ShardGeom& g) {
    PatchPos pp;
    pp.ar = (int)(p / g.P1);
    pp.b = p % g.P1;
    pp.bl = (pp.b + g.P1 - 1) % g.P1;
    pp.br = (pp.b + 1) % g.P1;
    pp.su = row_slot(pp.ar - 1, g);
    pp.sd = row_slot(pp.ar + 1, g);
    return pp;
}

// Index of an edge line element: line arrays are [slot][P1][me][N].
__device__ __forceinline__ size_t edge_ix(uint32_t slot, uint32_t b, uint32_t q, const ShardGeom& g,
                                          int N) {
    return (((size_t)slot * g.P1 + b) * g.me + q) * (size_t)N;
}

// Edge-line stores of the row edges: the halo lines (owned slot 1 of rowlo,
// owned slot R of rowhi) also go straight into the ring neighbours' halo
// slots when peers are attached (EdgeSet::peer_lo / peer_hi), so the step
// kernel itself performs the halo exchange over NVLink.
__device__ __forceinline__ void put_rowlo(const EdgeSet& e, const ShardGeom& g, uint32_t slot, uint32_t b, uint32_t q,
                                          int N, int j, double x) {
    e.rowlo[edge_ix(slot, b, q, g, N) + j] = x;
    if (slot == 1 && e.peer_lo) e.peer_lo[edge_ix(0, b, q, g, N) + j] = x;
}
__device__ __forceinline__ void put_rowhi(const EdgeSet& e, const ShardGeom& g, uint32_t slot, uint32_t b, uint32_t q,
                                          int N, int j, double x) {
    e.rowhi[edge_ix(slot, b, q, g, N) + j] = x;
    if (slot == g.R && e.peer_hi) e.peer_hi[edge_ix(0, b, q, g, N) + j] = x;
}

// ROW phase of the decode: row li of component (p, q) from the store into
// the tile (CSR scatter or raw copy), inverse transform along dim 1
// (idwt_nd, wavelet.hpp:200-223 does the last dimension first).  Returns
// whether the stored block is raw.
template <int N, int L>
__device__ __forceinline__ bool decode_row(double* T, int li, const DirEntry e,
                                           const unsigned char* store) {
    constexpr int TP = N + 2;
    const bool raw = (e.flags & DIR_RAW) != 0;
    const unsigned char* base = store + e.off;
    double* rowp = T + (li + 1) * TP + 1;
    if (e.flags & DIR_DEAD) {  // overflowed block (error already raised): zeros, never garbage
#pragma unroll
        for (int j = 0; j < N; ++j) rowp[j] = 0.0;
        return true;
    }
    if (e.flags & DIR_CONST) {  // constant raw block: the value itself is in the entry
        const double c = __longlong_as_double((long long)e.off);
#pragma unroll
        for (int j = 0; j < N; ++j) rowp[j] = c;
        return true;
    }
    if (raw) {
        // a raw block fills the whole tile interior; thread li copies COLUMN
        // li so that consecutive threads read consecutive addresses
        const double* d = reinterpret_cast<const double*>(base) + li;
#pragma unroll 8
        for (int i = 0; i < N; ++i) T[(i + 1) * TP + li + 1] = d[(size_t)i * N];
    } else {
        const double* v = reinterpret_cast<const double*>(base);
        const uint32_t* col = reinterpret_cast<const uint32_t*>(base + 8ull * e.nnz);
        const uint32_t* ro = col + e.nnz;
        const uint32_t k0 = ro[li], k1 = ro[li + 1];
        WG_CHECK(k0 <= k1 && k1 <= e.nnz && e.nnz <= (uint32_t)(N * N), 1);
#pragma unroll
        for (int j = 0; j < N; ++j) rowp[j] = 0.0;
        // an empty row inverse-transforms to +0.0 everywhere (every lifting
        // step maps zeros to +0.0): nothing more to do.  Well-compressed
        // patches keep their few coefficients in the coarse rows, so whole
        // warps of detail rows take this exit.
        if (k0 == k1) return false;
        for (uint32_t k = k0; k < k1; ++k) {
            WG_CHECK(col[k] < (uint32_t)N, 2);
            rowp[col[k]] = v[k];
        }
        double x[N];
#pragma unroll
        for (int r = 0; r < N; ++r) x[r] = rowp[corner_pos<N, L>(r)];
        idwt_line_reg<N, L>(x);
#pragma unroll
        for (int j = 0; j < N; ++j) rowp[j] = x[j];
    }
    return raw;
}

// Ghost ring of the tile from the neighbours' reconstructed edge lines
// (sync_ghosts, patchgrid.hpp:131-201: low ghost <- neighbour logical n-2,
// high ghost <- neighbour logical 1; corners from the diagonal neighbours).
template <int N>
__device__ __forceinline__ void fill_ghosts(double* T, int li, const EdgeSet& e, const PatchPos& pp,
                                            uint32_t q, const ShardGeom& g) {
    constexpr int TP = N + 2;
    const uint32_t own = row_slot(pp.ar, g);  // == ar + 1
    (void)own;
    T[(li + 1) * TP] = e.colhi[edge_ix(pp.ar, pp.bl, q, g, N) + li];
    T[(li + 1) * TP + N + 1] = e.collo[edge_ix(pp.ar, pp.br, q, g, N) + li];
    T[li + 1] = e.rowhi[edge_ix(pp.su, pp.b, q, g, N) + li];
    T[(N + 1) * TP + li + 1] = e.rowlo[edge_ix(pp.sd, pp.b, q, g, N) + li];
    if (li == 0) {
        T[0] = e.rowhi[edge_ix(pp.su, pp.bl, q, g, N) + N - 2];
        T[N + 1] = e.rowhi[edge_ix(pp.su, pp.br, q, g, N) + 1];
        T[(N + 1) * TP] = e.rowlo[edge_ix(pp.sd, pp.bl, q, g, N) + N - 2];
        T[(N + 1) * TP + N + 1] = e.rowlo[edge_ix(pp.sd, pp.br, q, g, N) + 1];
    }
}

// COLUMN phase of the decode: column j -> registers (natural order), inverse
// transform along dim 0 unless raw.
template <int N, int L>
__device__ __forceinline__ void decode_col(const double* T, int j, bool raw, double (&v)[N]) {
    constexpr int TP = N + 2;
    if (raw) {
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = T[(i + 1) * TP + j + 1];
    } else {
#pragma unroll
        for (int r = 0; r < N; ++r) v[r] = T[(corner_pos<N, L>(r) + 1) * TP + j + 1];
        idwt_line_reg<N, L>(v);
    }
}

template <int N>
__device__ __forceinline__ void store_col(double* T, int j, const double (&v)[N]) {
    constexpr int TP = N + 2;
#pragma unroll
    for (int i = 0; i < N; ++i) T[(i + 1) * TP + j + 1] = v[i];
}

// Forward transform along dim 0 of a register column, stored into the tile
// in corner layout.
template <int N, int L>
__device__ __forceinline__ void fwd_col_to_tile(double* T, int j, double (&v)[N]) {
    constexpr int TP = N + 2;
    dwt_line_reg<N, L>(v);
#pragma unroll
    for (int r = 0; r < N; ++r) T[(corner_pos<N, L>(r) + 1) * TP + j + 1] = v[r];
}

// ROW phase of the compression: forward transform along dim 1 of row i,
// threshold (threshold.hpp:51-86: samples untouched, strict <, v != 0),
// count kept and zeroed coefficients.  -0.0 becomes +0.0 like the CSR
// round trip of pipeline.hpp:234-237.
// dense_row (Codec::lz, else null): where row i of the block's coefficient
// array goes, in corner order, as apply_threshold leaves it
// (threshold.hpp:78-82: a killed value becomes +0.0, every other value —
// -0.0 included — is kept), for the LZ coder.  The kernels pass the tile's
// own row i (read into v above, free until the reconstruction) and copy the
// tiles out coalesced with tiles_to_dense.
template <int N, int L>
__device__ __forceinline__ void fwd_row_threshold(const double* T, int i, const double* thr,
                                                  double (&v)[N], unsigned& nz, unsigned& zr,
                                                  double* dense_row = nullptr) {
    constexpr int TP = N + 2;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v[jj] = T[(i + 1) * TP + jj + 1];
    dwt_line_reg<N, L>(v);
    const int bi = band_of_pos(N, L, i);
    double trow[L + 1];
#pragma unroll
    for (int bj = 0; bj <= L; ++bj) trow[bj] = thr[bi * (L + 1) + bj];
    nz = 0;
    zr = 0;
    if (dense_row) {  // Codec::lz only: one branch per row on the default path
#pragma unroll
        for (int r = 0; r < N; ++r) {
            const double x = v[r];
            dense_row[corner_pos<N, L>(r)] = (x != 0.0 && fabs(x) < trow[band_of_r<N, L>(r)]) ? 0.0 : x;
        }
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
        const double x = v[r];
        const bool nzx = x != 0.0;
        const bool kill = fabs(x) < trow[band_of_r<N, L>(r)];
        zr += (nzx && kill) ? 1u : 0u;
        const bool keep = nzx && !kill;
        v[r] = keep ? x : 0.0;
        nz += keep ? 1u : 0u;
    }
}

// Codec::lz staging: the interiors of `count` consecutive tiles (the
// coefficient arrays fwd_row_threshold left there) to dense[count][N*N],
// coalesced.  Between the row phase's scan barrier and the next barrier.
template <int N, int NT>
__device__ __forceinline__ void tiles_to_dense(const double* tiles, int tile_stride, int count, double* dense) {
    constexpr int TP = N + 2, NN = N * N;
    for (int k = threadIdx.x; k < count * NN; k += NT) {
        const int s = k / NN, r = k - s * NN, i = r / N, j = r - i * N;
        dense[k] = tiles[s * tile_stride + (i + 1) * TP + j + 1];
    }
}

// Ordered CSR write of row i (csr_encode, codec.hpp:37-60: row-major,
// ascending columns, u32 offsets from 0) at entry offset k.
template <int N, int L>
__device__ __forceinline__ void write_csr_row(unsigned char* base, uint32_t nnz_tot, int i, uint32_t k,
                                              unsigned nz, const double (&v)[N]) {
    double* vo = reinterpret_cast<double*>(base);
    uint32_t* co = reinterpret_cast<uint32_t*>(base + 8ull * nnz_tot);
    uint32_t* ro = co + nnz_tot;
    if (i == 0) ro[0] = 0;
    ro[i + 1] = k + nz;
    if (nz == 0) return;  // empty row (most detail rows of a well-compressed patch)
#pragma unroll
    for (int pc = 0; pc < N; ++pc) {
        const double x = v[interleaved_of<N, L>(pc)];
        if (x != 0.0) {
            vo[k] = x;
            co[k] = (uint32_t)pc;
            ++k;
        }
    }
}

// Inverse transform of a thresholded register row, stored into the tile.
template <int N, int L>
__device__ __forceinline__ void inv_row_to_tile(double* T, int i, double (&v)[N], unsigned nz = ~0u) {
    constexpr int TP = N + 2;
    if (nz == 0) {  // all coefficients zero: the inverse is +0.0 everywhere
#pragma unroll
        for (int jj = 0; jj < N; ++jj) T[(i + 1) * TP + jj + 1] = 0.0;
        return;
    }
    idwt_line_reg<N, L>(v);
#pragma unroll
    for (int jj = 0; jj < N; ++jj) T[(i + 1) * TP + jj + 1] = v[jj];
}

// Edge lines of the new state from a register column j (natural order).
template <int N>
__device__ __forceinline__ void write_edges(const EdgeSet& e, const PatchPos& pp, uint32_t q,
                                            const ShardGeom& g, int j, const double (&v)[N]) {
    put_rowlo(e, g, (uint32_t)(pp.ar + 1), pp.b, q, N, j, v[1]);
    put_rowhi(e, g, (uint32_t)(pp.ar + 1), pp.b, q, N, j, v[N - 2]);
    const size_t oc = edge_ix((uint32_t)pp.ar, pp.b, q, g, N);
    if (j == 1) {
#pragma unroll
        for (int i = 0; i < N; ++i) e.collo[oc + i] = v[i];
    }
    if (j == N - 2) {
#pragma unroll
        for (int i = 0; i < N; ++i) e.colhi[oc + i] = v[i];
    }
}

// D2Q9 variants: only the populations that cross a side (session.cuh).
template <int N>
__device__ __forceinline__ void fill_ghosts_lbm(double* T, int li, const EdgeSet& e, const PatchPos& pp, int q,
                                                const ShardGeom& g) {
    constexpr int TP = N + 2;
    const int cxq = lbm_cx(q), cyq = lbm_cy(q);
    WG_CHECK(pp.su <= g.R + 1 && pp.sd <= g.R + 1 && pp.b < g.P1 && pp.bl < g.P1 && pp.br < g.P1 && pp.ar >= 0 &&
                 (uint32_t)pp.ar < g.R, 3);
    if (cxq == 1) T[li + 1] = e.rowhi[edge_ix(pp.su, pp.b, lbm_slot_rowhi(q), g, N) + li];
    if (cxq == -1) T[(N + 1) * TP + li + 1] = e.rowlo[edge_ix(pp.sd, pp.b, lbm_slot_rowlo(q), g, N) + li];
    if (cyq == 1) T[(li + 1) * TP] = e.colhi[edge_ix(pp.ar, pp.bl, lbm_slot_colhi(q), g, N) + li];
    if (cyq == -1) T[(li + 1) * TP + N + 1] = e.collo[edge_ix(pp.ar, pp.br, lbm_slot_collo(q), g, N) + li];
    if (li == 0) {
        if (q == 5) T[0] = e.rowhi[edge_ix(pp.su, pp.bl, lbm_slot_rowhi(5), g, N) + N - 2];
        if (q == 7) T[N + 1] = e.rowhi[edge_ix(pp.su, pp.br, lbm_slot_rowhi(7), g, N) + 1];
        if (q == 8) T[(N + 1) * TP] = e.rowlo[edge_ix(pp.sd, pp.bl, lbm_slot_rowlo(8), g, N) + N - 2];
        if (q == 6) T[(N + 1) * TP + N + 1] = e.rowlo[edge_ix(pp.sd, pp.br, lbm_slot_rowlo(6), g, N) + 1];
    }
}

template <int N>
__device__ __forceinline__ void write_edges_lbm(const EdgeSet& e, const PatchPos& pp, int q, const ShardGeom& g,
                                                int j, const double (&v)[N]) {
    const int cxq = lbm_cx(q), cyq = lbm_cy(q);
    if (cxq == -1) put_rowlo(e, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowlo(q), N, j, v[1]);
    if (cxq == 1) put_rowhi(e, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowhi(q), N, j, v[N - 2]);
    if (cyq == -1 && j == 1) {
        double* d = e.collo + edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_collo(q), g, N);
#pragma unroll
        for (int i = 0; i < N; ++i) d[i] = v[i];
    }
    if (cyq == 1 && j == N - 2) {
        double* d = e.colhi + edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_colhi(q), g, N);
#pragma unroll
        for (int i = 0; i < N; ++i) d[i] = v[i];
    }
}

// D2Q9 edge lines of component q from the reconstructed TILE (logical cells
// at (i+1, j+1)); thread li writes element li of every line it owns, so the
// column lines are written in parallel and no register line stays live.
template <int N>
__device__ __forceinline__ void write_edges_lbm_tile(const EdgeSet& e, const PatchPos& pp, int q, const ShardGeom& g,
                                                     int li, const double* T) {
    constexpr int TP = N + 2;
    const int cxq = lbm_cx(q), cyq = lbm_cy(q);
    if (cxq == -1) put_rowlo(e, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowlo(q), N, li, T[2 * TP + li + 1]);
    if (cxq == 1) put_rowhi(e, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowhi(q), N, li, T[(N - 1) * TP + li + 1]);
    if (cyq == -1) e.collo[edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_collo(q), g, N) + li] = T[(li + 1) * TP + 2];
    if (cyq == 1) e.colhi[edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_colhi(q), g, N) + li] = T[(li + 1) * TP + N - 1];
}

// col_mass of tile column j (same weights and association).
template <int N>
__device__ __forceinline__ double tile_col_mass(const double* T, int j) {
    constexpr int TP = N + 2;
    const double wj = (j == 0 || j == N - 1) ? 0.5 : 1.0;
    double m[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double wi = (i == 0 || i == N - 1) ? 0.5 : 1.0;
        m[i & 3] += (wi * wj) * T[(i + 1) * TP + j + 1];
    }
    return (m[0] + m[1]) + (m[2] + m[3]);
}

// Squared error of tile column j against exact_transport (solver.hpp:264-287)
// at the step's time, over the global points this patch owns (its last row
// and column belong to the next patch, except at the global boundary).
__device__ __forceinline__ double wrap_unit_d(double x) {
    x = fmod(x, 1.0);
    return x < 0.0 ? x + 1.0 : x;
}

template <int N>
__device__ __forceinline__ double col_l2(const StepArgs& a, const PatchPos& pp, int j, const double (&v)[N]) {
    const uint64_t gi0 = (uint64_t)(a.g.row0 + pp.ar) * (N - 1), gj = (uint64_t)pp.b * (N - 1) + j;
    if (j == N - 1 && gj != a.l2_nx - 1) return 0.0;
    double py = wrap_unit_d((double)gj * a.l2_dx - a.l2_beta * a.time) - 0.5;
    if (py < -0.5) py += 1.0;
    if (py >= 0.5) py -= 1.0;
    double s = 0.0;
#pragma unroll 5
    for (int i = 0; i < N; ++i) {
        const uint64_t gi = gi0 + i;
        if (i == N - 1 && gi != a.l2_nx - 1) continue;
        double px = wrap_unit_d((double)gi * a.l2_dx - a.l2_alpha * a.time) - 0.5;
        if (px < -0.5) px += 1.0;
        if (px >= 0.5) px -= 1.0;
        const double d = v[i] - (1.0 + exp(-30.0 * (px * px + py * py)));
        s += d * d;
    }
    return s;
}

// Trapezoid-weighted column sum (global_mass weights, patchgrid.hpp:244-266),
// with four interleaved partial sums (fixed association: deterministic; the
// mass is a tolerance-checked diagnostic).
template <int N>
__device__ __forceinline__ double col_mass(int j, const double (&v)[N]) {
    const double wj = (j == 0 || j == N - 1) ? 0.5 : 1.0;
    double m[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double wi = (i == 0 || i == N - 1) ? 0.5 : 1.0;
        m[i & 3] += (wi * wj) * v[i];
    }
    return (m[0] + m[1]) + (m[2] + m[3]);
}

// Inclusive scan of one u64 per thread over the CTA (warp shuffles + one
// shared pass); result written to inc[threadIdx.x].  Contains barriers.
template <int NT>
__device__ __forceinline__ void cta_inclusive_scan(unsigned long long x, unsigned long long* inc,
                                                   bool after_barrier = false) {
    __shared__ unsigned long long wtot[NT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    // wtot may still be read by a previous scan (after_barrier: the caller
    // knows a CTA barrier separates the two)
    if (!after_barrier) __syncthreads();
    if (lane == 31) wtot[w] = x;
    __syncthreads();
    unsigned long long before = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k)
        if (k < w) before += wtot[k];
    inc[threadIdx.x] = x + before;
    __syncthreads();
}

// Deterministic sum of red[base .. base+n): fixed lane assignment and a
// fixed shuffle tree (called by a whole warp).
__device__ __forceinline__ double warp_sum_range(const double* red, int base, int n) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int k = lane; k < n; k += 32) s += red[base + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// Sum of every thread's partial over the CTA with a fixed association
// (xor-shuffle trees inside warps, warps in order): result valid in thread 0.
template <int NT>
__device__ __forceinline__ StepPartial cta_reduce_partial(StepPartial x) {
    __shared__ StepPartial wpart[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        x.comp_bytes += __shfl_xor_sync(0xffffffffu, x.comp_bytes, o);
        x.nnz += __shfl_xor_sync(0xffffffffu, x.nnz, o);
        x.zeroed += __shfl_xor_sync(0xffffffffu, x.zeroed, o);
        x.mass += __shfl_xor_sync(0xffffffffu, x.mass, o);
        x.mass_fv += __shfl_xor_sync(0xffffffffu, x.mass_fv, o);
        x.l2 += __shfl_xor_sync(0xffffffffu, x.l2, o);
    }
    if ((threadIdx.x & 31) == 0) wpart[threadIdx.x >> 5] = x;
    __syncthreads();
    StepPartial r{0, 0, 0, 0.0, 0.0, 0.0};
    if (threadIdx.x == 0) {
        for (int w = 0; w < NT / 32; ++w) {
            r.comp_bytes += wpart[w].comp_bytes;
            r.nnz += wpart[w].nnz;
            r.zeroed += wpart[w].zeroed;
            r.mass += wpart[w].mass;
            r.mass_fv += wpart[w].mass_fv;
            r.l2 += wpart[w].l2;
        }
    }
    return r;
}

// Per-CTA sub-allocator of the output pool: the CTA grabs `a.chunk` bytes
// with one global atomic and carves its blocks out of them, so most groups
// allocate without a global round trip.  Blocks larger than chunk/8 get an
// exact allocation, so the unused chunk tails stay below 1/8 of the bytes
// served from chunks plus one chunk per CTA.  Returns ~0 (and raises the
// error bit) on overflow.
struct ChunkState {
    unsigned long long cur, end;
};

__device__ __forceinline__ unsigned long long chunk_alloc(const StepArgs& a, ChunkState& cs,
                                                          unsigned long long bytes) {
    if (bytes == 0) return cs.cur;
    if (bytes * 8 > a.chunk) {
        const unsigned long long off = atomicAdd(a.bump_out, bytes);
        if (off + bytes > a.cap_out) {
            atomicOr(a.err, ERR_STORE_OVERFLOW);
            return ~0ull;
        }
        return off;
    }
    if (cs.cur + bytes > cs.end) {
        const unsigned long long c = atomicAdd(a.bump_out, (unsigned long long)a.chunk);
        if (c + a.chunk > a.cap_out) {
            atomicOr(a.err, ERR_STORE_OVERFLOW);
            cs.cur = cs.end = 0;
            return ~0ull;
        }
        cs.cur = c;
        cs.end = c + a.chunk;
    }
    const unsigned long long off = cs.cur;
    cs.cur += bytes;
    WG_CHECK(off + bytes <= a.cap_out, 5);
    return off;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Prefetch [p, p + bytes) into L2, lines split over `nthreads` threads.
__device__ __forceinline__ void prefetch_range(const unsigned char* p, unsigned long long bytes, int tid,
                                               int nthreads) {
    for (unsigned long long o = (unsigned long long)tid * 128; o < bytes; o += (unsigned long long)nthreads * 128)
        prefetch_l2(p + o);
}

// L2 prefetch of everything the decode of patch p will read: its stored
// block and the neighbours' edge lines (the ghost-ring sources).
template <int N>
__device__ __forceinline__ void prefetch_block(const StepArgs& a, const DirEntry e, int tid, int nthreads) {
    const unsigned long long bytes = (e.flags & DIR_RAW) ? (unsigned long long)N * N * 8
                                                          : 12ull * e.nnz + 4ull * (N + 1);
    if (!(e.flags & (DIR_DEAD | DIR_CONST))) prefetch_range(a.store_in + e.off, bytes, tid, nthreads);
}

// L2 prefetch of the neighbours' edge lines (all stored components) that
// the ghost ring of patch p will read.
template <int N>
__device__ __forceinline__ void prefetch_edges(const StepArgs& a, uint32_t p, int tid, int nthreads) {
    const PatchPos pp = patch_pos(p, a.g);
    const int lines = (int)((a.g.me * N * 8 + 127) / 128);
    const double* srcs[7] = {a.ein.colhi + edge_ix(pp.ar, pp.bl, 0, a.g, N),
                             a.ein.collo + edge_ix(pp.ar, pp.br, 0, a.g, N),
                             a.ein.rowhi + edge_ix(pp.su, pp.b, 0, a.g, N),
                             a.ein.rowlo + edge_ix(pp.sd, pp.b, 0, a.g, N),
                             a.ein.rowhi + edge_ix(pp.su, pp.bl, 0, a.g, N),
                             a.ein.rowlo + edge_ix(pp.sd, pp.br, 0, a.g, N),
                             a.ein.rowhi + edge_ix(pp.su, pp.br, 0, a.g, N)};
    for (int k = tid; k < 7 * lines; k += nthreads)
        prefetch_l2(reinterpret_cast<const unsigned char*>(srcs[k / lines]) + (k % lines) * 128);
}

// L2 prefetch of everything the decode of patch p (single component) reads.
template <int N>
__device__ __forceinline__ void prefetch_patch(const StepArgs& a, uint32_t p, const DirEntry e, uint32_t q,
                                               int tid, int nthreads) {
    (void)q;
    prefetch_block<N>(a, e, tid, nthreads);
    prefetch_edges<N>(a, p, tid, nthreads);
}

// The device clock of an SWE step, read by every CTA at its start (the
// inputs are written only by the previous launch, so the values are uniform).
struct SweClock {
    unsigned long long k;  // steps done before this one
    double t, dt;
    bool live;             // t < t_end (run() loop condition, pipeline.hpp:194)
};

__device__ __forceinline__ SweClock swe_clock(const StepArgs& a) {
    SweClock c;
    c.k = *a.swe_steps;
    c.t = a.swe_td[0];
    c.live = c.t < a.t_end - 1e-15;
    const double vmax = __longlong_as_double((long long)a.swe_vmax[c.k & 1]);
    if (c.live && !(vmax > 0.0) && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.err, ERR_ZERO_SPEED);
    double dt = a.cfl_dx / vmax;        // cfl_dt: cfg.cfl * cfg.dx() / vmax (solver.hpp:257)
    const double rest = a.t_end - c.t;
    c.dt = (rest < dt) ? rest : dt;     // std::min(dt, t_end - t) (pipeline.hpp:196)
    return c;
}

// End of a step, called by every CTA with its partial sums: the last CTA to
// finish reduces all partials in a fixed order (deterministic), writes the
// step's MetricsRow and resets the counter and the next pool's allocator.
// SWE (clk != nullptr): every CTA max-accumulates the wave speed of its
// patches of the new state; the last CTA advances the clock.
__device__ __forceinline__ void finalize_step(const StepArgs& a, const StepPartial& mine, double cta_vmax = 0.0,
                                              const SweClock* clk = nullptr) {
    __shared__ int am_last;
    if (threadIdx.x == 0) {
        a.partials[blockIdx.x] = mine;
        if (clk) atomicMax(a.swe_vmax + ((clk->k + 1) & 1), (unsigned long long)__double_as_longlong(cta_vmax));
        // (cumulative over the CTA's stores, the kernels end their patch
        // loops with a barrier): peer halo lines reach the neighbours before
        // the step is complete
        if (a.eout.peer_lo) __threadfence_system();
        else __threadfence();
        const unsigned prev = atomicAdd(a.done, 1u);
        am_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!am_last || threadIdx.x >= 32) return;
    __threadfence();
    if (!a.chunk_last) {  // a chunk of a step: partials stay for the next launch
        if (threadIdx.x == 0) *a.done = 0;
        return;
    }
    const int lane = threadIdx.x;
    unsigned long long cb = 0, nz = 0, zr = 0;
    double m = 0.0, mf = 0.0, l2 = 0.0;
    for (unsigned c = lane; c < gridDim.x; c += 32) {
        const StepPartial* pp = a.partials + c;
        cb += __ldcg(&pp->comp_bytes);
        nz += __ldcg(&pp->nnz);
        zr += __ldcg(&pp->zeroed);
        m += __ldcg(&pp->mass);
        mf += __ldcg(&pp->mass_fv);
        l2 += __ldcg(&pp->l2);
    }
    if (a.patch_mass) {  // per-patch masses, fixed order (dynamic patch scheduling)
        m = 0.0;
        mf = 0.0;
        for (unsigned p = lane; p < a.g.npatch; p += 32) {
            m += __ldcg(a.patch_mass + 2 * (size_t)p);
            mf += __ldcg(a.patch_mass + 2 * (size_t)p + 1);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cb += __shfl_xor_sync(0xffffffffu, cb, o);
        nz += __shfl_xor_sync(0xffffffffu, nz, o);
        zr += __shfl_xor_sync(0xffffffffu, zr, o);
        m += __shfl_xor_sync(0xffffffffu, m, o);
        mf += __shfl_xor_sync(0xffffffffu, mf, o);
        l2 += __shfl_xor_sync(0xffffffffu, l2, o);
    }
    if (lane == 0) {
        wg_metrics_row r;
        wg_metrics_row* row_out = a.row_out;
        double* mfv_out = a.mass_fv_out;
        r.step = a.step;
        r.time = a.time;
        if (clk) {  // device-side time stepping (SWE)
            row_out += clk->k;
            mfv_out += clk->k;
            r.step = clk->k + 1;
            r.time = clk->t + clk->dt;  // t += dt (pipeline.hpp:210)
            a.swe_td[0] = r.time;
            a.swe_td[1] = clk->dt;
            a.swe_vmax[clk->k & 1] = 0ull;  // read by every CTA already; accumulates step k + 1's output
            *a.swe_steps = clk->k + 1;
        }
        r.dense_bytes = a.compress ? a.dense_bytes : 0;
        r.compressed_bytes = a.compress ? cb : 0;
        r.ratio = (a.compress && cb > 0) ? (double)r.dense_bytes / (double)cb : 1.0;
        r.nnz = a.compress ? nz : 0;
        r.zeroed = a.compress ? zr : 0;
        r.global_mass = m;
        r.l2 = a.l2_on ? a.l2_scale * l2 : 0.0;  // area / size * sum (solver.hpp:302-304)
        *row_out = r;
        *mfv_out = mf;
        *a.done = 0;
        *a.bump_next = 0;
        if (a.work) *a.work = 0;
    }
}

// End of an l2 pass (transport, compute_l2): fixed-order reduction of the
// per-thread squared errors; the last CTA writes the step's row.l2.
template <int NT>
__device__ __forceinline__ void finalize_l2(const StepArgs& a, double mine) {
    __shared__ double wl2[NT / 32];
    __shared__ int am_last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0) wl2[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        double c = 0.0;
        for (int w = 0; w < NT / 32; ++w) c += wl2[w];
        a.partials[blockIdx.x].l2 = c;
        __threadfence();
        am_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!am_last || threadIdx.x >= 32) return;
    __threadfence();
    double s = 0.0;
    for (unsigned c = threadIdx.x; c < gridDim.x; c += 32) s += __ldcg(&a.partials[c].l2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) {
        a.row_out->l2 = a.l2_scale * s;  // area / size * sum (solver.hpp:302-304)
        *a.done = 0;
    }
}

}  // namespace wg
