// lbm_pair.cuh — the fused D2Q9 step: one patch per CTA PAIR (a 2-CTA
// thread-block cluster), the whole uncompressed patch in shared memory.
//
// A 65^2 x 9 fp64 patch is 304 KB: more than one SM's shared memory, less
// than two.  The pair splits it by population: rank 0 owns populations
// {1, 3, 5, 6}, rank 1 {2, 4, 7, 8}, and both hold a replica of the rest
// population 0 (no streaming, no edges).  Every CTA therefore has 4 x 65 +
// 33 (or 32) line jobs per pass — one per thread, population 0's from the
// next warp boundary (12 warps with the control warp) — and every phase
// except the collide is CTA-local:
//
//   D0  wait for the patch's CSR blocks (cp.async.bulk into shared memory,
//       issued while the previous patch was being processed; mbarrier)
//   D1  decode rows: a block whose stored coefficients are all among the
//       NS x NS coarsest samples (the common case) only scatters them;
//       otherwise CSR scatter + inverse transform along dim 1 of the
//       non-empty coefficient rows (a row that decodes to nothing is never
//       touched: the column pass reads it as +0.0 through a row mask)
//   D2  decode columns: inverse transform along dim 0 (samples-only blocks:
//       each column's row values by the predict chains, idwt_samples_at;
//       zero-detail levels skipped bit-exactly, lifting.cuh), ghost values
//       from the neighbours' edge lines, pull streaming as a register shift
//       -> the streamed population field in shared memory
//   C   BGK collide of this CTA's column half of the patch: 9 populations per
//       cell, the peer's 4 over distributed shared memory (DSMEM)
//   F1  forward transform along dim 0 (columns), corner layout, in place
//   F2  forward transform along dim 1 (rows) + threshold + nnz/zeroed counts
//   S   CTA scan -> CSR row offsets; the pair exchanges its counts through
//       a DSMEM mailbox (skip rule, pipeline.hpp:243-249, on the patch total)
//   W   CSR rows written straight from registers; edge lines (the next
//       step's ghost sources) by partial reconstruction: only the cones of
//       logical rows/columns 1 and n-2 are inverse transformed; mass from the
//       kept coefficients through the trapezoid functional of the inverse
//       (details integrate to zero: the sample coefficients carry the mass)
//
// The reconstruction of the reference's compress cycle (insert_logical of
// idwt_nd, pipeline.hpp:251-253) is not materialised: the next step decodes
// the stored coefficients anyway, and the edge lines it needs are computed
// bit-identically from the same lifting operations.  A patch whose cycle
// zeroes nothing is re-derived (decode + collide again, deterministic) and
// stored raw; its CSR blocks are never allocated.
//
// The D2Q9 scheme is NOT in the reference; its definition
// is shared with oracle/ref_shim.cpp and oracle/wg_oracle.c.
#pragma once

#include <cooperative_groups.h>

#include "patch_phases.cuh"

namespace wg {

namespace cg = cooperative_groups;

#ifndef WG_LBM_CELLS
#define WG_LBM_CELLS 3
#endif

// ---- PTX helpers: mbarrier, bulk async copy, cluster barriers ---------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WG_MBAR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WG_MBAR_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// arrive (release, cluster scope) on the barrier at the offset of `bar` in
// CTA `peer`'s shared memory: the arriving thread's earlier stores (DSMEM
// included) happen before the waiter's acquire
__device__ __forceinline__ void mbar_arrive_remote(unsigned long long* bar, unsigned peer) {
    uint32_t b;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b) : "r"(smem_u32(bar)), "r"(peer));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WG_MBAR_WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WG_MBAR_WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> this CTA's shared memory, completion counted on bar (bytes and
// both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 8-byte asynchronous global -> shared copy (LDGSTS): no register, no stall
// at issue; completed by cp_async_wait_all before the barrier that publishes it
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// generic-proxy accesses of shared memory before later async-proxy writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    cluster_arrive();
    cluster_wait();
}
// Cluster barrier after a CTA barrier: only warp 0 arrives with release
// semantics (cumulative over the CTA's writes it observed through the CTA
// barrier), the other warps arrive relaxed — one warp pays the fence.
__device__ __forceinline__ void cluster_sync_cta() {
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) cluster_arrive();
    else cluster_arrive_relaxed();
    cluster_wait();
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// ---- compile-time tables ----------------------------------------------------
// 128-bit position set (N <= 65 < 128).
struct Bits128 {
    unsigned long long lo, hi;
    __host__ __device__ constexpr bool has(int p) const { return p < 64 ? ((lo >> p) & 1ull) : ((hi >> (p - 64)) & 1ull); }
    __host__ __device__ constexpr void set(int p) {
        if (p < 64) lo |= 1ull << p;
        else hi |= 1ull << (p - 64);
    }
};

// Corner-layout positions of a line whose inverse transform feeds output
// position `ii` (the dependency cone of idwt_line_reg, wavelet.hpp:118-130).
template <int N, int L>
__host__ __device__ constexpr Bits128 inverse_cone(int ii) {
    Bits128 dep[N] = {};
    for (int r = 0; r < N; ++r) dep[r].set(r);
    for (int l = L; l >= 1; --l) {
        const int s = 1 << (l - 1);
        const int len = (N - 1) / s + 1;
        const int half = (len - 1) / 2;
        for (int k = 1; k < half; ++k) {
            dep[2 * k * s].lo |= dep[(2 * k - 1) * s].lo | dep[(2 * k + 1) * s].lo;
            dep[2 * k * s].hi |= dep[(2 * k - 1) * s].hi | dep[(2 * k + 1) * s].hi;
        }
        for (int k = 0; k < half; ++k) {
            dep[(2 * k + 1) * s].lo |= dep[2 * k * s].lo | dep[(2 * k + 2) * s].lo;
            dep[(2 * k + 1) * s].hi |= dep[2 * k * s].hi | dep[(2 * k + 2) * s].hi;
        }
    }
    Bits128 out{};
    for (int r = 0; r < N; ++r)
        if (dep[ii].has(r)) out.set(corner_pos<N, L>(r));
    return out;
}

// Threshold counts of one coefficient (apply_threshold, threshold.hpp:51-86:
// kept iff y != 0 && !(|y| < T), NaN kept): kept += 1, nonzero += 1, as two
// predicated adds (setp with predicate combination; |y| is an operand modifier).
__device__ __forceinline__ void thr_count(double y, double T, unsigned& kept, unsigned& nonzero) {
    asm("{\n\t.reg .pred p0, p1;\n\t.reg .f64 a;\n\t"
        "setp.ne.f64 p0, %2, 0d0000000000000000;\n\t"
        "abs.f64 a, %2;\n\t"
        "setp.geu.and.f64 p1, a, %3, p0;\n\t"
        "@p1 add.u32 %0, %0, 1;\n\t"
        "@p0 add.u32 %1, %1, 1;\n\t}"
        : "+r"(kept), "+r"(nonzero)
        : "d"(y), "d"(T));
}
// Register (interleaved) indices holding samples after L levels.
template <int N, int L>
__host__ __device__ constexpr Bits128 sample_bits() {
    Bits128 b{};
    for (int r = 0; r < N; ++r)
        if (r % (1 << L) == 0) b.set(r);
    return b;
}

// Output position II of the inverse line transform of a register line
// (only the dependency cone of II survives dead-code elimination).
template <int N, int L, int II>
__device__ __forceinline__ double idwt_at(const double (&x)[N]) {
    double y[N];
#pragma unroll
    for (int r = 0; r < N; ++r) y[r] = x[r];
    idwt_line_reg<N, L>(y);
    return y[II];
}

// Streamed column (pull streaming along dim 0: out[i] = v[i - cx], the
// ghost value at the row that enters) stored with element stride S.
template <int N, int S>
__device__ __forceinline__ void store_streamed(double* dst, const double (&v)[N], int cx, double ghost) {
    double* const d = dst + cx * S;  // out[i + cx] = v[i]
#pragma unroll
    for (int i = 1; i < N - 1; ++i) d[i * S] = v[i];
    if (cx >= 0) d[0] = v[0];
    if (cx <= 0) d[(N - 1) * S] = v[N - 1];
    if (cx == 1) dst[0] = ghost;
    if (cx == -1) dst[(N - 1) * S] = ghost;
}

// Output position p of the inverse line transform (idwt_line_reg<N, L, L>:
// every detail +0.0) of NS lines whose corner-layout positions 0..NS-1 hold
// the samples srow[l * NS + k] (interleaved positions k 2^L), all lines at
// once.  Only the chain of predicts that leads to p is evaluated: at each
// level the interval [a, a + 2h] around p is halved, its midpoint being
// lift_pred_inv(0, va, vb) exactly as in the full inverse, so the values are
// bit-identical.  Branch-free (selects): the lanes of a warp hold different p.
template <int N, int L, int NS>
__device__ __forceinline__ void idwt_samples_at(const double* srow, int p, double (&out)[NS]) {
    constexpr int S = 1 << L;
    const int k = min(p / S, NS - 2);  // the coarse interval [k S, (k + 1) S] holding p
    int a = k * S;
    double va[NS], vb[NS];
#pragma unroll
    for (int l = 0; l < NS; ++l) {
        va[l] = srow[l * NS + k];
        vb[l] = srow[l * NS + k + 1];
        out[l] = p == a ? va[l] : vb[l];  // p on a sample (the right end: p == (k + 1) S)
    }
#pragma unroll
    for (int h = S / 2; h >= 1; h /= 2) {
        const int mid = a + h;
        const bool hit = p == mid, right = p > mid;
#pragma unroll
        for (int l = 0; l < NS; ++l) {
            const double vm = lift_pred_inv(0.0, va[l], vb[l]);
            out[l] = hit ? vm : out[l];
            va[l] = right ? vm : va[l];
            vb[l] = right ? vb[l] : vm;
        }
        a = right ? mid : a;
    }
}

template <int N>
struct PairLayout {
    static constexpr int H0 = (N + 1) / 2;        // rank 0's half of population 0 (columns / rows)
    // population 0's line jobs start at a warp boundary (P0): with BUFD below,
    // no warp's line accesses conflict in shared-memory banks
    static constexpr int P0 = ((4 * N + 31) / 32) * 32;
    static constexpr int JOBS = P0 + H0;          // line jobs of rank 0 (rank 1: one fewer)
    // the line jobs' warps + one control warp (prefetch, allocation, mailbox,
    // the serial column-edge inverses) — free in registers: 9-12 warps all
    // get 168 registers per thread (3 warps per SM sub-partition)
    static constexpr int NT = ((JOBS + 31) / 32) * 32 + 32;
    static constexpr int CTL = NT - 32;  // first thread of the control warp
    static constexpr int NN = N * N;
    // doubles per population buffer: N^2 = 1 (mod 16) for N = 2^k + 1, so a
    // warp whose lanes straddle two buffers (the last columns / rows of one
    // population, the first of the next) spreads over the banks without a
    // conflict (2 BUFD = 2 (mod 32) words: the next buffer's lanes start
    // exactly where the previous one's end, modulo the 32 banks)
    static constexpr int BUFD = NN;
    static_assert(NN % 16 == 1, "bank-conflict-free buffer stride");
    static constexpr int NBUF = 5;                // slot 0: population 0 replica, slots 1..4: own populations
    static constexpr size_t kSmemMax = 232448;    // 227 KB per CTA (sm_100)
    static constexpr size_t kStatic = 8192;       // static shared memory of the kernel (bound, checked at load)
    // + the scan array, the column-edge partials of the 4 own populations and
    // the per-thread mass accumulators
    // (+ one pad double so that the staging area after them is 16-byte
    // aligned: the bulk copies land there)
    static constexpr int PAD = (NBUF * BUFD + 3 * NT + 4 * N) & 1;
    static constexpr size_t fixed_bytes() {
        return sizeof(double) * (size_t)NBUF * BUFD + 8ull * NT + sizeof(double) * 4 * (size_t)N +
               sizeof(double) * 2 * (size_t)NT + sizeof(double) * PAD;
    }
    static constexpr size_t stage_bytes() {
        const size_t room = kSmemMax - kStatic - fixed_bytes();
        const size_t want = (size_t)5 * (12 * NN + 4 * (N + 1) + 16);  // every block dense-CSR
        return ((want < room ? want : room) / 16) * 16;
    }
    static constexpr size_t smem_bytes() { return fixed_bytes() + stage_bytes(); }
};

enum : uint32_t { IN_CSR = 0, IN_RAW = 1, IN_DEAD = 2, IN_CONST = 3 };

// Where a slot's input block of the current patch lives.
struct SlotIn {
    const double* v;         // CSR values (staged copy or global)
    const uint32_t* col;
    const uint32_t* ro;
    const double* gv;        // the same block in global memory (re-derivation after the skip rule)
    const uint32_t* gcol;
    const uint32_t* gro;
    const double* raw;       // IN_RAW: dense N x N block in global memory (row pitch raw_ld)
    uint32_t nnz, kind, raw_ld;
};

// Population of slot s on rank r: rank 0 owns {1, 3, 5, 6}, rank 1 owns
// {2, 4, 7, 8} (two axis and two diagonal populations each: equal ghost and
// edge-line work), slot 0 is population 0 on both.
__host__ __device__ constexpr int pair_pop(int rank, int s) {
    return (int)(((rank == 0 ? 0x65310u : 0x87420u) >> (4 * s)) & 15u);
}
__host__ __device__ constexpr int pop_owner(int q) { return q == 0 ? -1 : (int)((0x194u >> q) & 1u); }  // rank
__host__ __device__ constexpr int pop_slot(int q) { return (int)((0x434322110ull >> (4 * q)) & 15u); }
static_assert(pair_pop(0, 1) == 1 && pair_pop(0, 2) == 3 && pair_pop(0, 3) == 5 && pair_pop(0, 4) == 6 &&
              pair_pop(1, 1) == 2 && pair_pop(1, 2) == 4 && pair_pop(1, 3) == 7 && pair_pop(1, 4) == 8);
static_assert(pop_owner(1) == 0 && pop_owner(3) == 0 && pop_owner(5) == 0 && pop_owner(6) == 0 &&
              pop_owner(2) == 1 && pop_owner(4) == 1 && pop_owner(7) == 1 && pop_owner(8) == 1);
static_assert(pop_slot(1) == 1 && pop_slot(3) == 2 && pop_slot(5) == 3 && pop_slot(6) == 4 && pop_slot(2) == 1 &&
              pop_slot(4) == 2 && pop_slot(7) == 3 && pop_slot(8) == 4);

// Two inverse variants (instruction-cache budget): every detail level empty
// (only the samples stored, the common well-compressed block: Z = L), or the
// general inverse (Z = 0; exact for any content).
template <int L, typename F>
__device__ __forceinline__ void with_z2(int z, F&& f) {
    if (z == L) f(std::integral_constant<int, L>{});
    else f(std::integral_constant<int, 0>{});
}

// ---- the kernel -------------------------------------------------------------
template <int N, int L, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairLayout<N>::NT, 1)
    k_lbm_pair(const __grid_constant__ StepArgs a) {
    using Lay = PairLayout<N>;
    constexpr int NT = Lay::NT, NN = N * N, BUFD = Lay::BUFD, H0 = Lay::H0, CTL = Lay::CTL;
    constexpr size_t STAGE = Lay::stage_bytes();
    constexpr Bits128 CONE_LO = inverse_cone<N, L>(1), CONE_HI = inverse_cone<N, L>(N - 2);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* bufs = reinterpret_cast<double*>(smem_raw);
    unsigned long long* inc = reinterpret_cast<unsigned long long*>(bufs + Lay::NBUF * BUFD);
    double* side = reinterpret_cast<double*>(inc + NT);  // [4][N] column-edge partials Y[r][1 or N-2]
    double* acc_m = side + 4 * N;                // per-thread mass of the reconstruction
    double* acc_f = acc_m + NT;                  // per-thread mass of the collided state
    unsigned char* stage = reinterpret_cast<unsigned char*>(acc_f + NT + Lay::PAD);

    __shared__ __align__(8) unsigned long long mbar;
    __shared__ __align__(8) unsigned long long mbm;  // rank 1: population 0's block offset delivered
    __shared__ __align__(16) DirEntry dnext[5];  // the next patch's directory entries (dir_ahead)
    __shared__ SlotIn slot_in[2][5];
    __shared__ Bits128 rmask[5];               // non-empty coefficient rows per slot
    // samples-only decode (the common well-compressed block: every stored
    // coefficient among the NS x NS coarsest samples): the samples per slot,
    // and per slot whether the block needs the general row decode instead
    constexpr int NS = ((N - 1) >> L) + 1;
    constexpr bool kSampFast = L >= 1 && NS >= 2 && NS <= 5;
    __shared__ double samp[5][kSampFast ? NS * NS : 1];
    __shared__ int slot_gen[5];
    __shared__ unsigned long long mail_tot[5];  // peer's per-slot (zeroed << 32 | nnz) totals
    __shared__ unsigned long long mail_off0;    // population 0 block offset (rank 0 -> rank 1)
    __shared__ int mail_ok0;
    __shared__ unsigned long long slot_tot[5];
    __shared__ uint64_t slot_off[5];
    __shared__ int slot_ok[5];
    __shared__ uint32_t slot_nnz[5];            // nnz of the block a slot writes into
    __shared__ uint32_t slot_k0[5];             // entry offset of this CTA's rows inside the block
    __shared__ int slot_top[5];                 // highest row holding a kept coefficient (-1: none)
    __shared__ ChunkState cs;
    __shared__ int skip_patch;
    __shared__ StepPartial part;                // this CTA's step sums (thread 0)
    __shared__ PatchPos ppos;
    __shared__ uint32_t cur_p;                  // the patch in flight (state lives in shared
    __shared__ int cur_it, cur_redo;            // memory: short register live ranges)
    __shared__ double red_m[NT / 32], red_f[NT / 32];
    __shared__ double gh_row[4][N];             // ghost value streamed in along dim 0, per output column
    __shared__ double gh_col[4][N];             // ghost column streamed in along dim 1
    __shared__ uint8_t ilv[N];                  // register (interleaved) index of a corner position

    const int t = threadIdx.x;
    const ShardGeom& g = a.g;
    const uint32_t npairs = gridDim.x / 2, pair = blockIdx.x / 2;

    // thread -> line job: own slot s (1..4) line li, or population 0 (slot 0) line li of this CTA's half
    struct Job {
        int s, li, q, cx, cy;
        bool on;
    };
    auto job_of = [&]() {
        const unsigned rank = cluster_rank();
        const int H = rank == 0 ? H0 : N - H0, lo = rank == 0 ? 0 : H0;
        Job jb{0, 0, 0, 0, 0, false};
        if (t < 4 * N) {
            jb.s = 1 + t / N;
            jb.li = t - (jb.s - 1) * N;
            jb.on = true;
        } else if (t >= Lay::P0 && t < Lay::P0 + H) {
            jb.li = lo + (t - Lay::P0);
            jb.on = true;
        }
        jb.q = pair_pop((int)rank, jb.s);
        jb.cx = lbm_cx(jb.q);
        jb.cy = lbm_cy(jb.q);
        return jb;
    };
    auto jb_on_d2 = [&]() { return t < 4 * N || (t >= Lay::P0 && t < Lay::P0 + (cluster_rank() == 0 ? H0 : N - H0)); };
    auto half_lo = [&]() { return cluster_rank() == 0 ? 0 : H0; };
    auto half_n = [&]() { return cluster_rank() == 0 ? H0 : N - H0; };
    auto peer_of = [&]() { return cluster_rank() ^ 1u; };

    // ---- input prefetch of patch p into descriptor set `par` (thread 0) ----
    // (`early`: the patch's directory entries were copied into dnext by
    // dir_ahead at the start of the current patch, so no global-load latency
    // lands on the control thread here)
    auto prefetch = [&](uint32_t p, int par, bool early = false) {
        const int rank = (int)cluster_rank();
        DirEntry e[5];
        if (early) cp_async_wait_all();
#pragma unroll
        for (int sl = 0; sl < 5; ++sl)  // independent loads in flight together
            e[sl] = (MODE != MODE_INIT && !a.raw_in) ? (early ? dnext[sl] : a.dir_in[(size_t)p * 9 + pair_pop(rank, sl)])
                                                      : DirEntry{0, 0u, DIR_DEAD};
        unsigned used = 0;
        unsigned char* src[5];
        unsigned nb[5];
        for (int sl = 0; sl < 5; ++sl) {
            const int qq = pair_pop(rank, sl);
            SlotIn d{};
            nb[sl] = 0;
            if (MODE != MODE_INIT && a.raw_in) {  // streamed input: the grid buffer's logical block
                constexpr size_t TP = N + 2;
                d.kind = IN_RAW;
                d.raw = a.raw_in + ((size_t)(p - a.p_begin) * 9 + qq) * TP * TP + TP + 1;
                d.raw_ld = (uint32_t)TP;
            } else if (e[sl].flags & DIR_DEAD) {
                d.kind = IN_DEAD;
            } else if (e[sl].flags & DIR_CONST) {  // constant raw block (value in the entry)
                d.kind = IN_CONST;
                d.nnz = (uint32_t)(e[sl].off & 0xffffffffull);
                d.raw_ld = (uint32_t)(e[sl].off >> 32);
            } else if (e[sl].flags & DIR_RAW) {
                d.kind = IN_RAW;
                d.raw = reinterpret_cast<const double*>(a.store_in + e[sl].off);
                d.raw_ld = (uint32_t)N;
            } else {
                d.kind = IN_CSR;
                d.nnz = e[sl].nnz;
                const unsigned char* gb = a.store_in + e[sl].off;
                d.gv = reinterpret_cast<const double*>(gb);
                d.gcol = reinterpret_cast<const uint32_t*>(gb + 8ull * e[sl].nnz);
                d.gro = d.gcol + e[sl].nnz;
                const unsigned bytes = (unsigned)round16(12ull * e[sl].nnz + 4ull * (N + 1));
                if (used + bytes <= STAGE) {
                    unsigned char* sb = stage + used;
                    src[sl] = const_cast<unsigned char*>(gb);
                    nb[sl] = bytes;
                    d.v = reinterpret_cast<const double*>(sb);
                    d.col = reinterpret_cast<const uint32_t*>(sb + 8ull * e[sl].nnz);
                    d.ro = d.col + e[sl].nnz;
                    used += bytes;
                } else {  // does not fit the staging area: decoded from global memory
                    d.v = d.gv;
                    d.col = d.gcol;
                    d.ro = d.gro;
                }
            }
            slot_in[par][sl] = d;
        }
        mbar_arrive_expect(&mbar, used);  // the transaction count first, then the copies
        for (int sl = 0; sl < 5; ++sl)
            if (nb[sl]) bulk_g2s(const_cast<double*>(slot_in[par][sl].v), src[sl], nb[sl], &mbar);
    };

    // The next patch's directory entries into dnext by cp.async (control
    // thread, at the start of a patch): consumed by prefetch(.., early) after D1.
    auto dir_ahead = [&](uint32_t p) {
        const int rank = (int)cluster_rank();
#pragma unroll
        for (int sl = 0; sl < 5; ++sl) {
            const DirEntry* src = a.dir_in + (size_t)p * 9 + pair_pop(rank, sl);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&dnext[sl])), "l"(src) : "memory");
        }
    };

    // The ghost values of the own populations of patch p (sync_ghosts,
    // patchgrid.hpp:131-201), gathered by all threads from the neighbours'
    // edge lines (the previous step's output): per output column j of D2 the
    // value streamed in along dim 0, L(-1, j - cy) (cx = +1) or L(N, j - cy)
    // (cx = -1), corners from the diagonal neighbours; and the column
    // streamed in along dim 1.  Issued at the end of the previous patch, so
    // its L2 latency overlaps that patch's tail.
    auto gather_ghosts = [&](uint32_t p) {
        if constexpr (MODE == MODE_STEP || MODE == MODE_STEP_LZ) {
            const int rank = (int)cluster_rank();
            const PatchPos pp = patch_pos(p, g);
            for (int k = t; k < 8 * N; k += NT) {
                const int which = k / (4 * N), rem = k - which * 4 * N, sl = 1 + rem / N, j = rem - (sl - 1) * N;
                const int q = pair_pop(rank, sl), cx = lbm_cx(q), cy = lbm_cy(q);
                if (which == 0) {
                    if (cx == 0) continue;
                    const int jc = j - cy;
                    const uint32_t bcol = jc < 0 ? pp.bl : (jc >= N ? pp.br : pp.b);
                    const int pos = jc < 0 ? N - 2 : (jc >= N ? 1 : jc);
                    cp_async8(&gh_row[sl - 1][j], cx == 1 ? a.ein.rowhi + edge_ix(pp.su, bcol, lbm_slot_rowhi(q), g, N) + pos
                                                          : a.ein.rowlo + edge_ix(pp.sd, bcol, lbm_slot_rowlo(q), g, N) + pos);
                } else {
                    if (cy == 0) continue;
                    cp_async8(&gh_col[sl - 1][j], cy == 1 ? a.ein.colhi + edge_ix(pp.ar, pp.bl, lbm_slot_colhi(q), g, N) + j
                                                          : a.ein.collo + edge_ix(pp.ar, pp.br, lbm_slot_collo(q), g, N) + j);
                }
            }
        }
    };

    for (int k = t; k < N; k += NT) ilv[k] = (uint8_t)interleaved_of<N, L>(k);
    if (t == CTL) {
        mbar_init(&mbar, 1);
        mbar_init(&mbm, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        cs.cur = cs.end = 0;
        part = a.chunk_first ? StepPartial{0, 0, 0, 0.0, 0.0, 0.0} : a.partials[blockIdx.x];
    }
    __syncthreads();
    cluster_sync_all();  // the peer CTA runs before any DSMEM access
    const uint32_t p_end = a.p_end;
    if (t == CTL && a.p_begin + pair < p_end) prefetch(a.p_begin + pair, 0);
    if (a.p_begin + pair < p_end) gather_ghosts(a.p_begin + pair);
    cp_async_wait_all();
    __syncthreads();
    WG_PHASE_MARK(-1);

    unsigned phase = 0, mbm_phase = 0;
    double tot_m = 0.0, tot_f = 0.0;  // this thread's mass contributions (reconstruction, scheme output)
    if (t == CTL) {
        cur_p = a.p_begin + pair;
        cur_it = 0;
        ppos = patch_pos(cur_p, g);
        cur_redo = 0;
    }
    if (t >= CTL && t < CTL + 5) {
        rmask[t - CTL] = Bits128{0ull, 0ull};
        slot_top[t - CTL] = -1;
        slot_gen[t - CTL] = kSampFast ? 0 : 1;
    }
    if constexpr (kSampFast)
        for (int k = t - CTL; k >= 0 && k < 5 * NS * NS; k += 32) (&samp[0][0])[k] = 0.0;
    __syncthreads();
    for (;;) {
        if (cur_p >= p_end) break;
        // D0: inputs arrived; row masks of the stored blocks and the ghost
        // values, gathered by all threads (no barrier: D1's covers them; the
        // per-patch state was reset at the end of the previous patch)
        WG_PHASE_MARK(12);
        mbar_wait(&mbar, phase);
        phase ^= 1u;
        if (MODE != MODE_INIT && t == CTL && !a.raw_in && cur_p + npairs < p_end) dir_ahead(cur_p + npairs);
        WG_PHASE_MARK(13);
        acc_m[t] = 0.0;
        acc_f[t] = 0.0;
        bool raw_now = false;  // this patch is stored raw (skip rule / no compression): uniform
        const int par = cur_it & 1;
        // produce the post-collide state (D1, D2, C); pass 1 re-derives the
        // state of a skip-rule patch after the transform overwrote it
        for (;;) {
            const int par = cur_it & 1;
            if constexpr (MODE == MODE_INIT) {
                // initial state generated on the device (CUDA libm, not bit-pinned
                // to the host IC) for grids whose raw state exceeds the store
                // budget; own populations fully, population 0 on the own half
                const int N1 = N - 1, rank = (int)cluster_rank(), lo = half_lo(), H = half_n();
                const PatchPos pp = ppos;
                for (int c = t; c < NN; c += NT) {
                    const int i = c / N, jj = c - i * N;
                    const uint64_t gi = ((uint64_t)(g.row0 + pp.ar) * N1 + i) % a.ic_period,
                                   gj = (uint64_t)pp.b * N1 + jj;
                    const double X = (double)gi * a.ic_inv, Y = (double)gj * a.ic_inv;
                    const double uy = X <= 0.5 ? a.ic_u0 * tanh(a.ic_kappa * (X - 0.25))
                                               : a.ic_u0 * tanh(a.ic_kappa * (0.75 - X));
                    const double ux = a.ic_delta * a.ic_u0 * sin(2.0 * 3.141592653589793 * (Y + 0.25));
                    const double usq = lbm_usq(ux, uy);
#pragma unroll
                    for (int sl = 0; sl < 5; ++sl) {
                        const int qq = pair_pop(rank, sl);
                        if (sl == 0 && (jj < lo || jj >= lo + H)) continue;
                        bufs[(size_t)sl * BUFD + c] = lbm_feq(qq, 1.0, lbm_cu(qq, ux, uy), usq);
                    }
                }
                __syncthreads();
                if (t == CTL && !cur_redo && cur_p + npairs < p_end) prefetch(cur_p + npairs, par ^ 1);
                cluster_sync_all();
            } else {
                WG_PHASE_MARK(14);
                if (cur_redo) {  // skip-rule re-derivation: this patch's ghosts again
                    cp_async_wait_all();
                    __syncthreads();
                    gather_ghosts(cur_p);
                    cp_async_wait_all();
                }
                // D1: decode rows (own slots: row li; population 0: every row,

                // strided).  The pull-streaming shift along dim 1 commutes with
                // the column transforms, so it is applied here: row r is stored
                // shifted by cy (B[r][j] = Y[r][j - cy]) and every column thread
                // of D2 then reads and writes only its own column.
                {
                    const Job jb = job_of();
                    const bool redo = cur_redo != 0;
                    auto decode_row = [&](double* Bs, const SlotIn& d, int r, int cy) {
                        if (d.kind != IN_CSR) return;
                        const double* vv = redo ? d.gv : d.v;
                        const uint32_t* cc = redo ? d.gcol : d.col;
                        const uint32_t* ro = redo ? d.gro : d.ro;
                        const uint32_t k0 = ro[r], k1 = ro[r + 1];
                        if (k0 == k1) return;
                        // the column pass reads only the rows that decode to something
                        if (r < 64) atomicOr(&rmask[&d - &slot_in[par][0]].lo, 1ull << r);
                        else atomicOr(&rmask[&d - &slot_in[par][0]].hi, 1ull << (r - 64));
                        WG_CHECK(k1 <= d.nnz && k0 < k1, 1);
                        double* rowp = Bs + (size_t)r * N;
                        // two variants: only sample columns stored (Z = L) or general
                        const int z = z_of_top(N, L, (int)cc[k1 - 1]) == L ? L : 0;
                        const int top = z_top(N, z);  // the positions the variant reads
                        for (int jj = 0; jj <= top; ++jj) rowp[jj] = 0.0;
                        for (uint32_t k = k0; k < k1; ++k) {
                            WG_CHECK(cc[k] < (uint32_t)N, 2);
                            rowp[cc[k]] = vv[k];
                        }
                        with_z2<L>(z, [&](auto ZC) {
                            constexpr int Z = decltype(ZC)::value;
                            double x[N];
#pragma unroll
                            for (int rr = 0; rr < N; ++rr)
                                x[rr] = corner_pos<N, L>(rr) <= z_top(N, Z) ? rowp[corner_pos<N, L>(rr)] : 0.0;
                            idwt_line_reg<N, L, Z>(x);
                            store_streamed<N, 1>(rowp, x, (MODE == MODE_DECODE) ? 0 : cy, 0.0);
                        });
                    };
                    // D1a: the rows of a samples-only block only scatter their
                    // samples (D2 interpolates them per column); any other stored
                    // row marks its block for the general row decode (D1b)
                    auto scan_row = [&](int sl, const SlotIn& d, int r) {
                        if (d.kind != IN_CSR) return;
                        const double* vv = redo ? d.gv : d.v;
                        const uint32_t* cc = redo ? d.gcol : d.col;
                        const uint32_t* ro = redo ? d.gro : d.ro;
                        const uint32_t k0 = ro[r], k1 = ro[r + 1];
                        if (k0 == k1) return;
                        if (!kSampFast || r >= NS || cc[k1 - 1] >= (uint32_t)NS) {
                            slot_gen[sl] = 1;
                            return;
                        }
                        for (uint32_t k = k0; k < k1; ++k) samp[sl][r * NS + cc[k]] = vv[k];
                    };
                    const int step = jb.s > 0 ? N : half_n();
                    if (jb.on)  // own slots one row, population 0 strided
                        for (int r = jb.s > 0 ? jb.li : t - Lay::P0; r < N; r += step) scan_row(jb.s, slot_in[par][jb.s], r);
                    __syncthreads();
                    if ((slot_gen[0] | slot_gen[1] | slot_gen[2] | slot_gen[3] | slot_gen[4]) != 0) {  // uniform
                        if (jb.on && slot_gen[jb.s]) {  // D1b: one call site (instruction cache)
                            double* Bs = bufs + (size_t)jb.s * BUFD;
                            for (int r = jb.s > 0 ? jb.li : t - Lay::P0; r < N; r += step)
                                decode_row(Bs, slot_in[par][jb.s], r, jb.cy);
                        }
                        __syncthreads();
                    }
                }
                WG_PHASE_MARK(21);
                // next patch's inputs: the staging area is free once D1 has run
                // (the skip rule's re-derivation reads the global copies)
                if (t == CTL && !cur_redo && cur_p + npairs < p_end) {
                    fence_proxy_async();
                    prefetch(cur_p + npairs, par ^ 1, !a.raw_in);
                }
                // D2: decode columns, ghosts, pull streaming along dim 0 (a
                // register shift), or the MODE_DECODE output.  Thread j owns
                // column j (already shifted along dim 1 by D1); the column that
                // streams in from outside (jc = j - cy off the patch) is the
                // neighbour's edge line.
                if (jb_on_d2()) {
                    const Job jb = job_of();
                    const int j = jb.li, cx = jb.cx, cy = jb.cy, q = jb.q;
                    double* const Bs = bufs + (size_t)jb.s * BUFD;
                    const int jc = (MODE == MODE_DECODE) ? j : j - cy;
                    const SlotIn& d = slot_in[par][jb.s];
                    const double ghost = (MODE != MODE_DECODE && cx != 0) ? gh_row[jb.s - 1][j] : 0.0;
                    auto emit = [&](const double (&v)[N]) {
                        if (MODE == MODE_DECODE) {
                            constexpr int TP = N + 2;
                            double* out = a.decode_out + ((size_t)(cur_p - a.p_begin) * 9 + q) * (size_t)TP * TP + TP + 1 + j;
#pragma unroll
                            for (int i = 0; i < N; ++i) out[i * TP] = v[i];
                        } else {
                            store_streamed<N, N>(Bs + j, v, cx, ghost);
                        }
                    };
                    double v[N];
                    if (jc < 0 || jc >= N) {  // a ghost column: the neighbour's edge line
                        const double* gl = gh_col[jb.s - 1];
#pragma unroll
                        for (int i = 0; i < N; ++i) v[i] = gl[i];
                        emit(v);
                    } else if (d.kind == IN_RAW) {
#pragma unroll
                        for (int i = 0; i < N; ++i) v[i] = d.raw[(size_t)i * d.raw_ld + jc];
                        emit(v);
                    } else if (d.kind == IN_DEAD || d.kind == IN_CONST) {
                        const double c = d.kind == IN_DEAD ? 0.0
                                                           : __longlong_as_double((long long)(((unsigned long long)d.raw_ld << 32) | d.nnz));
#pragma unroll
                        for (int i = 0; i < N; ++i) v[i] = c;
                        emit(v);
                    } else if (kSampFast && !slot_gen[jb.s]) {
                        // samples-only block: the D1 row values at this column
                        // straight from the samples (idwt_samples_at), then the
                        // column inverse — bit-identical to D1 + the masked path
                        double yr[NS];
                        idwt_samples_at<N, L, NS>(samp[jb.s], jc, yr);
#pragma unroll
                        for (int rr = 0; rr < N; ++rr) {
                            const int cp = corner_pos<N, L>(rr);
                            v[rr] = cp < NS ? yr[cp < NS ? cp : 0] : 0.0;
                        }
                        idwt_line_reg<N, L, L>(v);
                        emit(v);
                    } else {
                        const Bits128 m = rmask[jb.s];
                        int top = -1;
                        if (m.hi) top = 64 + 63 - __clzll((long long)m.hi);
                        else if (m.lo) top = 63 - __clzll((long long)m.lo);
                        with_z2<L>(z_of_top(N, L, top), [&](auto ZC) {
                            constexpr int Z = decltype(ZC)::value;
#pragma unroll
                            for (int rr = 0; rr < N; ++rr) {
                                const int cp = corner_pos<N, L>(rr);
                                v[rr] = (cp <= z_top(N, Z) && m.has(cp)) ? Bs[(size_t)cp * N + j] : 0.0;
                            }
                            idwt_line_reg<N, L, Z>(v);
                            emit(v);
                        });
                    }
                }
                if (MODE == MODE_DECODE) break;
                WG_PHASE_MARK(22);
                cluster_sync_cta();  // both halves streamed
                WG_PHASE_MARK(23);
                // D2 has read the ghosts: gather the next patch's (asynchronously,
                // completed at the end of this patch)
                if (cur_p + npairs < p_end) gather_ghosts(cur_p + npairs);
                // C: BGK collide of this CTA's column half (lbm_collide, physics.cuh);
                // the mass of the scheme output (strict check) as w * rho per
                // cell (BGK conserves it; a tolerance-checked diagnostic)
                {
                    const unsigned rank = cluster_rank(), peer = rank ^ 1u;
                    cg::cluster_group cluster = cg::this_cluster();
                    double* P[9];  // population pointers (the peer's populations through DSMEM)
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        const bool mine = k == 0 || pop_owner(k) == (int)rank;
                        const int sl = pop_slot(k);
                        P[k] = mine ? bufs + (size_t)sl * BUFD : cluster.map_shared_rank(bufs + (size_t)sl * BUFD, peer);
                    }
                    const bool redo = cur_redo != 0;
                    {
                        // one code path for both ranks: H0 columns from lo (rank 1's
                        // half is one column narrower: that column's cells are skipped)
                        constexpr int H = H0, cells = N * H;
                        const int lo = half_lo();
                        constexpr int K = WG_LBM_CELLS;  // cells per iteration (independent chains)
                        double mfv = 0.0;
                        for (int c0 = t; c0 < cells; c0 += K * NT) {
                            double f[K][9];
                            int o[K];
                            double w[K];
#pragma unroll
                            for (int u = 0; u < K; ++u) {
                                const int c = c0 + u * NT;
                                const int cc = c < cells ? c : c0;
                                const int i = cc / H, jj = min(lo + (cc - i * H), N - 1);
                                o[u] = i * N + jj;
                                w[u] = ((i == 0 || i == N - 1) ? 0.5 : 1.0) * ((jj == 0 || jj == N - 1) ? 0.5 : 1.0);
#pragma unroll
                                for (int k = 0; k < 9; ++k) f[u][k] = P[k][o[u]];
                            }
#pragma unroll
                            for (int u = 0; u < K; ++u) {
                                const double rho = lbm_collide(f[u], a.omega);
                                const int c = c0 + u * NT;
                                if (c < cells && lo + (c % H) < N) {
#pragma unroll
                                    for (int k = 0; k < 9; ++k) P[k][o[u]] = f[u][k];
                                    mfv += w[u] * rho;
                                }
                            }
                        }
                        if (!redo) acc_f[t] += mfv;
                    }
                }
                WG_PHASE_MARK(24);
                cluster_sync_cta();  // the peer's populations are written back
                WG_PHASE_MARK(25);
            }
            if (cur_redo || !a.compress) {  // the collided state, to be stored raw (uniform)
                raw_now = true;
                break;
            }

            // F1: forward transform along dim 0 (columns), corner layout, in place;
            // population 0's column half also into the peer's replica
            {
                const Job jb = job_of();
                if (jb.on) {
                    double* const Bs = bufs + (size_t)jb.s * BUFD;
                    const int j = jb.li;
                    double x[N];
#pragma unroll
                    for (int i = 0; i < N; ++i) x[i] = Bs[(size_t)i * N + j];
                    dwt_line_reg<N, L>(x);
#pragma unroll
                    for (int rr = 0; rr < N; ++rr) Bs[(size_t)corner_pos<N, L>(rr) * N + j] = x[rr];
                    if (jb.s == 0) {
                        cg::cluster_group cluster = cg::this_cluster();
                        double* const Bpeer0 = cluster.map_shared_rank(bufs, peer_of());
#pragma unroll
                        for (int rr = 0; rr < N; ++rr) Bpeer0[(size_t)corner_pos<N, L>(rr) * N + j] = x[rr];
                    }
                }
            }
            cluster_sync_cta();  // population 0's replicas hold both column halves
            WG_PHASE_MARK(26);
            // F2: forward transform along dim 1 (rows) + threshold (threshold.hpp:51-86);
            // the thresholded row is parked in its own buffer row across the barriers
            unsigned long long cnt = 0;  // zeroed << 32 | nnz of this row
            bool samp_only = true;       // every kept coefficient of the row is a sample (column)
            {
                const Job jb = job_of();
                if (jb.on) {
                    double* const rowp = bufs + (size_t)jb.s * BUFD + (size_t)jb.li * N;
                    const int r = jb.li;
                    double x[N];
#pragma unroll
                    for (int jj = 0; jj < N; ++jj) x[jj] = rowp[jj];
                    dwt_line_reg<N, L>(x);
                    const int bi = band_of_pos(N, L, r);
                    double trow[L + 1];
#pragma unroll
                    for (int bj = 0; bj <= L; ++bj) trow[bj] = a.thr[bi * (L + 1) + bj];
                    if (MODE == MODE_STEP_LZ) {  // apply_threshold's output (-0.0 kept) for the LZ sizes
                        double* lz = a.lz_dense + ((size_t)cur_p * 9 + jb.q) * NN + (size_t)r * N;
#pragma unroll
                        for (int rr = 0; rr < N; ++rr) {
                            const double y = x[rr];
                            lz[corner_pos<N, L>(rr)] = (y != 0.0 && fabs(y) < trow[band_of_r<N, L>(rr)]) ? 0.0 : y;
                        }
                    }
                    // counts: kept (y != 0 && !(|y| < T)) and nonzero, four
                    // independent counter pairs (two predicated adds per value)
                    // (ck[3]: the sample positions — every other position is a detail)
                    unsigned ck[4] = {0u, 0u, 0u, 0u}, cn[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int rr = 0; rr < N; ++rr)
                        thr_count(x[rr], trow[band_of_r<N, L>(rr)], ck[band_of_r<N, L>(rr) == 0 ? 3 : (rr & 1) + 1],
                                  cn[rr & 3]);
                    const unsigned nz = (ck[1] + ck[2]) + ck[3];
                    const unsigned zr = (cn[0] + cn[1]) + (cn[2] + cn[3]) - nz;
                    samp_only = (ck[1] + ck[2]) == 0u;  // no kept detail coefficient
                    // park the thresholded row for W (killed -> +0.0, -0.0 -> +0.0
                    // like the CSR round trip); a row without kept coefficients is
                    // needed only as zeros of a cone row of the row edge line
                    const bool cone_row = jb.s > 0 && jb.cx != 0 && (jb.cx == -1 ? CONE_LO : CONE_HI).has(r);
                    if (nz) {
#pragma unroll
                        for (int rr = 0; rr < N; ++rr) {
                            const double y = x[rr];
                            rowp[rr] = (y != 0.0 && !(fabs(y) < trow[band_of_r<N, L>(rr)])) ? y : 0.0;
                        }
                        atomicMax(&slot_top[jb.s], r);
                        // mass of the reconstruction: sum_rc a_r a_c C[r][c] (trapezoid
                        // functional of idwt_nd, host-computed exact dyadic values; for
                        // conservative levels only the samples carry mass)
                        const double ar = a.mass_a[r];
                        if (ar != 0.0) {
                            double acc = 0.0;
#pragma unroll
                            for (int rr = 0; rr < N; ++rr) acc += rowp[rr] * a.mass_a[corner_pos<N, L>(rr)];
                            acc_m[t] = ar * acc;
                        }
                    } else if (cone_row) {
#pragma unroll
                        for (int rr = 0; rr < N; ++rr) rowp[rr] = 0.0;
                    }
                    // column edge line of the reconstruction (own populations):
                    // Y[r][jj] = row inverse at jj = 1 (cy = -1) or N-2 (cy = +1)
                    if (jb.s > 0 && jb.cy != 0) {
                        double val = 0.0;
                        if (nz) {
                            double y[N];
#pragma unroll
                            for (int rr = 0; rr < N; ++rr) y[rr] = rowp[rr];  // only the cone is loaded
                            val = jb.cy == -1 ? idwt_at<N, L, 1>(y) : idwt_at<N, L, N - 2>(y);
                        }
                        side[(size_t)(jb.s - 1) * N + r] = val;
                    }
                    cnt = ((unsigned long long)zr << 32) | nz;
                }
            }
            WG_PHASE_MARK(27);
            // S: CTA scan of the counts in job order, per-slot totals, mailbox
            cta_inclusive_scan<NT>(cnt, inc, true);  // the previous patch's scan is barriers behind
            if (t >= CTL && t < CTL + 5) {
                const int u = t - CTL;
                const int first = u == 0 ? Lay::P0 : (u - 1) * N;
                const int n = u == 0 ? half_n() : N;
                const unsigned long long before = first == 0 ? 0ull : inc[first - 1];
                slot_tot[u] = inc[first + n - 1] - before;
                cg::cluster_group cluster = cg::this_cluster();
                cluster.map_shared_rank(mail_tot, peer_of())[u] = slot_tot[u];
            }
            cluster_sync_cta();  // M1: the pair's counts exchanged
            WG_PHASE_MARK(28);
            const bool cycle = a.thr_any != 0;
            if (t == CTL) {
                const unsigned rank = cluster_rank();
                unsigned long long zero = 0, nnz_m = 0, zr_m = 0;
                for (int sl = 0; sl < 5; ++sl) {
                    zero += (slot_tot[sl] >> 32) + (mail_tot[sl] >> 32);
                    nnz_m += slot_tot[sl] & 0xffffffffull;
                    zr_m += slot_tot[sl] >> 32;
                }
                // bytes: 12 nnz of the own rows + the row offsets of the blocks
                // this CTA allocates (population 0's by rank 0)
                part.comp_bytes += 12ull * nnz_m + 4ull * (N + 1) * (rank == 0 ? 5 : 4);
                part.nnz += nnz_m;
                part.zeroed += zr_m;
                skip_patch = (zero == 0) || !cycle;
                if (!skip_patch) {
                    // one allocation for the blocks this CTA owns (population 0's by rank 0)
                    const int s0 = rank == 0 ? 0 : 1;
                    uint64_t total = 0;
                    for (int sl = s0; sl < 5; ++sl) {
                        slot_nnz[sl] = (uint32_t)(slot_tot[sl] & 0xffffffffull) +
                                       (sl == 0 ? (uint32_t)(mail_tot[0] & 0xffffffffull) : 0u);
                        total += round16(12ull * slot_nnz[sl] + 4ull * (N + 1));
                    }
                    uint64_t off = chunk_alloc(a, cs, total);
                    const bool ok = off != ~0ull;
                    for (int sl = s0; sl < 5; ++sl) {
                        const int qq = pair_pop((int)rank, sl);
                        slot_ok[sl] = ok;
                        slot_off[sl] = off;
                        slot_k0[sl] = 0;
                        a.dir_out[(size_t)cur_p * 9 + qq] = ok ? DirEntry{off, slot_nnz[sl], 0u} : DirEntry{0, 0u, DIR_DEAD};
                        if (ok) off += round16(12ull * slot_nnz[sl] + 4ull * (N + 1));
                    }
                    cg::cluster_group cluster = cg::this_cluster();
                    if (rank == 0) {
                        *cluster.map_shared_rank(&mail_off0, peer_of()) = slot_off[0];
                        *cluster.map_shared_rank(&mail_ok0, peer_of()) = slot_ok[0];
                        mbar_arrive_remote(&mbm, peer_of());  // release: the two stores above first
                    } else {  // population 0: rank 0's rows come first in the block
                        slot_nnz[0] = (uint32_t)(slot_tot[0] & 0xffffffffull) + (uint32_t)(mail_tot[0] & 0xffffffffull);
                        slot_k0[0] = (uint32_t)(mail_tot[0] & 0xffffffffull);
                    }
                }
            }
            // M2: population 0's block offset, rank 0 -> rank 1 point to point
            // (a remote mbarrier arrival, no cluster barrier: rank 0 moves on)
            WG_PHASE_MARK(29);
            if (t == CTL && cluster_rank() == 1 && !skip_patch) {
                mbar_wait_acq_cluster(&mbm, mbm_phase);
                mbm_phase ^= 1u;
                slot_off[0] = mail_off0;
                slot_ok[0] = mail_ok0;
            }
            __syncthreads();
            if (!skip_patch) {
                // W: CSR blocks (csr_encode, codec.hpp:37-60) from the parked
                // rows: each thread its row offset; the entries of a warp's
                // non-empty rows written by the whole warp, one row at a time
                // (ballot of the non-zeros, popc prefix: row-major, ascending
                // columns); then the cone rows of the row edge line are
                // inverse transformed in place (a thread only touches its own
                // parked row)
                const Job jb = job_of();
                const unsigned nz = (unsigned)(cnt & 0xffffffffull);
                uint32_t k = 0;
                if (jb.on) {
                    const int s = jb.s;
                    const int first = s == 0 ? Lay::P0 : (s - 1) * N;
                    const unsigned long long before = first == 0 ? 0ull : inc[first - 1];
                    k = (uint32_t)((inc[t] - before) & 0xffffffffull) - nz + slot_k0[s];
                    if (slot_ok[s]) {  // row offsets: u32 from 0 (csr_encode)
                        uint32_t* ro = reinterpret_cast<uint32_t*>(a.store_out + slot_off[s] + 12ull * slot_nnz[s]);
                        if (jb.li == 0) ro[0] = 0;
                        ro[jb.li + 1] = k + nz;
                        WG_CHECK(slot_off[s] + 12ull * slot_nnz[s] + 4ull * (N + 1) <= a.cap_out &&
                                     k + nz <= slot_nnz[s], 10);
                    }
                }
                {
                    const int lane = t & 31;
                    unsigned todo = __ballot_sync(0xffffffffu, jb.on && nz != 0 && slot_ok[jb.s]);
                    // rows whose kept coefficients are all samples: only the
                    // first 32 corner columns can hold them (NS <= 32)
                    const unsigned sonly = __ballot_sync(0xffffffffu, samp_only);
                    while (todo) {
                        const int src = __ffs(todo) - 1;
                        todo &= todo - 1;
                        const int s_ = __shfl_sync(0xffffffffu, jb.s, src), r_ = __shfl_sync(0xffffffffu, jb.li, src);
                        uint32_t k_ = __shfl_sync(0xffffffffu, k, src);
                        const int cols = ((sonly >> src) & 1u) && ((N - 1) >> L) < 32 ? 32 : N;  // uniform
                        const double* row = bufs + (size_t)s_ * BUFD + (size_t)r_ * N;  // interleaved order
                        unsigned char* const blk = a.store_out + slot_off[s_];
                        double* vo = reinterpret_cast<double*>(blk);
                        uint32_t* co = reinterpret_cast<uint32_t*>(blk + 8ull * slot_nnz[s_]);
#pragma unroll
                        for (int base = 0; base < N; base += 32) {
                            if (base >= cols) break;
                            const int pc = base + lane;  // corner-layout column
                            const double xv = pc < N ? row[ilv[pc < N ? pc : 0]] : 0.0;
                            const unsigned m = __ballot_sync(0xffffffffu, xv != 0.0);
                            if (xv != 0.0) {
                                const uint32_t o = k_ + (uint32_t)__popc(m & ((1u << lane) - 1u));
                                vo[o] = xv;
                                co[o] = (uint32_t)pc;
                            }
                            k_ += (uint32_t)__popc(m);
                        }
                    }
                    __syncwarp();
                }
                if (jb.on && nz && jb.s > 0 && jb.cx != 0 && (jb.cx == -1 ? CONE_LO : CONE_HI).has(jb.li)) {
                    double* const rowp = bufs + (size_t)jb.s * BUFD + (size_t)jb.li * N;
                    with_z2<L>(samp_only ? L : 0, [&](auto ZC) {
                        double x[N];
#pragma unroll
                        for (int rr = 0; rr < N; ++rr) x[rr] = rowp[rr];
                        idwt_line_reg<N, L, decltype(ZC)::value>(x);
#pragma unroll
                        for (int jj = 0; jj < N; ++jj) rowp[jj] = x[jj];  // natural order: Y[r][.]
                    });
                }
                __syncthreads();
                WG_PHASE_MARK(30);
                if (jb.on && jb.s > 0) {
                    double* const Bs = bufs + (size_t)jb.s * BUFD;
                    const int j = jb.li, cx = jb.cx, cy = jb.cy, q = jb.q;
                    const PatchPos pp = ppos;
                    if (cx != 0) {  // row line: column j of the cone rows, inverse at 1 / N-2
                        double y[N];
                        if (cx == -1) {
#pragma unroll
                            for (int rr = 0; rr < N; ++rr) {
                                const int cp = corner_pos<N, L>(rr);
                                y[rr] = CONE_LO.has(cp) ? Bs[(size_t)cp * N + j] : 0.0;
                            }
                            put_rowlo(a.eout, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowlo(q), N, j,
                                      idwt_at<N, L, 1>(y));
                        } else {
#pragma unroll
                            for (int rr = 0; rr < N; ++rr) {
                                const int cp = corner_pos<N, L>(rr);
                                y[rr] = CONE_HI.has(cp) ? Bs[(size_t)cp * N + j] : 0.0;
                            }
                            put_rowhi(a.eout, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowhi(q), N, j,
                                      idwt_at<N, L, N - 2>(y));
                        }
                    }
                }
                if (t > CTL && t < CTL + 5) {  // column lines: the column inverse of the partials (control lanes)
                    const int sl = t - CTL, q = pair_pop((int)cluster_rank(), sl), cy = lbm_cy(q);
                    const PatchPos pp = ppos;
                    if (cy != 0) {
                        // rows without kept coefficients hold +0.0 partials: the
                        // zero-detail inverse variant of the top row applies
                        double* dst = cy == -1 ? a.eout.collo + edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_collo(q), g, N)
                                               : a.eout.colhi + edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_colhi(q), g, N);
                        const double* src = side + (size_t)(sl - 1) * N;
                        with_z2<L>(z_of_top(N, L, slot_top[sl]), [&](auto ZC) {
                            constexpr int Z = decltype(ZC)::value;
                            double y[N];
#pragma unroll
                            for (int rr = 0; rr < N; ++rr)
                                y[rr] = corner_pos<N, L>(rr) <= z_top(N, Z) ? src[corner_pos<N, L>(rr)] : 0.0;
                            idwt_line_reg<N, L, Z>(y);
#pragma unroll
                            for (int i = 0; i < N; ++i) dst[i] = y[i];
                        });
                    }
                }
                break;
            }
            if (t == CTL) cur_redo = 1;  // skip rule: the buffers hold the transform, re-derive the state
            __syncthreads();
        }
        if (MODE != MODE_DECODE && raw_now) {
            // skip rule / no compression: the collided state itself, stored raw
            const unsigned rank = cluster_rank();
            if (t == CTL) {
                for (int sl = (rank == 0 ? 0 : 1); sl < 5; ++sl) {
                    const int qq = pair_pop((int)rank, sl);
                    const uint64_t off = chunk_alloc(a, cs, round16((uint64_t)NN * 8));
                    slot_ok[sl] = off != ~0ull;
                    slot_off[sl] = off;
                    a.dir_out[(size_t)cur_p * 9 + qq] = slot_ok[sl] ? DirEntry{off, 0u, DIR_RAW} : DirEntry{0, 0u, DIR_DEAD};
                }
                if (rank == 0) {
                    cg::cluster_group cluster = cg::this_cluster();
                    *cluster.map_shared_rank(&mail_off0, peer_of()) = slot_off[0];
                    *cluster.map_shared_rank(&mail_ok0, peer_of()) = slot_ok[0];
                }
            }
            cluster_sync_all();  // (also: every thread has read cur_redo of this patch)
            if (t == CTL && rank == 1) {
                slot_off[0] = mail_off0;
                slot_ok[0] = mail_ok0;
            }
            if (t == CTL) cur_redo = 0;  // read again only after the next patch's barriers
            __syncthreads();
            double mass = 0.0;
            const int lo = half_lo(), H = half_n();
            for (int k = t; k < 5 * NN; k += NT) {
                const int sl = k / NN, e = k - sl * NN, i = e / N, jj = e - i * N;
                if (sl == 0 && (jj < lo || jj >= lo + H)) continue;  // population 0: own column half
                const double xv = bufs[(size_t)sl * BUFD + e];
                if (slot_ok[sl]) reinterpret_cast<double*>(a.store_out + slot_off[sl])[e] = xv;
                mass += (((i == 0 || i == N - 1) ? 0.5 : 1.0) * ((jj == 0 || jj == N - 1) ? 0.5 : 1.0)) * xv;
            }
            acc_m[t] = mass;
            const Job jb = job_of();
            if (jb.on && jb.s > 0) {  // edge lines straight from the state
                const double* Bs = bufs + (size_t)jb.s * BUFD;
                const int li = jb.li, q = jb.q;
                const PatchPos pp = ppos;
                if (jb.cx == -1) put_rowlo(a.eout, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowlo(q), N, li, Bs[(size_t)1 * N + li]);
                if (jb.cx == 1) put_rowhi(a.eout, g, (uint32_t)(pp.ar + 1), pp.b, lbm_slot_rowhi(q), N, li, Bs[(size_t)(N - 2) * N + li]);
                if (jb.cy == -1) a.eout.collo[edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_collo(q), g, N) + li] = Bs[(size_t)li * N + 1];
                if (jb.cy == 1) a.eout.colhi[edge_ix((uint32_t)pp.ar, pp.b, lbm_slot_colhi(q), g, N) + li] = Bs[(size_t)li * N + N - 2];
            }
        }
        cp_async_wait_all();  // the next patch's ghosts (issued after D2)
        // per-thread mass sums over this CTA's patches (a static sequence:
        // reduced once at the end, in a fixed order)
        if (MODE != MODE_DECODE) {
            tot_m += acc_m[t];
            tot_f += acc_f[t];
        }
        __syncthreads();  // buffers and descriptors free for the next patch
        WG_PHASE_MARK(31);
        if (t == CTL) {
            cur_p += npairs;
            ++cur_it;
            ppos = patch_pos(cur_p, g);
        }
        if (t >= CTL && t < CTL + 5) {
            rmask[t - CTL] = Bits128{0ull, 0ull};
            slot_top[t - CTL] = -1;
            slot_gen[t - CTL] = kSampFast ? 0 : 1;
        }
        if constexpr (kSampFast)
            for (int k = t - CTL; k >= 0 && k < 5 * NS * NS; k += 32) (&samp[0][0])[k] = 0.0;
        __syncthreads();
    }
    cluster_sync_all();  // no DSMEM access of an exited peer
    if (MODE == MODE_DECODE) return;
    __syncthreads();
    {  // the CTA's mass sums (fixed association: lanes, then warps in order)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            tot_m += __shfl_xor_sync(0xffffffffu, tot_m, o);
            tot_f += __shfl_xor_sync(0xffffffffu, tot_f, o);
        }
        if ((t & 31) == 0) {
            red_m[t >> 5] = tot_m;
            red_f[t >> 5] = tot_f;
        }
        __syncthreads();
        if (t == CTL) {
            double sm = 0.0, sf = 0.0;
            for (int w = 0; w < NT / 32; ++w) {
                sm += red_m[w];
                sf += red_f[w];
            }
            part.mass += sm;
            part.mass_fv += sf;
        }
        __syncthreads();
    }
    finalize_step(a, part);
}

}  // namespace wg
