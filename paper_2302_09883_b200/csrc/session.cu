// session.cu — the device-resident compressed patch store and its step loop
// (the B200 hot path), plus run() on top of it.
//
// One step (pipeline.hpp:194-289) is ONE kernel launch on the session
// stream: k_patch_step (transport) or k_lbm_step (D2Q9) runs the fused
// decode/ghost/scheme/DWT/threshold/CSR/reconstruction cycle of every patch,
// applies the skip rule (pipeline.hpp:243-249) in place, and its last CTA
// reduces the per-CTA partials into the step's MetricsRow (pipeline.hpp:
// 260-274) and resets the bump allocator of the other pool.  Nothing
// synchronises with the host inside the step loop.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "common.cuh"
#include "host_model.h"
#include "kernel_table.h"
#include "lz.cuh"
#include "patch_phases.cuh"

namespace wg {

void direction_speeds(double alpha, double beta, double* smax, double* smin);  // ops.cu
void lz_encode_device(const unsigned char* d_in, uint64_t n, uint64_t chunk, std::vector<uint64_t>& len,
                      std::vector<unsigned char>* payload);  // lz_ops.cu

namespace {

// ---- kernel table: kernel_table.h (one translation unit per scheme) ----------
}  // namespace

KernelSet select_kernels(int scheme, uint64_t n, int levels, uint64_t npatch) {
    KernelSet k{};
    bool ok = false;
    const char* what = "transport";
    if (scheme == WG_SCHEME_LBM_D2Q9) {
        ok = select_lbm_kernels(n, levels, k);
        what = "D2Q9";
    } else if (scheme == WG_SCHEME_SWE) {
        ok = select_swe_kernels(n, levels, k);
        what = "SWE";
    } else {
        int sms = 148, dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // C1-sized grids (64 patches of 33 points): one patch per CTA (more SMs busy)
        const bool small = n == 33 && npatch < 2ull * sms;
        ok = select_transport_kernels(n, levels, small, k);
    }
    if (!ok)
        raise(WG_INVALID_ARGUMENT, std::string("device session (") + what + "): patch side " + std::to_string(n) +
                                       " with " + std::to_string(levels) + " levels is not supported");
    return k;
}

namespace {

// The trapezoid functional of the inverse line transform in corner layout:
// out[k] = sum_i w_i (idwt_line e_k)_i with the global_mass weights w
// (patchgrid.hpp:244-266: 1/2 at both ends).  The inverse is linear and
// separable, so the trapezoid mass of idwt_nd(C) is sum_rc out[r] out[c]
// C[r][c].  The entries are small dyadic numbers, computed exactly; for
// conservative level counts the details' entries are exactly 0 (the detail
// functions integrate to zero), so only the samples carry mass.
void inverse_trapezoid_functional(uint32_t n, int levels, double* out) {
    const uint32_t m = n - 1;
    for (uint32_t k = 0; k < n; ++k) {
        std::vector<double> c(n, 0.0);
        c[k] = 1.0;
        std::vector<double> sig(c.begin(), c.begin() + (m >> levels) + 1);
        for (int l = levels; l >= 1; --l) {
            const uint32_t len = (m >> (l - 1)) + 1, half = (len - 1) / 2;
            const double* det = c.data() + (m >> l) + 1;
            std::vector<double> x(len);
            for (uint32_t j = 0; j <= half; ++j) {
                double e = sig[j];
                if (j >= 1 && j < half) {
                    const double w0 = (j - 1 == 0 || j - 1 == half - 1) ? 0.5 : 0.25;
                    const double w1 = (j == 0 || j == half - 1) ? 0.5 : 0.25;
                    e = e - (w0 * det[j - 1] + w1 * det[j]);
                }
                x[2 * j] = e;
            }
            for (uint32_t j = 0; j < half; ++j) x[2 * j + 1] = det[j] + (x[2 * j] + x[2 * j + 2]) / 2.0;
            sig.swap(x);
        }
        double s = 0.0;
        for (uint32_t i = 0; i < n; ++i) s += ((i == 0 || i == m) ? 0.5 : 1.0) * sig[i];
        out[k] = s;
    }
}

// ---- upload: raw store + edge lines from a grid buffer (one thread per
// logical element: consecutive threads read consecutive addresses, which
// matters when the source is page-locked host memory read over the bus) ----
// grid holds patches [p0, p0 + count) (a chunk of the shard's grid buffer).
__global__ void k_upload(const double* grid, uint32_t N, ShardGeom g, uint32_t p0, uint32_t count,
                         unsigned char* store, DirEntry* dir, EdgeSet e) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t per = (uint64_t)N * N;
    if (t >= (uint64_t)count * g.m * per) return;
    const uint64_t lq = t / per;                   // local patch * m + q
    const uint64_t pq = (uint64_t)p0 * g.m + lq;  // patch * m + q
    const uint32_t i = (uint32_t)((t % per) / N), j = (uint32_t)(t % N);
    const uint32_t p = (uint32_t)(pq / g.m), q = (uint32_t)(pq % g.m);
    const uint64_t TP = N + 2, tcount = TP * TP;
    const uint64_t block = round16(per * 8);
    const uint64_t off = pq * block;
    const double x = grid[lq * tcount + (i + 1) * TP + j + 1];
    reinterpret_cast<double*>(store + off)[(uint64_t)i * N + j] = x;
    if (i == 0 && j == 0) dir[pq] = DirEntry{off, 0u, DIR_RAW};
    const uint32_t ar = p / g.P1, b = p % g.P1;
    const bool lbm3 = g.me != g.m;  // D2Q9 edges with the 3 crossing populations
    const int s_rl = lbm3 ? lbm_slot_rowlo((int)q) : (int)q, s_rh = lbm3 ? lbm_slot_rowhi((int)q) : (int)q;
    const int s_cl = lbm3 ? lbm_slot_collo((int)q) : (int)q, s_ch = lbm3 ? lbm_slot_colhi((int)q) : (int)q;
    auto ix = [&](uint32_t slot, int c) { return (((uint64_t)slot * g.P1 + b) * g.me + c) * N; };
    if (i == 1 && s_rl >= 0) e.rowlo[ix(ar + 1, s_rl) + j] = x;
    if (i == N - 2 && s_rh >= 0) e.rowhi[ix(ar + 1, s_rh) + j] = x;
    if (j == 1 && s_cl >= 0) e.collo[ix(ar, s_cl) + i] = x;
    if (j == N - 2 && s_ch >= 0) e.colhi[ix(ar, s_ch) + i] = x;
}

// ---- edge lines of patches [p0, p0 + count) from their decoded grid buffer
// (the ghost-ring sources of the next step; same mapping as k_upload) -------
__global__ void k_edges_from_grid(const double* grid, uint32_t N, ShardGeom g, uint32_t p0, uint32_t count,
                                  EdgeSet e) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t per = (uint64_t)N * N;
    if (t >= (uint64_t)count * g.m * per) return;
    const uint64_t pq = t / per;
    const uint32_t i = (uint32_t)((t % per) / N), j = (uint32_t)(t % N);
    if (!(i == 1 || i == N - 2 || j == 1 || j == N - 2)) return;
    const uint32_t p = p0 + (uint32_t)(pq / g.m), q = (uint32_t)(pq % g.m);
    const uint64_t TP = N + 2, tcount = TP * TP;
    const double x = grid[pq * tcount + (i + 1) * TP + j + 1];
    const uint32_t ar = p / g.P1, b = p % g.P1;
    const bool lbm3 = g.me != g.m;
    const int s_rl = lbm3 ? lbm_slot_rowlo((int)q) : (int)q, s_rh = lbm3 ? lbm_slot_rowhi((int)q) : (int)q;
    const int s_cl = lbm3 ? lbm_slot_collo((int)q) : (int)q, s_ch = lbm3 ? lbm_slot_colhi((int)q) : (int)q;
    auto ix = [&](uint32_t slot, int c) { return (((uint64_t)slot * g.P1 + b) * g.me + c) * N; };
    if (i == 1 && s_rl >= 0) e.rowlo[ix(ar + 1, s_rl) + j] = x;
    if (i == N - 2 && s_rh >= 0) e.rowhi[ix(ar + 1, s_rh) + j] = x;
    if (j == 1 && s_cl >= 0) e.collo[ix(ar, s_cl) + i] = x;
    if (j == N - 2 && s_ch >= 0) e.colhi[ix(ar, s_ch) + i] = x;
}

// ---- SWE: the first time step from the uploaded state (cfl_dt,
// solver.hpp:242-258; dt = min(dt, t_end - 0), pipeline.hpp:195-196).  The
// max is exact, so a grid-wide atomic max of the (positive) double bits is
// the reference's value bit for bit.
__global__ void k_swe_vmax(const double* grid, uint32_t N, uint64_t npatch, double gravity,
                           unsigned long long* vmax_bits, unsigned* err) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t per = (uint64_t)N * N;
    double v = 0.0;
    if (t < npatch * per) {
        const uint64_t p = t / per;
        const uint32_t i = (uint32_t)((t % per) / N), j = (uint32_t)(t % N);
        const uint64_t TP = N + 2, tcount = TP * TP, o = (i + 1) * TP + j + 1;
        const double* base = grid + p * 3 * tcount;
        const double h = base[o];
        if (h <= 0.0) atomicOr(err, ERR_DOMAIN);
        const double c = sqrt(gravity * h);
        const double u = fabs(base[tcount + o] / h), w = fabs(base[2 * tcount + o] / h);
        v = fmax(u + c, w + c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) atomicMax(vmax_bits, (unsigned long long)__double_as_longlong(v));
}

// ---- Codec::lz metrics (codec.hpp:81-244): the byte size of lz_encode of
// every block's coefficient array — the warp parse of lz.cuh without
// emitting the bytes. ------------------------------------------------------

// The step's LZ row: the sizes are summed by atomics (integers: any order
// gives the same sum) and the last warp writes compressed_bytes and ratio
// (pipeline.hpp:270-272).  SWE (device clock): a launch is live only if the
// step kernel before it advanced the step counter; its row is rows_at[k - 1]
// and state[0] remembers the last row finalized, so a no-op launch changes
// nothing.
struct LzFinal {
    unsigned long long* state;  // [0] last SWE row done, [1] running sum, [2] warps done (both back to 0 after)
    wg_metrics_row* row;        // the step's row (transport, D2Q9)
    wg_metrics_row* rows_at;    // SWE: the row buffer shifted by the session's row0
    const unsigned long long* steps;  // SWE: the device step counter, else null
};

// LzStream::byte_size of every block (chunks of 64 KiB: 8 + payload each):
// one warp per block, a 16 KiB shared-memory hash table per warp, the block
// read through L2 (it was written by the step kernel just before).
constexpr int kLzWarps = 2;  // per CTA: 32 KiB of tables, 7 CTAs (14 warps) per SM
__global__ void __launch_bounds__(32 * kLzWarps) k_lz_sizes(const double* dense, uint64_t nblocks, uint32_t nn,
                                                            uint32_t chunk, LzFinal f) {
    __shared__ __align__(16) unsigned short tables[kLzWarps][8192];
    unsigned long long k = 0;
    if (f.steps) {
        k = *f.steps;
        if (k <= f.state[0]) return;  // uniform: the step launch was a no-op
    }
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
    const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
    unsigned short* table = tables[threadIdx.x / 32];
    unsigned long long sum = 0;
    for (uint64_t b = wid; b < nblocks; b += nw) {
        const unsigned char* in = reinterpret_cast<const unsigned char*>(dense + b * nn);
        const uint32_t bytes = nn * 8;
        // RunConfig::chunk_size (lz_encode, codec.hpp:223-235); a block is at
        // most 65^2 x 8 = 33800 bytes, so every chunk parses with 16-bit
        // table positions whatever the configured size
        for (uint32_t off = 0; off < bytes; off += chunk) {
            const uint32_t len = min(chunk, bytes - off);
            sum += 8 + lz_chunk_warp<unsigned short>(in + off, len, table, nullptr);
        }
    }
    if ((threadIdx.x & 31) != 0) return;
    atomicAdd(&f.state[1], sum);
    __threadfence();
    if (atomicAdd(&f.state[2], 1ull) != nw - 1) return;
    __threadfence();
    const unsigned long long tot = atomicAdd(&f.state[1], 0ull);
    wg_metrics_row* row = f.steps ? f.rows_at + (k - 1) : f.row;
    row->compressed_bytes = tot;
    row->ratio = tot > 0 ? (double)row->dense_bytes / (double)tot : 1.0;
    f.state[1] = 0;
    f.state[2] = 0;
    if (f.steps) f.state[0] = k;
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// Checkpoint: the raw blocks of a batch gathered back to back (block k from
// pool offset src[k], or the constant with the bits cst[k] when src[k] is
// ~0), for the device LZ encoder.
__global__ void k_gather_raw(const unsigned char* pool, const uint64_t* src, const unsigned long long* cst,
                             uint64_t rawb, unsigned char* dst) {
    const uint64_t k = blockIdx.x;
    unsigned char* d = dst + k * rawb;
    if (src[k] == ~0ull) {
        const double c = __longlong_as_double((long long)cst[k]);
        for (uint64_t i = threadIdx.x; i < rawb / 8; i += blockDim.x) reinterpret_cast<double*>(d)[i] = c;
    } else {
        const double* s = reinterpret_cast<const double*>(pool + src[k]);
        for (uint64_t i = threadIdx.x; i < rawb / 8; i += blockDim.x) reinterpret_cast<double*>(d)[i] = s[i];
    }
}

// ---- peer halo mode (multi-GPU): the step kernels store the halo lines into
// the ring neighbours' halo slots themselves (EdgeSet::peer_lo/peer_hi); a
// step may start once both neighbours delivered the same generation of edge
// lines, and announces its own when it is complete. -------------------------
__global__ void k_peer_signal(unsigned long long* to_above, unsigned long long* to_below, unsigned long long gen) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_above), "l"(gen) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_below), "l"(gen) : "memory");
}

// Bounded wait (10 s): a neighbour that never delivers becomes an error, not a hang.
__global__ void k_peer_wait(const unsigned long long* flags, unsigned long long gen, unsigned* err) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long a, b;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(flags) : "memory");
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(b) : "l"(flags + 1) : "memory");
        if (a >= gen && b >= gen) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10000000000ull) {
            atomicOr(err, ERR_PEER_TIMEOUT);
            return;
        }
        __nanosleep(200);
    }
}

__global__ void k_swe_clock_reset(double* td, unsigned long long* vmax_bits, unsigned long long* steps) {
    td[0] = 0.0;
    td[1] = 0.0;
    vmax_bits[1] = 0ull;  // vmax_bits[0]: the uploaded state's (k_swe_vmax)
    *steps = 0ull;
}

}  // namespace

// ---- strict mode: shared boundary cells of component 0 agree between the
// patches that own them (assemble(grid, 0), patchgrid.hpp:205-239: tolerance
// tol * max(|a|, |b|, 1)); grid = the decoded shard (grid-buffer layout).
// Only neighbours inside the shard are compared (assemble's global field has
// no periodic identification of its first and last points).
__global__ void k_check_shared(const double* grid, uint32_t N, ShardGeom g, double tol, unsigned* err) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t per = (uint64_t)g.m * (N + 2) * (N + 2), TP = N + 2;
    if (t >= (uint64_t)g.npatch * N * 2) return;
    const uint32_t p = (uint32_t)(t / (2ull * N)), k = (uint32_t)(t % N), side = (uint32_t)((t / N) & 1);
    const uint32_t ar = p / g.P1, b = p % g.P1;
    double x, y;
    if (side == 0) {  // right neighbour: my column N-1 == its column 0
        if (b + 1 >= g.P1) return;
        x = grid[p * per + (k + 1) * TP + N];
        y = grid[(uint64_t)(p + 1) * per + (k + 1) * TP + 1];
    } else {  // below neighbour: my row N-1 == its row 0
        if (ar + 1 >= g.R) return;
        x = grid[p * per + N * TP + k + 1];
        y = grid[(uint64_t)(p + g.P1) * per + TP + k + 1];
    }
    const double scale = fmax(fmax(fabs(x), fabs(y)), 1.0);
    if (!(fabs(x - y) <= tol * scale)) atomicOr(err, ERR_CONSISTENCY);
}

// ---- the session -------------------------------------------------------------
struct Session {
    wg_run_config cfg{};
    wg_shard shard{};
    RunGeometry geo;
    ShardGeom sg{};
    uint32_t N = 0;
    int levels = 0;
    KernelSet ks{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;

    // device memory
    unsigned char* store[2] = {nullptr, nullptr};
    DirEntry* dir[2] = {nullptr, nullptr};
    EdgeSet edges[2]{};
    double* edge_mem[2] = {nullptr, nullptr};
    StepPartial* partials = nullptr;     // per CTA of the step launch
    // peer halo mode: [0] edge generation delivered by the above neighbour, [1] by the below one
    unsigned long long* peer_flags = nullptr;
    unsigned long long* sig_above = nullptr;  // the above neighbour's word [1]
    unsigned long long* sig_below = nullptr;  // the below neighbour's word [0]
    unsigned long long peer_gen = 0;          // edge generations this session delivered
    bool peers = false;
    unsigned* done = nullptr;            // CTA completion counter
    double* scratch = nullptr;           // D2Q9 per-CTA staging (L2-resident)
    unsigned grid = 0;                   // launch grid of the step kernels
    unsigned long long* bump = nullptr;  // [2]
    unsigned* err = nullptr;
    unsigned* work = nullptr;       // SWE: dynamic patch counter
    double* patch_mass = nullptr;   // SWE: per-patch masses [npatch][2]
    wg_metrics_row* rows = nullptr;
    double* mass_fv = nullptr;
    uint64_t row_cap = 0;
    uint64_t cap = 0;  // bytes per pool
    uint64_t chunk = 0;  // per-CTA sub-allocation chunk
    uint64_t device_bytes = 0;
    // SWE device clock: [t, last dt] (f64), vmax bits [2], steps done (u64)
    unsigned long long* swe = nullptr;
    unsigned long long* phase = nullptr;  // per-phase cycle sums [32] (phase_mark, patch_phases.cuh)
    // Codec::lz metrics staging
    double* lz_dense = nullptr;
    unsigned long long* lz_done = nullptr;  // LzFinal::state
    uint32_t lz_ctas = 0;
    // pinned-host upload pipeline (created on first use)
    double* stage = nullptr;
    // row-chunk staging of the streamed first step / chunked download (D2Q9)
    double* rstage[3] = {nullptr, nullptr, nullptr};
    uint32_t rstage_rows = 0;
    cudaEvent_t rstage_ev[6] = {};
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t stage_ev[4] = {};
    uint64_t launched = 0;  // SWE step launches (steps past t_end are no-ops)
    uint64_t row0 = 0;      // step count at upload/load: rows[k] holds step row0 + k + 1

    int cur = 0;  // pool/edges holding the current state
    uint64_t step = 0;
    double time = 0.0;
    double thr[(kMaxLevels + 1) * (kMaxLevels + 1)] = {};
    double mass_a[kMaxN] = {};

    // optional per-launch timing of the fused kernel (bench roofline)
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_main;

    ~Session() { release(); }

    cudaEvent_t take_event() {
        cudaEvent_t e;
        if (!ev_pool.empty()) {
            e = ev_pool.back();
            ev_pool.pop_back();
        } else {
            WG_CUDA(cudaEventCreate(&e));
        }
        return e;
    }

    void clear_profile() {
        for (auto& pr : ev_main) {
            ev_pool.push_back(pr.first);
            ev_pool.push_back(pr.second);
        }
        ev_main.clear();
    }

    void release() {
        if (stream) cudaStreamSynchronize(stream);
        clear_profile();
        for (auto e : ev_pool) cudaEventDestroy(e);
        ev_pool.clear();
        for (int k = 0; k < 2; ++k) {
            cudaFree(store[k]);
            cudaFree(dir[k]);
            cudaFree(edge_mem[k]);
            store[k] = nullptr;
            dir[k] = nullptr;
            edge_mem[k] = nullptr;
        }
        cudaFree(partials);
        cudaFree(peer_flags);
        peer_flags = nullptr;
        cudaFree(done);
        cudaFree(work);
        work = nullptr;
        cudaFree(patch_mass);
        patch_mass = nullptr;
        cudaFree(scratch);
        scratch = nullptr;
        cudaFree(bump);
        cudaFree(err);
        cudaFree(rows);
        cudaFree(mass_fv);
        cudaFree(swe);
        swe = nullptr;
        cudaFree(phase);
        phase = nullptr;
        if (copy_stream) {
            cudaStreamSynchronize(copy_stream);
            for (auto& ev : stage_ev) cudaEventDestroy(ev);
            cudaStreamDestroy(copy_stream);
            copy_stream = nullptr;
        }
        cudaFree(stage);
        stage = nullptr;
        for (auto& b : rstage) {
            cudaFree(b);
            b = nullptr;
        }
        for (auto& ev : rstage_ev)
            if (ev) {
                cudaEventDestroy(ev);
                ev = nullptr;
            }
        cudaFree(lz_dense);
        cudaFree(lz_done);
        lz_done = nullptr;
        lz_dense = nullptr;
        partials = nullptr;
        done = nullptr;
        bump = nullptr;
        err = nullptr;
        rows = nullptr;
        mass_fv = nullptr;
        if (own_stream && stream) cudaStreamDestroy(stream);
        stream = nullptr;
    }

    template <typename T>
    T* dalloc(uint64_t count) {
        T* p = nullptr;
        if (count) {
            WG_CUDA(cudaMalloc(&p, count * sizeof(T)));
            device_bytes += count * sizeof(T);
        }
        return p;
    }

    bool is_swe() const { return cfg.scheme == WG_SCHEME_SWE; }
    // patches per staging chunk of a pinned-host upload (16 MB of grid buffer)
    // LZ chunk bytes (RunConfig::chunk_size), clamped to 32 bits: a block is
    // far smaller, so a larger chunk is the same single chunk
    uint32_t lz_chunk() const { return (uint32_t)std::min<uint64_t>(cfg.lz_chunk_size, 0xFFFFFFFFull); }
    uint32_t stage_chunk() const {
        return (uint32_t)std::max<uint64_t>(1, (16ull << 20) / ((uint64_t)sg.m * geo.tcount * 8));
    }
    double* swe_td() const { return reinterpret_cast<double*>(swe); }

    uint64_t halo_doubles() const { return (uint64_t)sg.P1 * sg.me * N; }

    void create(const wg_run_config& c, const wg_shard* sh, void* strm) {
        cfg = c;
        if (cfg.codec != 1 && cfg.codec != 2) raise(WG_INVALID_ARGUMENT, "unknown codec");
        if (cfg.codec == 2 && cfg.lz_chunk_size == 0) raise(WG_INVALID_ARGUMENT, "lz_encode: chunk_size must be > 0");

        if (cfg.scheme != WG_SCHEME_LBM_D2Q9) sim_validate(cfg);
        if (cfg.scheme == WG_SCHEME_LBM_D2Q9 && cfg.lbm_tau <= 0.5)
            raise(WG_INVALID_ARGUMENT, "LBM: tau must exceed 1/2");
        geo = run_geometry(cfg);
        if (geo.n[0] != geo.n[1]) raise(WG_INVALID_ARGUMENT, "device session: square patches only");
        N = (uint32_t)geo.n[0];
        levels = cfg.levels;
        const uint64_t dims[2] = {geo.n[0], geo.n[1]};
        plan_validate(dims, 2, levels);  // WaveletPlan{logical, levels}.validate(), pipeline.hpp:135-136
        if (cfg.c < 0.0) raise(WG_INVALID_ARGUMENT, "apply_threshold: c must be >= 0");
        if (cfg.threshold_mode < 0 || cfg.threshold_mode > 2)
            raise(WG_INVALID_ARGUMENT, "band_threshold: unknown mode");
        if (sh) shard = *sh;
        else {
            shard.rank = 0;
            shard.world = 1;
            WG_CUDA(cudaGetDevice(&shard.device));
            shard.row_begin = 0;
            shard.row_end = geo.splits[0];
        }
        if (shard.world < 1 || shard.row_begin >= shard.row_end || shard.row_end > geo.splits[0])
            raise(WG_INVALID_ARGUMENT, "wg_shard: bad patch-row range");
        WG_CUDA(cudaSetDevice(shard.device));
        if (strm) stream = static_cast<cudaStream_t>(strm);
        else {
            WG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
            own_stream = true;
        }
        sg.R = (uint32_t)(shard.row_end - shard.row_begin);
        sg.P1 = (uint32_t)geo.splits[1];
        sg.m = geo.m;
        sg.world = shard.world;
        sg.npatch = sg.R * sg.P1;
        sg.row0 = (uint32_t)shard.row_begin;
        ks = select_kernels(cfg.scheme, N, levels, (uint64_t)(shard.row_end - shard.row_begin) * geo.splits[1]);
        sg.me = ks.edges3 ? 3u : sg.m;
        {
            int per_sm = 0, sms = 0;
            WG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, shard.device));
            const uint64_t groups = (sg.npatch + ks.P - 1) / ks.P;
            uint64_t resident = 0;
            if (ks.cluster > 1) {  // co-resident clusters (one patch per cluster)
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3((unsigned)(ks.cluster * sms), 1, 1);
                lc.blockDim = dim3((unsigned)ks.threads, 1, 1);
                lc.dynamicSmemBytes = ks.smem;
                cudaLaunchAttribute at{};
                at.id = cudaLaunchAttributeClusterDimension;
                at.val.clusterDim.x = (unsigned)ks.cluster;
                at.val.clusterDim.y = 1;
                at.val.clusterDim.z = 1;
                lc.attrs = &at;
                lc.numAttrs = 1;
                int clusters = 0;
                WG_CUDA(cudaOccupancyMaxActiveClusters(&clusters, reinterpret_cast<const void*>(ks.main), &lc));
                resident = (uint64_t)std::max(clusters, 1);
            } else {
                WG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks.main, ks.threads, ks.smem));
                resident = (uint64_t)std::max(per_sm, 1) * sms;
            }
            if (const char* f = std::getenv("WG_GRID_WAVES"))  // test knob: fewer CTAs, many patches each
                resident = (uint64_t)std::max(1.0, std::atof(f) * (double)resident);
            grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(groups, resident)) * (unsigned)ks.cluster;
            if (ks.scratch_doubles) scratch = dalloc<double>((uint64_t)grid * ks.scratch_doubles);
        }
        // thresholds (threshold.hpp:31-47) — the "c == 0 or levels == 0"
        // early return of apply_threshold (threshold.hpp:53) is T = 0.
        if (cfg.c == 0.0 || levels == 0) std::fill(std::begin(thr), std::end(thr), 0.0);
        else threshold_table_2d(levels, cfg.threshold_mode, cfg.c, cfg.threshold_alpha, thr);
        inverse_trapezoid_functional(N, levels, mass_a);

        const uint64_t raw_block = round16((uint64_t)N * N * 8);
        const uint64_t blocks = (uint64_t)sg.npatch * sg.m;
        // per-CTA sub-allocation chunk: big enough to amortise the global
        // atomic, small enough that the unused tails (<= one chunk per CTA)
        // stay a small fraction of the pool
        chunk = std::clamp<uint64_t>(round16(blocks * raw_block / (8ull * grid)), 4096, 256 * 1024);
        // without a budget the pools hold the worst case, every block a dense
        // CSR block (12 N^2 + 4 (N + 1) bytes: 1.5x raw) — a valid run of the
        // reference never overflows the store, whatever the threshold
        const uint64_t csr_max = round16(12ull * N * N + 4ull * (N + 1));
        cap = cfg.store_budget_bytes ? cfg.store_budget_bytes / 2 : blocks * csr_max + (uint64_t)grid * chunk;
        cap = std::max<uint64_t>(cap, 16) & ~uint64_t(15);
        for (int k = 0; k < 2; ++k) {
            store[k] = dalloc<unsigned char>(cap);
            dir[k] = dalloc<DirEntry>(blocks);
            const uint64_t rowline = (uint64_t)(sg.R + 2) * sg.P1 * sg.me * N;
            const uint64_t colline = (uint64_t)sg.R * sg.P1 * sg.me * N;
            edge_mem[k] = dalloc<double>(2 * rowline + 2 * colline);
            WG_CUDA(cudaMemsetAsync(edge_mem[k], 0, (2 * rowline + 2 * colline) * sizeof(double), stream));
            edges[k].rowlo = edge_mem[k];
            edges[k].rowhi = edge_mem[k] + rowline;
            edges[k].collo = edge_mem[k] + 2 * rowline;
            edges[k].colhi = edge_mem[k] + 2 * rowline + colline;
        }
        partials = dalloc<StepPartial>(grid);
        peer_flags = dalloc<unsigned long long>(2);
        WG_CUDA(cudaMemsetAsync(peer_flags, 0, 2 * sizeof(unsigned long long), stream));
        done = dalloc<unsigned>(1);
        bump = dalloc<unsigned long long>(2);
        err = dalloc<unsigned>(1);
        WG_CUDA(cudaMemsetAsync(done, 0, sizeof(unsigned), stream));
        WG_CUDA(cudaMemsetAsync(bump, 0, 2 * sizeof(unsigned long long), stream));
        WG_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned), stream));
        if (is_swe()) {
            swe = dalloc<unsigned long long>(5);
            WG_CUDA(cudaMemsetAsync(swe, 0, 5 * sizeof(unsigned long long), stream));
            work = dalloc<unsigned>(1);
            WG_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned), stream));
            patch_mass = dalloc<double>(2 * (uint64_t)sg.npatch);
        }
        phase = dalloc<unsigned long long>(32);
        WG_CUDA(cudaMemsetAsync(phase, 0, 32 * sizeof(unsigned long long), stream));
        grow_rows(1024);
        // D2Q9: the row-chunk staging of the streamed first step and the
        // chunked download, allocated up front (<= 1 GB) so that no allocation
        // happens between a session's steps and its readback
        if (ks.cluster > 1) ensure_row_stage();
        if (cfg.codec == 2 && !cfg.no_compression) {  // Codec::lz metrics (the store itself stays CSR)
            if (!ks.main_lz) raise(WG_INVALID_ARGUMENT, "Codec::lz metrics: not available for this kernel variant");
            const uint64_t nb = (uint64_t)sg.npatch * sg.m;
            if (nb * N * N * 8 > (8ull << 30))
                raise(WG_INVALID_ARGUMENT, "Codec::lz metrics: grid too large for the coefficient staging");
            lz_dense = dalloc<double>(nb * N * N + 1);  // + 8 B tail padding for the word loads
            lz_done = dalloc<unsigned long long>(3);
            WG_CUDA(cudaMemsetAsync(lz_done, 0, 3 * sizeof(unsigned long long), stream));
            int lz_per_sm = 0, lz_sms = 0;
            WG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lz_per_sm, k_lz_sizes, 32 * kLzWarps, 0));
            WG_CUDA(cudaDeviceGetAttribute(&lz_sms, cudaDevAttrMultiProcessorCount, shard.device));
            lz_ctas = (uint32_t)std::min<uint64_t>((nb + kLzWarps - 1) / kLzWarps,
                                                   (uint64_t)std::max(lz_per_sm, 1) * lz_sms);
        }
        // the pinned-host upload pipeline (allocated here, outside any timed upload)
        stage = dalloc<double>(2 * (uint64_t)stage_chunk() * sg.m * geo.tcount);
        WG_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
        for (auto& ev : stage_ev) WG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }

    void grow_rows(uint64_t need) {
        if (need <= row_cap) return;
        uint64_t nc = std::max<uint64_t>(need, row_cap * 2);
        wg_metrics_row* nr = nullptr;
        double* nm = nullptr;
        WG_CUDA(cudaMalloc(&nr, nc * sizeof(wg_metrics_row)));
        WG_CUDA(cudaMalloc(&nm, nc * sizeof(double)));
        if (rows) {
            WG_CUDA(cudaMemcpyAsync(nr, rows, row_cap * sizeof(wg_metrics_row), cudaMemcpyDeviceToDevice, stream));
            WG_CUDA(cudaMemcpyAsync(nm, mass_fv, row_cap * sizeof(double), cudaMemcpyDeviceToDevice, stream));
            WG_CUDA(cudaStreamSynchronize(stream));
            cudaFree(rows);
            cudaFree(mass_fv);
            device_bytes -= row_cap * (sizeof(wg_metrics_row) + sizeof(double));
        }
        rows = nr;
        mass_fv = nm;
        device_bytes += nc * (sizeof(wg_metrics_row) + sizeof(double));
        row_cap = nc;
    }

    // The raw initial store from a grid buffer in device memory, or (pinned
    // != nullptr) streamed from page-locked host memory: chunks of patches
    // copied by the DMA engine on a second stream while the previous chunk
    // is being stored (double-buffered staging).
    void upload_dev(const double* dgrid, const double* pinned = nullptr) {
        const uint64_t raw_block = round16((uint64_t)N * N * 8);
        const uint64_t need = (uint64_t)sg.npatch * sg.m * raw_block;
        if (need > cap)
            raise(WG_OUT_OF_MEMORY, "initial state does not fit the compressed-store budget");
        cur = 0;
        if (is_swe()) WG_CUDA(cudaMemsetAsync(swe + 2, 0, sizeof(unsigned long long), stream));
        const uint64_t per = (uint64_t)sg.m * geo.tcount;  // doubles per patch in the grid buffer
        auto store_chunk = [&](const double* src, uint32_t p0, uint32_t cnt) {
            const uint64_t threads = (uint64_t)cnt * sg.m * N * N;
            k_upload<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(src, N, sg, p0, cnt, store[cur], dir[cur],
                                                                             edges[cur]);
            WG_LAUNCH_CHECK("upload");
            if (is_swe()) {
                const uint64_t cells = (uint64_t)cnt * N * N;
                k_swe_vmax<<<(unsigned)((cells + 255) / 256), 256, 0, stream>>>(src, N, cnt, cfg.gravity, swe + 2,
                                                                                err);
                WG_LAUNCH_CHECK("swe wave speed");
            }
        };
        if (!pinned) {
            store_chunk(dgrid, 0, sg.npatch);
        } else {
            const uint32_t chunk = stage_chunk();
            const uint32_t nch = (sg.npatch + chunk - 1) / chunk;
            cudaEvent_t* copied = stage_ev;
            cudaEvent_t* consumed = stage_ev + 2;
            WG_CUDA(cudaEventRecord(consumed[0], stream));  // earlier work on the session stream first
            WG_CUDA(cudaEventRecord(consumed[1], stream));
            for (uint32_t c = 0; c < nch; ++c) {
                const int k = c & 1;
                const uint32_t p0 = c * chunk, cnt = std::min<uint32_t>(chunk, sg.npatch - p0);
                double* buf = stage + (uint64_t)k * chunk * per;
                WG_CUDA(cudaStreamWaitEvent(copy_stream, consumed[k], 0));
                WG_CUDA(cudaMemcpyAsync(buf, pinned + (uint64_t)p0 * per, (uint64_t)cnt * per * 8,
                                        cudaMemcpyHostToDevice, copy_stream));
                WG_CUDA(cudaEventRecord(copied[k], copy_stream));
                WG_CUDA(cudaStreamWaitEvent(stream, copied[k], 0));
                store_chunk(buf, p0, cnt);
                WG_CUDA(cudaEventRecord(consumed[k], stream));
            }
        }
        k_set_u64<<<1, 1, 0, stream>>>(bump + cur, need);  // no host round trip: steps queue behind
        WG_LAUNCH_CHECK("upload bump");
        WG_CUDA(cudaMemsetAsync(bump + (1 - cur), 0, sizeof(unsigned long long), stream));
        if (is_swe()) {
            k_swe_clock_reset<<<1, 1, 0, stream>>>(swe_td(), swe + 2, swe + 4);
            WG_LAUNCH_CHECK("swe clock");
        }
        if (lz_done) k_set_u64<<<1, 1, 0, stream>>>(lz_done, 0ull);
        step = 0;
        launched = 0;
        row0 = 0;
        time = 0.0;
    }

    void upload_host(const double* hgrid) {
        // page-locked host memory is streamed in chunks by the DMA engine
        // (overlapped with storing the previous chunk); pageable memory is
        // copied whole first
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, hgrid) == cudaSuccess && at.type == cudaMemoryTypeHost &&
            at.devicePointer) {
            upload_dev(nullptr, hgrid);
            return;
        }
        cudaGetLastError();  // clear a failed attribute query on pageable memory
        const uint64_t n = (uint64_t)sg.npatch * sg.m * geo.tcount;
        DevBuf<double> d(n);
        WG_CUDA(cudaMemcpyAsync(d.p, hgrid, n * sizeof(double), cudaMemcpyHostToDevice, stream));
        upload_dev(d.p);
        WG_CUDA(cudaStreamSynchronize(stream));  // d dies with this scope
    }

    // Initial state generated and compressed on the device (no host grid):
    // the compression cycle of a step applied to the initial state.
    void init_device() {
        if (!ks.init) raise(WG_INVALID_ARGUMENT, "device initial state: D2Q9 full-line kernels only");
        cur = 1;  // the kernel writes pool 0 (dst = 1 - cur)
        WG_CUDA(cudaMemsetAsync(bump, 0, 2 * sizeof(unsigned long long), stream));
        StepArgs a = step_args(1, 0);
        a.omega = 1.0 / cfg.lbm_tau;
        a.ic_u0 = cfg.lbm_u0;
        a.ic_kappa = cfg.lbm_kappa;
        a.ic_delta = cfg.lbm_delta;
        a.ic_inv = 1.0 / static_cast<double>(cfg.nx - 1);
        a.ic_period = geo.tiles > 1 ? cfg.nx - 1 : ~0ull;
        grow_rows(1);
        a.row_out = rows;  // the IC's metrics row is scratch (step counter stays 0)
        a.mass_fv_out = mass_fv;
        ks.init<<<grid, ks.threads, ks.smem, stream>>>(a);
        WG_LAUNCH_CHECK("device initial state");
        cur = 0;
        step = 0;
        row0 = 0;
        time = 0.0;
        sync();
    }

    // Peer halo mode.  above_mem/below_mem: the neighbours' edge allocations
    // (both buffer parities) and flag words, mapped into this process.
    void peer_attach(double* const above_mem[2], uint32_t above_rows, unsigned long long* above_flags,
                     double* const below_mem[2], uint32_t below_rows, unsigned long long* below_flags) {
        if (is_swe()) raise(WG_INVALID_ARGUMENT, "peer halos: transport and D2Q9 sessions only (SWE all-reduces its CFL speed)");
        if (sg.R == 0) raise(WG_INVALID_ARGUMENT, "peer halos: empty shard");
        const uint64_t line = halo_doubles();
        for (int k = 0; k < 2; ++k) {
            if (!above_mem[k] || !below_mem[k]) raise(WG_INVALID_ARGUMENT, "peer halos: null edge allocation");
            edges[k].peer_lo = above_mem[k] + (uint64_t)(above_rows + 1) * line;  // above's rowlo slot R+1
            edges[k].peer_hi = below_mem[k] + (uint64_t)(below_rows + 2) * line;  // below's rowhi slot 0
        }
        sig_above = above_flags + 1;
        sig_below = below_flags + 0;
        peers = true;
    }

    void peer_signal() {
        k_peer_signal<<<1, 1, 0, stream>>>(sig_above, sig_below, peer_gen + 1);
        WG_LAUNCH_CHECK("peer signal");
        ++peer_gen;
    }

    // The current edge lines' halo rows to the neighbours (after upload /
    // load, which build the edges locally), once both neighbours reached
    // this session's generation.
    void peer_push() {
        if (!peers) raise(WG_INVALID_ARGUMENT, "peer halos: no peers attached");
        k_peer_wait<<<1, 1, 0, stream>>>(peer_flags, peer_gen, err);
        const EdgeSet& e = edges[cur];
        const uint64_t line = halo_doubles();
        WG_CUDA(cudaMemcpyAsync(e.peer_lo, e.rowlo + line, line * sizeof(double), cudaMemcpyDeviceToDevice, stream));
        WG_CUDA(cudaMemcpyAsync(e.peer_hi, e.rowhi + (uint64_t)sg.R * line, line * sizeof(double),
                                cudaMemcpyDeviceToDevice, stream));
        peer_signal();
        sync();
    }

    StepArgs step_args(int src, int dst) const {
        StepArgs a{};
        a.store_in = store[src];
        a.dir_in = dir[src];
        a.ein = edges[src];
        a.store_out = store[dst];
        a.dir_out = dir[dst];
        a.eout = edges[dst];
        a.bump_out = bump + dst;
        a.bump_next = bump + src;
        a.cap_out = cap;
        a.edge_row_elems = (uint64_t)(sg.R + 2) * sg.P1 * sg.me * N;
        a.edge_col_elems = (uint64_t)sg.R * sg.P1 * sg.me * N;
        a.chunk = chunk;
        a.err = err;
        a.partials = partials;
        a.done = done;
        a.work = work;
        a.patch_mass = patch_mass;
        a.scratch = scratch;
        a.g = sg;
        a.compress = cfg.no_compression ? 0 : 1;
        a.thr_any = (cfg.c > 0.0 && levels > 0) ? 1 : 0;
        a.dense_bytes = (uint64_t)sg.npatch * 8ull * N * N * sg.m;
        a.phase = phase;
        a.lz_dense = lz_dense;
        if (is_swe()) {
            a.swe_td = swe_td();
            a.swe_vmax = swe + 2;
            a.swe_steps = swe + 4;
            a.t_end = cfg.t_end;
            a.cfl_dx = cfg.cfl * sim_dx(cfg);  // cfg.cfl * cfg.dx() (solver.hpp:257)
            a.dx = sim_dx(cfg);
            a.gravity = cfg.gravity;
        }
        std::memcpy(a.thr, thr, sizeof(thr));
        std::memcpy(a.mass_a, mass_a, sizeof(mass_a));
        a.raw_in = nullptr;
        a.p_begin = 0;
        a.p_end = sg.npatch;
        a.chunk_first = 1;
        a.chunk_last = 1;
        return a;
    }

    // One step launch.  SWE: dt is ignored — the step runs with the device
    // clock's dt, or does nothing once t_end is reached.
    void do_step(double dt) {
        if (is_swe()) {
            do_swe_step();
            return;
        }
        const int src = cur, dst = 1 - cur;
        grow_rows(step - row0 + 1);
        StepArgs a = step_args(src, dst);
        direction_speeds(cfg.alpha, cfg.beta, a.smax, a.smin);
        a.r = dt / sim_dx(cfg);  // solver.hpp:212
        a.omega = 1.0 / cfg.lbm_tau;
        a.step = step + 1;
        a.time = time + dt;
        a.row_out = rows + (step - row0);
        a.mass_fv_out = mass_fv + (step - row0);

        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (profiling) {
            e0 = take_event();
            e1 = take_event();
            WG_CUDA(cudaEventRecord(e0, stream));
        }
        if (peers) k_peer_wait<<<1, 1, 0, stream>>>(peer_flags, peer_gen, err);
        (lz_dense ? ks.main_lz : ks.main)<<<grid, ks.threads, ks.smem, stream>>>(a);
        WG_LAUNCH_CHECK("fused step");
        if (peers) peer_signal();
        if (profiling) {
            WG_CUDA(cudaEventRecord(e1, stream));
            ev_main.emplace_back(e0, e1);
        }
        if (lz_dense) {  // Codec::lz: the step's compressed_bytes/ratio from the LZ stream sizes
            k_lz_sizes<<<lz_ctas, 32 * kLzWarps, 0, stream>>>(lz_dense, (uint64_t)sg.npatch * sg.m, N * N, lz_chunk(),
                                                               LzFinal{lz_done, a.row_out, nullptr, nullptr});
            WG_LAUNCH_CHECK("lz sizes");
        }
        if (ks.decode_l2 && cfg.compute_l2 && geo.tiles == 1) {
            // l2_error(assemble(grid, 0), exact_transport(t), cfg) of the new
            // state (pipeline.hpp:275-276): a decode pass over the output pool
            StepArgs b = step_args(dst, src);
            b.decode_out = nullptr;
            b.time = a.time;
            b.row_out = a.row_out;
            b.l2_on = 1;
            b.l2_nx = cfg.nx;
            b.l2_scale = cfg.domain_length * cfg.domain_length / static_cast<double>(cfg.nx * cfg.nx);
            b.l2_dx = sim_dx(cfg);
            b.l2_alpha = cfg.alpha;
            b.l2_beta = cfg.beta;
            ks.decode<<<grid, ks.threads, ks.smem, stream>>>(b);
            WG_LAUNCH_CHECK("l2 pass");
        }
        cur = dst;
        ++step;
        time += dt;
    }

    void do_swe_step() {
        grow_rows(launched - row0 + 1);
        const int src = cur, dst = 1 - cur;
        StepArgs a = step_args(src, dst);
        a.row_out = rows - row0;  // indexed by the device step counter (>= row0)
        a.mass_fv_out = mass_fv - row0;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (profiling) {
            e0 = take_event();
            e1 = take_event();
            WG_CUDA(cudaEventRecord(e0, stream));
        }
        (lz_dense ? ks.main_lz : ks.main)<<<grid, ks.threads, ks.smem, stream>>>(a);
        WG_LAUNCH_CHECK("fused swe step");
        if (lz_dense) {
            const uint64_t nb = (uint64_t)sg.npatch * sg.m;
            k_lz_sizes<<<lz_ctas, 32 * kLzWarps, 0, stream>>>(lz_dense, nb, N * N, lz_chunk(),
                                                               LzFinal{lz_done, nullptr, rows - row0, swe + 4});
            WG_LAUNCH_CHECK("lz sizes");
        }
        if (profiling) {
            WG_CUDA(cudaEventRecord(e1, stream));
            ev_main.emplace_back(e0, e1);
        }
        ++launched;
        // a no-op launch leaves both pools untouched: the host learns which
        // pool is current from the device step counter (sync())
        cur = dst;
    }

    void sync() {
        WG_CUDA(cudaStreamSynchronize(stream));
        unsigned e = 0;
        WG_CUDA(cudaMemcpy(&e, err, sizeof e, cudaMemcpyDeviceToHost));
        check_device_error(e);
        if (is_swe()) {
            unsigned long long h[5];
            WG_CUDA(cudaMemcpy(h, swe, sizeof h, cudaMemcpyDeviceToHost));
            double t;
            std::memcpy(&t, &h[0], sizeof t);
            step = h[4];
            time = t;
            cur = (int)(step & 1);  // step k writes pool k & 1 (pool 0 holds the upload)
            launched = step;
        }
    }

    // Row-chunk staging (D2Q9): three device buffers of rstage_rows patch
    // rows of the grid-buffer layout each (~512 MB), allocated on first use.
    uint64_t row_doubles() const { return (uint64_t)sg.P1 * sg.m * geo.tcount; }
    void ensure_row_stage() {
        if (rstage[0]) return;
        const uint64_t per_row = row_doubles() * 8;
        rstage_rows = (uint32_t)std::clamp<uint64_t>((512ull << 20) / std::max<uint64_t>(per_row, 1), 1, sg.R);
        if (const char* e = std::getenv("WG_STREAM_ROWS"))  // test knob: rows per chunk
            rstage_rows = (uint32_t)std::clamp<long>(std::atol(e), 1, (long)sg.R);
        for (auto& b : rstage) b = dalloc<double>((uint64_t)rstage_rows * row_doubles());
        for (auto& ev : rstage_ev) WG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }

    // The first step of a run straight from a host initial state (grid-buffer
    // layout, page-locked or pageable): the raw state is never stored.  Patch
    // rows stream through the device in chunks (DMA on the copy stream); the
    // edge lines of a chunk are built when it arrives, and the step kernel
    // runs on the previous chunk with its raw input read from the staging
    // buffer (StepArgs::raw_in), so the store holds only the compressed
    // result — the reference's step 1 on its raw initial grid (pipeline.hpp:
    // 138-155, 194-289) under a store budget smaller than the raw state (C4).
    void step_from_host(const double* hgrid, double dt) {
        if (ks.cluster < 2 || sg.world != 1 || is_swe())
            raise(WG_INVALID_ARGUMENT, "streamed first step: one-shard D2Q9 sessions only");
        ensure_row_stage();
        // the state of an upload (wg_session_upload), without the raw store
        cur = 0;
        step = 0;
        row0 = 0;
        time = 0.0;
        WG_CUDA(cudaMemsetAsync(bump, 0, 2 * sizeof(unsigned long long), stream));
        if (lz_done) k_set_u64<<<1, 1, 0, stream>>>(lz_done, 0ull);
        const uint32_t R = sg.R, RC = rstage_rows, C = (R + RC - 1) / RC;
        cudaEvent_t* copied = rstage_ev;
        cudaEvent_t* consumed = rstage_ev + 3;
        for (int k = 0; k < 3; ++k) WG_CUDA(cudaEventRecord(consumed[k], stream));
        auto dma_edges = [&](int b, uint32_t r0, uint32_t nr) {
            WG_CUDA(cudaStreamWaitEvent(copy_stream, consumed[b], 0));
            WG_CUDA(cudaMemcpyAsync(rstage[b], hgrid + (uint64_t)r0 * row_doubles(), (uint64_t)nr * row_doubles() * 8,
                                    cudaMemcpyHostToDevice, copy_stream));
            WG_CUDA(cudaEventRecord(copied[b], copy_stream));
            WG_CUDA(cudaStreamWaitEvent(stream, copied[b], 0));
            const uint64_t threads = (uint64_t)nr * sg.P1 * sg.m * N * N;
            k_edges_from_grid<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(rstage[b], N, sg, r0 * sg.P1,
                                                                                      nr * sg.P1, edges[cur]);
            WG_LAUNCH_CHECK("streamed edges");
        };
        if (C > 1) {  // the last patch row first: the periodic ghost source of row 0
            dma_edges(2, R - 1, 1);
            WG_CUDA(cudaEventRecord(consumed[2], stream));
        }
        dma_edges(0, 0, std::min(RC, R));
        grow_rows(1);
        StepArgs a = step_args(0, 1);
        a.omega = 1.0 / cfg.lbm_tau;
        a.step = 1;
        a.time = dt;
        a.row_out = rows;
        a.mass_fv_out = mass_fv;
        for (uint32_t c = 0; c < C; ++c) {
            const uint32_t r0 = c * RC, nr = std::min(RC, R - r0);
            if (c + 1 < C) dma_edges((int)((c + 1) % 3), r0 + RC, std::min(RC, R - r0 - RC));
            a.raw_in = rstage[c % 3];
            a.p_begin = r0 * sg.P1;
            a.p_end = (r0 + nr) * sg.P1;
            a.chunk_first = c == 0;
            a.chunk_last = c + 1 == C;
            (lz_dense ? ks.main_lz : ks.main)<<<grid, ks.threads, ks.smem, stream>>>(a);
            WG_LAUNCH_CHECK("streamed step");
            WG_CUDA(cudaEventRecord(consumed[c % 3], stream));
        }
        if (lz_dense) {
            k_lz_sizes<<<lz_ctas, 32 * kLzWarps, 0, stream>>>(lz_dense, (uint64_t)sg.npatch * sg.m, N * N, lz_chunk(),
                                                               LzFinal{lz_done, a.row_out, nullptr, nullptr});
            WG_LAUNCH_CHECK("lz sizes");
        }
        cur = 1;
        step = 1;
        time = dt;
    }

    void download(double* hgrid) {
        if (is_swe()) sync();  // the current pool follows the device step counter
        if (ks.cluster > 1) {  // D2Q9: decoded in row chunks through the staging buffers
            ensure_row_stage();
            const uint32_t R = sg.R, RC = rstage_rows;
            for (uint32_t r0 = 0, c = 0; r0 < R; r0 += RC, ++c) {
                const uint32_t nr = std::min(RC, R - r0);
                const int b = (int)(c % 2);
                WG_CUDA(cudaEventSynchronize(rstage_ev[3 + b]));  // its previous copy-out is done
                WG_CUDA(cudaMemsetAsync(rstage[b], 0, (uint64_t)nr * row_doubles() * 8, stream));
                StepArgs a = step_args(cur, 1 - cur);
                a.decode_out = rstage[b];
                a.p_begin = r0 * sg.P1;
                a.p_end = (r0 + nr) * sg.P1;
                ks.decode<<<grid, ks.threads, ks.smem, stream>>>(a);
                WG_LAUNCH_CHECK("decode");
                WG_CUDA(cudaMemcpyAsync(hgrid + (uint64_t)r0 * row_doubles(), rstage[b],
                                        (uint64_t)nr * row_doubles() * 8, cudaMemcpyDeviceToHost, stream));
                WG_CUDA(cudaEventRecord(rstage_ev[3 + b], stream));
            }
            sync();
            return;
        }
        const uint64_t n = (uint64_t)sg.npatch * sg.m * geo.tcount;
        DevBuf<double> d(n);
        WG_CUDA(cudaMemsetAsync(d.p, 0, n * sizeof(double), stream));
        StepArgs a = step_args(cur, 1 - cur);
        a.decode_out = d.p;
        ks.decode<<<grid, ks.threads, ks.smem, stream>>>(a);
        WG_LAUNCH_CHECK("decode");
        WG_CUDA(cudaMemcpyAsync(hgrid, d.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
        sync();
    }

    // Shares of the step kernel's phase clocks in RunSummary's categories
    // {step, dwt, threshold, codec} (phase ids: lbm_pair.cuh, patch_kernels.cuh,
    // swe_kernels.cuh; a row pass is half transform, half threshold).
    void phase_shares(double out[4]) {
        unsigned long long h[32];
        WG_CUDA(cudaMemcpy(h, phase, sizeof h, cudaMemcpyDeviceToHost));
        double w[4] = {0, 0, 0, 0};
        auto add = [&](int k, int cat, double f = 1.0) { w[cat] += f * (double)h[k]; };
        if (ks.cluster > 1) {  // D2Q9 pair kernel
            for (int k : {12, 13, 14, 21, 22, 23, 24, 25}) add(k, 0);
            add(26, 1);
            add(27, 1, 0.5);
            add(27, 2, 0.5);
            for (int k : {28, 29, 30}) add(k, 3);
            add(31, 1);
        } else if (is_swe()) {
            for (int k : {0, 1, 2, 9, 11, 13, 14}) add(k, 0);
            add(4, 1);
            add(5, 1, 0.5);
            add(5, 2, 0.5);
            add(8, 1);
            for (int k : {6, 7}) add(k, 3);
        } else {  // transport
            for (int k : {0, 1, 2, 3, 9, 10, 11}) add(k, 0);
            add(4, 1);
            add(5, 1, 0.5);
            add(5, 2, 0.5);
            add(8, 1);
            for (int k : {6, 7}) add(k, 3);
        }
        const double tot = w[0] + w[1] + w[2] + w[3];
        for (int k = 0; k < 4; ++k) out[k] = tot > 0 ? w[k] / tot : 0.0;
    }

    // assemble(grid, 0)'s consistency check on the current state (strict
    // mode, pipeline.hpp:278-283): decode, compare the shared cells on the
    // device; raises WG_CONSISTENCY at the next sync.
    void check_shared(double tol) {
        if (is_swe()) sync();
        const uint64_t n = (uint64_t)sg.npatch * sg.m * geo.tcount;
        DevBuf<double> d(n);
        WG_CUDA(cudaMemsetAsync(d.p, 0, n * sizeof(double), stream));
        StepArgs a = step_args(cur, 1 - cur);
        a.decode_out = d.p;
        ks.decode<<<grid, ks.threads, ks.smem, stream>>>(a);
        WG_LAUNCH_CHECK("decode (strict)");
        const uint64_t threads = (uint64_t)sg.npatch * N * 2;
        k_check_shared<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(d.p, N, sg, tol, err);
        WG_LAUNCH_CHECK("strict shared cells");
        sync();  // d dies with this scope; raises WG_CONSISTENCY
    }

    void metrics(wg_metrics_row* out, uint64_t max_rows, uint64_t* nrows) {
        sync();
        const uint64_t n = std::min<uint64_t>(step - row0, max_rows);
        if (out && n) WG_CUDA(cudaMemcpy(out, rows, n * sizeof(wg_metrics_row), cudaMemcpyDeviceToHost));
        if (nrows) *nrows = step - row0;
    }

    // ---- checkpoint / resume from the compressed store -------
    // File: a WGS1 header, then one WGC1 record per patch exactly as
    // save_wgc writes a CompressedPatch (codec.hpp:364-391): compressed
    // patches as Codec::csr records of their CSR blocks (the bytes the
    // reference would write), raw patches (skip rule / initial state) as
    // Codec::lz records with levels 0 whose chunks are literal-only LZ
    // sequences (codec.hpp:81-89, decodable by lz_decode; -0.0 survives).
    struct CkptHeader {
        char magic[4];
        uint32_t version;
        int32_t scheme, levels;
        uint64_t nx, splits[2], tile_rows, row_begin, row_end, npatch, m, n, step;
        double time, swe_last_dt;
        uint64_t swe_vmax_bits;
    };

    void save(const char* path) {
        sync();
        const uint64_t blocks = (uint64_t)sg.npatch * sg.m;
        std::vector<DirEntry> hd(blocks);
        WG_CUDA(cudaMemcpy(hd.data(), dir[cur], blocks * sizeof(DirEntry), cudaMemcpyDeviceToHost));
        unsigned long long used = 0;
        WG_CUDA(cudaMemcpy(&used, bump + cur, sizeof used, cudaMemcpyDeviceToHost));
        std::vector<unsigned char> pool(used);
        if (used) WG_CUDA(cudaMemcpy(pool.data(), store[cur], used, cudaMemcpyDeviceToHost));
        CkptHeader h{};
        std::memcpy(h.magic, "WGS1", 4);
        h.version = 1;
        h.scheme = cfg.scheme;
        h.levels = levels;
        h.nx = cfg.nx;
        h.splits[0] = cfg.splits[0];
        h.splits[1] = cfg.splits[1];
        h.tile_rows = geo.tiles;
        h.row_begin = shard.row_begin;
        h.row_end = shard.row_end;
        h.npatch = sg.npatch;
        h.m = sg.m;
        h.n = N;
        h.step = step;
        h.time = time;
        if (is_swe()) {
            unsigned long long c[5];
            WG_CUDA(cudaMemcpy(c, swe, sizeof c, cudaMemcpyDeviceToHost));
            std::memcpy(&h.swe_last_dt, &c[1], sizeof(double));
            h.swe_vmax_bits = c[2 + (step & 1)];
        }
        std::unique_ptr<FILE, int (*)(FILE*)> fh(std::fopen(path, "wb"), &std::fclose);
        FILE* f = fh.get();
        if (!f) raise(WG_INVALID_ARGUMENT, std::string("cannot open for writing: ") + path);
        std::vector<unsigned char> out;
        auto put = [&](const void* p, size_t nb) {
            const unsigned char* c = static_cast<const unsigned char*>(p);
            out.insert(out.end(), c, c + nb);
        };
        auto put32 = [&](uint32_t v) { put(&v, 4); };
        auto put64 = [&](uint64_t v) { put(&v, 8); };
        put(&h, sizeof h);
        const uint64_t nn = (uint64_t)N * N, rawb = nn * 8;
        // lz_encode of every raw block (one 64 KiB chunk each: a block is
        // smaller) by the device encoder (lz.cuh), in batches of <= 512 MB
        // taken in record order: the file's raw records are the reference's
        // own lz_encode output of the block bytes (codec.hpp:223-235)
        std::vector<uint64_t> raw_src;
        std::vector<unsigned long long> raw_cst;
        for (uint64_t p = 0; p < sg.npatch; ++p) {
            const DirEntry* e = &hd[p * sg.m];
            bool raw = false;
            for (uint32_t q = 0; q < sg.m; ++q) raw = raw || (e[q].flags & DIR_RAW);
            if (!raw) continue;
            for (uint32_t q = 0; q < sg.m; ++q) {
                const bool cst = (e[q].flags & DIR_CONST) != 0;
                raw_src.push_back(cst ? ~0ull : e[q].off);
                raw_cst.push_back(cst ? (unsigned long long)e[q].off : 0ull);
            }
        }
        const uint64_t batch = std::max<uint64_t>(1, (512ull << 20) / rawb);
        uint64_t raw_next = 0, batch_first = 0;
        std::vector<uint64_t> enc_len;
        std::vector<unsigned char> enc_pl;
        std::vector<uint64_t> enc_off;
        auto raw_payload = [&](const unsigned char** pl, uint64_t* len) {
            if (raw_next == batch_first + enc_len.size()) {  // encode the next batch
                batch_first = raw_next;
                const uint64_t nb = std::min<uint64_t>(batch, raw_src.size() - batch_first);
                DevBuf<uint64_t> d_src(nb);
                DevBuf<unsigned long long> d_cst(nb);
                d_src.upload(raw_src.data() + batch_first);
                d_cst.upload(raw_cst.data() + batch_first);
                DevBuf<unsigned char> d_raw(nb * rawb + 16);
                WG_CUDA(cudaMemset(d_raw.p + nb * rawb, 0, 16));
                k_gather_raw<<<(unsigned)nb, 256, 0, stream>>>(store[cur], d_src.p, d_cst.p, rawb, d_raw.p);
                WG_LAUNCH_CHECK("checkpoint gather");
                WG_CUDA(cudaStreamSynchronize(stream));
                lz_encode_device(d_raw.p, nb * rawb, rawb, enc_len, &enc_pl);
                enc_off.assign(nb, 0);
                for (uint64_t k = 1; k < nb; ++k) enc_off[k] = enc_off[k - 1] + enc_len[k - 1];
            }
            const uint64_t k = raw_next++ - batch_first;
            *pl = enc_pl.data() + enc_off[k];
            *len = enc_len[k];
        };
        for (uint64_t p = 0; p < sg.npatch; ++p) {
            const DirEntry* e = &hd[p * sg.m];
            bool raw = false;
            for (uint32_t q = 0; q < sg.m; ++q) {
                if (e[q].flags & DIR_DEAD)
                    raise(WG_OUT_OF_MEMORY, "checkpoint: the store holds blocks lost to an overflow");
                raw = raw || (e[q].flags & DIR_RAW);
            }
            put("WGC1", 4);
            put32(raw ? 2u : 1u);  // Codec::lz / Codec::csr
            put32(2);
            put32(N);
            put32(N);
            put32(sg.m);
            put32(raw ? 0u : (uint32_t)levels);
            for (uint32_t q = 0; q < sg.m; ++q) {
                const bool cst = (e[q].flags & DIR_CONST) != 0;
                if (!cst && e[q].off + (raw ? rawb : 12ull * e[q].nnz + 4ull * (N + 1)) > used)
                    raise(WG_CORRUPT_STREAM, "checkpoint: directory entry outside the pool");
                const unsigned char* b = pool.data() + (cst ? 0 : e[q].off);  // CSR blocks only (raw: encoded above)
                if (raw) {
                    if (!(e[q].flags & DIR_RAW)) raise(WG_LOGIC, "checkpoint: mixed raw/CSR patch");
                    const unsigned char* pl = nullptr;
                    uint64_t pl_len = 0;
                    raw_payload(&pl, &pl_len);
                    put64(64 * 1024);  // LzStream: chunk_size, one chunk (rawb < 64 KiB)
                    put64(1);
                    put32((uint32_t)rawb);
                    put32((uint32_t)pl_len);
                    put(pl, pl_len);
                } else {
                    const uint32_t nz = e[q].nnz;
                    put32(N);
                    put32(N);
                    put64(nz);
                    put(b, 8ull * nz);
                    put64(nz);
                    put(b + 8ull * nz, 4ull * nz);
                    put64(N + 1);
                    put(b + 12ull * nz, 4ull * (N + 1));
                }
            }
            if (out.size() > (64u << 20)) {
                if (std::fwrite(out.data(), 1, out.size(), f) != out.size())
                    raise(WG_INVALID_ARGUMENT, "checkpoint: write failed");
                out.clear();
            }
        }
        const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
        if (std::fclose(fh.release()) != 0 || !ok) raise(WG_INVALID_ARGUMENT, "checkpoint: write failed");
    }

    void load(const char* path) {
        FILE* f = std::fopen(path, "rb");
        if (!f) raise(WG_INVALID_ARGUMENT, std::string("cannot open: ") + path);
        std::vector<unsigned char> in;
        {
            unsigned char buf[1 << 16];
            size_t k;
            while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) in.insert(in.end(), buf, buf + k);
            std::fclose(f);
        }
        size_t pos = 0;
        auto get = [&](void* p, size_t nb) {
            if (pos + nb > in.size()) raise(WG_CORRUPT_STREAM, "unexpected end of stream");
            std::memcpy(p, in.data() + pos, nb);
            pos += nb;
        };
        auto get32 = [&] { uint32_t v; get(&v, 4); return v; };
        auto get64 = [&] { uint64_t v; get(&v, 8); return v; };
        CkptHeader h;
        get(&h, sizeof h);
        if (std::memcmp(h.magic, "WGS1", 4) != 0 || h.version != 1) raise(WG_CORRUPT_STREAM, "not a WGS1 checkpoint");
        if (h.scheme != cfg.scheme || h.levels != levels || h.nx != cfg.nx || h.splits[0] != cfg.splits[0] ||
            h.splits[1] != cfg.splits[1] || h.tile_rows != geo.tiles || h.row_begin != shard.row_begin ||
            h.row_end != shard.row_end || h.npatch != sg.npatch || h.m != sg.m || h.n != N)
            raise(WG_INVALID_ARGUMENT, "checkpoint: written for a different configuration or shard");
        const uint64_t blocks = (uint64_t)sg.npatch * sg.m, nn = (uint64_t)N * N, rawb = nn * 8;
        std::vector<DirEntry> hd(blocks);
        std::vector<unsigned char> pool;
        pool.reserve(std::min<uint64_t>(cap, in.size() + blocks * 16));
        for (uint64_t p = 0; p < sg.npatch; ++p) {
            char mg[4];
            get(mg, 4);
            if (std::memcmp(mg, "WGC1", 4) != 0) raise(WG_CORRUPT_STREAM, "not a WGC1 file");
            const uint32_t codec = get32();
            if (codec != 1 && codec != 2) raise(WG_CORRUPT_STREAM, "unknown codec id");
            const uint32_t nd = get32();
            if (nd != 2) raise(WG_INVALID_ARGUMENT, "checkpoint: patch rank");
            const uint32_t d0 = get32(), d1 = get32(), comps = get32(), lv = get32();
            if (d0 != N || d1 != N || comps != sg.m) raise(WG_INVALID_ARGUMENT, "checkpoint: patch shape");
            if ((codec == 1 && lv != (uint32_t)levels) || (codec == 2 && lv != 0))
                raise(WG_INVALID_ARGUMENT, "checkpoint: record levels do not match the session");
            for (uint32_t q = 0; q < sg.m; ++q) {
                const uint64_t off = round16(pool.size());
                pool.resize(off);
                DirEntry& e = hd[p * sg.m + q];
                e.off = off;
                if (codec == 1) {  // CsrBlock (codec.hpp:62-79 checks)
                    const uint32_t rows = get32(), cols = get32();
                    if (rows != N || cols != N) raise(WG_CORRUPT_STREAM, "csr_decode: block shape");
                    const uint64_t nv = get64();
                    if (nv > nn) raise(WG_CORRUPT_STREAM, "csr_decode: too many entries");
                    pool.resize(off + 12ull * nv + 4ull * (N + 1));
                    get(pool.data() + off, 8ull * nv);
                    if (get64() != nv) raise(WG_CORRUPT_STREAM, "csr_decode: v/col length mismatch");
                    get(pool.data() + off + 8ull * nv, 4ull * nv);
                    if (get64() != (uint64_t)N + 1) raise(WG_CORRUPT_STREAM, "csr_decode: row offsets");
                    uint32_t* ro = reinterpret_cast<uint32_t*>(pool.data() + off + 12ull * nv);
                    get(ro, 4ull * (N + 1));
                    const uint32_t* co = reinterpret_cast<const uint32_t*>(pool.data() + off + 8ull * nv);
                    if (ro[0] != 0 || ro[N] != nv) raise(WG_CORRUPT_STREAM, "csr_decode: row offsets");
                    for (uint32_t r = 0; r < N; ++r)
                        if (ro[r] > ro[r + 1]) raise(WG_CORRUPT_STREAM, "csr_decode: row offsets");
                    for (uint32_t r = 0; r < N; ++r)  // columns in range and strictly increasing per row
                        for (uint32_t k = ro[r]; k < ro[r + 1]; ++k)
                            if (co[k] >= N || (k > ro[r] && co[k] <= co[k - 1]))
                                raise(WG_CORRUPT_STREAM, "csr_decode: bad column index");
                    e.nnz = (uint32_t)nv;
                    e.flags = 0;
                } else {  // LzStream (lz_decode, codec.hpp:177-244) of the raw block
                    pool.resize(off + rawb);
                    unsigned char* dst = pool.data() + off;
                    uint64_t done = 0;
                    const uint64_t chunk = get64(), nch = get64();
                    (void)chunk;
                    for (uint64_t c = 0; c < nch; ++c) {
                        const uint32_t raw_len = get32(), enc = get32();
                        if (pos + enc > in.size()) raise(WG_CORRUPT_STREAM, "truncated LZ chunk");
                        if (done + raw_len > rawb) raise(WG_CORRUPT_STREAM, "decode_patch: payload size mismatch");
                        const unsigned char* src = in.data() + pos;
                        size_t sp = 0;
                        uint64_t o = 0;
                        auto length = [&](size_t base) {
                            size_t len = base;
                            if (base == 15) {
                                unsigned char b;
                                do {
                                    if (sp >= enc) raise(WG_CORRUPT_STREAM, "lz_decode: truncated chunk");
                                    b = src[sp++];
                                    len += b;
                                } while (b == 255);
                            }
                            return len;
                        };
                        while (o < raw_len) {
                            if (sp >= enc) raise(WG_CORRUPT_STREAM, "lz_decode: truncated chunk");
                            const unsigned char token = src[sp++];
                            const size_t lit = length(token >> 4);
                            if (sp + lit > enc || o + lit > raw_len) raise(WG_CORRUPT_STREAM, "lz_decode: truncated chunk");
                            std::memcpy(dst + done + o, src + sp, lit);
                            sp += lit;
                            o += lit;
                            if (o == raw_len) break;
                            if (sp + 2 > enc) raise(WG_CORRUPT_STREAM, "lz_decode: truncated chunk");
                            const size_t moff = src[sp] | ((size_t)src[sp + 1] << 8);
                            sp += 2;
                            const size_t ml = length(token & 0x0f) + 4;
                            if (moff == 0 || moff > o) raise(WG_CORRUPT_STREAM, "lz_decode: bad match offset");
                            if (o + ml > raw_len) raise(WG_CORRUPT_STREAM, "lz_decode: raw_len overrun");
                            for (size_t i = 0; i < ml; ++i) dst[done + o + i] = dst[done + o - moff + i];
                            o += ml;
                        }
                        if (sp != enc) raise(WG_CORRUPT_STREAM, "lz_decode: trailing bytes");
                        pos += enc;
                        done += raw_len;
                    }
                    if (done != rawb) raise(WG_CORRUPT_STREAM, "decode_patch: payload size mismatch");
                    e.nnz = 0;
                    e.flags = DIR_RAW;
                }
            }
        }
        if (pos != in.size()) raise(WG_CORRUPT_STREAM, "checkpoint: trailing bytes");
        const uint64_t used = round16(pool.size());
        if (used > cap) raise(WG_OUT_OF_MEMORY, "checkpoint does not fit the compressed-store budget");
        pool.resize(used);
        // the pool parity follows the step count (SWE derives it on the device)
        const int k = (int)(h.step & 1);
        WG_CUDA(cudaMemcpy(store[k], pool.data(), used, cudaMemcpyHostToDevice));
        WG_CUDA(cudaMemcpy(dir[k], hd.data(), blocks * sizeof(DirEntry), cudaMemcpyHostToDevice));
        const unsigned long long bu[2] = {k == 0 ? used : 0ull, k == 1 ? used : 0ull};
        WG_CUDA(cudaMemcpy(bump, bu, sizeof bu, cudaMemcpyHostToDevice));
        cur = k;
        // edge lines: decode patch batches, copy their boundary lines
        const uint64_t tcount = (uint64_t)(N + 2) * (N + 2);
        const uint32_t batch = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(sg.npatch, (256ull << 20) /
                                                                                                (8 * sg.m * tcount)));
        DevBuf<double> buf((uint64_t)batch * sg.m * tcount);
        for (uint32_t p0 = 0; p0 < sg.npatch; p0 += batch) {
            const uint32_t cnt = std::min<uint32_t>(batch, sg.npatch - p0);
            StepArgs a = step_args(k, 1 - k);
            a.dir_in = dir[k] + (uint64_t)p0 * sg.m;
            a.g.npatch = cnt;
            a.decode_out = buf.p;
            ks.decode<<<grid, ks.threads, ks.smem, stream>>>(a);
            WG_LAUNCH_CHECK("checkpoint decode");
            const uint64_t th = (uint64_t)cnt * sg.m * N * N;
            k_edges_from_grid<<<(unsigned)((th + 255) / 256), 256, 0, stream>>>(buf.p, N, sg, p0, cnt, edges[k]);
            WG_LAUNCH_CHECK("checkpoint edges");
        }
        step = h.step;
        row0 = h.step;
        launched = h.step;
        time = h.time;
        if (is_swe()) {
            unsigned long long c[5] = {0, 0, 0, 0, h.step};
            std::memcpy(&c[0], &h.time, sizeof(double));
            std::memcpy(&c[1], &h.swe_last_dt, sizeof(double));
            c[2 + (h.step & 1)] = h.swe_vmax_bits;
            WG_CUDA(cudaMemcpyAsync(swe, c, sizeof c, cudaMemcpyHostToDevice, stream));
        }
        if (lz_done) k_set_u64<<<1, 1, 0, stream>>>(lz_done, h.step);
        sync();
    }

    void patch_csr(uint64_t p, uint32_t q, double* v, uint32_t* col, uint32_t* row, uint64_t* nnz,
                   int32_t* raw) {
        if (p >= sg.npatch || q >= sg.m) raise(WG_OUT_OF_RANGE, "patch_csr: patch/component");
        sync();
        DirEntry e;
        WG_CUDA(cudaMemcpy(&e, dir[cur] + p * sg.m + q, sizeof e, cudaMemcpyDeviceToHost));
        const bool is_raw = e.flags & DIR_RAW;
        if (raw) *raw = is_raw ? 1 : 0;
        if (nnz) *nnz = is_raw ? (uint64_t)N * N : e.nnz;
        const unsigned char* base = store[cur] + e.off;
        if (e.flags & DIR_CONST) {  // constant block: the value is in the entry
            double c;
            std::memcpy(&c, &e.off, 8);
            if (v) std::fill(v, v + (size_t)N * N, c);
            return;
        }
        if (is_raw) {
            if (v) WG_CUDA(cudaMemcpy(v, base, (size_t)N * N * 8, cudaMemcpyDeviceToHost));
            return;
        }
        if (v) WG_CUDA(cudaMemcpy(v, base, 8ull * e.nnz, cudaMemcpyDeviceToHost));
        if (col) WG_CUDA(cudaMemcpy(col, base + 8ull * e.nnz, 4ull * e.nnz, cudaMemcpyDeviceToHost));
        if (row) WG_CUDA(cudaMemcpy(row, base + 12ull * e.nnz, 4ull * (N + 1), cudaMemcpyDeviceToHost));
    }
};

}  // namespace wg

using namespace wg;

extern "C" {

wg_status wg_session_create(const wg_run_config* cfg, const wg_shard* shard, void* stream,
                            wg_session** out) {
    return guard([&] {
        auto s = std::make_unique<Session>();
        s->create(*cfg, shard, stream);
        *out = reinterpret_cast<wg_session*>(s.release());
    });
}

wg_status wg_session_destroy(wg_session* s) {
    return guard([&] { delete reinterpret_cast<Session*>(s); });
}

wg_status wg_session_info_get(const wg_session* sp, wg_session_info* info) {
    return guard([&] {
        const Session* s = reinterpret_cast<const Session*>(sp);
        info->npatch_local = s->sg.npatch;
        info->patch_n = s->N;
        info->components = s->sg.m;
        info->halo_doubles = s->halo_doubles();
        info->store_capacity_bytes = s->cap;
        info->device_bytes = s->device_bytes;
        info->cells_per_step = (uint64_t)s->sg.R * (s->N - 1) * (uint64_t)s->sg.P1 * (s->N - 1);
    });
}

wg_status wg_session_upload(wg_session* s, const double* host_grid) {
    return guard([&] { reinterpret_cast<Session*>(s)->upload_host(host_grid); });
}

wg_status wg_dev_session_upload(wg_session* s, const double* dev_grid) {
    return guard([&] { reinterpret_cast<Session*>(s)->upload_dev(dev_grid); });
}

wg_status wg_session_step_host(wg_session* s, const double* host_grid, double dt) {
    return guard([&] {
        if (!s || !host_grid) raise(WG_INVALID_ARGUMENT, "wg_session_step_host: null argument");
        reinterpret_cast<Session*>(s)->step_from_host(host_grid, dt);
    });
}

wg_status wg_session_check_shared(wg_session* s, double tol) {
    return guard([&] { reinterpret_cast<Session*>(s)->check_shared(tol); });
}

wg_status wg_session_init_device(wg_session* s) {
    return guard([&] { reinterpret_cast<Session*>(s)->init_device(); });
}

wg_status wg_session_step(wg_session* s, double dt) {
    return guard([&] { reinterpret_cast<Session*>(s)->do_step(dt); });
}

wg_status wg_session_halo(wg_session* sp, double** send_lo, double** send_hi, double** recv_lo,
                          double** recv_hi) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        const EdgeSet& e = s->edges[s->cur];
        const uint64_t line = s->halo_doubles();
        if (send_lo) *send_lo = e.rowlo + 1 * line;              // slot 1: first owned row
        if (send_hi) *send_hi = e.rowhi + (uint64_t)s->sg.R * line;  // slot R: last owned row
        if (recv_lo) *recv_lo = e.rowhi;                         // slot 0: halo above
        if (recv_hi) *recv_hi = e.rowlo + (uint64_t)(s->sg.R + 1) * line;  // slot R+1: halo below
    });
}

wg_status wg_session_peer_export(wg_session* sp, void** edge_mem0, void** edge_mem1, void** flags, uint32_t* rows) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        if (edge_mem0) *edge_mem0 = s->edge_mem[0];
        if (edge_mem1) *edge_mem1 = s->edge_mem[1];
        if (flags) *flags = s->peer_flags;
        if (rows) *rows = s->sg.R;
    });
}

wg_status wg_session_peer_attach(wg_session* sp, void* above_mem0, void* above_mem1, void* above_flags,
                                 uint32_t above_rows, void* below_mem0, void* below_mem1, void* below_flags,
                                 uint32_t below_rows) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        double* const am[2] = {static_cast<double*>(above_mem0), static_cast<double*>(above_mem1)};
        double* const bm[2] = {static_cast<double*>(below_mem0), static_cast<double*>(below_mem1)};
        if (!above_flags || !below_flags) raise(WG_INVALID_ARGUMENT, "peer halos: null flag words");
        s->peer_attach(am, above_rows, static_cast<unsigned long long*>(above_flags), bm, below_rows,
                       static_cast<unsigned long long*>(below_flags));
    });
}

wg_status wg_session_peer_push(wg_session* s) {
    return guard([&] { reinterpret_cast<Session*>(s)->peer_push(); });
}

wg_status wg_ipc_handle(void* dev_ptr, unsigned char out[64]) {
    return guard([&] {
        cudaIpcMemHandle_t h;
        WG_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(out, &h, 64);
    });
}

wg_status wg_ipc_open(const unsigned char in[64], void** dev_ptr) {
    return guard([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, in, 64);
        WG_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

wg_status wg_ipc_close(void* dev_ptr) {
    return guard([&] { WG_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

wg_status wg_session_cfl_vmax(wg_session* sp, unsigned long long** vmax_bits) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        if (!s->is_swe()) raise(WG_INVALID_ARGUMENT, "wg_session_cfl_vmax: SWE sessions only");
        *vmax_bits = s->swe + 2 + (s->launched & 1);
    });
}

wg_status wg_session_save(wg_session* s, const char* path) {
    return guard([&] { reinterpret_cast<Session*>(s)->save(path); });
}

wg_status wg_session_load(wg_session* s, const char* path) {
    return guard([&] { reinterpret_cast<Session*>(s)->load(path); });
}

wg_status wg_session_metrics(wg_session* s, wg_metrics_row* rows, uint64_t max_rows, uint64_t* nrows) {
    return guard([&] { reinterpret_cast<Session*>(s)->metrics(rows, max_rows, nrows); });
}

wg_status wg_session_download(wg_session* s, double* host_grid) {
    return guard([&] { reinterpret_cast<Session*>(s)->download(host_grid); });
}

wg_status wg_session_patch_csr(wg_session* s, uint64_t patch, uint32_t comp, double* v, uint32_t* col,
                               uint32_t* row, uint64_t* nnz, int32_t* raw) {
    return guard([&] { reinterpret_cast<Session*>(s)->patch_csr(patch, comp, v, col, row, nnz, raw); });
}

wg_status wg_session_sync(wg_session* s) {
    return guard([&] { reinterpret_cast<Session*>(s)->sync(); });
}

wg_status wg_session_last_row(wg_session* sp, wg_metrics_row* row) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        if (s->is_swe()) s->sync();
        if (s->step <= s->row0) raise(WG_LOGIC, "no step has run");
        WG_CUDA(cudaMemcpyAsync(row, s->rows + (s->step - 1 - s->row0), sizeof(wg_metrics_row), cudaMemcpyDeviceToHost,
                                s->stream));
        s->sync();
    });
}

wg_status wg_session_last_row_async(wg_session* sp, wg_metrics_row* row) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        const uint64_t done = s->is_swe() ? s->launched : s->step;  // SWE: the last launch's row
        if (done <= s->row0) raise(WG_LOGIC, "no step has run");
        WG_CUDA(cudaMemcpyAsync(row, s->rows + (done - 1 - s->row0), sizeof(wg_metrics_row), cudaMemcpyDeviceToHost,
                                s->stream));
    });
}

// Summed per-phase cycles of thread 0 of every CTA (phase_mark)
// of every CTA of the session's step launches; `reset` zeroes them.  Not
// part of the product ABI.
wg_status wg_debug_phase_cycles(wg_session* sp, uint64_t* out, int32_t n, int32_t reset) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        if (!s->phase) raise(WG_LOGIC, "no phase buffer");
        s->sync();
        unsigned long long h[32];
        WG_CUDA(cudaMemcpy(h, s->phase, sizeof h, cudaMemcpyDeviceToHost));
        for (int k = 0; k < n && k < 32; ++k) out[k] = h[k];
        if (reset) WG_CUDA(cudaMemset(s->phase, 0, sizeof h));
    });
}

wg_status wg_session_profile(wg_session* sp, int32_t enable) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        s->sync();
        s->clear_profile();
        s->profiling = enable != 0;
    });
}

wg_status wg_session_profile_read(wg_session* sp, double* main_ms, uint64_t* launches) {
    return guard([&] {
        Session* s = reinterpret_cast<Session*>(sp);
        s->sync();
        double tot = 0.0;
        for (auto& pr : s->ev_main) {
            float ms = 0.f;
            WG_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
            tot += ms;
        }
        if (main_ms) *main_ms = tot;
        if (launches) *launches = s->ev_main.size();
    });
}

// run(RunConfig) (pipeline.hpp:129-305) on one device through a session.
wg_status wg_run_hooked(const wg_run_config* cfg, wg_metrics_row* rows, uint64_t max_rows, uint64_t* nrows,
                        double* final_grid, wg_run_summary* summary, wg_step_hook hook, void* user) {
    return guard([&] {
        if (cfg->scheme != WG_SCHEME_LBM_D2Q9) sim_validate(*cfg);
        const RunGeometry g = run_geometry(*cfg);
        std::vector<double> dts;
        if (cfg->scheme == WG_SCHEME_TRANSPORT) dts = transport_dts(*cfg);
        else if (cfg->scheme == WG_SCHEME_LBM_D2Q9) dts.assign(cfg->lbm_steps, 1.0);
        Session s;
        s.create(*cfg, nullptr, nullptr);
        std::vector<double> grid(g.npatch * g.m * g.tcount);
        initial_state(*cfg, 0, g.splits[0], grid.data());
        cudaEvent_t e0, e1;
        WG_CUDA(cudaEventCreate(&e0));
        WG_CUDA(cudaEventCreate(&e1));
        // a raw initial state larger than the store budget streams into step 1
        const bool streamed = cfg->scheme == WG_SCHEME_LBM_D2Q9 && !dts.empty() &&
                              (uint64_t)s.sg.npatch * s.sg.m * round16((uint64_t)s.N * s.N * 8) > s.cap;
        if (!streamed) s.upload_host(grid.data());
        WG_CUDA(cudaMemsetAsync(s.phase, 0, 32 * sizeof(unsigned long long), s.stream));
        WG_CUDA(cudaEventRecord(e0, s.stream));
        if (streamed) {
            s.step_from_host(grid.data(), dts[0]);
            dts.erase(dts.begin());
        }
        // the caller's per-step hook (metrics file, observer, snapshots:
        // pipeline.hpp:285-288): the step's row, then the state on request
        if (hook && !final_grid) raise(WG_INVALID_ARGUMENT, "wg_run_hooked: a hook needs the final_grid buffer");
        auto after_step = [&] {
            if (!hook) return;
            wg_metrics_row row{};
            s.sync();
            WG_CUDA(cudaMemcpy(&row, s.rows + (s.step - 1 - s.row0), sizeof row, cudaMemcpyDeviceToHost));
            if (cfg->strict && !cfg->no_compression) {  // the mass half, before the observer sees the row
                double mfv = 0.0;
                WG_CUDA(cudaMemcpy(&mfv, s.mass_fv + (s.step - 1 - s.row0), sizeof mfv, cudaMemcpyDeviceToHost));
                if (std::abs(row.global_mass - mfv) > 1e-12 * std::max(std::abs(mfv), 1.0))
                    raise(WG_CONSISTENCY, "strict: compression cycle changed global mass");
            }
            int k = hook(user, &row, nullptr);
            if (k == WG_HOOK_WANT_GRID) {
                s.download(final_grid);
                k = hook(user, &row, final_grid);
            }
            if (k < 0) raise(WG_ABORTED, "run stopped by its step hook");
        };
        if (streamed) after_step();
        if (s.is_swe()) {
            // the step count is known only on the device: launch batches
            // sized from the current dt, then read the clock back
            s.sync();
            while (s.time < cfg->t_end - 1e-15) {
                double td[2];  // [t, dt of the last step]
                WG_CUDA(cudaMemcpy(td, s.swe_td(), sizeof td, cudaMemcpyDeviceToHost));
                const double est = td[1] > 0.0 ? std::ceil((cfg->t_end - td[0]) / td[1]) : 16.0;
                const uint64_t batch = (cfg->strict || hook) ? 1 : (uint64_t)std::clamp(est, 1.0, 512.0);
                const uint64_t before = s.step;
                for (uint64_t k = 0; k < batch; ++k) s.do_step(0.0);
                s.sync();
                if (cfg->strict && !cfg->no_compression) s.check_shared(1e-12);
                if (s.step == before) raise(WG_LOGIC, "SWE step loop made no progress");
                after_step();
            }
        } else {
            for (double dt : dts) {
                s.do_step(dt);
                // strict (pipeline.hpp:278-283): assemble(grid, 0) every step
                if (cfg->strict && !cfg->no_compression) s.check_shared(1e-12);
                after_step();
            }
        }
        WG_CUDA(cudaEventRecord(e1, s.stream));
        s.sync();
        float ms = 0.f;
        WG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        std::vector<wg_metrics_row> r(s.step);
        uint64_t n = 0;
        s.metrics(r.data(), r.size(), &n);
        if (cfg->strict && !cfg->no_compression) {  // pipeline.hpp:278-283 (mass half)
            std::vector<double> mfv(s.step);
            if (s.step)
                WG_CUDA(cudaMemcpy(mfv.data(), s.mass_fv, s.step * sizeof(double), cudaMemcpyDeviceToHost));
            for (uint64_t k = 0; k < s.step; ++k) {
                const double scale = std::max(std::abs(mfv[k]), 1.0);
                if (std::abs(r[k].global_mass - mfv[k]) > 1e-12 * scale)
                    raise(WG_CONSISTENCY, "strict: compression cycle changed global mass");
            }
        }
        if (nrows) *nrows = n;
        if (rows)
            for (uint64_t k = 0; k < n && k < max_rows; ++k) rows[k] = r[k];
        if (final_grid) s.download(final_grid);
        if (summary) {
            std::memset(summary, 0, sizeof(*summary));
            double sum = 0.0;
            for (auto& x : r) sum += x.ratio;
            summary->avg_ratio = r.empty() ? 1.0 : sum / (double)r.size();
            summary->total_seconds = ms * 1e-3;
            // RunSummary's phase split (pipeline.hpp:52-63, 188-189, 229-255)
            // from the fused kernel's phase clocks: the scheme phases (decode,
            // ghosts, FV / collide, raw stores) are the step, the forward
            // transforms and the edge reconstruction the dwt, the threshold
            // half of the row pass the threshold, scan / allocation / CSR the
            // codec — each a share of the measured run time
            double share[4] = {0, 0, 0, 0};  // step, dwt, threshold, codec
            s.phase_shares(share);
            summary->step_seconds = share[0] * ms * 1e-3;
            summary->dwt_seconds = share[1] * ms * 1e-3;
            summary->threshold_seconds = share[2] * ms * 1e-3;
            summary->codec_seconds = share[3] * ms * 1e-3;
            summary->t_final = s.time;
            summary->steps = s.step;
        }
    });
}

wg_status wg_run(const wg_run_config* cfg, wg_metrics_row* rows, uint64_t max_rows, uint64_t* nrows,
                 double* final_grid, wg_run_summary* summary) {
    return wg_run_hooked(cfg, rows, max_rows, nrows, final_grid, summary, nullptr, nullptr);
}

}  // extern "C"
