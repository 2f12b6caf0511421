/*
 * wavegrid_b200.h — C ABI of the B200 compressed stencil loop.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `wavegrid` (/root/reference/proj/include/wavegrid/, header-only C++20
 * CPU library).  Every entry point below replaces one reference function; the
 * reference interface it stands for is cited as file:line (paths relative to
 * proj/include/wavegrid/).  The C++ host layer (include/wavegrid_b200.hpp)
 * rethrows the status codes as the reference's exception types, and the
 * Python layer (paper_2302_09883_b200/) does the same with Python exceptions.
 *
 * Conventions
 *  - plain pointers and sizes, no C++ or torch types; every function returns a
 *    wg_status; wg_last_error() gives the message of the last failure on the
 *    calling thread.
 *  - host pointers unless the name starts with wg_dev_ (device pointers, run
 *    asynchronously on the given cudaStream_t passed as void*).
 *  - arrays are row-major with the last dimension fastest (field.hpp:11-44).
 *  - a "grid buffer" holds a PatchGrid (patchgrid.hpp:38-55) as one array:
 *    patches in row-major split order (patch_flat, patchgrid.hpp:50-54), then
 *    components, then the true (logical + 2 ghost ring) array of each
 *    component (Patch::comps, patchgrid.hpp:26-36).
 *
 * Three shared objects export (subsets of) these symbols with identical
 * semantics: the product paper_2302_09883_b200/libwavegrid_b200.so (sm_100a
 * CUDA), and the test oracles oracle/libwg_oracle.so (plain C restatement)
 * and oracle/_ref/libwg_ref.so (the reference headers compiled unchanged).
 */
#ifndef WAVEGRID_B200_H
#define WAVEGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WG_ABI_VERSION 1

/* ---- status codes: the reference's exception types ---------- */
typedef enum wg_status {
    WG_OK = 0,
    WG_INVALID_ARGUMENT = 1, /* std::invalid_argument                      */
    WG_CORRUPT_STREAM = 2,   /* corrupt_stream_error, codec.hpp:16-18       */
    WG_CONSISTENCY = 3,      /* consistency_error, patchgrid.hpp:19-21      */
    WG_RIEMANN = 4,          /* riemann_error, solver.hpp:16-18             */
    WG_DOMAIN = 5,           /* std::domain_error, solver.hpp:108-109,248   */
    WG_CUDA = 6,             /* CUDA runtime / launch failure (no fallback) */
    WG_OUT_OF_MEMORY = 7,    /* device memory or compressed-store budget    */
    WG_OUT_OF_RANGE = 8,     /* std::out_of_range, wavelet.hpp:164          */
    WG_LOGIC = 9,            /* std::logic_error                            */
    WG_ABORTED = 10          /* a wg_run_hooked hook stopped the run        */
} wg_status;

/* Copies the message of the last failure on this thread (NUL-terminated). */
size_t wg_last_error(char* buf, size_t cap);
/* Name of the implementation: "b200-sm100a", "oracle-c" or "reference". */
const char* wg_impl_name(void);
int wg_abi_version(void);

/* ---- enums mirroring the reference ------------------------------------- */
typedef enum wg_threshold_mode { /* threshold.hpp:14 */
    WG_THRESHOLD_CONSTANT = 0,
    WG_THRESHOLD_ACCUMULATION = 1,
    WG_THRESHOLD_CAPPED = 2
} wg_threshold_mode;

typedef enum wg_scheme { /* solver.hpp:24 (+ the north star's D2Q9 LBM) */
    WG_SCHEME_TRANSPORT = 0,
    WG_SCHEME_SWE = 1,
    WG_SCHEME_LBM_D2Q9 = 2 /* NOT in the reference: builder-defined */
} wg_scheme;

/* ---- wavelet (wavelet.hpp) ---------------------------------------------- */

/* dwt_nd(field, WaveletPlan{dims, levels}) -> CoefficientSet.values
 * (wavelet.hpp:175-198).  `in` and `out` hold prod(dims) doubles; they may
 * alias.  rank <= 8.  Errors: WaveletPlan::validate (wavelet.hpp:137-144). */
wg_status wg_dwt_nd(const double* in, double* out, const uint64_t* dims,
                    uint32_t rank, int32_t levels);

/* idwt_nd(CoefficientSet{plan, values}) -> Field.values (wavelet.hpp:200-223). */
wg_status wg_idwt_nd(const double* in, double* out, const uint64_t* dims,
                     uint32_t rank, int32_t levels);

/* band_threshold(scales, ThresholdSpec) (threshold.hpp:31-47). Host only. */
wg_status wg_band_threshold(const int32_t* scales, uint32_t rank, int32_t mode,
                            double c, double alpha, double* out);

/* apply_threshold(CoefficientSet&, ThresholdSpec) (threshold.hpp:51-86):
 * in place on prod(dims) coefficients; *zeroed receives the return value. */
wg_status wg_apply_threshold(double* coeffs, const uint64_t* dims, uint32_t rank,
                             int32_t levels, int32_t mode, double c,
                             double alpha, uint64_t* zeroed);

/* ---- CSR codec (codec.hpp) ---------------------------------------------- */

/* csr_encode(dense, rows, cols) (codec.hpp:37-60).  v/col need room for
 * `capacity` entries (rows*cols always suffices); row needs rows+1.
 * *nnz receives the entry count. */
wg_status wg_csr_encode(const double* dense, uint64_t rows, uint64_t cols,
                        double* v, uint32_t* col, uint32_t* row,
                        uint64_t capacity, uint64_t* nnz);

/* csr_decode(CsrBlock) (codec.hpp:62-79); `row` has row_len entries (the
 * reference checks row.size() == rows+1).  Validation failures return
 * WG_CORRUPT_STREAM exactly where the reference throws. */
wg_status wg_csr_decode(const double* v, const uint32_t* col, uint64_t nnz,
                        const uint32_t* row, uint64_t row_len, uint32_t rows,
                        uint32_t cols, double* dense);

/* ---- Codec::lz (codec.hpp:81-244) --------------------------------------
 * lz_encode(data[n], chunk) (codec.hpp:223-235): chunk k covers bytes
 * [k chunk, min((k + 1) chunk, n)); its lz_encode_chunk payload
 * (codec.hpp:127-175) is written at out + the sum of the previous payload
 * lengths, its length to enc_len[k] (room for ceil(n / chunk) entries);
 * *out_len = the total.  out == NULL: lengths only.  chunk == 0:
 * WG_INVALID_ARGUMENT (as lz_encode); cap < total: WG_OUT_OF_RANGE. */
wg_status wg_lz_encode(const uint8_t* data, uint64_t n, uint64_t chunk, uint8_t* out,
                       uint64_t cap, uint64_t* enc_len, uint64_t* out_len);
/* lz_decode (codec.hpp:237-244): chunk k's payload (enc_len[k] bytes, the
 * chunks back to back in payload) decoded to its raw length
 * min(chunk, n - k chunk) into out[n]; lz_decode_chunk's checks
 * (codec.hpp:177-220) -> WG_CORRUPT_STREAM. */
wg_status wg_lz_decode(const uint8_t* payload, const uint64_t* enc_len, uint64_t chunk,
                       uint8_t* out, uint64_t n);

/* ---- patch grid (patchgrid.hpp) ----------------------------------------- */

typedef struct wg_grid_desc { /* PatchGrid, patchgrid.hpp:38-55 */
    uint32_t rank;            /* 1..3 */
    uint32_t components;
    int32_t periodic;
    int32_t _pad;
    uint64_t global_dims[3];
    uint64_t splits[3];
} wg_grid_desc;

/* decompose() validation and geometry (patchgrid.hpp:59-103): fills the
 * logical extent per dimension, the patch count and the grid-buffer size. */
wg_status wg_grid_geometry(const wg_grid_desc* g, uint64_t* patch_logical,
                           uint64_t* npatch, uint64_t* grid_doubles);

/* sync_ghosts(PatchGrid&) (patchgrid.hpp:131-201) on a grid buffer. */
wg_status wg_sync_ghosts(const wg_grid_desc* g, double* grid);

/* global_mass(grid, comp) (patchgrid.hpp:244-266). */
wg_status wg_global_mass(const wg_grid_desc* g, const double* grid,
                         uint32_t comp, double* out);

/* fv_step<Flux>(cur, next, flux, dt, dx) (solver.hpp:207-231) applied to
 * every patch of a 2-D grid buffer (scheme transport or swe).  `next`
 * receives the logical cells; its ghost ring is left untouched. */
wg_status wg_fv_step(const wg_grid_desc* g, const double* cur, double* next,
                     int32_t scheme, double alpha, double beta, double gravity,
                     double dt, double dx);

/* Builder-defined D2Q9 BGK pull-stream + collide on every patch of a 2-D,
 * 9-component grid buffer (NOT in the reference). */
wg_status wg_lbm_step(const wg_grid_desc* g, const double* cur, double* next,
                      double tau);

/* ---- the experiment loop (pipeline.hpp) ---------------------------------- */

typedef struct wg_run_config { /* RunConfig + SimConfig, pipeline.hpp:23-38, solver.hpp:26-46 */
    int32_t scheme;           /* wg_scheme                                   */
    int32_t levels;           /* RunConfig::levels (default 4)               */
    uint64_t nx;              /* SimConfig::nx: global points per dimension  */
    uint64_t splits[2];       /* SimConfig::splits                           */
    double cfl, t_end, alpha, beta, gravity, domain_length;
    int32_t threshold_mode;   /* ThresholdSpec::mode (default capped)        */
    int32_t codec;            /* 1 = Codec::csr; 2 = Codec::lz (device session:
                                 the store stays CSR — both codecs are
                                 lossless — and every step's compressed_bytes
                                 and ratio are the exact lz_encode sizes,
                                 codec.hpp:81-244)                           */
    double c, threshold_alpha;/* ThresholdSpec::c, ::alpha                    */
    int32_t no_compression;
    int32_t strict;
    uint32_t threads;         /* reference thread pool size (CPU oracles)    */
    int32_t compute_l2;       /* transport l2 diagnostic every step (ref: 1) */
    /* D2Q9 LBM (builder-defined; ignored by transport/swe) */
    uint64_t lbm_steps;       /* number of LBM steps (t_end is not used)     */
    double lbm_tau, lbm_u0, lbm_kappa, lbm_delta;
    /* compressed-store budget in bytes for the device session (0 = auto)   */
    uint64_t store_budget_bytes;
    /* device session only: the square grid replicated `tile_rows` times
     * along dim 0 (periodic copies, identical initial state in each; 0 or 1
     * = the reference's grid).  Weak scaling: one copy per rank.            */
    uint64_t tile_rows;
    /* RunConfig::chunk_size (pipeline.hpp:28): LZ chunk bytes of Codec::lz
     * (lz_encode, codec.hpp:223-235); 0 is rejected with Codec::lz like
     * lz_encode rejects it.  Default 64 KiB.                                 */
    uint64_t lz_chunk_size;
} wg_run_config;

typedef struct wg_metrics_row { /* MetricsRow, pipeline.hpp:40-50 */
    uint64_t step;
    double time;
    uint64_t dense_bytes;
    uint64_t compressed_bytes;
    double ratio;
    uint64_t nnz;
    uint64_t zeroed;
    double global_mass;
    double l2;
} wg_metrics_row;

typedef struct wg_run_summary { /* RunSummary, pipeline.hpp:52-63 */
    double avg_ratio;
    double total_seconds;
    double step_seconds;
    double dwt_seconds;
    double threshold_seconds;
    double codec_seconds;
    double t_final;
    uint64_t steps;
} wg_run_summary;

/* Fill *cfg with the reference defaults (RunConfig{}, SimConfig{}). */
void wg_run_config_default(wg_run_config* cfg);

/* Number of steps run() will take for cfg (the dt sequence of
 * pipeline.hpp:194-196 for transport; lbm_steps for LBM; SWE: unknown -> 0). */
wg_status wg_run_step_count(const wg_run_config* cfg, uint64_t* steps);

/* Size of the grid buffer for cfg (decompose({nx,nx}, splits, m)). */
wg_status wg_run_grid_doubles(const wg_run_config* cfg, uint64_t* grid_doubles);

/* The initial state of run() (pipeline.hpp:138-155; the shear layer for LBM)
 * written into a grid buffer (logical cells; ghosts zero). */
wg_status wg_run_initial_state(const wg_run_config* cfg, double* grid);

/* run(RunConfig) -> RunResult (pipeline.hpp:129-305).  rows: room for
 * max_rows metrics rows, *nrows receives the step count.  final_grid
 * (nullable) receives RunResult::grid as a grid buffer (logical cells are
 * the contract; ghost rings hold whatever the last sync left). */
wg_status wg_run(const wg_run_config* cfg, wg_metrics_row* rows,
                 uint64_t max_rows, uint64_t* nrows, double* final_grid,
                 wg_run_summary* summary);

/* run() with the harness hooks of pipeline.hpp:161-181, 285-288 (metrics
 * file, observer, snapshots) left to the caller.  After every step's metrics
 * row (where run() writes the metrics line, calls the observer and takes
 * snapshots) hook(user, row, NULL) is called; it returns WG_HOOK_CONTINUE,
 * WG_HOOK_WANT_GRID (called again as hook(user, row, grid) with the current
 * state as a grid buffer, valid during the call; the product copies it into
 * final_grid, which must then be non-NULL) or WG_HOOK_ABORT (the run stops
 * and returns WG_ABORTED; the caller rethrows what its hook caught).  The
 * return value of the second call is CONTINUE or ABORT.  hook == NULL is
 * wg_run. */
enum { WG_HOOK_CONTINUE = 0, WG_HOOK_WANT_GRID = 1, WG_HOOK_ABORT = -1 };
typedef int (*wg_step_hook)(void* user, const wg_metrics_row* row, const double* grid);
wg_status wg_run_hooked(const wg_run_config* cfg, wg_metrics_row* rows,
                        uint64_t max_rows, uint64_t* nrows, double* final_grid,
                        wg_run_summary* summary, wg_step_hook hook, void* user);

/* ---- device-resident session (the B200 hot path) ------------------------ */
/* The state lives ONLY as a compressed patch store in HBM; one step =
 * ghost lines -> decode -> scheme step -> DWT -> threshold -> CSR -> edge
 * reconstruction, fused per patch.  Exported by the product only. */

typedef struct wg_session wg_session;

typedef struct wg_shard { /* patch-row ownership for multi-GPU */
    int32_t rank, world;
    int32_t device;           /* CUDA device ordinal                         */
    int32_t _pad;
    uint64_t row_begin, row_end; /* owned patch rows [begin, end)            */
} wg_shard;

typedef struct wg_session_info {
    uint64_t npatch_local;    /* patches owned by this shard                 */
    uint64_t patch_n;         /* logical points per patch side (2^k+1)       */
    uint64_t components;
    uint64_t halo_doubles;    /* doubles in one halo line block (P1*m*n)     */
    uint64_t store_capacity_bytes;
    uint64_t device_bytes;    /* total device memory held by the session     */
    uint64_t cells_per_step;  /* unique cells advanced per step (this shard) */
} wg_session_info;

wg_status wg_session_create(const wg_run_config* cfg, const wg_shard* shard,
                            void* stream, wg_session** out);
wg_status wg_session_destroy(wg_session* s);
wg_status wg_session_info_get(const wg_session* s, wg_session_info* info);

/* Upload a grid buffer holding this shard's patches (logical cells are
 * read) as the raw initial store; resets step and time to 0. */
wg_status wg_session_upload(wg_session* s, const double* host_grid);
/* Same from a device grid buffer (async on the session stream). */
wg_status wg_dev_session_upload(wg_session* s, const double* dev_grid);

/* Step 1 of a run straight from a host grid buffer holding the initial
 * state (this shard's patches, grid-buffer layout; page-locked memory is
 * streamed by the DMA engine): the raw state never enters the store, so a
 * store budget smaller than the raw state (C4) still starts from the
 * reference's raw initial grid (pipeline.hpp:138-155, 194-289) — the same
 * result as wg_session_upload + wg_session_step.  Resets step and time,
 * then performs step 1 with `dt`.  One-shard D2Q9 sessions. */
wg_status wg_session_step_host(wg_session* s, const double* host_grid, double dt);

/* assemble(grid, 0)'s consistency check (patchgrid.hpp:205-239) on the
 * current state: every shared boundary cell of component 0 agrees between
 * the patches of this shard that own it to tol * max(|a|, |b|, 1); returns
 * WG_CONSISTENCY otherwise (run() applies it every step in strict mode,
 * pipeline.hpp:278-283). */
wg_status wg_session_check_shared(wg_session* s, double tol);

/* Generate the initial state of cfg ON THE DEVICE and store it through the
 * compression cycle (for grids whose raw state does not fit the store
 * budget, C4/C5).  Unlike wg_session_upload the first step then starts from
 * the compressed initial state, and the device libm (tanh/sin) is not
 * bit-identical to the host's: results are not pinned to run().  D2Q9. */
wg_status wg_session_init_device(wg_session* s);

/* Advance one step with time step dt (ignored for LBM and SWE).  After it
 * returns (asynchronously), the halo send blocks of the next step are ready.
 * SWE keeps its clock on the device: each step takes dt = cfl dx / vmax
 * (cfl_dt, solver.hpp:242-258) clipped to t_end - t, and steps launched
 * once t >= t_end are no-ops (run()'s loop, pipeline.hpp:194-196);
 * wg_session_metrics reports the steps actually taken. */
wg_status wg_session_step(wg_session* s, double dt);

/* Checkpoint / resume straight from the compressed store.
 * The file is a "WGS1" header (configuration, shard, step, time, SWE
 * clock) followed by one WGC1 record per patch in the reference's
 * container format (save_wgc, codec.hpp:364-391): compressed patches as
 * Codec::csr records holding their CSR blocks byte for byte, raw patches
 * (skip rule, initial state) as Codec::lz records with levels 0 made of
 * literal-only LZ sequences, so load_wgc/decode_patch of the reference
 * read every record.  wg_session_load restores a session created with the
 * same configuration and shard; stepping on continues bit-identically.
 * wg_session_metrics then reports the rows of the steps after the load. */
wg_status wg_session_save(wg_session* s, const char* path);
wg_status wg_session_load(wg_session* s, const char* path);

/* Measured fp64 FMA throughput of the current device in TFLOP/s (2 flops
 * per DFMA; SURVEY §8d's compute ceiling, reported next to the roofline). */
wg_status wg_dev_fp64_probe(uint64_t iters, double* tflops);

/* SWE, world > 1: the max wave speed the NEXT step's dt is computed from
 * (IEEE bits of a non-negative double, so an int64 MAX is the double max).
 * Multi-GPU callers all-reduce it with MAX after every upload and step —
 * the per-step CFL all-reduce of SURVEY §8e.  Device pointer, 1 element. */
wg_status wg_session_cfl_vmax(wg_session* s, unsigned long long** vmax_bits);

/* Halo blocks for multi-GPU (world > 1).  send_lo: logical row 1 of every
 * patch of the first owned patch row; send_hi: logical row n-2 of the last
 * owned patch row; recv_lo receives the rank above's send_hi, recv_hi the
 * rank below's send_lo.  Each is info.halo_doubles doubles on the device.
 * With world == 1 the session wraps them itself. */
wg_status wg_session_halo(wg_session* s, double** send_lo, double** send_hi,
                          double** recv_lo, double** recv_hi);

/* Peer halo mode (multi-GPU over NVLink, transport and D2Q9; replaces the
 * host-driven exchange of the blocks above — the halo exchange of
 * sync_ghosts, patchgrid.hpp:131-201, across shards).  The step kernel
 * stores the halo lines straight into the ring neighbours' halo slots; a
 * step waits (on the device, bounded: WG_LOGIC after 10 s) until both
 * neighbours delivered the same generation of edge lines and announces its
 * own when complete, so no host exchange or NCCL call sits between steps.
 *   export: this session's two edge allocations, its 2 flag words, its rows;
 *   attach: the neighbours' exports, mapped into this process (the same
 *     pointers in one process, or wg_ipc_open of wg_ipc_handle across
 *     processes); above = rank - 1, below = rank + 1 (mod world);
 *   push: after upload / load (every rank, after a barrier): the current
 *     halo lines to the neighbours. */
wg_status wg_session_peer_export(wg_session* s, void** edge_mem0, void** edge_mem1, void** flags,
                                 uint32_t* rows);
wg_status wg_session_peer_attach(wg_session* s, void* above_mem0, void* above_mem1, void* above_flags,
                                 uint32_t above_rows, void* below_mem0, void* below_mem1,
                                 void* below_flags, uint32_t below_rows);
wg_status wg_session_peer_push(wg_session* s);
/* CUDA IPC of a device allocation (64-byte handle) for the peer mode. */
wg_status wg_ipc_handle(void* dev_ptr, unsigned char out[64]);
wg_status wg_ipc_open(const unsigned char in[64], void** dev_ptr);
wg_status wg_ipc_close(void* dev_ptr);

/* Per-step metrics rows accumulated on the device since upload (nsteps rows;
 * this shard's partial sums — multi-GPU callers all-reduce them). */
wg_status wg_session_metrics(wg_session* s, wg_metrics_row* rows,
                             uint64_t max_rows, uint64_t* nrows);

/* The latest step's metrics row, read back to the host (synchronises the
 * session stream: the per-step device->host result read of the e2e path). */
wg_status wg_session_last_row(wg_session* s, wg_metrics_row* row);

/* The same read enqueued on the session stream without synchronising: the
 * row lands in `row` (page-locked host memory) once the stream reaches it
 * (after wg_session_sync).  The per-step result read of a pipelined loop.
 * SWE: the row of the last launch — undefined if that launch was a no-op
 * (t_end already reached); wg_session_metrics reports the live steps. */
wg_status wg_session_last_row_async(wg_session* s, wg_metrics_row* row);

/* Decode the current state into a host grid buffer (logical cells). */
wg_status wg_session_download(wg_session* s, double* host_grid);

/* CSR block of (patch, comp) of the current store: counts first (pass NULL
 * arrays to query nnz), raw=1 when the patch is stored uncompressed (skip
 * rule, pipeline.hpp:243-249) — then v holds n*n dense values. */
wg_status wg_session_patch_csr(wg_session* s, uint64_t patch, uint32_t comp,
                               double* v, uint32_t* col, uint32_t* row,
                               uint64_t* nnz, int32_t* raw);

/* Synchronise the session stream and return the device error word. */
wg_status wg_session_sync(wg_session* s);

/* Bench instrumentation: when enabled, CUDA events bracket every launch of
 * the fused step kernel on the session stream; _read returns the summed
 * device time (ms) and the launch count since the last enable. */
wg_status wg_session_profile(wg_session* s, int32_t enable);
wg_status wg_session_profile_read(wg_session* s, double* main_ms, uint64_t* launches);

/* ---- device per-op entry points (async; for benches and torch callers) -- */
wg_status wg_dev_dwt2d(const double* in, double* out, uint64_t n0, uint64_t n1,
                       int32_t levels, uint64_t batch, void* stream);
wg_status wg_dev_idwt2d(const double* in, double* out, uint64_t n0, uint64_t n1,
                        int32_t levels, uint64_t batch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WAVEGRID_B200_H */
