// wavegrid_b200_reference.hpp — the drop-in a reference maintainer adds.
//
// Binds the reference's own C++ types (wavegrid/*.hpp: Field, WaveletPlan,
// CoefficientSet, ThresholdSpec, CsrBlock, PatchGrid, RunConfig, MetricsRow,
// RunResult) to the C ABI of include/wavegrid_b200.h, so a caller of the
// reference switches the hot path by calling wavegrid::b200::X where it
// called wavegrid::X — same arguments, same results, same exception types.
// Requires the reference headers on the include path; links against
// paper_2302_09883_b200/libwavegrid_b200.so (sm_100a) or, for CPU checks,
// any other library exporting the same ABI (oracle/libwg_oracle.so).
//
// Functions replaced (reference file:line, relative to
// proj/include/wavegrid/):
//   dwt_nd          wavelet.hpp:175-198     idwt_nd        wavelet.hpp:200-223
//   apply_threshold threshold.hpp:51-86     band_threshold threshold.hpp:31-47
//   csr_encode      codec.hpp:37-60         csr_decode     codec.hpp:62-79
//   lz_encode       codec.hpp:223-235       lz_decode      codec.hpp:237-244
//   sync_ghosts     patchgrid.hpp:131-201   global_mass    patchgrid.hpp:244-266
//   fv_step (every patch of a grid)         solver.hpp:207-231
//   run             pipeline.hpp:129-305    (+ Session: the device-resident loop)
#pragma once

#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "wavegrid/codec.hpp"
#include "wavegrid/patchgrid.hpp"
#include "wavegrid/pipeline.hpp"
#include "wavegrid/solver.hpp"
#include "wavegrid/threshold.hpp"
#include "wavegrid/wavelet.hpp"
#include "wavegrid_b200.h"

namespace wavegrid::b200 {

// wg_status -> the reference's exception types (codec.hpp:16,
// patchgrid.hpp:19, solver.hpp:16 and the std types they throw).
inline void check(wg_status s) {
    if (s == WG_OK) return;
    char msg[1024];
    wg_last_error(msg, sizeof msg);
    switch (s) {
        case WG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case WG_CORRUPT_STREAM: throw corrupt_stream_error(msg);
        case WG_CONSISTENCY: throw consistency_error(msg);
        case WG_RIEMANN: throw riemann_error(msg);
        case WG_DOMAIN: throw std::domain_error(msg);
        case WG_OUT_OF_RANGE: throw std::out_of_range(msg);
        case WG_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

// ---- wavelet / threshold / codec ------------------------------------------

inline CoefficientSet dwt_nd(const Field& field, const WaveletPlan& plan) {
    if (field.dims != plan.dims) throw std::invalid_argument("dwt_nd: plan/field dimension mismatch");
    std::vector<uint64_t> d(plan.dims.begin(), plan.dims.end());
    CoefficientSet cs{plan, std::vector<double>(field.values.size())};
    check(wg_dwt_nd(field.values.data(), cs.values.data(), d.data(), (uint32_t)d.size(), plan.levels));
    return cs;
}

inline Field idwt_nd(const CoefficientSet& coeffs) {
    std::vector<uint64_t> d(coeffs.plan.dims.begin(), coeffs.plan.dims.end());
    Field f;
    f.dims = coeffs.plan.dims;
    f.values.resize(coeffs.values.size());
    check(wg_idwt_nd(coeffs.values.data(), f.values.data(), d.data(), (uint32_t)d.size(), coeffs.plan.levels));
    return f;
}

inline double band_threshold(std::span<const int> scales, const ThresholdSpec& spec) {
    double out = 0.0;
    check(wg_band_threshold(scales.data(), (uint32_t)scales.size(), (int32_t)spec.mode, spec.c, spec.alpha, &out));
    return out;
}

inline std::size_t apply_threshold(CoefficientSet& coeffs, const ThresholdSpec& spec) {
    std::vector<uint64_t> d(coeffs.plan.dims.begin(), coeffs.plan.dims.end());
    uint64_t zeroed = 0;
    check(wg_apply_threshold(coeffs.values.data(), d.data(), (uint32_t)d.size(), coeffs.plan.levels,
                             (int32_t)spec.mode, spec.c, spec.alpha, &zeroed));
    return (std::size_t)zeroed;
}

inline CsrBlock csr_encode(std::span<const double> dense, std::size_t rows, std::size_t cols) {
    if (dense.size() != rows * cols) throw std::invalid_argument("csr_encode: size mismatch");
    CsrBlock b;
    b.rows = (uint32_t)rows;
    b.cols = (uint32_t)cols;
    b.v.resize(dense.size());
    b.col.resize(dense.size());
    b.row.resize(rows + 1);
    uint64_t nnz = 0;
    check(wg_csr_encode(dense.data(), rows, cols, b.v.data(), b.col.data(), b.row.data(), dense.size(), &nnz));
    b.v.resize(nnz);
    b.col.resize(nnz);
    return b;
}

inline std::vector<double> csr_decode(const CsrBlock& b) {
    if (b.v.size() != b.col.size()) throw corrupt_stream_error("csr_decode: v/col length mismatch");
    std::vector<double> dense((std::size_t)b.rows * b.cols);
    check(wg_csr_decode(b.v.data(), b.col.data(), b.v.size(), b.row.data(), b.row.size(), b.rows, b.cols,
                        dense.data()));
    return dense;
}

// lz_encode / lz_decode (codec.hpp:223-244) through wg_lz_encode /
// wg_lz_decode: same LzStream, same bytes, same exceptions.
inline LzStream lz_encode(std::span<const std::uint8_t> data, std::size_t chunk_size) {
    const uint64_t n = data.size();
    const uint64_t nc = chunk_size ? (n + chunk_size - 1) / chunk_size : 0;
    std::vector<uint64_t> lens(nc ? nc : 1);
    uint64_t tot = 0;
    check(wg_lz_encode(data.data(), n, chunk_size, nullptr, 0, lens.data(), &tot));
    std::vector<std::uint8_t> bytes(tot ? tot : 1);
    check(wg_lz_encode(data.data(), n, chunk_size, bytes.data(), tot, lens.data(), &tot));
    LzStream s;
    s.chunk_size = chunk_size;
    uint64_t at = 0;
    for (uint64_t k = 0; k < nc; ++k) {
        LzChunk c;
        c.raw_len = static_cast<std::uint32_t>(std::min<uint64_t>(chunk_size, n - k * chunk_size));
        c.payload.assign(bytes.begin() + (std::ptrdiff_t)at, bytes.begin() + (std::ptrdiff_t)(at + lens[k]));
        at += lens[k];
        s.chunks.push_back(std::move(c));
    }
    return s;
}

inline std::vector<std::uint8_t> lz_decode(const LzStream& s) {
    std::vector<std::uint8_t> out;
    for (const LzChunk& c : s.chunks) {  // every chunk with its own raw length
        if (c.raw_len == 0) {
            if (!c.payload.empty()) throw corrupt_stream_error("lz_decode: trailing bytes");
            continue;
        }
        std::vector<std::uint8_t> d(c.raw_len);
        const uint64_t len = c.payload.size();
        check(wg_lz_decode(c.payload.data(), &len, c.raw_len, d.data(), c.raw_len));
        out.insert(out.end(), d.begin(), d.end());
    }
    return out;
}

// ---- patch grids: PatchGrid <-> the ABI's flat grid buffer ------------------
// Grid buffer = [patch (row-major split order)][component][true cells]
// (patchgrid.hpp:26-55), i.e. the concatenation of every Patch::comps[c].

inline wg_grid_desc grid_desc(const PatchGrid& g) {
    wg_grid_desc d{};
    d.rank = (uint32_t)g.global_dims.size();
    d.components = (uint32_t)g.components;
    d.periodic = g.periodic ? 1 : 0;
    for (uint32_t k = 0; k < d.rank && k < 3; ++k) {
        d.global_dims[k] = g.global_dims[k];
        d.splits[k] = g.splits[k];
    }
    return d;
}

inline std::vector<double> pack(const PatchGrid& g) {
    std::vector<double> buf;
    for (const auto& p : g.patches)
        for (const auto& f : p.comps) buf.insert(buf.end(), f.values.begin(), f.values.end());
    return buf;
}

inline void unpack(std::span<const double> buf, PatchGrid& g) {
    std::size_t o = 0;
    for (auto& p : g.patches)
        for (auto& f : p.comps) {
            if (o + f.values.size() > buf.size()) throw std::logic_error("unpack: buffer too short");
            std::memcpy(f.values.data(), buf.data() + o, f.values.size() * sizeof(double));
            o += f.values.size();
        }
}

inline void sync_ghosts(PatchGrid& g) {
    const wg_grid_desc d = grid_desc(g);
    std::vector<double> buf = pack(g);
    check(wg_sync_ghosts(&d, buf.data()));
    unpack(buf, g);
}

inline double global_mass(const PatchGrid& g, std::size_t comp) {
    const wg_grid_desc d = grid_desc(g);
    const std::vector<double> buf = pack(g);
    double m = 0.0;
    check(wg_global_mass(&d, buf.data(), (uint32_t)comp, &m));
    return m;
}

// fv_step<Flux> applied to every patch of `cur` into `next` (same layout).
inline void fv_step(const PatchGrid& cur, PatchGrid& next, Scheme scheme, const SimConfig& sim, double dt) {
    const wg_grid_desc d = grid_desc(cur);
    const std::vector<double> a = pack(cur);
    std::vector<double> b = pack(next);
    check(wg_fv_step(&d, a.data(), b.data(), scheme == Scheme::swe ? WG_SCHEME_SWE : WG_SCHEME_TRANSPORT,
                     sim.alpha, sim.beta, sim.gravity, dt, sim.dx()));
    unpack(b, next);
}

// ---- run(RunConfig) ---------------------------------------------------------

inline wg_run_config to_c(const RunConfig& rc) {
    wg_run_config c;
    wg_run_config_default(&c);
    c.scheme = rc.sim.scheme == Scheme::swe ? WG_SCHEME_SWE : WG_SCHEME_TRANSPORT;
    c.levels = rc.levels;
    c.nx = rc.sim.nx;
    if (rc.sim.splits.size() != 2) throw std::invalid_argument("b200::run: 2-D grids only");
    c.splits[0] = rc.sim.splits[0];
    c.splits[1] = rc.sim.splits[1];
    c.cfl = rc.sim.cfl;
    c.t_end = rc.sim.t_end;
    c.alpha = rc.sim.alpha;
    c.beta = rc.sim.beta;
    c.gravity = rc.sim.gravity;
    c.domain_length = rc.sim.domain_length;
    c.threshold_mode = (int32_t)rc.spec.mode;
    c.codec = (int32_t)rc.codec;
    c.c = rc.spec.c;
    c.threshold_alpha = rc.spec.alpha;
    c.no_compression = rc.no_compression ? 1 : 0;
    c.strict = rc.strict ? 1 : 0;
    c.threads = rc.threads;
    c.compute_l2 = 1;
    c.lz_chunk_size = rc.chunk_size;
    return c;
}

inline MetricsRow from_c(const wg_metrics_row& r) {
    MetricsRow m;
    m.step = r.step;
    m.time = r.time;
    m.dense_bytes = r.dense_bytes;
    m.compressed_bytes = r.compressed_bytes;
    m.ratio = r.ratio;
    m.nnz = r.nnz;
    m.zeroed = r.zeroed;
    m.global_mass = r.global_mass;
    m.l2 = r.l2;
    return m;
}

namespace detail_b200 {

// The harness around run()'s loop (pipeline.hpp:161-181, 285-288): metrics
// CSV, observer and snapshots, driven by wg_run_hooked's per-step hook.  The
// state is copied back only for the steps where the observer or a snapshot
// needs it.
struct RunHooks {
    const RunConfig& rc;
    std::ofstream metrics;
    std::vector<char> snap_done;
    PatchGrid grid;
    std::exception_ptr err;

    explicit RunHooks(const RunConfig& c)
        : rc(c), snap_done(c.snapshot_times.size(), 0),
          grid(decompose({c.sim.nx, c.sim.nx}, c.sim.splits, c.sim.component_count())) {}

    bool snapshot_due(double t) const {
        for (std::size_t k = 0; k < rc.snapshot_times.size(); ++k)
            if (!snap_done[k] && !(t < rc.snapshot_times[k] - 1e-9)) return true;
        return false;
    }
    void maybe_snapshot(double t) {  // pipeline.hpp:168-181
        for (std::size_t k = 0; k < rc.snapshot_times.size(); ++k) {
            if (snap_done[k] || t < rc.snapshot_times[k] - 1e-9) continue;
            snap_done[k] = 1;
            std::vector<Field> comps;
            for (std::size_t c = 0; c < grid.components; ++c) comps.push_back(assemble(grid, c));
            char name[64];
            std::snprintf(name, sizeof(name), "t%.3f", rc.snapshot_times[k]);
            save_wgrd(rc.snapshot_prefix + name + ".wgrd", comps);
            if (rc.csv_snapshots) wavegrid::detail::write_field_csv(rc.snapshot_prefix + name + ".csv", comps[0]);
        }
    }
    int on_step(const wg_metrics_row& r, const double* state) {
        const MetricsRow row = from_c(r);
        if (!state) {
            if (metrics.is_open()) wavegrid::detail::write_metrics_row(metrics, row);
            return (rc.observer || snapshot_due(row.time)) ? WG_HOOK_WANT_GRID : WG_HOOK_CONTINUE;
        }
        std::size_t n = 0;
        for (const auto& p : grid.patches)
            for (const auto& f : p.comps) n += f.values.size();
        unpack(std::span<const double>(state, n), grid);
        if (rc.observer) rc.observer(grid, row);
        maybe_snapshot(row.time);
        return WG_HOOK_CONTINUE;
    }
    static int trampoline(void* user, const wg_metrics_row* row, const double* state) {
        auto* h = static_cast<RunHooks*>(user);
        try {
            return h->on_step(*row, state);
        } catch (...) {  // rethrown by run() once the library has unwound
            h->err = std::current_exception();
            return WG_HOOK_ABORT;
        }
    }
};

}  // namespace detail_b200

// run() on the device, with the reference's harness: the metrics file, the
// per-step observer and the snapshots (pipeline.hpp:161-181, 285-288) are
// served through wg_run_hooked; an exception thrown by the observer
// propagates out of run() like the reference's.
inline RunResult run(const RunConfig& rc) {
    rc.sim.validate();
    const wg_run_config c = to_c(rc);
    uint64_t steps = 0, doubles = 0;
    check(wg_run_step_count(&c, &steps));
    check(wg_run_grid_doubles(&c, &doubles));
    const bool hooked = !rc.metrics_path.empty() || !rc.snapshot_times.empty() || bool(rc.observer);
    std::unique_ptr<detail_b200::RunHooks> h;
    if (hooked) {
        h = std::make_unique<detail_b200::RunHooks>(rc);
        if (!rc.metrics_path.empty()) {
            h->metrics.open(rc.metrics_path);
            if (!h->metrics) throw std::runtime_error("cannot open metrics file: " + rc.metrics_path);
            wavegrid::detail::write_metrics_header(h->metrics);
        }
        if (h->snapshot_due(0.0)) {  // maybe_snapshot(0.0) on the initial state
            std::vector<double> init(doubles);
            check(wg_run_initial_state(&c, init.data()));
            unpack(init, h->grid);
            h->maybe_snapshot(0.0);
        }
    }
    std::vector<wg_metrics_row> rows(steps ? steps : (1u << 20));
    std::vector<double> grid(doubles);
    wg_run_summary s{};
    uint64_t n = 0;
    const wg_status st = wg_run_hooked(&c, rows.data(), rows.size(), &n, grid.data(), &s,
                                       hooked ? &detail_b200::RunHooks::trampoline : nullptr, h.get());
    if (h) h->metrics.close();
    if (st == WG_ABORTED && h && h->err) std::rethrow_exception(h->err);
    check(st);
    RunResult res;
    for (uint64_t k = 0; k < n && k < rows.size(); ++k) res.rows.push_back(from_c(rows[k]));
    res.summary.avg_ratio = s.avg_ratio;
    res.summary.total_seconds = s.total_seconds;
    res.summary.step_seconds = s.step_seconds;
    res.summary.dwt_seconds = s.dwt_seconds;
    res.summary.threshold_seconds = s.threshold_seconds;
    res.summary.codec_seconds = s.codec_seconds;
    res.grid = decompose({rc.sim.nx, rc.sim.nx}, rc.sim.splits, rc.sim.component_count());
    unpack(grid, res.grid);
    res.t_final = s.t_final;
    return res;
}

// sweep(SweepConfig) (pipeline.hpp:360-401) with every run on the device:
// the same grid of (codec, level, threshold) runs, metrics files and
// summary.csv, the runs going through b200::run.
inline std::vector<SweepEntry> sweep(const SweepConfig& sc) {
    namespace fs = std::filesystem;
    if (!sc.out_dir.empty()) fs::create_directories(sc.out_dir);
    std::vector<SweepEntry> table;
    for (const Codec codec : sc.codecs)
        for (const int level : sc.levels)
            for (const double c : sc.thresholds) {
                RunConfig rc = sc.base;
                rc.codec = codec;
                rc.levels = level;
                rc.spec.c = c;
                char file[128];
                std::snprintf(file, sizeof file, "run_%s_L%d_c%g.csv", codec == Codec::lz ? "lz" : "csr", level, c);
                rc.metrics_path = sc.out_dir.empty() ? std::string(file) : (fs::path(sc.out_dir) / file).string();
                const RunResult r = b200::run(rc);
                SweepEntry e;
                e.codec = codec;
                e.level = level;
                e.threshold = c;
                e.avg_ratio = r.summary.avg_ratio;
                e.final_l2 = r.rows.empty() ? 0.0 : r.rows.back().l2;
                e.metrics_file = rc.metrics_path;
                table.push_back(std::move(e));
            }
    if (!sc.out_dir.empty()) {
        std::ofstream os((fs::path(sc.out_dir) / "summary.csv").string());
        os << "codec,level,threshold,avg_ratio,final_l2_error,metrics_file\n";
        for (const SweepEntry& e : table) {
            char line[256];
            std::snprintf(line, sizeof line, "%s,%d,%.17g,%.17g,%.17g,", e.codec == Codec::lz ? "lz" : "csr", e.level,
                          e.threshold, e.avg_ratio, e.final_l2);
            os << line << e.metrics_file << '\n';
        }
    }
    return table;
}

// ---- the device-resident loop ------------------------------------------------

// RAII over wg_session_*: the state lives compressed in HBM; step() is one
// fused kernel launch; nothing is copied back until rows()/download().
class Session {
  public:
    explicit Session(const RunConfig& rc, void* stream = nullptr) : cfg_(to_c(rc)) {
        check(wg_session_create(&cfg_, nullptr, stream, &s_));
    }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;
    ~Session() {
        if (s_) wg_session_destroy(s_);
    }
    void upload(const PatchGrid& g) {
        const std::vector<double> buf = pack(g);
        check(wg_session_upload(s_, buf.data()));
    }
    void step(double dt) { check(wg_session_step(s_, dt)); }  // dt ignored for SWE (device CFL clock)
    std::vector<MetricsRow> rows() {
        uint64_t n = 0;
        check(wg_session_metrics(s_, nullptr, 0, &n));
        std::vector<wg_metrics_row> r(n);
        check(wg_session_metrics(s_, r.data(), n, &n));
        std::vector<MetricsRow> out;
        for (const auto& x : r) out.push_back(from_c(x));
        return out;
    }
    void download(PatchGrid& g) {
        std::vector<double> buf(pack(g).size());
        check(wg_session_download(s_, buf.data()));
        unpack(buf, g);
    }

  private:
    wg_run_config cfg_;
    wg_session* s_ = nullptr;
};

}  // namespace wavegrid::b200
