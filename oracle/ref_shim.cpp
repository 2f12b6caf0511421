// oracle/ref_shim.cpp — TEST INFRASTRUCTURE, not product code.
//
// Exposes the UNMODIFIED reference library (/root/reference/proj/include/
// wavegrid/*.hpp, header-only C++20) through the C ABI of
// include/wavegrid_b200.h, so that tests/ and bench.py's reference arm can
// call the reference CPU implementation with the same arguments as the B200
// product.  Built by oracle/Makefile into oracle/_ref/libwg_ref.so with the
// reference's CMake Release flags (-std=c++20 -O3, no -march: no FMA
// contraction, proj/CMakeLists.txt:3-7).  Nothing here is copied from the
// reference; its headers are included from where they lie.
//
// The D2Q9 LBM step below is NOT in the reference: it is
// the builder's definition, written against the reference's
// own Patch / sync_ghosts / compression functions, exactly as SURVEY.md §8c
// asks ("must use the reference's Patch, sync_ghosts and compression
// functions unchanged").  Its parity is therefore "unpinned" by the reference.
#include <wavegrid/pipeline.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <numbers>
#include <string>
#include <thread>

#include "wavegrid_b200.h"

using namespace wavegrid;

namespace {

thread_local std::string g_err;

// thrown by a wg_run_hooked observer whose hook asked to stop
struct HookAbort {};

template <typename F>
wg_status guard(F&& f) {
    try {
        f();
        return WG_OK;
    } catch (const HookAbort&) {
        g_err = "run stopped by its step hook";
        return WG_ABORTED;
    } catch (const consistency_error& e) {
        g_err = e.what();
        return WG_CONSISTENCY;
    } catch (const corrupt_stream_error& e) {
        g_err = e.what();
        return WG_CORRUPT_STREAM;
    } catch (const riemann_error& e) {
        g_err = e.what();
        return WG_RIEMANN;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return WG_DOMAIN;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return WG_OUT_OF_RANGE;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return WG_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return WG_LOGIC;
    }
}

std::vector<std::size_t> to_dims(const uint64_t* d, uint32_t rank) {
    return std::vector<std::size_t>(d, d + rank);
}

PatchGrid grid_from_desc(const wg_grid_desc* g) {
    if (!g || g->rank == 0 || g->rank > 3)
        throw std::invalid_argument("wg_grid_desc: rank must be 1..3");
    return decompose(to_dims(g->global_dims, g->rank), to_dims(g->splits, g->rank),
                     g->components, g->periodic != 0);
}

std::size_t patch_true_count(const Patch& p) { return Field::count(p.true_dims); }

void load_grid(PatchGrid& grid, const double* buf) {
    std::size_t off = 0;
    for (auto& p : grid.patches)
        for (auto& f : p.comps) {
            std::memcpy(f.values.data(), buf + off, f.values.size() * sizeof(double));
            off += f.values.size();
        }
}

void store_grid(const PatchGrid& grid, double* buf) {
    std::size_t off = 0;
    for (const auto& p : grid.patches)
        for (const auto& f : p.comps) {
            std::memcpy(buf + off, f.values.data(), f.values.size() * sizeof(double));
            off += f.values.size();
        }
}

ThresholdMode to_mode(int32_t m) {
    switch (m) {
        case WG_THRESHOLD_CONSTANT: return ThresholdMode::constant;
        case WG_THRESHOLD_ACCUMULATION: return ThresholdMode::accumulation;
        case WG_THRESHOLD_CAPPED: return ThresholdMode::capped;
    }
    throw std::invalid_argument("unknown threshold mode");
}

// ---------------------------------------------------------------------------
// Builder-defined D2Q9 BGK. Same operation order in
// oracle/wg_oracle.c and the CUDA kernels; no FMA contraction.
// ---------------------------------------------------------------------------
constexpr int kCx[9] = {0, 1, -1, 0, 0, 1, -1, 1, -1};
constexpr int kCy[9] = {0, 0, 0, 1, -1, 1, -1, -1, 1};
constexpr double kW[9] = {4.0 / 9.0,  1.0 / 9.0,  1.0 / 9.0,  1.0 / 9.0, 1.0 / 9.0,
                          1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0};

inline void lbm_cu(double ux, double uy, double cu[9]) {
    cu[0] = 0.0;
    cu[1] = ux;
    cu[2] = -ux;
    cu[3] = uy;
    cu[4] = -uy;
    cu[5] = ux + uy;
    cu[6] = -(ux + uy);
    cu[7] = ux - uy;
    cu[8] = uy - ux;
}

// D2Q9 BGK in its FMA form: std::fma is correctly rounded.
inline double lbm_usq(double ux, double uy) { return std::fma(ux, ux, uy * uy); }

inline double lbm_feq(int q, double rho, double cu, double usq) {
    const double t = std::fma(cu, std::fma(4.5, cu, 3.0), std::fma(-1.5, usq, 1.0));
    return (kW[q] * rho) * t;
}

inline void lbm_collide(const double f[9], double omega, double out[9]) {
    const double rho = ((((((((f[0] + f[1]) + f[2]) + f[3]) + f[4]) + f[5]) + f[6]) + f[7]) + f[8]);
    const double jx = ((f[1] - f[2]) + (f[5] - f[6])) + (f[7] - f[8]);
    const double jy = ((f[3] - f[4]) + (f[5] - f[6])) + (f[8] - f[7]);
    const double inv = 1.0 / rho;
    const double ux = jx * inv, uy = jy * inv;
    const double usq = lbm_usq(ux, uy);
    double cu[9];
    lbm_cu(ux, uy, cu);
    for (int q = 0; q < 9; ++q) out[q] = std::fma(omega, lbm_feq(q, rho, cu[q], usq) - f[q], f[q]);
}

// One pull-stream + collide on every logical cell of a 2-D, 9-component
// patch; mirrors the fv_step contract (solver.hpp:207-231): reads the true
// array of `cur` (ghost ring included, corners needed), writes the logical
// cells of `next`.
void lbm_step(const Patch& cur, Patch& next, double omega) {
    const std::size_t nx = cur.true_dims[0], ny = cur.true_dims[1];
    double f[9], out[9];
    for (std::size_t i = 1; i + 1 < nx; ++i)
        for (std::size_t j = 1; j + 1 < ny; ++j) {
            for (int q = 0; q < 9; ++q)
                f[q] = cur.comps[q].values[(i - kCx[q]) * ny + (j - kCy[q])];
            lbm_collide(f, omega, out);
            for (int q = 0; q < 9; ++q) next.comps[q].values[i * ny + j] = out[q];
        }
}

// Shear-layer initial condition: rho = 1, u_y = U0 tanh(k(X-1/4))
// for X <= 1/2 else U0 tanh(k(3/4-X)), u_x = d U0 sin(2 pi (Y + 1/4)).
void lbm_initial(PatchGrid& grid, const wg_run_config& c) {
    const double inv = 1.0 / static_cast<double>(c.nx - 1);
    for (int q = 0; q < 9; ++q) {
        fill(grid, q, [&](std::span<const std::size_t> gi) {
            const double X = static_cast<double>(gi[0]) * inv;
            const double Y = static_cast<double>(gi[1]) * inv;
            const double uy = X <= 0.5 ? c.lbm_u0 * std::tanh(c.lbm_kappa * (X - 0.25))
                                       : c.lbm_u0 * std::tanh(c.lbm_kappa * (0.75 - X));
            const double ux =
                c.lbm_delta * c.lbm_u0 * std::sin(2.0 * std::numbers::pi * (Y + 0.25));
            double cu[9];
            lbm_cu(ux, uy, cu);
            return lbm_feq(q, 1.0, cu[q], lbm_usq(ux, uy));
        });
    }
}

RunConfig to_run_config(const wg_run_config* c) {
    RunConfig rc;
    rc.sim.scheme = c->scheme == WG_SCHEME_SWE ? Scheme::swe : Scheme::transport;
    rc.sim.nx = c->nx;
    rc.sim.splits = {c->splits[0], c->splits[1]};
    rc.sim.cfl = c->cfl;
    rc.sim.t_end = c->t_end;
    rc.sim.alpha = c->alpha;
    rc.sim.beta = c->beta;
    rc.sim.gravity = c->gravity;
    rc.sim.domain_length = c->domain_length;
    rc.levels = c->levels;
    rc.spec = ThresholdSpec{to_mode(c->threshold_mode), c->c, c->threshold_alpha};
    if (c->codec != 1 && c->codec != 2) throw std::invalid_argument("unknown codec");
    rc.codec = c->codec == 2 ? Codec::lz : Codec::csr;
    rc.chunk_size = c->lz_chunk_size;
    rc.no_compression = c->no_compression != 0;
    rc.strict = c->strict != 0;
    rc.threads = c->threads ? c->threads : 1;
    return rc;
}

void copy_row(const MetricsRow& r, wg_metrics_row* o) {
    o->step = r.step;
    o->time = r.time;
    o->dense_bytes = r.dense_bytes;
    o->compressed_bytes = r.compressed_bytes;
    o->ratio = r.ratio;
    o->nnz = r.nnz;
    o->zeroed = r.zeroed;
    o->global_mass = r.global_mass;
    o->l2 = r.l2;
}

// The LBM experiment loop in the shape of run() (pipeline.hpp:129-305):
// sync_ghosts -> lbm_step per patch -> swap -> the per-patch compression
// cycle of pipeline.hpp:217-257 verbatim in structure (reference functions)
// -> metrics with global mass summed over the 9 populations.
using Observer = std::function<void(const PatchGrid&, const MetricsRow&)>;

RunResult run_lbm(const wg_run_config* c, const Observer& observer = {}) {
    if (c->lbm_tau <= 0.5) throw std::invalid_argument("LBM: tau must exceed 1/2");
    const std::size_t m = 9;
    PatchGrid grid = decompose({c->nx, c->nx}, {c->splits[0], c->splits[1]}, m);
    WaveletPlan plan{grid.patches[0].logical, c->levels};
    plan.validate();
    const ThresholdSpec spec{to_mode(c->threshold_mode), c->c, c->threshold_alpha};
    lbm_initial(grid, *c);
    PatchGrid scratch = grid;
    const double omega = 1.0 / c->lbm_tau;
    const unsigned threads = c->threads ? c->threads : 1;
    RunResult res;
    const std::size_t npatch = grid.patches.size();
    struct PatchStats {
        std::size_t dense = 0, comp = 0, nnz = 0, zeroed = 0;
    };
    std::vector<PatchStats> stats(npatch);
    detail::PhaseTimer total_timer;
    for (std::uint64_t step = 1; step <= c->lbm_steps; ++step) {
        sync_ghosts(grid);
        detail::PhaseTimer step_timer;
        detail::for_each_patch(npatch, threads, [&](std::size_t pi) {
            lbm_step(grid.patches[pi], scratch.patches[pi], omega);
        });
        std::swap(grid.patches, scratch.patches);
        res.summary.step_seconds += step_timer.lap();
        if (!c->no_compression) {
            detail::for_each_patch(npatch, threads, [&](std::size_t pi) {
                Patch& p = grid.patches[pi];
                std::vector<std::vector<double>> comps(m);
                std::vector<Field> original;
                for (std::size_t q = 0; q < m; ++q) original.push_back(extract_logical(p, q));
                std::vector<CoefficientSet> coeffs;
                for (std::size_t q = 0; q < m; ++q) coeffs.push_back(dwt_nd(original[q], plan));
                std::size_t zeroed = 0;
                for (auto& cs : coeffs) zeroed += apply_threshold(cs, spec);
                for (std::size_t q = 0; q < m; ++q) comps[q] = std::move(coeffs[q].values);
                const CompressedPatch enc = encode_patch(comps, plan.dims, static_cast<std::uint32_t>(c->levels),
                                                         c->codec == 2 ? Codec::lz : Codec::csr, c->lz_chunk_size);
                auto decoded = decode_patch(enc);
                std::size_t nnz = 0;
                for (const auto& d : decoded)
                    for (double v : d)
                        if (v != 0.0) ++nnz;
                if (zeroed == 0) {
                    for (std::size_t q = 0; q < m; ++q) insert_logical(p, q, original[q]);
                } else {
                    for (std::size_t q = 0; q < m; ++q)
                        insert_logical(p, q, idwt_nd(CoefficientSet{plan, std::move(decoded[q])}));
                }
                stats[pi] = {enc.dense_bytes(), enc.compressed_bytes(), nnz, zeroed};
            });
        }
        MetricsRow row;
        row.step = step;
        row.time = static_cast<double>(step);
        if (!c->no_compression) {
            for (const auto& s : stats) {
                row.dense_bytes += s.dense;
                row.compressed_bytes += s.comp;
                row.nnz += s.nnz;
                row.zeroed += s.zeroed;
            }
            row.ratio = row.compressed_bytes > 0
                            ? static_cast<double>(row.dense_bytes) / row.compressed_bytes
                            : 1.0;
        }
        double mass = 0.0;
        for (std::size_t q = 0; q < m; ++q) mass += global_mass(grid, q);
        row.global_mass = mass;
        if (observer) observer(grid, row);  // pipeline.hpp:285-286
        res.rows.push_back(row);
    }
    res.summary.total_seconds = total_timer.lap();
    if (!res.rows.empty()) {
        double sum = 0.0;
        for (const auto& r : res.rows) sum += r.ratio;
        res.summary.avg_ratio = sum / static_cast<double>(res.rows.size());
    }
    res.t_final = static_cast<double>(c->lbm_steps);
    res.grid = std::move(grid);
    return res;
}

// The reference's observer (pipeline.hpp:36-37, 286) forwarding to a
// wg_step_hook: the row first, the state only when the hook asks for it.
Observer hook_observer(wg_step_hook hook, void* user) {
    if (!hook) return {};
    return [hook, user](const PatchGrid& g, const MetricsRow& r) {
        wg_metrics_row row;
        copy_row(r, &row);
        int k = hook(user, &row, nullptr);
        if (k == WG_HOOK_WANT_GRID) {
            std::size_t n = 0;
            for (const auto& p : g.patches)
                for (const auto& f : p.comps) n += f.values.size();
            std::vector<double> buf(n);
            store_grid(g, buf.data());
            k = hook(user, &row, buf.data());
        }
        if (k < 0) throw HookAbort{};
    };
}

}  // namespace

extern "C" {

size_t wg_last_error(char* buf, size_t cap) {
    if (buf && cap) {
        std::snprintf(buf, cap, "%s", g_err.c_str());
    }
    return g_err.size();
}

const char* wg_impl_name(void) { return "reference"; }
int wg_abi_version(void) { return WG_ABI_VERSION; }

wg_status wg_dwt_nd(const double* in, double* out, const uint64_t* dims, uint32_t rank,
                    int32_t levels) {
    return guard([&] {
        const auto d = to_dims(dims, rank);
        const std::size_t n = Field::count(d);
        Field f{d, std::vector<double>(in, in + n)};
        const CoefficientSet cs = dwt_nd(f, WaveletPlan{d, levels});
        std::memcpy(out, cs.values.data(), n * sizeof(double));
    });
}

wg_status wg_idwt_nd(const double* in, double* out, const uint64_t* dims, uint32_t rank,
                     int32_t levels) {
    return guard([&] {
        const auto d = to_dims(dims, rank);
        const std::size_t n = Field::count(d);
        const Field f = idwt_nd(CoefficientSet{WaveletPlan{d, levels},
                                               std::vector<double>(in, in + n)});
        std::memcpy(out, f.values.data(), n * sizeof(double));
    });
}

wg_status wg_band_threshold(const int32_t* scales, uint32_t rank, int32_t mode, double c,
                            double alpha, double* out) {
    return guard([&] {
        const std::vector<int> s(scales, scales + rank);
        *out = band_threshold(s, ThresholdSpec{to_mode(mode), c, alpha});
    });
}

wg_status wg_apply_threshold(double* coeffs, const uint64_t* dims, uint32_t rank,
                             int32_t levels, int32_t mode, double c, double alpha,
                             uint64_t* zeroed) {
    return guard([&] {
        const auto d = to_dims(dims, rank);
        const std::size_t n = Field::count(d);
        CoefficientSet cs{WaveletPlan{d, levels}, std::vector<double>(coeffs, coeffs + n)};
        const std::size_t z = apply_threshold(cs, ThresholdSpec{to_mode(mode), c, alpha});
        std::memcpy(coeffs, cs.values.data(), n * sizeof(double));
        if (zeroed) *zeroed = z;
    });
}

wg_status wg_csr_encode(const double* dense, uint64_t rows, uint64_t cols, double* v,
                        uint32_t* col, uint32_t* row, uint64_t capacity, uint64_t* nnz) {
    return guard([&] {
        const std::size_t n = static_cast<std::size_t>(rows * cols);
        const CsrBlock b = csr_encode(std::span<const double>(dense, n), rows, cols);
        if (b.nnz() > capacity) throw std::invalid_argument("wg_csr_encode: capacity");
        std::memcpy(v, b.v.data(), b.v.size() * sizeof(double));
        std::memcpy(col, b.col.data(), b.col.size() * sizeof(uint32_t));
        std::memcpy(row, b.row.data(), b.row.size() * sizeof(uint32_t));
        *nnz = b.nnz();
    });
}

wg_status wg_csr_decode(const double* v, const uint32_t* col, uint64_t nnz,
                        const uint32_t* row, uint64_t row_len, uint32_t rows, uint32_t cols,
                        double* dense) {
    return guard([&] {
        CsrBlock b;
        b.v.assign(v, v + nnz);
        b.col.assign(col, col + nnz);
        b.row.assign(row, row + row_len);
        b.rows = rows;
        b.cols = cols;
        const auto d = csr_decode(b);
        std::memcpy(dense, d.data(), d.size() * sizeof(double));
    });
}

wg_status wg_grid_geometry(const wg_grid_desc* g, uint64_t* patch_logical, uint64_t* npatch,
                           uint64_t* grid_doubles) {
    return guard([&] {
        const PatchGrid grid = grid_from_desc(g);
        for (uint32_t d = 0; d < g->rank; ++d) patch_logical[d] = grid.patch_logical(d);
        *npatch = grid.patches.size();
        std::size_t total = 0;
        for (const auto& p : grid.patches) total += patch_true_count(p) * grid.components;
        *grid_doubles = total;
    });
}

wg_status wg_sync_ghosts(const wg_grid_desc* g, double* buf) {
    return guard([&] {
        PatchGrid grid = grid_from_desc(g);
        load_grid(grid, buf);
        sync_ghosts(grid);
        store_grid(grid, buf);
    });
}

wg_status wg_global_mass(const wg_grid_desc* g, const double* buf, uint32_t comp,
                         double* out) {
    return guard([&] {
        PatchGrid grid = grid_from_desc(g);
        load_grid(grid, buf);
        *out = global_mass(grid, comp);
    });
}

wg_status wg_fv_step(const wg_grid_desc* g, const double* cur, double* next, int32_t scheme,
                     double alpha, double beta, double gravity, double dt, double dx) {
    return guard([&] {
        if (g->rank != 2) throw std::invalid_argument("fv_step: 2-D grids only");
        PatchGrid a = grid_from_desc(g), b = grid_from_desc(g);
        load_grid(a, cur);
        load_grid(b, next);
        for (std::size_t pi = 0; pi < a.patches.size(); ++pi) {
            if (scheme == WG_SCHEME_TRANSPORT)
                fv_step(a.patches[pi], b.patches[pi], TransportFlux{alpha, beta}, dt, dx);
            else if (scheme == WG_SCHEME_SWE)
                fv_step(a.patches[pi], b.patches[pi], SweFlux{gravity}, dt, dx);
            else
                throw std::invalid_argument("fv_step: unknown scheme");
        }
        store_grid(b, next);
    });
}

wg_status wg_lbm_step(const wg_grid_desc* g, const double* cur, double* next, double tau) {
    return guard([&] {
        if (g->rank != 2 || g->components != 9)
            throw std::invalid_argument("lbm_step: 2-D, 9 components");
        PatchGrid a = grid_from_desc(g), b = grid_from_desc(g);
        load_grid(a, cur);
        load_grid(b, next);
        for (std::size_t pi = 0; pi < a.patches.size(); ++pi)
            lbm_step(a.patches[pi], b.patches[pi], 1.0 / tau);
        store_grid(b, next);
    });
}

void wg_run_config_default(wg_run_config* c) {
    const RunConfig rc;
    std::memset(c, 0, sizeof(*c));
    c->scheme = WG_SCHEME_TRANSPORT;
    c->levels = rc.levels;
    c->nx = rc.sim.nx;
    c->splits[0] = rc.sim.splits[0];
    c->splits[1] = rc.sim.splits[1];
    c->cfl = rc.sim.cfl;
    c->t_end = rc.sim.t_end;
    c->alpha = rc.sim.alpha;
    c->beta = rc.sim.beta;
    c->gravity = rc.sim.gravity;
    c->domain_length = rc.sim.domain_length;
    c->threshold_mode = WG_THRESHOLD_CAPPED;
    c->codec = 1;
    c->c = rc.spec.c;
    c->threshold_alpha = rc.spec.alpha;
    c->threads = rc.threads;
    c->compute_l2 = 1;
    c->lbm_steps = 100;
    c->lbm_tau = 0.6;
    c->lbm_u0 = 0.05;
    c->lbm_kappa = 80.0;
    c->lbm_delta = 0.05;
    c->lz_chunk_size = 64 * 1024;
}

wg_status wg_run_step_count(const wg_run_config* c, uint64_t* steps) {
    return guard([&] {
        if (c->scheme == WG_SCHEME_LBM_D2Q9) {
            *steps = c->lbm_steps;
            return;
        }
        if (c->scheme != WG_SCHEME_TRANSPORT) {
            *steps = 0;
            return;
        }
        const RunConfig rc = to_run_config(c);
        rc.sim.validate();
        const double dt0 = rc.sim.cfl * rc.sim.dx() / std::max(rc.sim.alpha, rc.sim.beta);
        double t = 0.0;
        uint64_t n = 0;
        while (t < rc.sim.t_end - 1e-15) {
            t += std::min(dt0, rc.sim.t_end - t);
            ++n;
        }
        *steps = n;
    });
}

wg_status wg_run_grid_doubles(const wg_run_config* c, uint64_t* n) {
    return guard([&] {
        const std::size_t m =
            c->scheme == WG_SCHEME_LBM_D2Q9 ? 9 : (c->scheme == WG_SCHEME_SWE ? 3 : 1);
        const PatchGrid g = decompose({c->nx, c->nx}, {c->splits[0], c->splits[1]}, m);
        std::size_t total = 0;
        for (const auto& p : g.patches) total += patch_true_count(p) * m;
        *n = total;
    });
}

wg_status wg_run_initial_state(const wg_run_config* c, double* out) {
    return guard([&] {
        if (c->scheme == WG_SCHEME_LBM_D2Q9) {
            PatchGrid g = decompose({c->nx, c->nx}, {c->splits[0], c->splits[1]}, 9);
            lbm_initial(g, *c);
            store_grid(g, out);
            return;
        }
        const RunConfig rc = to_run_config(c);
        const std::size_t m = rc.sim.component_count();
        PatchGrid grid = decompose({rc.sim.nx, rc.sim.nx}, rc.sim.splits, m);
        const double dx = rc.sim.dx();
        if (rc.sim.scheme == Scheme::transport) {  // pipeline.hpp:139-143
            const Field init = exact_transport(0.0, rc.sim);
            fill(grid, 0, [&](std::span<const std::size_t> gi) {
                return init.values[gi[0] * rc.sim.nx + gi[1]];
            });
        } else {  // pipeline.hpp:144-155
            fill(grid, 0, [&](std::span<const std::size_t> gi) {
                const double x = gi[0] * dx / rc.sim.domain_length;
                const double y = gi[1] * dx / rc.sim.domain_length;
                const bool inside = std::abs(x - 0.5) <= 0.25 && std::abs(y - 0.5) <= 0.25;
                return inside ? 2.0 : 1.0;
            });
            fill(grid, 1, [](auto) { return 0.0; });
            fill(grid, 2, [](auto) { return 0.0; });
        }
        store_grid(grid, out);
    });
}

// lz_encode / lz_decode of the reference (codec.hpp:223-244)
wg_status wg_lz_encode(const uint8_t* data, uint64_t n, uint64_t chunk, uint8_t* out, uint64_t cap,
                       uint64_t* enc_len, uint64_t* out_len) {
    return guard([&] {
        const LzStream st = lz_encode(std::span<const std::uint8_t>(data, n), chunk);
        uint64_t tot = 0;
        for (std::size_t k = 0; k < st.chunks.size(); ++k) {
            if (enc_len) enc_len[k] = st.chunks[k].payload.size();
            if (out) {
                if (tot + st.chunks[k].payload.size() > cap) throw std::out_of_range("lz_encode: output buffer too small");
                std::memcpy(out + tot, st.chunks[k].payload.data(), st.chunks[k].payload.size());
            }
            tot += st.chunks[k].payload.size();
        }
        if (out_len) *out_len = tot;
    });
}

wg_status wg_lz_decode(const uint8_t* payload, const uint64_t* enc_len, uint64_t chunk, uint8_t* out, uint64_t n) {
    return guard([&] {
        if (chunk == 0) throw std::invalid_argument("lz_decode: chunk_size must be > 0");
        LzStream st;
        st.chunk_size = chunk;
        uint64_t p = 0, k = 0;
        for (uint64_t off = 0; off < n; off += chunk, ++k) {
            LzChunk c;
            c.raw_len = static_cast<std::uint32_t>(std::min<uint64_t>(chunk, n - off));
            c.payload.assign(payload + p, payload + p + enc_len[k]);
            p += enc_len[k];
            st.chunks.push_back(std::move(c));
        }
        const std::vector<std::uint8_t> d = lz_decode(st);
        if (d.size() != n) throw corrupt_stream_error("lz_decode: size mismatch");
        std::memcpy(out, d.data(), n);
    });
}

wg_status wg_run_hooked(const wg_run_config* c, wg_metrics_row* rows, uint64_t max_rows,
                        uint64_t* nrows, double* final_grid, wg_run_summary* summary, wg_step_hook hook,
                        void* user) {
    return guard([&] {
        RunResult r;
        if (c->scheme == WG_SCHEME_LBM_D2Q9) {
            r = run_lbm(c, hook_observer(hook, user));
        } else {
            RunConfig rc = to_run_config(c);
            rc.observer = hook_observer(hook, user);
            r = run(rc);
        }
        if (nrows) *nrows = r.rows.size();
        if (rows)
            for (std::size_t i = 0; i < r.rows.size() && i < max_rows; ++i)
                copy_row(r.rows[i], rows + i);
        if (final_grid) store_grid(r.grid, final_grid);
        if (summary) {
            summary->avg_ratio = r.summary.avg_ratio;
            summary->total_seconds = r.summary.total_seconds;
            summary->step_seconds = r.summary.step_seconds;
            summary->dwt_seconds = r.summary.dwt_seconds;
            summary->threshold_seconds = r.summary.threshold_seconds;
            summary->codec_seconds = r.summary.codec_seconds;
            summary->t_final = r.t_final;
            summary->steps = r.rows.size();
        }
    });
}

wg_status wg_run(const wg_run_config* c, wg_metrics_row* rows, uint64_t max_rows,
                 uint64_t* nrows, double* final_grid, wg_run_summary* summary) {
    return wg_run_hooked(c, rows, max_rows, nrows, final_grid, summary, nullptr, nullptr);
}

}  // extern "C"
