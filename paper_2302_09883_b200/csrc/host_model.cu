// host_model.cu — host-side model code of the product: configuration
// defaults, the run() time-step sequence, initial conditions and the band
// threshold table.  These run once per run (not per cell-step); they are
// written against the reference's definitions, cited per function, and use
// the same glibc libm (exp, sin, tanh, pow) as the reference so that the
// initial state and the thresholds are bit-identical (SURVEY §8 hard parts:
// "Generate ICs with exp/sin on the host").
#include <atomic>
#include <cmath>
#include <thread>
#include <vector>
#include <cstring>
#include <numbers>
#include <string>
#include <vector>

#include "common.cuh"
#include "host_model.h"
#include "physics.cuh"

namespace wg {

thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

bool valid_signal_length(uint64_t n) { return n >= 2 && ((n - 1) & (n - 2)) == 0; }
int signal_level(uint64_t n) { return __builtin_ctzll(n - 1); }

// WaveletPlan::validate (wavelet.hpp:137-144)
void plan_validate(const uint64_t* dims, uint32_t rank, int levels) {
    if (levels < 0) raise(WG_INVALID_ARGUMENT, "WaveletPlan: negative level count");
    for (uint32_t d = 0; d < rank; ++d) {
        if (!valid_signal_length(dims[d])) raise(WG_INVALID_ARGUMENT, "signal length must be 2^j + 1");
        if (levels > signal_level(dims[d]))
            raise(WG_INVALID_ARGUMENT, "WaveletPlan: levels exceed dimension depth");
    }
}

// band_threshold (threshold.hpp:31-47)
double band_threshold(const int* scales, uint32_t rank, int mode, double c, double alpha) {
    switch (mode) {
        case WG_THRESHOLD_CONSTANT: return c;
        case WG_THRESHOLD_ACCUMULATION: {
            int sum = 0;
            for (uint32_t d = 0; d < rank; ++d) sum += scales[d];
            return c * std::pow(alpha, sum);
        }
        case WG_THRESHOLD_CAPPED: {
            int mx = 0;
            for (uint32_t d = 0; d < rank; ++d) mx = std::max(mx, scales[d]);
            return c * std::pow(alpha, mx);
        }
    }
    raise(WG_INVALID_ARGUMENT, "band_threshold: unknown mode");
}

// 2-D table T[bi][bj], band index 0 = sample, 1 + scale otherwise.  The
// sample x sample corner gets T = 0 so that `|v| < T` never fires there
// (samples are never touched, threshold.hpp:78).
void threshold_table_2d(int levels, int mode, double c, double alpha, double* out) {
    const int nb = levels + 1;
    for (int bi = 0; bi < nb; ++bi)
        for (int bj = 0; bj < nb; ++bj) {
            const int s[2] = {bi ? bi - 1 : 0, bj ? bj - 1 : 0};
            out[bi * nb + bj] = (bi == 0 && bj == 0) ? 0.0 : band_threshold(s, 2, mode, c, alpha);
        }
}

uint32_t scheme_components(int scheme) {
    switch (scheme) {
        case WG_SCHEME_TRANSPORT: return 1;
        case WG_SCHEME_SWE: return 3;
        case WG_SCHEME_LBM_D2Q9: return 9;
    }
    raise(WG_INVALID_ARGUMENT, "unknown scheme");
}

// SimConfig::validate (solver.hpp:40-45)
void sim_validate(const wg_run_config& c) {
    if (c.cfl <= 0.0 || c.cfl > 1.0) raise(WG_INVALID_ARGUMENT, "SimConfig: CFL must be in (0, 1]");
    if (c.nx < 2) raise(WG_INVALID_ARGUMENT, "SimConfig: nx too small");
    if (c.t_end < 0.0) raise(WG_INVALID_ARGUMENT, "SimConfig: negative t_end");
}

double sim_dx(const wg_run_config& c) { return c.domain_length / static_cast<double>(c.nx - 1); }

// decompose({nx, nx}, splits, m) geometry (patchgrid.hpp:59-103)
RunGeometry run_geometry(const wg_run_config& c) {
    RunGeometry g;
    g.m = scheme_components(c.scheme);
    g.tiles = c.tile_rows > 1 ? c.tile_rows : 1;
    for (int d = 0; d < 2; ++d) {
        const uint64_t G = c.nx, P = c.splits[d];
        if (P == 0 || G < 2 || (G - 1) % P != 0)
            raise(WG_INVALID_ARGUMENT, "decompose: dimension not divisible by splits");
        const uint64_t n = (G - 1) / P + 1;
        if (!valid_signal_length(n))
            raise(WG_INVALID_ARGUMENT, "decompose: patch logical length is not 2^k+1");
        g.splits[d] = P;
        g.n[d] = n;
    }
    g.splits[0] *= g.tiles;  // periodic copies stacked along dim 0
    g.npatch = g.splits[0] * g.splits[1];
    g.tcount = (g.n[0] + 2) * (g.n[1] + 2);
    return g;
}

// The transport dt sequence of run() (pipeline.hpp:194-196, cfl_dt
// solver.hpp:235-241).
std::vector<double> transport_dts(const wg_run_config& c) {
    sim_validate(c);
    const double vmax = std::max(c.alpha, c.beta);
    if (vmax <= 0.0) raise(WG_INVALID_ARGUMENT, "cfl_dt: nonpositive speed");
    const double dt0 = c.cfl * sim_dx(c) / vmax;
    std::vector<double> dts;
    double t = 0.0;
    while (t < c.t_end - 1e-15) {
        const double dt = std::min(dt0, c.t_end - t);
        dts.push_back(dt);
        t += dt;
    }
    return dts;
}

// exact_transport (solver.hpp:264-287) at one global point.
double exact_transport_at(const wg_run_config& c, double t, uint64_t i, uint64_t j) {
    auto wrap_unit = [](double x) {
        x = std::fmod(x, 1.0);
        return x < 0.0 ? x + 1.0 : x;
    };
    const double dx = sim_dx(c);
    double px = wrap_unit(i * dx - c.alpha * t) - 0.5;
    double py = wrap_unit(j * dx - c.beta * t) - 0.5;
    if (px < -0.5) px += 1.0;
    if (px >= 0.5) px -= 1.0;
    if (py < -0.5) py += 1.0;
    if (py >= 0.5) py -= 1.0;
    return 1.0 + std::exp(-30.0 * (px * px + py * py));
}

// Initial state of run() (pipeline.hpp:138-155) and the LBM shear layer
// for the patches whose rows lie in [row_begin, row_end),
// written into a grid buffer of those patches (logical cells; ghosts 0).
void initial_state(const wg_run_config& c, uint64_t row_begin, uint64_t row_end, double* buf) {
    const RunGeometry g = run_geometry(c);
    const uint64_t n0 = g.n[0], n1 = g.n[1], ty = n1 + 2;
    const double dx = sim_dx(c);
    const double inv = 1.0 / static_cast<double>(c.nx - 1);
    // D2Q9 shear layer: u_y depends on the row coordinate only, u_x on the
    // column only — each libm value is evaluated once per index (the same
    // expression, so the same bits as evaluating it per point)
    std::vector<double> uy_of, ux_of;
    if (c.scheme == WG_SCHEME_LBM_D2Q9) {
        uy_of.resize(c.nx);
        ux_of.resize(c.nx);
        for (uint64_t k = 0; k < c.nx; ++k) {
            const double X = static_cast<double>(k) * inv, Y = X;
            uy_of[k] = X <= 0.5 ? c.lbm_u0 * std::tanh(c.lbm_kappa * (X - 0.25))
                                : c.lbm_u0 * std::tanh(c.lbm_kappa * (0.75 - X));
            ux_of[k] = c.lbm_delta * c.lbm_u0 * std::sin(2.0 * std::numbers::pi * (Y + 0.25));
        }
    }
    auto fill_row = [&](uint64_t a) {
        for (uint64_t b = 0; b < g.splits[1]; ++b) {
            const uint64_t p = (a - row_begin) * g.splits[1] + b;
            double* base = buf + p * g.m * g.tcount;
            std::memset(base, 0, sizeof(double) * g.m * g.tcount);
            for (uint64_t i = 1; i <= n0; ++i)
                for (uint64_t j = 1; j <= n1; ++j) {
                    // tiled grids repeat the square problem along dim 0 (the
                    // reference's own grid, tiles == 1, is evaluated unreduced)
                    const uint64_t graw = a * (n0 - 1) + i - 1;
                    const uint64_t gi = g.tiles > 1 ? graw % (c.nx - 1) : graw, gj = b * (n1 - 1) + j - 1;
                    const uint64_t off = i * ty + j;
                    if (c.scheme == WG_SCHEME_TRANSPORT) {
                        base[off] = exact_transport_at(c, 0.0, gi, gj);
                    } else if (c.scheme == WG_SCHEME_SWE) {
                        const double x = gi * dx / c.domain_length;
                        const double y = gj * dx / c.domain_length;
                        const bool inside = std::abs(x - 0.5) <= 0.25 && std::abs(y - 0.5) <= 0.25;
                        base[off] = inside ? 2.0 : 1.0;
                    } else {
                        const double uy = uy_of[gi], ux = ux_of[gj];
                        const double usq = lbm_usq(ux, uy);
                        for (int q = 0; q < 9; ++q)
                            base[q * g.tcount + off] = lbm_feq(q, 1.0, lbm_cu(q, ux, uy), usq);
                    }
                }
        }
    };
    // patch rows in parallel (host threads; large grids: C4 is 21 GB)
    const uint64_t rows = row_end - row_begin;
    const unsigned nt = (unsigned)std::min<uint64_t>(rows, std::max(1u, std::thread::hardware_concurrency()));
    if (nt <= 1 || rows * g.splits[1] * g.m * g.tcount < (1ull << 22)) {
        for (uint64_t a = row_begin; a < row_end; ++a) fill_row(a);
        return;
    }
    std::atomic<uint64_t> next{row_begin};
    std::vector<std::thread> pool;
    for (unsigned k = 0; k < nt; ++k)
        pool.emplace_back([&] {
            for (uint64_t a; (a = next.fetch_add(1)) < row_end;) fill_row(a);
        });
    for (auto& th : pool) th.join();
}

}  // namespace wg

using namespace wg;

extern "C" {

size_t wg_last_error(char* buf, size_t cap) {
    if (buf && cap) std::snprintf(buf, cap, "%s", g_last_error.c_str());
    return g_last_error.size();
}

const char* wg_impl_name(void) { return "b200-sm100a"; }
int wg_abi_version(void) { return WG_ABI_VERSION; }

void wg_run_config_default(wg_run_config* c) {  // RunConfig{}, SimConfig{}
    std::memset(c, 0, sizeof(*c));
    c->scheme = WG_SCHEME_TRANSPORT;
    c->levels = 4;
    c->nx = 129;
    c->splits[0] = c->splits[1] = 2;
    c->cfl = 0.45;
    c->t_end = 0.5;
    c->alpha = 0.9;
    c->beta = 0.9;
    c->gravity = 9.81;
    c->domain_length = 1.0;
    c->threshold_mode = WG_THRESHOLD_CAPPED;
    c->codec = 1;
    c->c = 0.0;
    c->threshold_alpha = 2.0;
    c->threads = 1;
    c->compute_l2 = 1;
    c->lbm_steps = 100;
    c->lbm_tau = 0.6;
    c->lbm_u0 = 0.05;
    c->lbm_kappa = 80.0;
    c->lbm_delta = 0.05;
    c->lz_chunk_size = 64 * 1024;
}

wg_status wg_band_threshold(const int32_t* scales, uint32_t rank, int32_t mode, double c,
                            double alpha, double* out) {
    return guard([&] { *out = band_threshold(scales, rank, mode, c, alpha); });
}

wg_status wg_run_step_count(const wg_run_config* c, uint64_t* steps) {
    return guard([&] {
        if (c->scheme == WG_SCHEME_LBM_D2Q9) *steps = c->lbm_steps;
        else if (c->scheme == WG_SCHEME_TRANSPORT) *steps = transport_dts(*c).size();
        else *steps = 0;
    });
}

wg_status wg_run_grid_doubles(const wg_run_config* c, uint64_t* n) {
    return guard([&] {
        const RunGeometry g = run_geometry(*c);
        *n = g.npatch * g.m * g.tcount;
    });
}

wg_status wg_run_initial_state(const wg_run_config* c, double* grid) {
    return guard([&] {
        const RunGeometry g = run_geometry(*c);
        initial_state(*c, 0, g.splits[0], grid);
    });
}

}  // extern "C"
