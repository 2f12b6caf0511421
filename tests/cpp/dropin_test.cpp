// dropin_test.cpp — the reference's own C++ API against the B200 library.
//
// Built by tests/cpp/Makefile against the reference headers (this
// container only) and linked against a library exporting the C ABI:
//   _bin/dropin_oracle   -> oracle/libwg_oracle.so   (CPU, tests/test_dropin.py)
//   _bin/dropin_product  -> libwavegrid_b200.so      (B200, tests/test_gpu_dropin.py)
// For every check the reference function (wavegrid::X) and the drop-in
// (wavegrid::b200::X) run on the same inputs and must agree bit for bit;
// exception types must match.  Prints "DROPIN OK <checks>" on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "wavegrid_b200_reference.hpp"

namespace wg = wavegrid;
static int g_checks = 0;

#define EXPECT(cond)                                                              \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(cond)) {                                                            \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static int check_ops(bool device_session) {
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    // dwt_nd / idwt_nd / apply_threshold / csr on a 2-D field (wavelet.hpp:175-223)
    for (int levels : {0, 1, 3, 5}) {
        wg::Field f({33, 65});
        for (auto& x : f.values) x = U(rng);
        const wg::WaveletPlan plan{f.dims, levels};
        const auto a = wg::dwt_nd(f, plan);
        const auto b = wg::b200::dwt_nd(f, plan);
        EXPECT(same_bits(a.values, b.values));
        EXPECT(same_bits(wg::idwt_nd(a).values, wg::b200::idwt_nd(b).values));
        for (auto mode : {wg::ThresholdMode::constant, wg::ThresholdMode::accumulation, wg::ThresholdMode::capped}) {
            const wg::ThresholdSpec spec{mode, 0.05, 2.0};
            auto ca = a, cb = b;
            EXPECT(wg::apply_threshold(ca, spec) == wg::b200::apply_threshold(cb, spec));
            EXPECT(same_bits(ca.values, cb.values));
            const auto ea = wg::csr_encode(ca.values, 33, 65);
            const auto eb = wg::b200::csr_encode(cb.values, 33, 65);
            EXPECT(ea.v == eb.v && ea.col == eb.col && ea.row == eb.row);
            EXPECT(same_bits(wg::csr_decode(ea), wg::b200::csr_decode(eb)));
        }
        const int sc[2] = {1, 3};
        const wg::ThresholdSpec spec{wg::ThresholdMode::accumulation, 1e-3, 2.0};
        EXPECT(wg::band_threshold(sc, spec) == wg::b200::band_threshold(sc, spec));
    }
    // exception types (wavelet.hpp:137-144, codec.hpp:62-79)
    {
        wg::Field f({9, 9});
        EXPECT(throws<std::invalid_argument>([&] { wg::b200::dwt_nd(f, wg::WaveletPlan{f.dims, 4}); }));
        wg::CsrBlock bad{{1.0}, {5}, {0, 1, 1}, 2, 2};
        EXPECT(throws<wg::corrupt_stream_error>([&] { wg::b200::csr_decode(bad); }));
    }
    // sync_ghosts / global_mass / fv_step on a decomposed grid (patchgrid.hpp, solver.hpp)
    for (auto scheme : {wg::Scheme::transport, wg::Scheme::swe}) {
        wg::SimConfig sim;
        sim.scheme = scheme;
        sim.nx = 65;
        sim.splits = {2, 2};
        const std::size_t m = sim.component_count();
        auto g = wg::decompose({65, 65}, {2, 2}, m);
        for (std::size_t c = 0; c < m; ++c)
            wg::fill(g, c, [&](std::span<const std::size_t> gi) {
                return c == 0 ? 1.5 + 0.25 * std::sin(0.1 * gi[0] + 0.2 * gi[1]) : 0.01 * std::cos(0.3 * gi[0]);
            });
        auto g2 = g;
        wg::sync_ghosts(g);
        wg::b200::sync_ghosts(g2);
        EXPECT(same_bits(wg::b200::pack(g), wg::b200::pack(g2)));
        for (std::size_t c = 0; c < m; ++c) {  // summation order differs on the device: 1e-12
            const double ma = wg::global_mass(g, c), mb = wg::b200::global_mass(g2, c);
            EXPECT(std::abs(ma - mb) <= 1e-12 * std::max(1.0, std::abs(ma)));
        }
        auto n1 = g, n2 = g;
        const double dt = 1e-3;
        for (std::size_t p = 0; p < g.patches.size(); ++p) {
            if (scheme == wg::Scheme::transport)
                wg::fv_step(g.patches[p], n1.patches[p], wg::TransportFlux{sim.alpha, sim.beta}, dt, sim.dx());
            else
                wg::fv_step(g.patches[p], n1.patches[p], wg::SweFlux{sim.gravity}, dt, sim.dx());
        }
        wg::b200::fv_step(g, n2, scheme, sim, dt);
        EXPECT(same_bits(wg::b200::pack(n1), wg::b200::pack(n2)));
    }
    // run(RunConfig) (pipeline.hpp:129-305): rows, summary and grid
    struct Case {
        wg::Scheme scheme;
        std::size_t nx, split;
        int levels;
        wg::ThresholdMode mode;
        double c, t_end;
    };
    for (const Case& k : {Case{wg::Scheme::transport, 129, 4, 4, wg::ThresholdMode::capped, 1e-3, 0.02},
                          Case{wg::Scheme::transport, 65, 2, 3, wg::ThresholdMode::constant, 0.0, 0.02},
                          Case{wg::Scheme::swe, 65, 2, 3, wg::ThresholdMode::constant, 5e-4, 0.01}}) {
        wg::RunConfig rc;
        rc.sim.scheme = k.scheme;
        rc.sim.nx = k.nx;
        rc.sim.splits = {k.split, k.split};
        rc.sim.t_end = k.t_end;
        rc.levels = k.levels;
        rc.spec = {k.mode, k.c, 2.0};
        const auto ra = wg::run(rc);
        const auto rb = wg::b200::run(rc);
        EXPECT(ra.rows.size() == rb.rows.size());
        for (std::size_t s = 0; s < ra.rows.size(); ++s) {
            const auto &x = ra.rows[s], &y = rb.rows[s];
            EXPECT(x.step == y.step && x.time == y.time && x.nnz == y.nnz && x.zeroed == y.zeroed);
            EXPECT(x.dense_bytes == y.dense_bytes && x.compressed_bytes == y.compressed_bytes && x.ratio == y.ratio);
            EXPECT(std::abs(x.global_mass - y.global_mass) <= 1e-12 * std::max(1.0, std::abs(x.global_mass)));
        }
        if (k.scheme == wg::Scheme::transport)  // l2_error every step (device exp: 1e-12)
            for (std::size_t s = 0; s < ra.rows.size(); ++s)
                EXPECT(std::abs(ra.rows[s].l2 - rb.rows[s].l2) <= 1e-12 * ra.rows[s].l2);
        EXPECT(ra.t_final == rb.t_final);
        for (std::size_t c = 0; c < rc.sim.component_count(); ++c)
            EXPECT(same_bits(wg::assemble(ra.grid, c).values, wg::assemble(rb.grid, c).values));
    }
    {  // Codec::lz (codec.hpp:81-244): the same state, the LZ stream sizes as metrics
        wg::RunConfig rc;
        rc.sim.nx = 129;
        rc.sim.splits = {2, 2};
        rc.sim.t_end = 0.01;
        rc.spec = {wg::ThresholdMode::capped, 1e-3, 2.0};
        rc.codec = wg::Codec::lz;
        const auto ra = wg::run(rc);
        const auto rb = wg::b200::run(rc);
        EXPECT(ra.rows.size() == rb.rows.size());
        for (std::size_t s = 0; s < ra.rows.size(); ++s)
            EXPECT(ra.rows[s].compressed_bytes == rb.rows[s].compressed_bytes && ra.rows[s].ratio == rb.rows[s].ratio);
    }
    if (device_session) {
#ifdef WG_DROPIN_SESSION
        // the device-resident loop: same rows and state as run()
        wg::RunConfig rc;
        rc.sim.nx = 129;
        rc.sim.splits = {4, 4};
        rc.sim.t_end = 0.02;
        rc.spec = {wg::ThresholdMode::capped, 1e-3, 2.0};
        const auto ref = wg::run(rc);
        auto g = wg::decompose({129, 129}, {4, 4}, 1);
        const wg::Field init = wg::exact_transport(0.0, rc.sim);
        wg::fill(g, 0, [&](std::span<const std::size_t> gi) { return init.values[gi[0] * 129 + gi[1]]; });
        wg::b200::Session s(rc);
        s.upload(g);
        double t = 0.0;
        for (std::size_t k = 0; k < ref.rows.size(); ++k) {
            const double dt = std::min(wg::cfl_dt(g, rc.sim), rc.sim.t_end - t);
            s.step(dt);
            t += dt;
        }
        const auto rows = s.rows();
        EXPECT(rows.size() == ref.rows.size());
        for (std::size_t k = 0; k < rows.size(); ++k) EXPECT(rows[k].nnz == ref.rows[k].nnz && rows[k].time == ref.rows[k].time);
        s.download(g);
        EXPECT(same_bits(wg::assemble(ref.grid, 0).values, wg::assemble(g, 0).values));
#endif
    }
    return 0;
}

int main(int argc, char** argv) {
    const bool session = argc > 1 && std::strcmp(argv[1], "--session") == 0;
    const int rc = check_ops(session);
    if (rc == 0) std::printf("DROPIN OK %d\n", g_checks);
    return rc;
}
