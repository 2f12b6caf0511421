/*
 * oracle/wg_oracle.c — TEST INFRASTRUCTURE: CPU restatement of the reference
 * algorithm for the compressed stencil loop, in plain C11.
 *
 * This file is the CHECKER used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py.  It is never linked into, called by, or used
 * as a fallback for the product (paper_2302_09883_b200/libwavegrid_b200.so).
 *
 * Each function restates one reference function (paths relative to
 * /root/reference/proj/include/wavegrid/) with the same floating-point
 * operation order, so that its results are bit-identical to the reference
 * compiled with the reference's Release flags (-O3, no -march, no FMA; this
 * file is built with -ffp-contract=off).  Parity of this restatement is
 * PINNED by tests/test_oracle.py against oracle/_ref/libwg_ref.so (the
 * reference headers compiled unchanged) and the golden vectors in
 * tests/golden/ generated from it (tests/golden/make_golden.py).
 *
 * The D2Q9 LBM functions are NOT in the reference: they
 * restate the builder's definition in oracle/ref_shim.cpp;
 * for them parity with the reference is unpinned.
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "wavegrid_b200.h"

static _Thread_local char g_err[256];

static wg_status fail(wg_status s, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return s;
}

size_t wg_last_error(char* buf, size_t cap) {
    if (buf && cap) snprintf(buf, cap, "%s", g_err);
    return strlen(g_err);
}
const char* wg_impl_name(void) { return "oracle-c"; }
int wg_abi_version(void) { return WG_ABI_VERSION; }

/* std::max / std::min semantics (not fmax/fmin: signed zeros, NaN). */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

/* ---- wavelet.hpp ----------------------------------------------------- */

/* valid_signal_length, wavelet.hpp:16-18 */
static int valid_len(uint64_t n) { return n >= 2 && ((n - 1) & (n - 2)) == 0; }
/* signal_level, wavelet.hpp:20-24 */
static int level_of(uint64_t n) { return __builtin_ctzll(n - 1); }

/* lift_weight, wavelet.hpp:31-33 */
static inline double lift_w(uint64_t k, uint64_t half) {
    return (k == 0 || k == half - 1) ? 0.5 : 0.25;
}

/* dwt_step_1d, wavelet.hpp:48-63 (s has n = 2 half + 1 entries). */
static void dwt_step(const double* s, uint64_t n, double* coarse, double* det) {
    const uint64_t half = (n - 1) / 2;
    for (uint64_t k = 0; k < half; ++k)
        det[k] = s[2 * k + 1] - (s[2 * k] + s[2 * k + 2]) / 2.0; /* predict, :36-38 */
    coarse[0] = s[0];
    coarse[half] = s[n - 1];
    for (uint64_t k = 1; k < half; ++k) /* update, :40-42 */
        coarse[k] = s[2 * k] + (lift_w(k - 1, half) * det[k - 1] + lift_w(k, half) * det[k]);
}

/* idwt_step_1d, wavelet.hpp:74-90 */
static void idwt_step(const double* coarse, const double* det, uint64_t half, double* s) {
    s[0] = coarse[0];
    s[2 * half] = coarse[half];
    for (uint64_t k = 1; k < half; ++k)
        s[2 * k] = coarse[k] - (lift_w(k - 1, half) * det[k - 1] + lift_w(k, half) * det[k]);
    for (uint64_t k = 0; k < half; ++k) s[2 * k + 1] = det[k] + (s[2 * k] + s[2 * k + 2]) / 2.0;
}

/* dwt_line, wavelet.hpp:102-116: corner layout [samples | coarse..fine]. */
static void dwt_line(double* line, uint64_t n, int levels, double* tmp) {
    uint64_t b = n;
    for (int l = 0; l < levels; ++l) {
        const uint64_t half = (b - 1) / 2;
        double* coarse = tmp;
        double* det = tmp + half + 1;
        dwt_step(line, b, coarse, det);
        memcpy(line, tmp, (2 * half + 1) * sizeof(double));
        b = half + 1;
    }
}

/* idwt_line, wavelet.hpp:118-130 */
static void idwt_line(double* line, uint64_t n, int levels, double* tmp) {
    for (int l = levels; l >= 1; --l) {
        const uint64_t bl = ((n - 1) >> l) + 1;
        const uint64_t bl1 = ((n - 1) >> (l - 1)) + 1;
        idwt_step(line, line + bl, bl - 1, tmp);
        memcpy(line, tmp, bl1 * sizeof(double));
    }
}

/* WaveletPlan::validate, wavelet.hpp:137-144 */
static wg_status plan_validate(const uint64_t* dims, uint32_t rank, int32_t levels) {
    if (levels < 0) return fail(WG_INVALID_ARGUMENT, "WaveletPlan: negative level count");
    for (uint32_t d = 0; d < rank; ++d) {
        if (!valid_len(dims[d])) return fail(WG_INVALID_ARGUMENT, "signal length must be 2^j + 1");
        if (levels > level_of(dims[d]))
            return fail(WG_INVALID_ARGUMENT, "WaveletPlan: levels exceed dimension depth");
    }
    return WG_OK;
}

static uint64_t count_of(const uint64_t* dims, uint32_t rank) {
    uint64_t n = 1;
    for (uint32_t d = 0; d < rank; ++d) n *= dims[d];
    return n;
}

/* Apply a line transform along every dimension (forward: 0..rank-1,
 * dwt_nd wavelet.hpp:175-198; inverse: rank-1..0, idwt_nd :200-223). */
static wg_status transform_nd(const double* in, double* out, const uint64_t* dims,
                              uint32_t rank, int32_t levels, int inverse) {
    if (rank == 0 || rank > 8) return fail(WG_INVALID_ARGUMENT, "rank must be 1..8");
    wg_status st = plan_validate(dims, rank, levels);
    if (st) return st;
    const uint64_t total = count_of(dims, rank);
    if (out != in) memmove(out, in, total * sizeof(double));
    if (levels == 0) return WG_OK;
    uint64_t strides[8];
    strides[rank - 1] = 1;
    for (uint32_t d = rank - 1; d-- > 0;) strides[d] = strides[d + 1] * dims[d + 1];
    uint64_t maxn = 0;
    for (uint32_t d = 0; d < rank; ++d) maxn = dims[d] > maxn ? dims[d] : maxn;
    double* line = malloc(sizeof(double) * maxn);
    double* tmp = malloc(sizeof(double) * maxn);
    for (uint32_t s = 0; s < rank; ++s) {
        const uint32_t d = inverse ? rank - 1 - s : s;
        const uint64_t n = dims[d];
        for (uint64_t base_flat = 0; base_flat < total; ++base_flat) {
            /* lines along d start where the d-coordinate is 0 */
            if ((base_flat / strides[d]) % n != 0) continue;
            for (uint64_t i = 0; i < n; ++i) line[i] = out[base_flat + i * strides[d]];
            if (inverse) idwt_line(line, n, levels, tmp);
            else dwt_line(line, n, levels, tmp);
            for (uint64_t i = 0; i < n; ++i) out[base_flat + i * strides[d]] = line[i];
        }
    }
    free(line);
    free(tmp);
    return WG_OK;
}

wg_status wg_dwt_nd(const double* in, double* out, const uint64_t* dims, uint32_t rank,
                    int32_t levels) {
    return transform_nd(in, out, dims, rank, levels, 0);
}

wg_status wg_idwt_nd(const double* in, double* out, const uint64_t* dims, uint32_t rank,
                     int32_t levels) {
    return transform_nd(in, out, dims, rank, levels, 1);
}

/* ---- threshold.hpp -------------------------------------------------- */

/* band_threshold, threshold.hpp:31-47 */
static double band_thr(const int32_t* scales, uint32_t rank, int32_t mode, double c,
                       double alpha) {
    if (mode == WG_THRESHOLD_CONSTANT) return c;
    if (mode == WG_THRESHOLD_ACCUMULATION) {
        int sum = 0;
        for (uint32_t d = 0; d < rank; ++d) sum += scales[d];
        return c * pow(alpha, (double)sum);
    }
    int mx = 0;
    for (uint32_t d = 0; d < rank; ++d) mx = scales[d] > mx ? scales[d] : mx;
    return c * pow(alpha, (double)mx);
}

wg_status wg_band_threshold(const int32_t* scales, uint32_t rank, int32_t mode, double c,
                            double alpha, double* out) {
    if (mode < 0 || mode > 2) return fail(WG_INVALID_ARGUMENT, "band_threshold: unknown mode");
    *out = band_thr(scales, rank, mode, c, alpha);
    return WG_OK;
}

/* CoefficientSet::band, wavelet.hpp:162-170: returns -1 for a sample,
 * else the normalised scale (coarsest detail band = 0). */
static int band_of(uint64_t n, int32_t levels, uint64_t pos) {
    const uint64_t m = n - 1;
    if (levels == 0 || pos <= (m >> levels)) return -1;
    for (int l = levels; l >= 1; --l)
        if (pos <= (m >> (l - 1))) return levels - l;
    return -2; /* logic_error in the reference */
}

/* apply_threshold, threshold.hpp:51-86 */
wg_status wg_apply_threshold(double* v, const uint64_t* dims, uint32_t rank, int32_t levels,
                             int32_t mode, double c, double alpha, uint64_t* zeroed) {
    if (c < 0.0) return fail(WG_INVALID_ARGUMENT, "apply_threshold: c must be >= 0");
    if (zeroed) *zeroed = 0;
    if (c == 0.0 || levels == 0) return WG_OK;
    if (rank == 0 || rank > 8) return fail(WG_INVALID_ARGUMENT, "rank must be 1..8");
    if (mode < 0 || mode > 2) return fail(WG_INVALID_ARGUMENT, "band_threshold: unknown mode");
    uint64_t strides[8];
    strides[rank - 1] = 1;
    for (uint32_t d = rank - 1; d-- > 0;) strides[d] = strides[d + 1] * dims[d + 1];
    const uint64_t total = count_of(dims, rank);
    uint64_t z = 0;
    int32_t scales[8];
    for (uint64_t flat = 0; flat < total; ++flat) {
        uint64_t rem = flat;
        int any = 0;
        for (uint32_t d = 0; d < rank; ++d) {
            const int b = band_of(dims[d], levels, rem / strides[d]);
            if (b == -2) return fail(WG_LOGIC, "CoefficientSet::band: corrupt band map");
            rem %= strides[d];
            any |= b >= 0;
            scales[d] = b >= 0 ? b : 0;
        }
        if (!any) continue;
        if (v[flat] != 0.0 && fabs(v[flat]) < band_thr(scales, rank, mode, c, alpha)) {
            v[flat] = 0.0;
            ++z;
        }
    }
    if (zeroed) *zeroed = z;
    return WG_OK;
}

/* ---- codec.hpp (CSR) ----------------------------------------------- */

/* csr_encode, codec.hpp:37-60 */
wg_status wg_csr_encode(const double* dense, uint64_t rows, uint64_t cols, double* v,
                        uint32_t* col, uint32_t* row, uint64_t capacity, uint64_t* nnz) {
    if (rows == 0 || cols == 0) return fail(WG_INVALID_ARGUMENT, "csr_encode: bad shape");
    if (rows > 0xFFFFFFFFull - 1 || cols > 0xFFFFFFFFull)
        return fail(WG_INVALID_ARGUMENT, "csr_encode: shape overflows 32-bit indices");
    uint64_t k = 0;
    row[0] = 0;
    for (uint64_t r = 0; r < rows; ++r) {
        for (uint64_t c = 0; c < cols; ++c) {
            const double x = dense[r * cols + c];
            if (x != 0.0) {
                if (k >= capacity) return fail(WG_INVALID_ARGUMENT, "wg_csr_encode: capacity");
                v[k] = x;
                col[k] = (uint32_t)c;
                ++k;
            }
        }
        row[r + 1] = (uint32_t)k;
    }
    *nnz = k;
    return WG_OK;
}

/* csr_decode, codec.hpp:62-79 */
wg_status wg_csr_decode(const double* v, const uint32_t* col, uint64_t nnz,
                        const uint32_t* row, uint64_t row_len, uint32_t rows, uint32_t cols,
                        double* dense) {
    if (row_len != (uint64_t)rows + 1u || row[0] != 0 || row[row_len - 1] != nnz)
        return fail(WG_CORRUPT_STREAM, "csr_decode: invalid block structure");
    memset(dense, 0, sizeof(double) * (uint64_t)rows * cols);
    for (uint32_t r = 0; r < rows; ++r) {
        if (row[r] > row[r + 1])
            return fail(WG_CORRUPT_STREAM, "csr_decode: row offsets not nondecreasing");
        uint32_t prev = 0;
        for (uint32_t i = row[r]; i < row[r + 1]; ++i) {
            if (col[i] >= cols || (i > row[r] && col[i] <= prev))
                return fail(WG_CORRUPT_STREAM, "csr_decode: bad column index");
            prev = col[i];
            dense[(uint64_t)r * cols + col[i]] = v[i];
        }
    }
    (void)v;
    return WG_OK;
}

/* ---- patchgrid.hpp -------------------------------------------------- */

typedef struct grid_t {
    uint32_t rank, m;
    int periodic;
    uint64_t gdims[3], splits[3], n[3], tdims[3], tstr[3];
    uint64_t npatch, tcount; /* true cells per component */
} grid_t;

/* decompose, patchgrid.hpp:59-103 (validation + geometry only) */
static wg_status grid_init(const wg_grid_desc* d, grid_t* g) {
    if (!d || d->rank == 0 || d->rank > 3)
        return fail(WG_INVALID_ARGUMENT, "wg_grid_desc: rank must be 1..3");
    memset(g, 0, sizeof *g);
    g->rank = d->rank;
    g->m = d->components;
    g->periodic = d->periodic != 0;
    g->npatch = 1;
    for (uint32_t k = 0; k < d->rank; ++k) {
        const uint64_t G = d->global_dims[k], P = d->splits[k];
        if (P == 0 || G < 2 || (G - 1) % P != 0)
            return fail(WG_INVALID_ARGUMENT, "decompose: dimension not divisible by splits");
        const uint64_t n = (G - 1) / P + 1;
        if (!valid_len(n))
            return fail(WG_INVALID_ARGUMENT, "decompose: patch logical length is not 2^k+1");
        g->gdims[k] = G;
        g->splits[k] = P;
        g->n[k] = n;
        g->tdims[k] = n + 2;
        g->npatch *= P;
    }
    g->tcount = 1;
    for (uint32_t k = g->rank; k-- > 0;) {
        g->tstr[k] = g->tcount;
        g->tcount *= g->tdims[k];
    }
    return WG_OK;
}

static inline double* comp_ptr(const grid_t* g, double* buf, uint64_t p, uint32_t c) {
    return buf + (p * g->m + c) * g->tcount;
}

static void patch_coord(const grid_t* g, uint64_t p, uint64_t* coord) {
    for (uint32_t k = g->rank; k-- > 0;) {
        coord[k] = p % g->splits[k];
        p /= g->splits[k];
    }
}

static uint64_t patch_flat(const grid_t* g, const uint64_t* coord) {
    uint64_t f = 0;
    for (uint32_t k = 0; k < g->rank; ++k) f = f * g->splits[k] + coord[k];
    return f;
}

wg_status wg_grid_geometry(const wg_grid_desc* d, uint64_t* patch_logical, uint64_t* npatch,
                           uint64_t* grid_doubles) {
    grid_t g;
    wg_status st = grid_init(d, &g);
    if (st) return st;
    for (uint32_t k = 0; k < g.rank; ++k) patch_logical[k] = g.n[k];
    *npatch = g.npatch;
    *grid_doubles = g.npatch * g.m * g.tcount;
    return WG_OK;
}

/* sync_ghosts, patchgrid.hpp:131-201 */
static void sync_ghosts_g(const grid_t* g, double* buf) {
    uint64_t coord[3], ncoord[3], idx[3], lo[3], hi[3];
    for (uint32_t d = 0; d < g->rank; ++d) {
        const uint64_t n = g->n[d];
        for (uint64_t pi = 0; pi < g->npatch; ++pi) {
            patch_coord(g, pi, coord);
            for (int side = 0; side < 2; ++side) {
                const int low = side == 0;
                int has = 1;
                memcpy(ncoord, coord, sizeof coord);
                if (low) {
                    if (coord[d] > 0) ncoord[d] = coord[d] - 1;
                    else if (g->periodic) ncoord[d] = g->splits[d] - 1;
                    else has = 0;
                } else {
                    if (coord[d] + 1 < g->splits[d]) ncoord[d] = coord[d] + 1;
                    else if (g->periodic) ncoord[d] = 0;
                    else has = 0;
                }
                const uint64_t src_patch = has ? patch_flat(g, ncoord) : pi;
                const uint64_t tdst = low ? 0 : n + 1;
                const uint64_t tsrc = has ? (low ? n - 1 : 2) : (low ? 1 : n);
                for (uint32_t e = 0; e < g->rank; ++e) {
                    lo[e] = e < d ? 0 : 1;
                    hi[e] = e < d ? g->tdims[e] - 1 : g->n[e];
                }
                memcpy(idx, lo, sizeof lo);
                idx[d] = tdst;
                int more = 1;
                while (more) {
                    uint64_t fdst = 0, fsrc = 0;
                    for (uint32_t e = 0; e < g->rank; ++e) {
                        fdst += idx[e] * g->tstr[e];
                        fsrc += (e == d ? tsrc : idx[e]) * g->tstr[e];
                    }
                    for (uint32_t c = 0; c < g->m; ++c)
                        comp_ptr(g, buf, pi, c)[fdst] = comp_ptr(g, buf, src_patch, c)[fsrc];
                    more = 0;
                    for (uint32_t e = g->rank; e-- > 0;) {
                        if (e == d) continue;
                        if (++idx[e] <= hi[e]) {
                            more = 1;
                            break;
                        }
                        idx[e] = lo[e];
                    }
                }
            }
        }
    }
}

wg_status wg_sync_ghosts(const wg_grid_desc* d, double* buf) {
    grid_t g;
    wg_status st = grid_init(d, &g);
    if (st) return st;
    sync_ghosts_g(&g, buf);
    return WG_OK;
}

/* global_mass, patchgrid.hpp:244-266 (serial, patch order, row-major). */
static double global_mass_g(const grid_t* g, const double* buf, uint32_t comp) {
    double total = 0.0;
    uint64_t idx[3];
    for (uint64_t p = 0; p < g->npatch; ++p) {
        const double* f = comp_ptr(g, (double*)buf, p, comp);
        for (uint32_t k = 0; k < g->rank; ++k) idx[k] = 1;
        int more = 1;
        while (more) {
            double w = 1.0;
            uint64_t flat = 0;
            for (uint32_t k = 0; k < g->rank; ++k) {
                if (idx[k] == 1 || idx[k] == g->n[k]) w *= 0.5;
                flat += idx[k] * g->tstr[k];
            }
            total += w * f[flat];
            more = 0;
            for (uint32_t k = g->rank; k-- > 0;) {
                if (++idx[k] <= g->n[k]) {
                    more = 1;
                    break;
                }
                idx[k] = 1;
            }
        }
    }
    return total;
}

wg_status wg_global_mass(const wg_grid_desc* d, const double* buf, uint32_t comp,
                         double* out) {
    grid_t g;
    wg_status st = grid_init(d, &g);
    if (st) return st;
    if (comp >= g.m) return fail(WG_INVALID_ARGUMENT, "global_mass: component");
    *out = global_mass_g(&g, buf, comp);
    return WG_OK;
}

/* assemble, patchgrid.hpp:205-239 (2-D), with the shared-cell check. */
static wg_status assemble_g(const grid_t* g, const double* buf, uint32_t comp, double tol,
                            double* out, char* seen) {
    const uint64_t G0 = g->gdims[0], G1 = g->gdims[1];
    memset(seen, 0, G0 * G1);
    uint64_t coord[3];
    for (uint64_t p = 0; p < g->npatch; ++p) {
        patch_coord(g, p, coord);
        const uint64_t o0 = coord[0] * (g->n[0] - 1), o1 = coord[1] * (g->n[1] - 1);
        const double* f = comp_ptr(g, (double*)buf, p, comp);
        for (uint64_t i = 1; i <= g->n[0]; ++i)
            for (uint64_t j = 1; j <= g->n[1]; ++j) {
                const uint64_t gf = (o0 + i - 1) * G1 + (o1 + j - 1);
                const double v = f[i * g->tdims[1] + j];
                if (seen[gf]) {
                    const double ref = out[gf];
                    const double scale = smax(smax(fabs(ref), fabs(v)), 1.0);
                    if (fabs(ref - v) > tol * scale)
                        return fail(WG_CONSISTENCY, "assemble: shared cells disagree");
                } else {
                    out[gf] = v;
                    seen[gf] = 1;
                }
            }
    }
    return WG_OK;
}

/* ---- solver.hpp ----------------------------------------------------- */

static const int kDirs[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}}; /* solver.hpp:21-22 */

/* flux_upwind, solver.hpp:53-57 */
static inline double flux_upwind(double wl, double wr, const int* n, double a, double b) {
    const double speed = a * (double)n[0] + b * (double)n[1];
    return wl * smax(speed, 0.0) + wr * smin(speed, 0.0);
}

/* phi_side / phi_side_deriv, solver.hpp:86-95 */
static inline double phi_side(double h, double hs, double g) {
    if (h <= hs) return 2.0 * (sqrt(g * h) - sqrt(g * hs));
    return (h - hs) * sqrt(g * (h + hs) / (2.0 * h * hs));
}
static inline double phi_side_deriv(double h, double hs, double g) {
    if (h <= hs) return sqrt(g / h);
    const double a = sqrt(g * (h + hs) / (2.0 * h * hs));
    return a - (h - hs) * g / (4.0 * a * h * h);
}

/* SweRiemann::solve_hstar, solver.hpp:107-124 */
static wg_status solve_hstar(double g, double hl, double ul, double hr, double ur,
                             double* out) {
    if (hl <= 0.0 || hr <= 0.0) return fail(WG_DOMAIN, "SweRiemann: water depth must be positive");
    const double cl = sqrt(g * hl), cr = sqrt(g * hr);
#ifdef WG_NEWTON_SQUARE_MUL
    /* test-only variant (libwg_oracle_sq.so): the Newton start squared by a
     * multiplication, as the device does — isolates the one place where
     * glibc pow(x, 2) and a correctly rounded x * x can differ by an ulp */
    const double b = 0.5 * (cl + cr) + 0.25 * (ul - ur);
    double h = (b * b) / g;
#else
    double h = pow(0.5 * (cl + cr) + 0.25 * (ul - ur), 2) / g;
#endif
    h = smax(h, 1e-12);
    for (int it = 0; it < 100; ++it) {
        const double f = phi_side(h, hl, g) + phi_side(h, hr, g) + ur - ul;
        const double df = phi_side_deriv(h, hl, g) + phi_side_deriv(h, hr, g);
        double dh = f / df;
        if (h - dh <= 0.0) dh = h / 2.0;
        h -= dh;
        if (fabs(dh) < 1e-10) {
            *out = h;
            return WG_OK;
        }
    }
    return fail(WG_RIEMANN, "SweRiemann: Newton iteration did not converge");
}

/* SweRiemann::sample, solver.hpp:128-164 */
static wg_status swe_sample(double g, double hl, double ul, double utl, double hr, double ur,
                            double utr, double xi, double* o) {
    double hs;
    wg_status st = solve_hstar(g, hl, ul, hr, ur, &hs);
    if (st) return st;
    const double us = 0.5 * (ul + ur) + 0.5 * (phi_side(hs, hr, g) - phi_side(hs, hl, g));
    const double ut = xi <= us ? utl : utr;
    o[2] = ut;
    if (xi <= us) {
        const double cl = sqrt(g * hl), cs = sqrt(g * hs);
        if (hs > hl) {
            const double sl = ul - cl * sqrt(0.5 * (hs + hl) * hs / (hl * hl));
            if (xi <= sl) { o[0] = hl; o[1] = ul; return WG_OK; }
            o[0] = hs; o[1] = us; return WG_OK;
        }
        const double head = ul - cl, tail = us - cs;
        if (xi <= head) { o[0] = hl; o[1] = ul; return WG_OK; }
        if (xi >= tail) { o[0] = hs; o[1] = us; return WG_OK; }
        const double u = (ul + 2.0 * cl + 2.0 * xi) / 3.0;
        const double c = (ul + 2.0 * cl - xi) / 3.0;
        o[0] = c * c / g; o[1] = u; return WG_OK;
    }
    const double crr = sqrt(g * hr), cs = sqrt(g * hs);
    if (hs > hr) {
        const double sr = ur + crr * sqrt(0.5 * (hs + hr) * hs / (hr * hr));
        if (xi >= sr) { o[0] = hr; o[1] = ur; return WG_OK; }
        o[0] = hs; o[1] = us; return WG_OK;
    }
    const double head = ur + crr, tail = us + cs;
    if (xi >= head) { o[0] = hr; o[1] = ur; return WG_OK; }
    if (xi <= tail) { o[0] = hs; o[1] = us; return WG_OK; }
    const double u = (ur - 2.0 * crr + 2.0 * xi) / 3.0;
    const double c = (-ur + 2.0 * crr + xi) / 3.0;
    o[0] = c * c / g; o[1] = u; return WG_OK;
}

/* flux_godunov_swe, solver.hpp:169-189 */
static wg_status flux_swe(const double* wl, const double* wr, const int* n, double g,
                          double* f) {
    const double hl = wl[0], hr = wr[0];
    if (hl <= 0.0 || hr <= 0.0)
        return fail(WG_DOMAIN, "flux_godunov_swe: water depth must be positive");
    const double nx = (double)n[0], ny = (double)n[1];
    const double ul = (wl[1] * nx + wl[2] * ny) / hl;
    const double utl = (-wl[1] * ny + wl[2] * nx) / hl;
    const double ur = (wr[1] * nx + wr[2] * ny) / hr;
    const double utr = (-wr[1] * ny + wr[2] * nx) / hr;
    double s[3];
    wg_status st = swe_sample(g, hl, ul, utl, hr, ur, utr, 0.0, s);
    if (st) return st;
    const double h = s[0], un = s[1], ut = s[2];
    const double fn_mass = h * un;
    const double fn_mom = h * un * un + 0.5 * g * h * h;
    const double ft_mom = h * un * ut;
    f[0] = fn_mass;
    f[1] = fn_mom * nx - ft_mom * ny;
    f[2] = fn_mom * ny + ft_mom * nx;
    return WG_OK;
}

/* fv_step<Flux>, solver.hpp:207-231, one patch (m = 1 or 3). */
static wg_status fv_step_patch(const grid_t* g, const double* cur, double* next, uint64_t p,
                               int scheme, double a, double b, double grav, double dt,
                               double dx) {
    const uint32_t m = g->m;
    const uint64_t nx = g->tdims[0], ny = g->tdims[1];
    const double r = dt / dx;
    double w[3], wn[3], out[3], f[3];
    for (uint64_t i = 1; i + 1 < nx; ++i)
        for (uint64_t j = 1; j + 1 < ny; ++j) {
            for (uint32_t c = 0; c < m; ++c) w[c] = comp_ptr(g, (double*)cur, p, c)[i * ny + j];
            for (uint32_t c = 0; c < m; ++c) out[c] = w[c];
            for (int k = 0; k < 4; ++k) {
                const uint64_t ii = i + (uint64_t)(int64_t)kDirs[k][0];
                const uint64_t jj = j + (uint64_t)(int64_t)kDirs[k][1];
                for (uint32_t c = 0; c < m; ++c)
                    wn[c] = comp_ptr(g, (double*)cur, p, c)[ii * ny + jj];
                if (scheme == WG_SCHEME_TRANSPORT) {
                    f[0] = flux_upwind(w[0], wn[0], kDirs[k], a, b);
                } else {
                    wg_status st = flux_swe(w, wn, kDirs[k], grav, f);
                    if (st) return st;
                }
                for (uint32_t c = 0; c < m; ++c) out[c] -= r * f[c];
            }
            for (uint32_t c = 0; c < m; ++c) comp_ptr(g, next, p, c)[i * ny + j] = out[c];
        }
    return WG_OK;
}

wg_status wg_fv_step(const wg_grid_desc* d, const double* cur, double* next, int32_t scheme,
                     double alpha, double beta, double gravity, double dt, double dx) {
    grid_t g;
    wg_status st = grid_init(d, &g);
    if (st) return st;
    if (g.rank != 2) return fail(WG_INVALID_ARGUMENT, "fv_step: 2-D grids only");
    if (scheme != WG_SCHEME_TRANSPORT && scheme != WG_SCHEME_SWE)
        return fail(WG_INVALID_ARGUMENT, "fv_step: unknown scheme");
    if (g.m != (scheme == WG_SCHEME_SWE ? 3u : 1u))
        return fail(WG_INVALID_ARGUMENT, "fv_step: component count");
    for (uint64_t p = 0; p < g.npatch; ++p) {
        st = fv_step_patch(&g, cur, next, p, scheme, alpha, beta, gravity, dt, dx);
        if (st) return st;
    }
    return WG_OK;
}

/* ---- D2Q9 LBM (builder-defined; mirrors oracle/ref_shim.cpp) -------- */

static const int kCx[9] = {0, 1, -1, 0, 0, 1, -1, 1, -1};
static const int kCy[9] = {0, 0, 0, 1, -1, 1, -1, -1, 1};
static const double kW[9] = {4.0 / 9.0,  1.0 / 9.0,  1.0 / 9.0,  1.0 / 9.0, 1.0 / 9.0,
                             1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0};

static void lbm_cu(double ux, double uy, double* cu) {
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

/* D2Q9 BGK in its FMA form (csrc/physics.cuh): C99 fma() is
 * correctly rounded, so this restatement and the device agree bit for bit. */
static inline double lbm_usq(double ux, double uy) { return fma(ux, ux, uy * uy); }

static inline double lbm_feq(int q, double rho, double cu, double usq) {
    const double t = fma(cu, fma(4.5, cu, 3.0), fma(-1.5, usq, 1.0));
    return (kW[q] * rho) * t;
}

static void lbm_collide(const double* f, double omega, double* out) {
    const double rho = ((((((((f[0] + f[1]) + f[2]) + f[3]) + f[4]) + f[5]) + f[6]) + f[7]) + f[8]);
    const double jx = ((f[1] - f[2]) + (f[5] - f[6])) + (f[7] - f[8]);
    const double jy = ((f[3] - f[4]) + (f[5] - f[6])) + (f[8] - f[7]);
    const double inv = 1.0 / rho;
    const double ux = jx * inv, uy = jy * inv;
    const double usq = lbm_usq(ux, uy);
    double cu[9];
    lbm_cu(ux, uy, cu);
    for (int q = 0; q < 9; ++q) out[q] = fma(omega, lbm_feq(q, rho, cu[q], usq) - f[q], f[q]);
}

static void lbm_step_patch(const grid_t* g, const double* cur, double* next, uint64_t p,
                           double omega) {
    const uint64_t nx = g->tdims[0], ny = g->tdims[1];
    double f[9], out[9];
    for (uint64_t i = 1; i + 1 < nx; ++i)
        for (uint64_t j = 1; j + 1 < ny; ++j) {
            for (int q = 0; q < 9; ++q)
                f[q] = comp_ptr(g, (double*)cur, p, q)[(i - kCx[q]) * ny + (j - kCy[q])];
            lbm_collide(f, omega, out);
            for (int q = 0; q < 9; ++q) comp_ptr(g, next, p, q)[i * ny + j] = out[q];
        }
}

wg_status wg_lbm_step(const wg_grid_desc* d, const double* cur, double* next, double tau) {
    grid_t g;
    wg_status st = grid_init(d, &g);
    if (st) return st;
    if (g.rank != 2 || g.m != 9) return fail(WG_INVALID_ARGUMENT, "lbm_step: 2-D, 9 components");
    for (uint64_t p = 0; p < g.npatch; ++p) lbm_step_patch(&g, cur, next, p, 1.0 / tau);
    return WG_OK;
}

/* ---- pipeline.hpp: run() -------------------------------------------- */

void wg_run_config_default(wg_run_config* c) { /* RunConfig{}, SimConfig{} */
    memset(c, 0, sizeof *c);
    c->scheme = WG_SCHEME_TRANSPORT;
    c->levels = 4;
    c->nx = 129;
    c->splits[0] = 2;
    c->splits[1] = 2;
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

static uint32_t comps_of(int scheme) {
    return scheme == WG_SCHEME_LBM_D2Q9 ? 9u : (scheme == WG_SCHEME_SWE ? 3u : 1u);
}

static wg_status run_grid(const wg_run_config* c, grid_t* g) {
    wg_grid_desc d;
    memset(&d, 0, sizeof d);
    d.rank = 2;
    d.components = comps_of(c->scheme);
    d.periodic = 1;
    d.global_dims[0] = d.global_dims[1] = c->nx;
    d.splits[0] = c->splits[0];
    d.splits[1] = c->splits[1];
    return grid_init(&d, g);
}

/* SimConfig::validate, solver.hpp:40-45 */
static wg_status sim_validate(const wg_run_config* c) {
    if (c->cfl <= 0.0 || c->cfl > 1.0) return fail(WG_INVALID_ARGUMENT, "SimConfig: CFL must be in (0, 1]");
    if (c->nx < 2) return fail(WG_INVALID_ARGUMENT, "SimConfig: nx too small");
    if (c->t_end < 0.0) return fail(WG_INVALID_ARGUMENT, "SimConfig: negative t_end");
    return WG_OK;
}

static inline double sim_dx(const wg_run_config* c) {
    return c->domain_length / (double)(c->nx - 1);
}

wg_status wg_run_step_count(const wg_run_config* c, uint64_t* steps) {
    if (c->scheme == WG_SCHEME_LBM_D2Q9) {
        *steps = c->lbm_steps;
        return WG_OK;
    }
    if (c->scheme != WG_SCHEME_TRANSPORT) {
        *steps = 0;
        return WG_OK;
    }
    wg_status st = sim_validate(c);
    if (st) return st;
    const double dt0 = c->cfl * sim_dx(c) / smax(c->alpha, c->beta);
    double t = 0.0;
    uint64_t n = 0;
    while (t < c->t_end - 1e-15) {
        t += smin(dt0, c->t_end - t);
        ++n;
    }
    *steps = n;
    return WG_OK;
}

wg_status wg_run_grid_doubles(const wg_run_config* c, uint64_t* n) {
    grid_t g;
    wg_status st = run_grid(c, &g);
    if (st) return st;
    *n = g.npatch * g.m * g.tcount;
    return WG_OK;
}

/* wrap_unit / exact_transport, solver.hpp:264-287 (value at global (i,j)). */
static inline double wrap_unit(double x) {
    x = fmod(x, 1.0);
    return x < 0.0 ? x + 1.0 : x;
}
static double exact_transport_at(const wg_run_config* c, double t, uint64_t i, uint64_t j) {
    const double dx = sim_dx(c);
    double px = wrap_unit((double)i * dx - c->alpha * t) - 0.5;
    double py = wrap_unit((double)j * dx - c->beta * t) - 0.5;
    if (px < -0.5) px += 1.0;
    if (px >= 0.5) px -= 1.0;
    if (py < -0.5) py += 1.0;
    if (py >= 0.5) py -= 1.0;
    return 1.0 + exp(-30.0 * (px * px + py * py));
}

/* fill(), patchgrid.hpp:106-126, with the run() initial states
 * (pipeline.hpp:138-155) and the LBM shear layer. */
wg_status wg_run_initial_state(const wg_run_config* c, double* buf) {
    grid_t g;
    wg_status st = run_grid(c, &g);
    if (st) return st;
    memset(buf, 0, sizeof(double) * g.npatch * g.m * g.tcount);
    const double dx = sim_dx(c);
    const double inv = 1.0 / (double)(c->nx - 1);
    uint64_t coord[3];
    for (uint64_t p = 0; p < g.npatch; ++p) {
        patch_coord(&g, p, coord);
        for (uint64_t i = 1; i <= g.n[0]; ++i)
            for (uint64_t j = 1; j <= g.n[1]; ++j) {
                const uint64_t gi = coord[0] * (g.n[0] - 1) + i - 1;
                const uint64_t gj = coord[1] * (g.n[1] - 1) + j - 1;
                const uint64_t off = i * g.tdims[1] + j;
                if (c->scheme == WG_SCHEME_TRANSPORT) {
                    comp_ptr(&g, buf, p, 0)[off] = exact_transport_at(c, 0.0, gi, gj);
                } else if (c->scheme == WG_SCHEME_SWE) {
                    const double x = (double)gi * dx / c->domain_length;
                    const double y = (double)gj * dx / c->domain_length;
                    const int inside = fabs(x - 0.5) <= 0.25 && fabs(y - 0.5) <= 0.25;
                    comp_ptr(&g, buf, p, 0)[off] = inside ? 2.0 : 1.0;
                } else {
                    const double X = (double)gi * inv, Y = (double)gj * inv;
                    const double uy = X <= 0.5 ? c->lbm_u0 * tanh(c->lbm_kappa * (X - 0.25))
                                               : c->lbm_u0 * tanh(c->lbm_kappa * (0.75 - X));
                    const double ux =
                        c->lbm_delta * c->lbm_u0 * sin(2.0 * 3.141592653589793 * (Y + 0.25));
                    double cu[9];
                    lbm_cu(ux, uy, cu);
                    for (int q = 0; q < 9; ++q)
                        comp_ptr(&g, buf, p, q)[off] = lbm_feq(q, 1.0, cu[q], lbm_usq(ux, uy));
                }
            }
    }
    return WG_OK;
}

/* cfl_dt, solver.hpp:235-258 */
static wg_status cfl_dt_g(const wg_run_config* c, const grid_t* g, const double* buf,
                          double* dt) {
    wg_status st = sim_validate(c);
    if (st) return st;
    if (c->scheme == WG_SCHEME_TRANSPORT) {
        const double vmax = smax(c->alpha, c->beta);
        if (vmax <= 0.0) return fail(WG_INVALID_ARGUMENT, "cfl_dt: nonpositive speed");
        *dt = c->cfl * sim_dx(c) / vmax;
        return WG_OK;
    }
    double vmax = 0.0;
    const uint64_t ny = g->tdims[1];
    for (uint64_t p = 0; p < g->npatch; ++p) {
        const double* h0 = comp_ptr(g, (double*)buf, p, 0);
        const double* h1 = comp_ptr(g, (double*)buf, p, 1);
        const double* h2 = comp_ptr(g, (double*)buf, p, 2);
        for (uint64_t i = 1; i <= g->n[0]; ++i)
            for (uint64_t j = 1; j <= g->n[1]; ++j) {
                const double h = h0[i * ny + j];
                if (h <= 0.0) return fail(WG_DOMAIN, "cfl_dt: nonpositive depth");
                const double cc = sqrt(c->gravity * h);
                const double u = fabs(h1[i * ny + j] / h);
                const double v = fabs(h2[i * ny + j] / h);
                /* std::max({vmax, u + c, v + c}) : first largest wins */
                double mx = vmax;
                if (mx < u + cc) mx = u + cc;
                if (mx < v + cc) mx = v + cc;
                vmax = mx;
            }
    }
    if (vmax <= 0.0) return fail(WG_INVALID_ARGUMENT, "cfl_dt: zero wave speed");
    *dt = c->cfl * sim_dx(c) / vmax;
    return WG_OK;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* The per-patch compression cycle of run(), pipeline.hpp:217-257:
 * extract_logical -> dwt_nd -> apply_threshold -> encode/decode (CSR) ->
 * nnz count -> skip rule -> idwt_nd -> insert_logical. */
/* lz_encode_chunk (codec.hpp:127-175): the greedy LZ parse of one chunk
 * (13-bit hash of 4 bytes, minimum match 4, offsets <= 65535, literal/match
 * lengths extended with 255-bytes); returns the payload length and writes
 * the payload to out when out != NULL. */
static uint64_t lz_put_len(unsigned char* out, uint64_t o, uint64_t len) { /* lz_put_length, codec.hpp:113-119 */
    while (len >= 255) {
        if (out) out[o] = 255;
        ++o;
        len -= 255;
    }
    if (out) out[o] = (unsigned char)len;
    return o + 1;
}
static uint64_t lz_put_seq(unsigned char* out, uint64_t o, const unsigned char* in, uint64_t anchor, uint64_t lit,
                           int64_t ml, uint64_t offset) {
    const unsigned ln = lit < 15 ? (unsigned)lit : 15u;
    const unsigned mn = ml < 0 ? 0u : (ml < 15 ? (unsigned)ml : 15u);
    if (out) out[o] = (unsigned char)((ln << 4) | mn);
    ++o;
    if (ln == 15) o = lz_put_len(out, o, lit - 15);
    if (out) memcpy(out + o, in + anchor, lit);
    o += lit;
    if (ml < 0) return o;
    if (out) {
        out[o] = (unsigned char)(offset & 0xff);
        out[o + 1] = (unsigned char)(offset >> 8);
    }
    o += 2;
    if (mn == 15) o = lz_put_len(out, o, (uint64_t)ml - 15);
    return o;
}
static uint64_t lz_chunk_encode(const unsigned char* in, uint64_t n, unsigned char* out) {
    static int64_t table[1u << 13];
    for (uint32_t k = 0; k < (1u << 13); ++k) table[k] = -1;
    uint64_t anchor = 0, pos = 0, o = 0;
    while (n >= 4 && pos + 4 <= n) {
        uint32_t v;
        memcpy(&v, in + pos, 4);
        const uint32_t h = (v * 2654435761u) >> 19;
        const int64_t cand = table[h];
        table[h] = (int64_t)pos;
        if (cand >= 0 && pos - (uint64_t)cand <= 65535 && memcmp(in + cand, in + pos, 4) == 0) {
            uint64_t len = 4;
            while (pos + len < n && in[cand + len] == in[pos + len]) ++len;
            o = lz_put_seq(out, o, in, anchor, pos - anchor, (int64_t)(len - 4), pos - (uint64_t)cand);
            pos += len;
            anchor = pos;
            continue;
        }
        ++pos;
    }
    if (anchor < n) o = lz_put_seq(out, o, in, anchor, n - anchor, -1, 0);
    return o;
}
static uint64_t lz_chunk_payload(const unsigned char* in, uint64_t n) { return lz_chunk_encode(in, n, NULL); }

/* lz_decode_chunk (codec.hpp:177-220): 0 or the reason (1 truncated,
 * 2 raw_len overrun, 3 bad match offset, 4 trailing bytes). */
static int lz_get_len(const unsigned char* in, uint64_t in_len, uint64_t* p, uint64_t base, uint64_t* len) {
    *len = base;
    if (base == 15) {
        unsigned b;
        do {
            if (*p + 1 > in_len) return 1;
            b = in[(*p)++];
            *len += b;
        } while (b == 255);
    }
    return 0;
}
static int lz_chunk_decode(const unsigned char* in, uint64_t in_len, uint64_t raw_len, unsigned char* out) {
    uint64_t p = 0, o = 0;
    while (o < raw_len) {
        if (p + 1 > in_len) return 1;
        const unsigned token = in[p++];
        uint64_t lit, ml;
        if (lz_get_len(in, in_len, &p, token >> 4, &lit)) return 1;
        if (p + lit > in_len) return 1;
        if (o + lit > raw_len) return 2;
        memcpy(out + o, in + p, lit);
        p += lit;
        o += lit;
        if (o == raw_len) break;
        if (p + 2 > in_len) return 1;
        const uint64_t offset = (uint64_t)in[p] | ((uint64_t)in[p + 1] << 8);
        p += 2;
        if (lz_get_len(in, in_len, &p, token & 0x0f, &ml)) return 1;
        ml += 4;
        if (offset == 0 || offset > o) return 3;
        if (o + ml > raw_len) return 2;
        for (uint64_t i = 0; i < ml; ++i) out[o + i] = out[o - offset + i];
        o += ml;
    }
    return p != in_len ? 4 : 0;
}

wg_status wg_lz_encode(const uint8_t* data, uint64_t n, uint64_t chunk, uint8_t* out, uint64_t cap,
                       uint64_t* enc_len, uint64_t* out_len) {
    if (chunk == 0) return fail(WG_INVALID_ARGUMENT, "lz_encode: chunk_size must be > 0");
    uint64_t tot = 0, k = 0;
    for (uint64_t off = 0; off < n; off += chunk, ++k) { /* lz_encode, codec.hpp:223-235 */
        const uint64_t len = n - off < chunk ? n - off : chunk;
        const uint64_t m = lz_chunk_payload(data + off, len);
        if (enc_len) enc_len[k] = m;
        if (out) {
            if (tot + m > cap) return fail(WG_OUT_OF_RANGE, "lz_encode: output buffer too small");
            lz_chunk_encode(data + off, len, out + tot);
        }
        tot += m;
    }
    if (out_len) *out_len = tot;
    return WG_OK;
}

wg_status wg_lz_decode(const uint8_t* payload, const uint64_t* enc_len, uint64_t chunk, uint8_t* out, uint64_t n) {
    static const char* why[] = {"", "lz_decode: truncated chunk", "lz_decode: raw_len overrun",
                                "lz_decode: bad match offset", "lz_decode: trailing bytes"};
    if (chunk == 0) return fail(WG_INVALID_ARGUMENT, "lz_decode: chunk_size must be > 0");
    uint64_t p = 0, k = 0;
    for (uint64_t off = 0; off < n; off += chunk, ++k) { /* lz_decode, codec.hpp:237-244 */
        const uint64_t len = n - off < chunk ? n - off : chunk;
        const int e = lz_chunk_decode(payload + p, enc_len[k], len, out + off);
        if (e) return fail(WG_CORRUPT_STREAM, why[e]);
        p += enc_len[k];
    }
    return WG_OK;
}

/* LzStream::byte_size of lz_encode(bytes, chunk) (codec.hpp:99-105, 223-235). */
static uint64_t lz_stream_size(const double* a, uint64_t count, uint64_t chunk) {
    const unsigned char* b = (const unsigned char*)a;
    const uint64_t bytes = count * 8;
    uint64_t s = 0;
    for (uint64_t off = 0; off < bytes; off += chunk)
        s += 8 + lz_chunk_payload(b + off, bytes - off < chunk ? bytes - off : chunk);
    return s;
}

static wg_status compress_patch(const wg_run_config* c, const grid_t* g, double* buf,
                                uint64_t p, double* work, uint64_t* st_comp, uint64_t* st_nnz,
                                uint64_t* st_zeroed) {
    const uint64_t n0 = g->n[0], n1 = g->n[1], ny = g->tdims[1];
    const uint64_t dims[2] = {n0, n1};
    const uint32_t m = g->m;
    uint64_t zeroed = 0, nnz = 0, comp_bytes = 0;
    double* orig = work;              /* m * n0 * n1 */
    double* coef = work + m * n0 * n1; /* m * n0 * n1 */
    for (uint32_t q = 0; q < m; ++q) {
        const double* f = comp_ptr(g, buf, p, q);
        double* o = orig + q * n0 * n1;
        for (uint64_t i = 0; i < n0; ++i)
            for (uint64_t j = 0; j < n1; ++j) o[i * n1 + j] = f[(i + 1) * ny + (j + 1)];
        double* cs = coef + q * n0 * n1;
        wg_status st = wg_dwt_nd(o, cs, dims, 2, c->levels);
        if (st) return st;
    }
    for (uint32_t q = 0; q < m; ++q) {
        uint64_t z = 0;
        wg_status st = wg_apply_threshold(coef + q * n0 * n1, dims, 2, c->levels,
                                          c->threshold_mode, c->c, c->threshold_alpha, &z);
        if (st) return st;
        zeroed += z;
    }
    for (uint32_t q = 0; q < m; ++q) { /* CSR round trip: bytes, nnz, -0.0 -> +0.0 */
        double* cs = coef + q * n0 * n1;
        if (c->codec == 2) comp_bytes += lz_stream_size(cs, n0 * n1, c->lz_chunk_size); /* Codec::lz: the thresholded bytes */
        uint64_t k = 0;
        for (uint64_t e = 0; e < n0 * n1; ++e) {
            if (cs[e] != 0.0) ++k;
            else cs[e] = 0.0;
        }
        nnz += k;
        if (c->codec == 1) comp_bytes += 12 * k + 4 * (n0 + 1); /* CsrBlock::byte_size, codec.hpp:33 */
    }
    for (uint32_t q = 0; q < m; ++q) {
        double* f = comp_ptr(g, buf, p, q);
        double* src = orig + q * n0 * n1;
        if (zeroed != 0) {
            wg_status st = wg_idwt_nd(coef + q * n0 * n1, coef + q * n0 * n1, dims, 2, c->levels);
            if (st) return st;
            src = coef + q * n0 * n1;
        }
        for (uint64_t i = 0; i < n0; ++i)
            for (uint64_t j = 0; j < n1; ++j) f[(i + 1) * ny + (j + 1)] = src[i * n1 + j];
    }
    *st_comp = comp_bytes;
    *st_nnz = nnz;
    *st_zeroed = zeroed;
    return WG_OK;
}

/* run(RunConfig), pipeline.hpp:129-305 (single thread; the thread count of
 * the reference does not change results, test_pipeline.cpp:55-71). */
/* run(), pipeline.hpp:129-305; the hook is called where run() writes the
 * metrics line and calls the observer (pipeline.hpp:285-286). */
wg_status wg_run_hooked(const wg_run_config* c, wg_metrics_row* rows, uint64_t max_rows,
                        uint64_t* nrows, double* final_grid, wg_run_summary* summary,
                        wg_step_hook hook, void* user) {
    grid_t g;
    wg_status st;
    if (c->scheme != WG_SCHEME_LBM_D2Q9 && (st = sim_validate(c))) return st;
    if ((st = run_grid(c, &g))) return st;
    if ((st = plan_validate(g.n, 2, c->levels))) return st;
    if (c->codec != 1 && c->codec != 2) return fail(WG_INVALID_ARGUMENT, "unknown codec");
    if (c->codec == 2 && c->lz_chunk_size == 0)
        return fail(WG_INVALID_ARGUMENT, "lz_encode: chunk_size must be > 0");
    if (c->scheme == WG_SCHEME_LBM_D2Q9 && c->lbm_tau <= 0.5)
        return fail(WG_INVALID_ARGUMENT, "LBM: tau must exceed 1/2");
    const uint64_t total = g.npatch * g.m * g.tcount;
    double* grid = calloc(total, sizeof(double));
    double* scratch = calloc(total, sizeof(double));
    double* work = malloc(sizeof(double) * 2 * g.m * g.n[0] * g.n[1]);
    double* asm_buf = malloc(sizeof(double) * c->nx * c->nx);
    char* seen = malloc(c->nx * c->nx);
    st = wg_run_initial_state(c, grid);
    if (!st) memcpy(scratch, grid, total * sizeof(double)); /* PatchGrid scratch = grid */
    const double dx = sim_dx(c);
    const uint64_t dense_patch = 8 * g.n[0] * g.n[1] * g.m; /* CompressedPatch::dense_bytes */
    double t = 0.0, step_s = 0.0, ratio_sum = 0.0;
    uint64_t step = 0;
    const double t_start = now_s();
    while (!st) {
        double dt = 1.0;
        if (c->scheme == WG_SCHEME_LBM_D2Q9) {
            if (step >= c->lbm_steps) break;
        } else {
            if (!(t < c->t_end - 1e-15)) break;
            if ((st = cfl_dt_g(c, &g, grid, &dt))) break;
            dt = smin(dt, c->t_end - t);
        }
        sync_ghosts_g(&g, grid);
        const double t0 = now_s();
        for (uint64_t p = 0; p < g.npatch && !st; ++p) {
            if (c->scheme == WG_SCHEME_LBM_D2Q9)
                lbm_step_patch(&g, grid, scratch, p, 1.0 / c->lbm_tau);
            else
                st = fv_step_patch(&g, grid, scratch, p, c->scheme, c->alpha, c->beta,
                                   c->gravity, dt, dx);
        }
        if (st) break;
        double* sw = grid; /* std::swap(grid.patches, scratch.patches) */
        grid = scratch;
        scratch = sw;
        step_s += now_s() - t0;
        t += dt;
        ++step;
        double mass_before = 0.0;
        if (c->strict) mass_before = global_mass_g(&g, grid, 0);
        wg_metrics_row row;
        memset(&row, 0, sizeof row);
        row.step = step;
        row.time = c->scheme == WG_SCHEME_LBM_D2Q9 ? (double)step : t;
        row.ratio = 1.0;
        if (!c->no_compression) {
            for (uint64_t p = 0; p < g.npatch && !st; ++p) {
                uint64_t cb = 0, nz = 0, zr = 0;
                st = compress_patch(c, &g, grid, p, work, &cb, &nz, &zr);
                row.dense_bytes += dense_patch;
                row.compressed_bytes += cb;
                row.nnz += nz;
                row.zeroed += zr;
            }
            if (st) break;
            row.ratio = row.compressed_bytes > 0
                            ? (double)row.dense_bytes / (double)row.compressed_bytes
                            : 1.0;
        }
        if (c->scheme == WG_SCHEME_LBM_D2Q9) {
            double mass = 0.0;
            for (uint32_t q = 0; q < 9; ++q) mass += global_mass_g(&g, grid, q);
            row.global_mass = mass;
        } else {
            row.global_mass = global_mass_g(&g, grid, 0);
        }
        if (c->scheme == WG_SCHEME_TRANSPORT && c->compute_l2) { /* l2_error, solver.hpp:290-300 */
            if ((st = assemble_g(&g, grid, 0, 1e-12, asm_buf, seen))) break;
            double sum = 0.0;
            for (uint64_t i = 0; i < c->nx; ++i)
                for (uint64_t j = 0; j < c->nx; ++j) {
                    const double d = asm_buf[i * c->nx + j] - exact_transport_at(c, t, i, j);
                    sum += d * d;
                }
            const double area = c->domain_length * c->domain_length;
            row.l2 = area / (double)(c->nx * c->nx) * sum;
        }
        if (c->strict && !c->no_compression) {
            const double scale = smax(fabs(mass_before), 1.0);
            if (fabs(row.global_mass - mass_before) > 1e-12 * scale) {
                st = fail(WG_CONSISTENCY, "strict: compression cycle changed global mass");
                break;
            }
            if ((st = assemble_g(&g, grid, 0, 1e-12, asm_buf, seen))) break;
        }
        if (hook) {
            int k = hook(user, &row, NULL);
            if (k == WG_HOOK_WANT_GRID) k = hook(user, &row, grid);
            if (k < 0) {
                st = fail(WG_ABORTED, "run stopped by its step hook");
                break;
            }
        }
        if (rows && step <= max_rows) rows[step - 1] = row;
        ratio_sum += row.ratio;
    }
    if (!st) {
        if (nrows) *nrows = step;
        if (final_grid) memcpy(final_grid, grid, total * sizeof(double));
        if (summary) {
            memset(summary, 0, sizeof *summary);
            summary->avg_ratio = step ? ratio_sum / (double)step : 1.0;
            summary->total_seconds = now_s() - t_start;
            summary->step_seconds = step_s;
            summary->t_final = t;
            summary->steps = step;
        }
    }
    free(grid);
    free(scratch);
    free(work);
    free(asm_buf);
    free(seen);
    return st;
}

wg_status wg_run(const wg_run_config* c, wg_metrics_row* rows, uint64_t max_rows,
                 uint64_t* nrows, double* final_grid, wg_run_summary* summary) {
    return wg_run_hooked(c, rows, max_rows, nrows, final_grid, summary, NULL, NULL);
}
