// physics.cuh — the scheme updates (device), in the reference's exact
// operation order.  Compiled with -fmad=false: no FMA contraction, matching
// the reference's x86-64 Release build.
#pragma once

#include <cmath>

namespace wg {

// ---- transport: flux_upwind, solver.hpp:53-57 --------------------------------
// smax/smin are std::max(speed, 0.0) / std::min(speed, 0.0) of the direction,
// computed once on the host with the reference's formula.
__host__ __device__ __forceinline__ double flux_upwind(double wl, double wr, double smax,
                                                        double smin) {
    return wl * smax + wr * smin;
}

// ---- shallow water: solver.hpp:74-199 ---------------------------------------
struct SweStatus {
    int err;  // 0 ok, 1 domain, 2 riemann
};

__device__ __forceinline__ double phi_side(double h, double hs, double g) {
    if (h <= hs) return 2.0 * (sqrt(g * h) - sqrt(g * hs));
    return (h - hs) * sqrt(g * (h + hs) / (2.0 * h * hs));
}

__device__ __forceinline__ double phi_side_deriv(double h, double hs, double g) {
    if (h <= hs) return sqrt(g / h);
    const double a = sqrt(g * (h + hs) / (2.0 * h * hs));
    return a - (h - hs) * g / (4.0 * a * h * h);
}

// SweRiemann::solve_hstar, solver.hpp:107-124 (std::pow(x, 2) as x * x).
__device__ __forceinline__ double solve_hstar(double g, double hl, double ul, double hr,
                                              double ur, int& err) {
    if (hl <= 0.0 || hr <= 0.0) {
        err = 1;
        return 1.0;
    }
    const double cl = sqrt(g * hl), cr = sqrt(g * hr);
    const double b = 0.5 * (cl + cr) + 0.25 * (ul - ur);
    double h = (b * b) / g;
    h = (h < 1e-12) ? 1e-12 : h;
    for (int it = 0; it < 100; ++it) {
        const double f = phi_side(h, hl, g) + phi_side(h, hr, g) + ur - ul;
        const double df = phi_side_deriv(h, hl, g) + phi_side_deriv(h, hr, g);
        double dh = f / df;
        if (h - dh <= 0.0) dh = h / 2.0;
        h -= dh;
        if (fabs(dh) < 1e-10) return h;
    }
    err = 2;
    return h;
}

// flux_godunov_swe at xi = 0, solver.hpp:128-189.
__device__ __forceinline__ void flux_swe(const double* wl, const double* wr, int nxi, int nyi,
                                         double g, double* f, int& err) {
    const double hl = wl[0], hr = wr[0];
    if (hl <= 0.0 || hr <= 0.0) {
        err = 1;
        f[0] = f[1] = f[2] = 0.0;
        return;
    }
    const double nx = (double)nxi, ny = (double)nyi;
    const double ul = (wl[1] * nx + wl[2] * ny) / hl;
    const double utl = (-wl[1] * ny + wl[2] * nx) / hl;
    const double ur = (wr[1] * nx + wr[2] * ny) / hr;
    const double utr = (-wr[1] * ny + wr[2] * nx) / hr;
    const double xi = 0.0;
    const double hs = solve_hstar(g, hl, ul, hr, ur, err);
    const double us = 0.5 * (ul + ur) + 0.5 * (phi_side(hs, hr, g) - phi_side(hs, hl, g));
    const double ut = xi <= us ? utl : utr;
    double h, un;
    if (xi <= us) {
        const double cl = sqrt(g * hl), cs = sqrt(g * hs);
        if (hs > hl) {
            const double sl = ul - cl * sqrt(0.5 * (hs + hl) * hs / (hl * hl));
            if (xi <= sl) { h = hl; un = ul; }
            else { h = hs; un = us; }
        } else {
            const double head = ul - cl, tail = us - cs;
            if (xi <= head) { h = hl; un = ul; }
            else if (xi >= tail) { h = hs; un = us; }
            else {
                const double u = (ul + 2.0 * cl + 2.0 * xi) / 3.0;
                const double c = (ul + 2.0 * cl - xi) / 3.0;
                h = c * c / g;
                un = u;
            }
        }
    } else {
        const double crr = sqrt(g * hr), cs = sqrt(g * hs);
        if (hs > hr) {
            const double sr = ur + crr * sqrt(0.5 * (hs + hr) * hs / (hr * hr));
            if (xi >= sr) { h = hr; un = ur; }
            else { h = hs; un = us; }
        } else {
            const double head = ur + crr, tail = us + cs;
            if (xi >= head) { h = hr; un = ur; }
            else if (xi <= tail) { h = hs; un = us; }
            else {
                const double u = (ur - 2.0 * crr + 2.0 * xi) / 3.0;
                const double c = (-ur + 2.0 * crr + xi) / 3.0;
                h = c * c / g;
                un = u;
            }
        }
    }
    const double fn_mass = h * un;
    const double fn_mom = h * un * un + 0.5 * g * h * h;
    const double ft_mom = h * un * ut;
    f[0] = fn_mass;
    f[1] = fn_mom * nx - ft_mom * ny;
    f[2] = fn_mom * ny + ft_mom * nx;
}

// ---- the four faces of one cell, solved in lock-step -------------------------
// Same arithmetic as flux_swe (every value below is produced by the very
// expression the reference evaluates, so the results are bit-identical), with
// two changes that only remove work or add parallelism:
//  * common subexpressions are computed once: sqrt(g h) and sqrt(g / h) are
//    shared by both sides of the Newton function, the shock factor
//    sqrt(g (h + hs) / (2 h hs)) by phi_side and phi_side_deriv, and
//    sqrt(g hl), sqrt(g hr) (the cl, cr of solve_hstar) by the whole solve;
//  * the 4 Newton iterations of a cell (faces +x, -x, +y, -y) advance
//    together, each stopping at its own convergence (or after its own 100
//    iterations), so a thread has 4 independent dependency chains in flight.
// f[k] receives the flux of face k; err as flux_swe (1 domain, 2 riemann).
__device__ __forceinline__ void swe_cell_fluxes(const double (&w)[3], const double (&wn)[4][3], double g,
                                                double (&f)[4][3], int& err) {
    constexpr double NX[4] = {1.0, -1.0, 0.0, 0.0}, NY[4] = {0.0, 0.0, 1.0, -1.0};
    const double hl = w[0];
    double hr[4], ul[4], utl[4], ur[4], utr[4], cr[4], h[4];
    unsigned act = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        hr[k] = wn[k][0];
        f[k][0] = f[k][1] = f[k][2] = 0.0;
        if (hl <= 0.0 || hr[k] <= 0.0) {  // flux_godunov_swe / solve_hstar domain checks
            err = 1;
            continue;
        }
        act |= 1u << k;
    }
    if (!act) return;
    const double cl = sqrt(g * hl);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        ul[k] = (w[1] * NX[k] + w[2] * NY[k]) / hl;
        utl[k] = (-w[1] * NY[k] + w[2] * NX[k]) / hl;
        ur[k] = (wn[k][1] * NX[k] + wn[k][2] * NY[k]) / hr[k];
        utr[k] = (-wn[k][1] * NY[k] + wn[k][2] * NX[k]) / hr[k];
        cr[k] = sqrt(g * hr[k]);
        const double b = 0.5 * (cl + cr[k]) + 0.25 * (ul[k] - ur[k]);
        const double h0 = (b * b) / g;  // std::pow(b, 2) / g
        h[k] = (h0 < 1e-12) ? 1e-12 : h0;
    }
    const unsigned valid = act;
    for (int it = 0; it < 100 && act; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!((act >> k) & 1u)) continue;
            const double hk = h[k];
            const bool rl = hk <= hl, rr = hk <= hr[k];
            double sgh = 0.0, sgoh = 0.0;
            if (rl || rr) {
                sgh = sqrt(g * hk);
                sgoh = sqrt(g / hk);
            }
            double pl, dl, pr, dr;
            if (rl) {
                pl = 2.0 * (sgh - cl);
                dl = sgoh;
            } else {
                const double a = sqrt(g * (hk + hl) / (2.0 * hk * hl));
                pl = (hk - hl) * a;
                dl = a - (hk - hl) * g / (4.0 * a * hk * hk);
            }
            if (rr) {
                pr = 2.0 * (sgh - cr[k]);
                dr = sgoh;
            } else {
                const double a = sqrt(g * (hk + hr[k]) / (2.0 * hk * hr[k]));
                pr = (hk - hr[k]) * a;
                dr = a - (hk - hr[k]) * g / (4.0 * a * hk * hk);
            }
            const double fk = pl + pr + ur[k] - ul[k];
            const double dfk = dl + dr;
            double dh = fk / dfk;
            if (hk - dh <= 0.0) dh = hk / 2.0;
            h[k] = hk - dh;
            if (fabs(dh) < 1e-10) act &= ~(1u << k);
        }
    }
    if (act) err = 2;  // SweRiemann: Newton iteration did not converge
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!((valid >> k) & 1u)) continue;
        const double hs = h[k], xi = 0.0;
        const double cs = sqrt(g * hs);
        const double phr = (hs <= hr[k]) ? 2.0 * (cs - cr[k])
                                          : (hs - hr[k]) * sqrt(g * (hs + hr[k]) / (2.0 * hs * hr[k]));
        const double phl = (hs <= hl) ? 2.0 * (cs - cl) : (hs - hl) * sqrt(g * (hs + hl) / (2.0 * hs * hl));
        const double us = 0.5 * (ul[k] + ur[k]) + 0.5 * (phr - phl);
        const double ut = xi <= us ? utl[k] : utr[k];
        double H, U;
        if (xi <= us) {
            if (hs > hl) {
                const double sl = ul[k] - cl * sqrt(0.5 * (hs + hl) * hs / (hl * hl));
                if (xi <= sl) { H = hl; U = ul[k]; }
                else { H = hs; U = us; }
            } else {
                const double head = ul[k] - cl, tail = us - cs;
                if (xi <= head) { H = hl; U = ul[k]; }
                else if (xi >= tail) { H = hs; U = us; }
                else {
                    const double u = (ul[k] + 2.0 * cl + 2.0 * xi) / 3.0;
                    const double c = (ul[k] + 2.0 * cl - xi) / 3.0;
                    H = c * c / g;
                    U = u;
                }
            }
        } else {
            if (hs > hr[k]) {
                const double sr = ur[k] + cr[k] * sqrt(0.5 * (hs + hr[k]) * hs / (hr[k] * hr[k]));
                if (xi >= sr) { H = hr[k]; U = ur[k]; }
                else { H = hs; U = us; }
            } else {
                const double head = ur[k] + cr[k], tail = us + cs;
                if (xi >= head) { H = hr[k]; U = ur[k]; }
                else if (xi <= tail) { H = hs; U = us; }
                else {
                    const double u = (ur[k] - 2.0 * cr[k] + 2.0 * xi) / 3.0;
                    const double c = (-ur[k] + 2.0 * cr[k] + xi) / 3.0;
                    H = c * c / g;
                    U = u;
                }
            }
        }
        const double fn_mass = H * U;
        const double fn_mom = H * U * U + 0.5 * g * H * H;
        const double ft_mom = H * U * ut;
        f[k][0] = fn_mass;
        f[k][1] = fn_mom * NX[k] - ft_mom * NY[k];
        f[k][2] = fn_mom * NY[k] + ft_mom * NX[k];
    }
}

// ---- D2Q9 BGK (builder-defined, oracle/ref_shim.cpp) -------
// q: 0 rest, 1 +x, 2 -x, 3 +y, 4 -y, 5 (+1,+1), 6 (-1,-1), 7 (+1,-1), 8 (-1,+1)
// (c + 1) packed in 2 bits per q: a branch-free lookup for a runtime q
constexpr unsigned kLbmCxP = (1u << 0) | (2u << 2) | (0u << 4) | (1u << 6) | (1u << 8) | (2u << 10) | (0u << 12) |
                             (2u << 14) | (0u << 16);
constexpr unsigned kLbmCyP = (1u << 0) | (1u << 2) | (1u << 4) | (2u << 6) | (0u << 8) | (2u << 10) | (0u << 12) |
                             (0u << 14) | (2u << 16);
__host__ __device__ constexpr int lbm_cx(int q) { return (int)((kLbmCxP >> (2 * q)) & 3u) - 1; }
__host__ __device__ constexpr int lbm_cy(int q) { return (int)((kLbmCyP >> (2 * q)) & 3u) - 1; }
static_assert(lbm_cx(1) == 1 && lbm_cx(2) == -1 && lbm_cx(5) == 1 && lbm_cx(6) == -1 && lbm_cx(7) == 1 &&
              lbm_cx(8) == -1 && lbm_cx(0) == 0 && lbm_cx(3) == 0 && lbm_cx(4) == 0);
static_assert(lbm_cy(3) == 1 && lbm_cy(4) == -1 && lbm_cy(5) == 1 && lbm_cy(6) == -1 && lbm_cy(7) == -1 &&
              lbm_cy(8) == 1 && lbm_cy(0) == 0 && lbm_cy(1) == 0 && lbm_cy(2) == 0);
__host__ __device__ constexpr double lbm_w(int q) {
    return q == 0 ? 4.0 / 9.0 : (q < 5 ? 1.0 / 9.0 : 1.0 / 36.0);
}

__host__ __device__ __forceinline__ double lbm_cu(int q, double ux, double uy) {
    switch (q) {
        case 0: return 0.0;
        case 1: return ux;
        case 2: return -ux;
        case 3: return uy;
        case 4: return -uy;
        case 5: return ux + uy;
        case 6: return -(ux + uy);
        case 7: return ux - uy;
        default: return uy - ux;
    }
}

// Equilibrium, FMA form (the scheme's definition):
//   feq_q = (w_q rho) * fma(cu, fma(4.5, cu, 3.0), fma(-1.5, usq, 1.0))
//         = w_q rho (1 + 3 cu + 4.5 cu^2 - 1.5 u^2),  usq = fma(ux, ux, uy * uy)
// Every fma is an explicit correctly rounded fused multiply-add (the C
// oracles call C99 fma()), so host and device agree bit for bit.
__host__ __device__ __forceinline__ double lbm_usq(double ux, double uy) { return fma(ux, ux, uy * uy); }
__host__ __device__ __forceinline__ double lbm_feq(int q, double rho, double cu, double usq) {
    const double t = fma(cu, fma(4.5, cu, 3.0), fma(-1.5, usq, 1.0));
    return (lbm_w(q) * rho) * t;
}

// BGK collide of the 9 pulled populations f (in place); returns the density.
//   rho = sum_q f_q (sequential), j = (x, y) momentum sums, u = j * (1 / rho)
//   f_q <- fma(omega, feq_q - f_q, f_q)          (= f - (f - feq) omega)
// The moments of the collide: density (returned) and velocity.
__host__ __device__ __forceinline__ double lbm_moments(const double (&f)[9], double& ux, double& uy) {
    const double rho = ((((((((f[0] + f[1]) + f[2]) + f[3]) + f[4]) + f[5]) + f[6]) + f[7]) + f[8]);
    const double jx = ((f[1] - f[2]) + (f[5] - f[6])) + (f[7] - f[8]);
    const double jy = ((f[3] - f[4]) + (f[5] - f[6])) + (f[8] - f[7]);
    const double inv = 1.0 / rho;
    ux = jx * inv;
    uy = jy * inv;
    return rho;
}
// The relaxation of one population toward its equilibrium.
__host__ __device__ __forceinline__ double lbm_relax(int q, double fq, double rho, double ux, double uy, double usq,
                                                     double omega) {
    return fma(omega, lbm_feq(q, rho, lbm_cu(q, ux, uy), usq) - fq, fq);
}
__host__ __device__ __forceinline__ double lbm_collide(double (&f)[9], double omega) {
    double ux, uy;
    const double rho = lbm_moments(f, ux, uy);
    const double usq = lbm_usq(ux, uy);
#pragma unroll
    for (int q = 0; q < 9; ++q) f[q] = lbm_relax(q, f[q], rho, ux, uy, usq, omega);
    return rho;
}

}  // namespace wg
