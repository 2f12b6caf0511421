// ops.cu — per-op device kernels behind the host-buffer C ABI (isolation
// parity for dwt_nd, idwt_nd, apply_threshold, csr_encode/decode,
// sync_ghosts, global_mass, fv_step and the LBM step).  These are generic
// (any rank, any 2^k+1 length) and follow the reference operation order
// exactly; the fused, register-resident hot path is in session.cu.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "host_model.h"
#include "lifting.cuh"
#include "physics.cuh"

namespace wg {
namespace {

// ---- generic line transform: one CTA per line, line staged in SMEM -------
struct LineGeom {
    uint64_t n;       // line length
    uint64_t stride;  // element stride of the line
    uint64_t inner;   // product of dims after d (== stride)
};

__device__ __forceinline__ uint64_t line_base(uint64_t line, const LineGeom& g) {
    const uint64_t outer = line / g.inner, in = line % g.inner;
    return outer * g.n * g.inner + in;
}

// dwt_line (wavelet.hpp:102-116) on one line: dwt_step_1d level by level,
// coarse to the front and details behind it.
__global__ void k_dwt_lines(double* data, LineGeom g, int levels) {
    extern __shared__ double sm[];
    double* s = sm;
    double* tmp = sm + g.n;
    const uint64_t base = line_base(blockIdx.x, g);
    for (uint64_t i = threadIdx.x; i < g.n; i += blockDim.x) s[i] = data[base + i * g.stride];
    __syncthreads();
    uint64_t b = g.n;
    for (int l = 0; l < levels; ++l) {
        const uint64_t half = (b - 1) / 2;
        double* coarse = tmp;
        double* det = tmp + half + 1;
        for (uint64_t k = threadIdx.x; k < half; k += blockDim.x)
            det[k] = s[2 * k + 1] - (s[2 * k] + s[2 * k + 2]) / 2.0;
        __syncthreads();
        for (uint64_t k = threadIdx.x; k <= half; k += blockDim.x) {
            if (k == 0) coarse[0] = s[0];
            else if (k == half) coarse[half] = s[b - 1];
            else
                coarse[k] = s[2 * k] + (lift_w((int)k - 1, (int)half) * det[k - 1] +
                                        lift_w((int)k, (int)half) * det[k]);
        }
        __syncthreads();
        for (uint64_t k = threadIdx.x; k < b; k += blockDim.x) s[k] = tmp[k];
        __syncthreads();
        b = half + 1;
    }
    for (uint64_t i = threadIdx.x; i < g.n; i += blockDim.x) data[base + i * g.stride] = s[i];
}

// idwt_line (wavelet.hpp:118-130)
__global__ void k_idwt_lines(double* data, LineGeom g, int levels) {
    extern __shared__ double sm[];
    double* s = sm;
    double* out = sm + g.n;
    const uint64_t base = line_base(blockIdx.x, g);
    for (uint64_t i = threadIdx.x; i < g.n; i += blockDim.x) s[i] = data[base + i * g.stride];
    __syncthreads();
    for (int l = levels; l >= 1; --l) {
        const uint64_t bl = ((g.n - 1) >> l) + 1;
        const uint64_t bl1 = ((g.n - 1) >> (l - 1)) + 1;
        const uint64_t half = bl - 1;
        const double* coarse = s;
        const double* det = s + bl;
        for (uint64_t k = threadIdx.x; k <= half; k += blockDim.x) {
            if (k == 0) out[0] = coarse[0];
            else if (k == half) out[2 * half] = coarse[half];
            else
                out[2 * k] = coarse[k] - (lift_w((int)k - 1, (int)half) * det[k - 1] +
                                          lift_w((int)k, (int)half) * det[k]);
        }
        __syncthreads();
        for (uint64_t k = threadIdx.x; k < half; k += blockDim.x)
            out[2 * k + 1] = det[k] + (out[2 * k] + out[2 * k + 2]) / 2.0;
        __syncthreads();
        for (uint64_t k = threadIdx.x; k < bl1; k += blockDim.x) s[k] = out[k];
        __syncthreads();
    }
    for (uint64_t i = threadIdx.x; i < g.n; i += blockDim.x) data[base + i * g.stride] = s[i];
}

void transform_nd_dev(double* d_data, const uint64_t* dims, uint32_t rank, int levels,
                      bool inverse, uint32_t first_dim = 0, cudaStream_t stream = 0) {
    uint64_t total = 1;
    for (uint32_t d = 0; d < rank; ++d) total *= dims[d];
    for (uint32_t s = first_dim; s < rank; ++s) {
        const uint32_t d = inverse ? rank - 1 - (s - first_dim) : s;
        LineGeom g;
        g.n = dims[d];
        g.inner = 1;
        for (uint32_t e = d + 1; e < rank; ++e) g.inner *= dims[e];
        g.stride = g.inner;
        const uint64_t nlines = total / g.n;
        const size_t smem = 2 * g.n * sizeof(double);
        if (smem > 200 * 1024) raise(WG_INVALID_ARGUMENT, "line too long for the device transform");
        auto kern = inverse ? k_idwt_lines : k_dwt_lines;
        if (smem > 48 * 1024)
            WG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (nlines > 0x7fffffffull) raise(WG_INVALID_ARGUMENT, "too many lines");
        kern<<<(unsigned)nlines, 128, smem, stream>>>(d_data, g, levels);
        WG_LAUNCH_CHECK("line transform");
    }
}

// ---- apply_threshold (threshold.hpp:51-86), one thread per coefficient ---
struct ThrArgs {
    uint64_t dims[kMaxRank];
    uint64_t strides[kMaxRank];
    uint32_t rank;
    int levels;
    int mode;
    double table[128];  // by key: 0 (constant), max scale (capped), sum (accumulation)
};

__global__ void k_threshold(double* v, uint64_t total, ThrArgs a, unsigned long long* zeroed) {
    const uint64_t flat = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    unsigned long long z = 0;
    if (flat < total) {
        uint64_t rem = flat;
        bool any = false;
        int key = 0;
        for (uint32_t d = 0; d < a.rank; ++d) {
            const int b = band_of_pos((int)a.dims[d], a.levels, (int)(rem / a.strides[d]));
            rem %= a.strides[d];
            const int s = b ? b - 1 : 0;
            any |= b != 0;
            if (a.mode == WG_THRESHOLD_CAPPED) key = key > s ? key : s;
            else if (a.mode == WG_THRESHOLD_ACCUMULATION) key += s;
        }
        if (any) {
            const double x = v[flat];
            if (x != 0.0 && fabs(x) < a.table[key]) {
                v[flat] = 0.0;
                z = 1;
            }
        }
    }
    // warp-aggregated count
    const unsigned mask = __ballot_sync(0xffffffffu, z != 0);
    if ((threadIdx.x & 31) == 0 && mask) atomicAdd(zeroed, (unsigned long long)__popc(mask));
}

// ---- CSR (codec.hpp:37-79) ------------------------------------------------
// Row counts with one warp per row (ballot/popc), then an exclusive scan of
// the row counts, then the ordered write of values and column indices.
__global__ void k_csr_count(const double* dense, uint64_t rows, uint64_t cols, uint32_t* cnt) {
    const uint64_t r = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    uint32_t c = 0;
    for (uint64_t j0 = 0; j0 < cols; j0 += 32) {
        const uint64_t j = j0 + lane;
        const bool nz = j < cols && dense[r * cols + j] != 0.0;
        c += __popc(__ballot_sync(0xffffffffu, nz));
    }
    if (lane == 0) cnt[r] = c;
}

// single-CTA exclusive scan of `n` u32 counts into row[0..n] (row[0] = 0)
__global__ void k_scan_rows(const uint32_t* cnt, uint64_t n, uint32_t* row) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) {
        carry = 0;
        row[0] = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint64_t base = 0; base < n; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        uint32_t x = i < n ? cnt[i] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            warp_tot[lane] = t;
        }
        __syncthreads();
        const uint32_t incl = x + (wid ? warp_tot[wid - 1] : 0) + carry;
        if (i < n) row[i + 1] = incl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
}

__global__ void k_csr_write(const double* dense, uint64_t rows, uint64_t cols, const uint32_t* row,
                            double* v, uint32_t* col) {
    const uint64_t r = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    uint32_t k = row[r];
    for (uint64_t j0 = 0; j0 < cols; j0 += 32) {
        const uint64_t j = j0 + lane;
        const double x = j < cols ? dense[r * cols + j] : 0.0;
        const bool nz = j < cols && x != 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, nz);
        if (nz) {
            const uint32_t at = k + __popc(m & ((1u << lane) - 1u));
            v[at] = x;
            col[at] = (uint32_t)j;
        }
        k += __popc(m);
    }
}

// csr_decode validation (codec.hpp:63-74) and scatter, one thread per row.
__global__ void k_csr_decode(const double* v, const uint32_t* col, const uint32_t* row,
                             uint32_t rows, uint32_t cols, double* dense, unsigned* err) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const uint32_t b = row[r], e = row[r + 1];
    if (b > e) {
        atomicOr(err, ERR_CORRUPT);
        return;
    }
    uint32_t prev = 0;
    for (uint32_t i = b; i < e; ++i) {
        if (col[i] >= cols || (i > b && col[i] <= prev)) {
            atomicOr(err, ERR_CORRUPT);
            return;
        }
        prev = col[i];
        dense[(uint64_t)r * cols + col[i]] = v[i];
    }
}

// ---- patch grid ---------------------------------------------------------------
struct GridGeom {
    uint32_t rank, m;
    int periodic;
    uint64_t splits[3], n[3], tdims[3], tstr[3];
    uint64_t npatch, tcount;
};

GridGeom grid_geom(const wg_grid_desc* d) {
    if (!d || d->rank == 0 || d->rank > 3) raise(WG_INVALID_ARGUMENT, "wg_grid_desc: rank must be 1..3");
    GridGeom g{};
    g.rank = d->rank;
    g.m = d->components;
    g.periodic = d->periodic != 0;
    g.npatch = 1;
    for (uint32_t k = 0; k < d->rank; ++k) {
        const uint64_t G = d->global_dims[k], P = d->splits[k];
        if (P == 0 || G < 2 || (G - 1) % P != 0)
            raise(WG_INVALID_ARGUMENT, "decompose: dimension not divisible by splits");
        const uint64_t n = (G - 1) / P + 1;
        if (!valid_signal_length(n)) raise(WG_INVALID_ARGUMENT, "decompose: patch logical length is not 2^k+1");
        g.splits[k] = P;
        g.n[k] = n;
        g.tdims[k] = n + 2;
        g.npatch *= P;
    }
    g.tcount = 1;
    for (uint32_t k = g.rank; k-- > 0;) {
        g.tstr[k] = g.tcount;
        g.tcount *= g.tdims[k];
    }
    return g;
}

// sync_ghosts dimension pass d (patchgrid.hpp:131-201): thread per
// (patch, side, cross index); dims < d span their full true range (ghosts
// included), dims > d their logical range.
__global__ void k_sync_pass(double* buf, GridGeom g, uint32_t d, uint64_t cross_count) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t total = g.npatch * 2 * cross_count;
    if (t >= total) return;
    uint64_t rest = t;
    const uint64_t cross = rest % cross_count;
    rest /= cross_count;
    const int side = (int)(rest % 2);
    const uint64_t p = rest / 2;
    uint64_t coord[3], ncoord[3], idx[3];
    uint64_t q = p;
    for (uint32_t k = g.rank; k-- > 0;) {
        coord[k] = q % g.splits[k];
        q /= g.splits[k];
    }
    uint64_t c2 = cross;
    for (uint32_t e = g.rank; e-- > 0;) {
        if (e == d) continue;
        const uint64_t lo = e < d ? 0 : 1;
        const uint64_t cnt = e < d ? g.tdims[e] : g.n[e];
        idx[e] = lo + c2 % cnt;
        c2 /= cnt;
    }
    const bool low = side == 0;
    bool has = true;
    for (uint32_t k = 0; k < g.rank; ++k) ncoord[k] = coord[k];
    if (low) {
        if (coord[d] > 0) ncoord[d] = coord[d] - 1;
        else if (g.periodic) ncoord[d] = g.splits[d] - 1;
        else has = false;
    } else {
        if (coord[d] + 1 < g.splits[d]) ncoord[d] = coord[d] + 1;
        else if (g.periodic) ncoord[d] = 0;
        else has = false;
    }
    uint64_t src = p;
    if (has) {
        src = 0;
        for (uint32_t k = 0; k < g.rank; ++k) src = src * g.splits[k] + ncoord[k];
    }
    const uint64_t n = g.n[d];
    const uint64_t tdst = low ? 0 : n + 1;
    const uint64_t tsrc = has ? (low ? n - 1 : 2) : (low ? 1 : n);
    uint64_t fdst = 0, fsrc = 0;
    for (uint32_t e = 0; e < g.rank; ++e) {
        fdst += (e == d ? tdst : idx[e]) * g.tstr[e];
        fsrc += (e == d ? tsrc : idx[e]) * g.tstr[e];
    }
    for (uint32_t c = 0; c < g.m; ++c)
        buf[(p * g.m + c) * g.tcount + fdst] = buf[(src * g.m + c) * g.tcount + fsrc];
}

// global_mass partial per patch (patchgrid.hpp:244-266)
__global__ void k_mass_partial(const double* buf, GridGeom g, uint32_t comp, double* part) {
    const uint64_t p = blockIdx.x;
    const double* f = buf + (p * g.m + comp) * g.tcount;
    uint64_t logical = 1;
    for (uint32_t k = 0; k < g.rank; ++k) logical *= g.n[k];
    double acc = 0.0;
    for (uint64_t c = threadIdx.x; c < logical; c += blockDim.x) {
        uint64_t rem = c, flat = 0;
        double w = 1.0;
        for (uint32_t k = g.rank; k-- > 0;) {
            const uint64_t i = rem % g.n[k] + 1;
            rem /= g.n[k];
            if (i == 1 || i == g.n[k]) w *= 0.5;
            flat += i * g.tstr[k];
        }
        acc += w * f[flat];
    }
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[p] = red[0];
}

__global__ void k_sum_ordered(const double* part, uint64_t n, double* out) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += part[i];
    *out = s;
}

// fv_step (solver.hpp:207-231): thread per logical cell of a 2-D patch.
struct FvArgs {
    GridGeom g;
    int scheme;
    double smax[4], smin[4];
    double r, gravity;
};

__global__ void k_fv_step(const double* cur, double* next, FvArgs a, unsigned* err) {
    const uint64_t n0 = a.g.n[0], n1 = a.g.n[1], ny = a.g.tdims[1];
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t per = n0 * n1;
    if (t >= a.g.npatch * per) return;
    const uint64_t p = t / per, c = t % per;
    const uint64_t i = c / n1 + 1, j = c % n1 + 1;
    const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
    const uint32_t m = a.g.m;
    const double* base = cur + p * m * a.g.tcount;
    if (a.scheme == WG_SCHEME_TRANSPORT) {
        const double w = base[i * ny + j];
        double out = w;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double wn = base[(i + di[k]) * ny + (j + dj[k])];
            out -= a.r * flux_upwind(w, wn, a.smax[k], a.smin[k]);
        }
        next[p * m * a.g.tcount + i * ny + j] = out;
    } else {
        double w[3], wn[3], out[3], f[3];
        for (uint32_t q = 0; q < 3; ++q) out[q] = w[q] = base[q * a.g.tcount + i * ny + j];
        int e = 0;
        for (int k = 0; k < 4; ++k) {
            for (uint32_t q = 0; q < 3; ++q) wn[q] = base[q * a.g.tcount + (i + di[k]) * ny + (j + dj[k])];
            flux_swe(w, wn, di[k], dj[k], a.gravity, f, e);
            for (uint32_t q = 0; q < 3; ++q) out[q] -= a.r * f[q];
        }
        if (e) atomicOr(err, e == 1 ? ERR_DOMAIN : ERR_RIEMANN);
        for (uint32_t q = 0; q < 3; ++q) next[(p * m + q) * a.g.tcount + i * ny + j] = out[q];
    }
}

__global__ void k_lbm_step(const double* cur, double* next, GridGeom g, double omega) {
    const uint64_t n0 = g.n[0], n1 = g.n[1], ny = g.tdims[1];
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t per = n0 * n1;
    if (t >= g.npatch * per) return;
    const uint64_t p = t / per, c = t % per;
    const uint64_t i = c / n1 + 1, j = c % n1 + 1;
    double f[9];
#pragma unroll
    for (int q = 0; q < 9; ++q)
        f[q] = cur[(p * 9 + q) * g.tcount + (i - lbm_cx(q)) * ny + (j - lbm_cy(q))];
    lbm_collide(f, omega);
#pragma unroll
    for (int q = 0; q < 9; ++q) next[(p * 9 + q) * g.tcount + i * ny + j] = f[q];
}

unsigned read_err(unsigned* d_err) {
    unsigned e = 0;
    WG_CUDA(cudaMemcpy(&e, d_err, sizeof e, cudaMemcpyDeviceToHost));
    return e;
}

unsigned grid_blocks(uint64_t n, unsigned bs) {
    const uint64_t b = (n + bs - 1) / bs;
    if (b > 0x7fffffffull) raise(WG_INVALID_ARGUMENT, "problem too large for one launch");
    return (unsigned)std::max<uint64_t>(b, 1);
}

}  // namespace

// shared with session.cu: direction speeds of the four faces
void direction_speeds(double alpha, double beta, double* smax, double* smin) {
    const int dirs[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};  // solver.hpp:21-22
    for (int k = 0; k < 4; ++k) {
        const double speed = alpha * dirs[k][0] + beta * dirs[k][1];  // flux_upwind, solver.hpp:55
        smax[k] = std::max(speed, 0.0);
        smin[k] = std::min(speed, 0.0);
    }
}

}  // namespace wg

using namespace wg;

extern "C" {

wg_status wg_dwt_nd(const double* in, double* out, const uint64_t* dims, uint32_t rank,
                    int32_t levels) {
    return guard([&] {
        if (rank == 0 || rank > kMaxRank) raise(WG_INVALID_ARGUMENT, "rank must be 1..8");
        plan_validate(dims, rank, levels);
        uint64_t total = 1;
        for (uint32_t d = 0; d < rank; ++d) total *= dims[d];
        DevBuf<double> buf(total);
        buf.upload(in);
        if (levels > 0) transform_nd_dev(buf.p, dims, rank, levels, false);
        buf.download(out);
    });
}

wg_status wg_idwt_nd(const double* in, double* out, const uint64_t* dims, uint32_t rank,
                     int32_t levels) {
    return guard([&] {
        if (rank == 0 || rank > kMaxRank) raise(WG_INVALID_ARGUMENT, "rank must be 1..8");
        plan_validate(dims, rank, levels);
        uint64_t total = 1;
        for (uint32_t d = 0; d < rank; ++d) total *= dims[d];
        DevBuf<double> buf(total);
        buf.upload(in);
        if (levels > 0) transform_nd_dev(buf.p, dims, rank, levels, true);
        buf.download(out);
    });
}

wg_status wg_apply_threshold(double* coeffs, const uint64_t* dims, uint32_t rank, int32_t levels,
                             int32_t mode, double c, double alpha, uint64_t* zeroed) {
    return guard([&] {
        if (c < 0.0) raise(WG_INVALID_ARGUMENT, "apply_threshold: c must be >= 0");
        if (zeroed) *zeroed = 0;
        if (c == 0.0 || levels == 0) return;  // threshold.hpp:53
        if (rank == 0 || rank > kMaxRank) raise(WG_INVALID_ARGUMENT, "rank must be 1..8");
        if (mode < 0 || mode > 2) raise(WG_INVALID_ARGUMENT, "band_threshold: unknown mode");
        ThrArgs a{};
        a.rank = rank;
        a.levels = levels;
        a.mode = mode;
        uint64_t total = 1;
        for (uint32_t d = rank; d-- > 0;) {
            a.dims[d] = dims[d];
            a.strides[d] = total;
            total *= dims[d];
        }
        const int maxkey = mode == WG_THRESHOLD_ACCUMULATION ? (int)rank * levels : levels;
        if (maxkey >= 128) raise(WG_INVALID_ARGUMENT, "too many threshold keys");
        for (int k = 0; k <= maxkey; ++k) {
            int s[kMaxRank] = {0};
            s[0] = k;  // capped: max = k; accumulation: sum = k; constant: c
            a.table[k] = band_threshold(s, rank, mode, c, alpha);
        }
        DevBuf<double> buf(total);
        DevBuf<unsigned long long> z(1);
        buf.upload(coeffs);
        WG_CUDA(cudaMemset(z.p, 0, sizeof(unsigned long long)));
        k_threshold<<<grid_blocks(total, 256), 256>>>(buf.p, total, a, z.p);
        WG_LAUNCH_CHECK("apply_threshold");
        buf.download(coeffs);
        unsigned long long hz = 0;
        z.download(&hz);
        if (zeroed) *zeroed = hz;
    });
}

wg_status wg_csr_encode(const double* dense, uint64_t rows, uint64_t cols, double* v, uint32_t* col,
                        uint32_t* row, uint64_t capacity, uint64_t* nnz) {
    return guard([&] {
        if (rows == 0 || cols == 0) raise(WG_INVALID_ARGUMENT, "csr_encode: bad shape");
        if (rows > 0xFFFFFFFFull - 1 || cols > 0xFFFFFFFFull)
            raise(WG_INVALID_ARGUMENT, "csr_encode: shape overflows 32-bit indices");
        DevBuf<double> d(rows * cols);
        DevBuf<uint32_t> cnt(rows), r(rows + 1);
        d.upload(dense);
        k_csr_count<<<grid_blocks(rows, 8), 256>>>(d.p, rows, cols, cnt.p);
        WG_LAUNCH_CHECK("csr count");
        k_scan_rows<<<1, 1024>>>(cnt.p, rows, r.p);
        WG_LAUNCH_CHECK("csr scan");
        uint32_t total = 0;
        WG_CUDA(cudaMemcpy(&total, r.p + rows, sizeof total, cudaMemcpyDeviceToHost));
        if (total > capacity) raise(WG_INVALID_ARGUMENT, "wg_csr_encode: capacity");
        DevBuf<double> dv(total);
        DevBuf<uint32_t> dc(total);
        if (total) {
            k_csr_write<<<grid_blocks(rows, 8), 256>>>(d.p, rows, cols, r.p, dv.p, dc.p);
            WG_LAUNCH_CHECK("csr write");
        }
        dv.download(v);
        dc.download(col);
        r.download(row);
        *nnz = total;
    });
}

wg_status wg_csr_decode(const double* v, const uint32_t* col, uint64_t nnz, const uint32_t* row,
                        uint64_t row_len, uint32_t rows, uint32_t cols, double* dense) {
    return guard([&] {
        if (row_len != (uint64_t)rows + 1u || row[0] != 0 || row[row_len - 1] != nnz)
            raise(WG_CORRUPT_STREAM, "csr_decode: invalid block structure");
        DevBuf<double> dv(nnz), out((uint64_t)rows * cols);
        DevBuf<uint32_t> dc(nnz), dr(row_len);
        DevBuf<unsigned> err(1);
        dv.upload(v);
        dc.upload(col);
        dr.upload(row);
        WG_CUDA(cudaMemset(out.p, 0, out.n * sizeof(double)));
        WG_CUDA(cudaMemset(err.p, 0, sizeof(unsigned)));
        k_csr_decode<<<grid_blocks(rows, 128), 128>>>(dv.p, dc.p, dr.p, rows, cols, out.p, err.p);
        WG_LAUNCH_CHECK("csr decode");
        const unsigned e = read_err(err.p);
        if (e) raise(WG_CORRUPT_STREAM, "csr_decode: bad column index or row offsets");
        out.download(dense);
    });
}

wg_status wg_grid_geometry(const wg_grid_desc* d, uint64_t* patch_logical, uint64_t* npatch,
                           uint64_t* grid_doubles) {
    return guard([&] {
        const GridGeom g = grid_geom(d);
        for (uint32_t k = 0; k < g.rank; ++k) patch_logical[k] = g.n[k];
        *npatch = g.npatch;
        *grid_doubles = g.npatch * g.m * g.tcount;
    });
}

wg_status wg_sync_ghosts(const wg_grid_desc* d, double* grid) {
    return guard([&] {
        const GridGeom g = grid_geom(d);
        const uint64_t total = g.npatch * g.m * g.tcount;
        DevBuf<double> buf(total);
        buf.upload(grid);
        for (uint32_t dim = 0; dim < g.rank; ++dim) {
            uint64_t cross = 1;
            for (uint32_t e = 0; e < g.rank; ++e)
                if (e != dim) cross *= e < dim ? g.tdims[e] : g.n[e];
            const uint64_t threads = g.npatch * 2 * cross;
            k_sync_pass<<<grid_blocks(threads, 256), 256>>>(buf.p, g, dim, cross);
            WG_LAUNCH_CHECK("sync_ghosts");
        }
        buf.download(grid);
    });
}

wg_status wg_global_mass(const wg_grid_desc* d, const double* grid, uint32_t comp, double* out) {
    return guard([&] {
        const GridGeom g = grid_geom(d);
        if (comp >= g.m) raise(WG_INVALID_ARGUMENT, "global_mass: component");
        DevBuf<double> buf(g.npatch * g.m * g.tcount), part(g.npatch), res(1);
        buf.upload(grid);
        k_mass_partial<<<(unsigned)g.npatch, 256>>>(buf.p, g, comp, part.p);
        k_sum_ordered<<<1, 1>>>(part.p, g.npatch, res.p);
        WG_LAUNCH_CHECK("global_mass");
        res.download(out);
    });
}

wg_status wg_fv_step(const wg_grid_desc* d, const double* cur, double* next, int32_t scheme,
                     double alpha, double beta, double gravity, double dt, double dx) {
    return guard([&] {
        const GridGeom g = grid_geom(d);
        if (g.rank != 2) raise(WG_INVALID_ARGUMENT, "fv_step: 2-D grids only");
        if (scheme != WG_SCHEME_TRANSPORT && scheme != WG_SCHEME_SWE)
            raise(WG_INVALID_ARGUMENT, "fv_step: unknown scheme");
        if (g.m != (scheme == WG_SCHEME_SWE ? 3u : 1u)) raise(WG_INVALID_ARGUMENT, "fv_step: component count");
        FvArgs a{};
        a.g = g;
        a.scheme = scheme;
        direction_speeds(alpha, beta, a.smax, a.smin);
        a.r = dt / dx;  // solver.hpp:212
        a.gravity = gravity;
        const uint64_t total = g.npatch * g.m * g.tcount;
        DevBuf<double> c(total), n(total);
        DevBuf<unsigned> err(1);
        c.upload(cur);
        n.upload(next);
        WG_CUDA(cudaMemset(err.p, 0, sizeof(unsigned)));
        const uint64_t cells = g.npatch * g.n[0] * g.n[1];
        k_fv_step<<<grid_blocks(cells, 128), 128>>>(c.p, n.p, a, err.p);
        WG_LAUNCH_CHECK("fv_step");
        check_device_error(read_err(err.p));
        n.download(next);
    });
}

// Batched 2-D transforms on device buffers (batch x n0 x n1), async on `stream`.
wg_status wg_dev_dwt2d(const double* in, double* out, uint64_t n0, uint64_t n1, int32_t levels,
                       uint64_t batch, void* stream) {
    return guard([&] {
        const uint64_t dims[3] = {batch, n0, n1};
        plan_validate(dims + 1, 2, levels);
        auto st = static_cast<cudaStream_t>(stream);
        if (out != in) WG_CUDA(cudaMemcpyAsync(out, in, batch * n0 * n1 * 8, cudaMemcpyDeviceToDevice, st));
        if (levels > 0 && batch > 0) transform_nd_dev(out, dims, 3, levels, false, 1, st);
    });
}

wg_status wg_dev_idwt2d(const double* in, double* out, uint64_t n0, uint64_t n1, int32_t levels,
                        uint64_t batch, void* stream) {
    return guard([&] {
        const uint64_t dims[3] = {batch, n0, n1};
        plan_validate(dims + 1, 2, levels);
        auto st = static_cast<cudaStream_t>(stream);
        if (out != in) WG_CUDA(cudaMemcpyAsync(out, in, batch * n0 * n1 * 8, cudaMemcpyDeviceToDevice, st));
        if (levels > 0 && batch > 0) transform_nd_dev(out, dims, 3, levels, true, 1, st);
    });
}

wg_status wg_lbm_step(const wg_grid_desc* d, const double* cur, double* next, double tau) {
    return guard([&] {
        const GridGeom g = grid_geom(d);
        if (g.rank != 2 || g.m != 9) raise(WG_INVALID_ARGUMENT, "lbm_step: 2-D, 9 components");
        const uint64_t total = g.npatch * g.m * g.tcount;
        DevBuf<double> c(total), n(total);
        c.upload(cur);
        n.upload(next);
        const uint64_t cells = g.npatch * g.n[0] * g.n[1];
        k_lbm_step<<<grid_blocks(cells, 128), 128>>>(c.p, n.p, g, 1.0 / tau);
        WG_LAUNCH_CHECK("lbm_step");
        n.download(next);
    });
}

// fp64 issue ceiling of this GPU (SURVEY §8d "measure the fp64 compute
// ceiling with a microbenchmark"): 8 independent DFMA chains per thread,
// enough CTAs to fill every SM; *tflops = 2 * FMAs / second.
__global__ void k_fp64_probe(double* sink, uint64_t iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) sink[0] = s;  // keeps the chains live
}

wg_status wg_dev_fp64_probe(uint64_t iters, double* tflops) {
    return guard([&] {
        int sms = 0, dev = 0;
        WG_CUDA(cudaGetDevice(&dev));
        WG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int blocks = sms * 8, threads = 256;
        DevBuf<double> sink(1);
        cudaEvent_t e0, e1;
        WG_CUDA(cudaEventCreate(&e0));
        WG_CUDA(cudaEventCreate(&e1));
        k_fp64_probe<<<blocks, threads>>>(sink.p, iters / 10 + 1, 0.999999, 1e-7);  // warm-up
        WG_CUDA(cudaEventRecord(e0));
        k_fp64_probe<<<blocks, threads>>>(sink.p, iters, 0.999999, 1e-7);
        WG_CUDA(cudaEventRecord(e1));
        WG_CUDA(cudaEventSynchronize(e1));
        WG_LAUNCH_CHECK("fp64 probe");
        float ms = 0.f;
        WG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *tflops = 2.0 * 8.0 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
    });
}

}  // extern "C"
